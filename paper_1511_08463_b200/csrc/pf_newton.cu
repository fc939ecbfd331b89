// pf_newton.cu -- coupled (u, alpha) reduced-space active-set Newton (solver.py:274-330).
#include "pf_internal.cuh"

namespace pf {
int newton_solve(Ctx* c, const double*, const double*, const double*, double*, double*, const pf_vi_opts*,
                 pf_vi_report*, cudaStream_t) {
    return set_error(c, PF_EINVAL, "coupled Newton not built yet");
}
}  // namespace pf
