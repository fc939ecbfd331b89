// pf_core.cu -- context, workspace, vector kernels and the device solvers behind the C ABI.
//
// Solvers keep all scalars on the device (scal[]); the host loop only polls a done/fail flag
// every `check_every` iterations (one 64-byte D2H read), so Krylov iterations run back to back.
// Reference semantics:
//   PCG       linalg.py:106-152  (stop ||r|| <= max(rtol ||b||, atol); breakdown on p'Ap<=0, r'z<=0)
//   rsls      vi.py:187-264      (active set, projected Armijo search, steepest-descent fallback)
//   AM pieces solver.py:129-216  (half-steps, over-relaxation with midpoint backtracking)
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "pf_internal.cuh"

namespace pf {

static thread_local std::string g_create_error;

int set_error(Ctx* c, int code, const std::string& msg) {
    if (c) c->err = msg;
    else g_create_error = msg;
    return code;
}
int check_cuda(Ctx* c, cudaError_t e, const char* where) {
    if (e == cudaSuccess) return PF_OK;
    return set_error(c, PF_ECUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

int prof_begin(Ctx* c, cudaStream_t st) {
    if (!c->prof.on) return -1;
    const int idx = (int)c->prof.log.size();
    while ((int)c->prof.ev.size() < 2 * (idx + 1)) {
        cudaEvent_t e;
        if (cudaEventCreate(&e) != cudaSuccess) return -1;
        c->prof.ev.push_back(e);
    }
    cudaEventRecord(c->prof.ev[2 * idx], st);
    return idx;
}
void prof_end(Ctx* c, cudaStream_t st, int slot, int kind, double bytes) {
    if (slot < 0) return;
    cudaEventRecord(c->prof.ev[2 * slot + 1], st);
    c->prof.log.push_back(ProfEntry{kind, slot, bytes});
}

#define PF_TRY(x)                       \
    do {                                \
        int _rc = (x);                  \
        if (_rc != PF_OK) return _rc;   \
    } while (0)
#define PF_CU(c, x, where) PF_TRY(check_cuda((c), (x), (where)))

// ---- vector kernels ------------------------------------------------------------------------
constexpr int kVecBlock = 256;
static int vec_blocks(long long n) {
    long long b = (n + kVecBlock - 1) / kVecBlock;
    return (int)std::max(1LL, std::min(b, (long long)148 * 8));
}

__device__ __forceinline__ bool solver_live(const double* s) { return s[S_DONE] == 0.0 && s[S_FAIL] == 0.0; }

// r = b - q ; z = dinv r ; rr, rz.  Last block: ||b||, target, convergence at iteration 0.
__global__ void k_cg_init(long long n, const double* __restrict__ b, const double* __restrict__ q,
                          const double* __restrict__ dinv, double* __restrict__ r, double* __restrict__ z,
                          double* s, RedBuf rb, double rtol, double atol, double maxit, int zero_x0) {
    double acc[2] = {0.0, 0.0};
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const double ri = b[i] - (zero_x0 ? 0.0 : q[i]);
        r[i] = ri;
        acc[0] += ri * ri;
        if (dinv) {
            const double zi = dinv[i] * ri;
            z[i] = zi;
            acc[1] += ri * zi;
        }
    }
    const bool check_rz = dinv != nullptr;
    grid_reduce<2>(acc, rb, 4, [=](double* t) {
        const double bn = sqrt(s[S_AUX0]);
        s[S_BNORM] = bn;
        s[S_TARGET] = fmax(rtol * bn, atol);
        s[S_RNORM] = sqrt(t[0]);
        s[S_ITER] = 0.0;
        s[S_MAXIT] = maxit;
        s[S_DONE] = 0.0;
        s[S_FAIL] = 0.0;
        s[S_BETA] = 0.0;
        s[S_RZ] = t[1];
        if (zero_x0 && bn == 0.0) { s[S_DONE] = 2.0; return; }  // x = 0 exactly (linalg.py:119-120)
        if (s[S_RNORM] <= s[S_TARGET]) { s[S_DONE] = 1.0; return; }
        if (check_rz && !(t[1] > 0.0)) s[S_FAIL] = 2.0;
    });
}

// preconditioned-PCG pieces for an external preconditioner (GMG): x += gamma p; r -= gamma q; |r|
__global__ void k_cg_update_nz(long long n, double* __restrict__ x, double* __restrict__ r,
                               const double* __restrict__ p, const double* __restrict__ q, double* s, RedBuf rb) {
    if (!solver_live(s)) return;
    const double gm = s[S_GAMMA];
    double acc[1] = {0.0};
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        x[i] += gm * p[i];
        const double ri = r[i] - gm * q[i];
        r[i] = ri;
        acc[0] += ri * ri;
    }
    grid_reduce<1>(acc, rb, 5, [=](double* t) {
        const double rn = sqrt(t[0]);
        s[S_RNORM] = rn;
        s[S_ITER] += 1.0;
        if (rn <= s[S_TARGET]) { s[S_DONE] = 1.0; return; }
        if (s[S_ITER] >= s[S_MAXIT]) s[S_DONE] = 3.0;
    });
}
// GMG-PCG update with the V-cycle's level-0 cheb0 fused in (per vertex, 2 dofs):
// x += gamma p ; r -= gamma q ; |r| ; res = D0^-1 r ; d0 = z = res / theta
__global__ void k_cg_update_gmg(long long nv, double* __restrict__ x, double* __restrict__ r,
                                const double* __restrict__ p, const double* __restrict__ q, double* s, RedBuf rb,
                                const double* __restrict__ Dinv, double* __restrict__ res, double* __restrict__ d0,
                                double* __restrict__ z, const double* lam, double ratio) {
    if (!solver_live(s)) return;
    const double gm = s[S_GAMMA];
    const Cheb c = cheb_of(lam, ratio);
    double acc[1] = {0.0};
    for (long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x; v < nv;
         v += (long long)gridDim.x * blockDim.x) {
        double2 xv = reinterpret_cast<double2*>(x)[v];
        const double2 pv = reinterpret_cast<const double2*>(p)[v];
        const double2 qv = reinterpret_cast<const double2*>(q)[v];
        double2 rv = reinterpret_cast<double2*>(r)[v];
        xv.x += gm * pv.x;
        xv.y += gm * pv.y;
        rv.x = rv.x - gm * qv.x;
        rv.y = rv.y - gm * qv.y;
        reinterpret_cast<double2*>(x)[v] = xv;
        reinterpret_cast<double2*>(r)[v] = rv;
        acc[0] += rv.x * rv.x + rv.y * rv.y;
        const double2 rr = bmul(Dinv, nv, v, rv.x, rv.y);
        const double2 dd = make_double2(rr.x / c.theta, rr.y / c.theta);
        reinterpret_cast<double2*>(res)[v] = rr;
        reinterpret_cast<double2*>(d0)[v] = dd;
        reinterpret_cast<double2*>(z)[v] = dd;
    }
    grid_reduce<1>(acc, rb, 5, [=](double* t) {
        const double rn = sqrt(t[0]);
        s[S_RNORM] = rn;
        s[S_ITER] += 1.0;
        if (rn <= s[S_TARGET]) { s[S_DONE] = 1.0; return; }
        if (s[S_ITER] >= s[S_MAXIT]) s[S_DONE] = 3.0;
    });
}

// rz = r . z ; first: S_RZ = rz ; else beta = rz / rz_old  (breakdown if rz <= 0)
__global__ void k_cg_rz(long long n, const double* __restrict__ r, const double* __restrict__ z, double* s,
                        RedBuf rb, int first) {
    if (!solver_live(s)) return;
    double acc[1] = {0.0};
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        acc[0] += r[i] * z[i];
    grid_reduce<1>(acc, rb, 6, [=](double* t) {
        if (!(t[0] > 0.0)) { s[S_FAIL] = 2.0; return; }
        if (!first) s[S_BETA] = t[0] / s[S_RZ];
        s[S_RZ] = t[0];
    });
}

// x += gamma p ; r -= gamma q ; z = dinv r ; reductions -> beta / convergence (linalg.py:137-150)
__global__ void k_cg_update(long long n, double* __restrict__ x, double* __restrict__ r,
                            double* __restrict__ z, const double* __restrict__ p,
                            const double* __restrict__ q, const double* __restrict__ dinv, double* s,
                            RedBuf rb) {
    if (!solver_live(s)) return;
    const double gm = s[S_GAMMA];
    double acc[2] = {0.0, 0.0};
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        x[i] += gm * p[i];
        const double ri = r[i] - gm * q[i];
        r[i] = ri;
        const double zi = dinv[i] * ri;
        z[i] = zi;
        acc[0] += ri * ri;
        acc[1] += ri * zi;
    }
    grid_reduce<2>(acc, rb, 5, [=](double* t) {
        const double rn = sqrt(t[0]);
        s[S_RNORM] = rn;
        s[S_ITER] += 1.0;
        if (rn <= s[S_TARGET]) { s[S_DONE] = 1.0; return; }
        if (!(t[1] > 0.0)) { s[S_FAIL] = 2.0; return; }
        s[S_BETA] = t[1] / s[S_RZ];
        s[S_RZ] = t[1];
        if (s[S_ITER] >= s[S_MAXIT]) s[S_DONE] = 3.0;
    });
}

__global__ void k_relax_u(long long nv, long long nc, int nvy, int nx, int ny, const double* __restrict__ up,
                          const double* __restrict__ us, double om, double* __restrict__ uo,
                          const unsigned char* __restrict__ mask, const double* __restrict__ ubar, int has_bc,
                          int snap_only) {
    for (long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x; v < nv;
         v += (long long)gridDim.x * blockDim.x) {
        double2 a;
        if (snap_only) {
            a = reinterpret_cast<const double2*>(uo)[v];
        } else {
            const double2 p = reinterpret_cast<const double2*>(up)[v];
            const double2 q = reinterpret_cast<const double2*>(us)[v];
            a = make_double2(p.x + om * (q.x - p.x), p.y + om * (q.y - p.y));
        }
        if (has_bc && v < nc) {
            const int i = (int)(v / nvy), j = (int)(v % nvy);
            if (i == 0 || i == nx || j == 0 || j == ny) {
                const unsigned m = mask[v];
                if (m) {
                    const double2 b = reinterpret_cast<const double2*>(ubar)[v];
                    if (m & 1u) a.x = b.x;
                    if (m & 2u) a.y = b.y;
                }
            }
        }
        reinterpret_cast<double2*>(uo)[v] = a;
    }
}

// over-relaxed damage candidates: bit k of the OR-reduced word is set if candidate k is
// infeasible somewhere (solver.py:202-213); k = 0..59, omega_k = (1 + omega_{k-1}) / 2.
__global__ void k_relax_bits(long long n, const double* __restrict__ ap, const double* __restrict__ as,
                             const double* __restrict__ lb, double omega, unsigned long long* bits) {
    unsigned long long m = 0ull;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const double a0 = ap[i], d = as[i] - a0, l = lb[i];
        double w = omega;
        for (int k = 0; k < 60; ++k) {
            if (k > 0 && w == 1.0) break;
            const double cand = a0 + w * d;
            if (cand < l || cand > 1.0) m |= (1ull << k);
            w = 0.5 * (1.0 + w);
        }
    }
    unsigned lo = __reduce_or_sync(PF_FULL, (unsigned)(m & 0xffffffffull));
    unsigned hi = __reduce_or_sync(PF_FULL, (unsigned)(m >> 32));
    if ((threadIdx.x & 31) == 0 && (lo | hi)) atomicOr(bits, ((unsigned long long)hi << 32) | lo);
}

__global__ void k_relax_apply(long long n, const double* __restrict__ ap, const double* __restrict__ as,
                              const double* __restrict__ lb, double omega, const unsigned long long* bits,
                              double* __restrict__ out, unsigned long long* dmax, double* s) {
    double wb;
    int kk;
    bool star;
    choose_omega(omega, bits[0], wb, kk, star);
    double dm = 0.0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const double a0 = ap[i];
        const double cand = star ? as[i] : a0 + wb * (as[i] - a0);
        const double a = fmin(fmax(cand, lb[i]), 1.0);
        out[i] = a;
        dm = fmax(dm, fabs(a - a0));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) dm = fmax(dm, __shfl_xor_sync(PF_FULL, dm, o));
    if ((threadIdx.x & 31) == 0 && dm > 0.0) atomicMax(dmax, (unsigned long long)__double_as_longlong(dm));
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        s[S_OMEGABAR] = wb;
        s[S_AUX1] = (double)kk;
    }
}

// x = clip(x0, lb, 1) and max|x| (vi.py:197-201)
__global__ void k_clip_max(long long n, const double* __restrict__ x0, const double* __restrict__ lb,
                           double* __restrict__ x, unsigned long long* xmax) {
    double m = 0.0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const double v = fmin(fmax(x0[i], lb[i]), 1.0);
        x[i] = v;
        m = fmax(m, fabs(v));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(PF_FULL, m, o));
    if ((threadIdx.x & 31) == 0 && m > 0.0) atomicMax(xmax, (unsigned long long)__double_as_longlong(m));
}

// activity classification (vi.py:127-141) + masked right-hand side rhs = F on N, 0 on A.
// zeta = zero_tol, or 1e-10 (1 + |x0|_inf) as vi.py:198-201 (|x0|_inf from k_clip_max)
__global__ void k_set_zeta(const unsigned long long* xmax, double* s, double zero_tol) {
    s[S_ZETA] = zero_tol > 0.0 ? zero_tol : 1e-10 * (1.0 + __longlong_as_double((long long)*xmax));
}

__global__ void k_classify(long long n, const double* __restrict__ x, const double* __restrict__ F,
                           const double* __restrict__ lb, unsigned char* __restrict__ act,
                           double* __restrict__ rhs, double* s, RedBuf rb) {
    const double zeta = s[S_ZETA];
    double acc[2] = {0.0, 0.0};
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const double xv = x[i], Fv = F[i];
        const bool lo = (xv - lb[i] <= zeta) && (Fv > 0.0);
        const bool up = (1.0 - xv <= zeta) && (Fv < 0.0) && !lo;
        const bool a = lo || up;
        act[i] = lo ? 1 : (up ? 2 : 0);
        rhs[i] = a ? 0.0 : Fv;
        acc[0] += a ? 0.0 : 1.0;
        acc[1] += a ? 0.0 : Fv * Fv;
    }
    grid_reduce<2>(acc, rb, 6, [=](double* t) {
        s[S_NINACT] = t[0];
        s[S_AUX0] = t[1];  // |rhs|^2 for the inner PCG stopping rule
    });
}

// projected-Jacobi direction of the damage QP: d = -D^-1 F  (damage_solve, crawl mode)
__global__ void k_pj_dir(long long n, const double* __restrict__ dinv, const double* __restrict__ F,
                         double* __restrict__ d) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        d[i] = -dinv[i] * F[i];
}

__global__ void k_scale(long long n, double* __restrict__ x, double a) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        x[i] *= a;
}

// merit-gradient ingredients for the two-sided box (vi.py:144-178): p, q partials and w = q*phi.
__device__ __forceinline__ void fb_part(double a, double b, double& pa, double& pb) {
    const double rho = hypot(a, b);
    if (rho > 0.0) { pa = a / rho - 1.0; pb = b / rho - 1.0; }
    else { pa = 0.70710678118654752440 - 1.0; pb = pa; }
}
__global__ void k_merit_parts(long long n, const double* __restrict__ x, const double* __restrict__ F,
                              const double* __restrict__ lb, double* __restrict__ pphi,
                              double* __restrict__ w) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const double xv = x[i], Fv = F[i], sl = 1.0 - xv;
        const double inner = hypot(sl, -Fv) - sl + Fv;
        double pao, pbo, pai, pbi;
        fb_part(xv - lb[i], inner, pao, pbo);
        fb_part(sl, -Fv, pai, pbi);
        const double ph = hypot(xv - lb[i], inner) - (xv - lb[i]) - inner;
        const double p = pao - pbo * pai;
        const double q = -pbo * pbi;
        pphi[i] = p * ph;
        w[i] = q * ph;
    }
}
// g = 2 (p phi + Kaa w) in place on kw; reduces |g|^2
__global__ void k_grad_finish(long long n, const double* __restrict__ pphi, double* __restrict__ kw,
                              double* s, RedBuf rb) {
    double acc[1] = {0.0};
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const double gv = 2.0 * (pphi[i] + kw[i]);
        kw[i] = gv;
        acc[0] += gv * gv;
    }
    grid_reduce<1>(acc, rb, 7, [=](double* t) { s[S_GNORM2] = t[0]; });
}

// ---- host helpers ---------------------------------------------------------------------------
int read_scal(Ctx* c, cudaStream_t st, int first, int count) {
    PF_CU(c, cudaMemcpyAsync(c->h_scal + first, c->scal + first, sizeof(double) * count,
                             cudaMemcpyDeviceToHost, st), "scalar readback");
    PF_CU(c, cudaStreamSynchronize(st), "stream sync");
    return PF_OK;
}
int set_scal(Ctx* c, cudaStream_t st, int slot, double v) {
    c->h_scal[64 + (slot & 63)] = v;
    // small synchronous-ordered upload via cudaMemcpyAsync from pinned memory
    PF_CU(c, cudaMemcpyAsync(c->scal + slot, c->h_scal + 64 + (slot & 63), sizeof(double),
                             cudaMemcpyHostToDevice, st), "scalar upload");
    return PF_OK;
}

// ---- generic PCG on device --------------------------------------------------------------------
int vec_blocks_n(long long n) { return vec_blocks(n); }
void classify(Ctx* c, long long n, const double* x, const double* F, const double* lb, unsigned char* act,
              double* rhs, cudaStream_t st) {
    const RedBuf rb{c->partials, c->tickets, c->scal};
    k_classify<<<vec_blocks(n), kVecBlock, 0, st>>>(n, x, F, lb, act, rhs, c->scal, rb);
    c->launches++;
}
void merit_parts(Ctx* c, long long n, const double* x, const double* F, const double* lb, double* pphi,
                 double* w, cudaStream_t st) {
    k_merit_parts<<<vec_blocks(n), kVecBlock, 0, st>>>(n, x, F, lb, pphi, w);
    c->launches++;
}

// last node of the device-side Krylov loop body: continue while the solver is live
__global__ void k_loop_cond(cudaGraphConditionalHandle h, const double* s) {
    if (threadIdx.x == 0) cudaGraphSetConditional(h, (s[S_DONE] == 0.0 && s[S_FAIL] == 0.0) ? 1u : 0u);
}

// report + error mapping once the Krylov loop stopped (scalars already read back)
static int pcg_finish(Ctx* c, const PcgBuffers& B, pf_lin_report* rep, cudaStream_t st) {
    rep->iterations = (long long)c->h_scal[S_ITER];
    rep->final_residual_norm = c->h_scal[S_RNORM];
    rep->b_norm = c->h_scal[S_BNORM];
    rep->converged = (c->h_scal[S_FAIL] == 0.0) && (c->h_scal[S_RNORM] <= c->h_scal[S_TARGET] ||
                                                    c->h_scal[S_DONE] == 2.0);
    rep->status = PF_OK;
    if (c->h_scal[S_DONE] == 2.0) {
        PF_CU(c, cudaMemsetAsync(B.x, 0, sizeof(double) * B.n, st), "memset");
        rep->iterations = 0;
        rep->final_residual_norm = 0.0;
    }
    if (c->h_scal[S_FAIL] != 0.0) {
        char msg[160];
        if (c->h_scal[S_FAIL] == 1.0)
            snprintf(msg, sizeof msg, "cg: p'Ap = %.3e <= 0 at iteration %lld (operator not positive definite)",
                     c->h_scal[S_PAP], (long long)c->h_scal[S_ITER] + 1);
        else
            snprintf(msg, sizeof msg, "cg: preconditioner not SPD at iteration %lld",
                     (long long)c->h_scal[S_ITER]);
        rep->status = PF_EBREAKDOWN;
        return set_error(c, PF_EBREAKDOWN, msg);
    }
    return PF_OK;
}


int pcg_run(Ctx* c, int kind, const PcgBuffers& B, const double* coef, const unsigned char* act,
                   double rtol, double atol, long long maxit, int zero_x0, int check_every,
                   pf_lin_report* rep, cudaStream_t st) {
    const RedBuf rb{c->partials, c->tickets, c->scal};
    const int vb = vec_blocks(B.n);
    const bool gmg = (kind == 2);
    // q = A x0 (if warm)
    if (!zero_x0) {
        if (kind == 0 || kind == 2) PF_TRY(launch_Kuu(c, coef, B.x, B.q, PF_BC_ELIMINATE, st));
        else PF_TRY(launch_Kaa(c, coef, B.x, B.q, act, st));
    } else {
        PF_CU(c, cudaMemsetAsync(B.x, 0, sizeof(double) * B.n, st), "memset");
    }
    {
        const int ps = prof_begin(c, st);
        k_cg_init<<<vb, kVecBlock, 0, st>>>(B.n, B.b, B.q, gmg ? nullptr : B.dinv, B.r, B.z, c->scal, rb, rtol,
                                            atol, (double)maxit, zero_x0);
        prof_end(c, st, ps, K_CG_VEC, 8.0 * B.n * 5);
    }
    c->launches++;
    PF_CU(c, cudaGetLastError(), "cg init");
    if (gmg) {
        bool rzd = false;
        if (c->dim == 3) PF_TRY(gmg3_vcycle(c, B.r, B.z, st, c->scal));
        else PF_TRY(gmg_vcycle(c, B.r, B.z, st, c->scal, false, 1, &rzd));
        if (!rzd) {
            k_cg_rz<<<vb, kVecBlock, 0, st>>>(B.n, B.r, B.z, c->scal, rb, 1);
            c->launches++;
        }
    }
    // No host poll here: the persistent and graph loops below check the done/fail flags on the
    // device (the start-up may already have converged); only the eager loop needs them now.
    const bool graphs = c->use_graphs && !c->prof.on;
    const bool persistent = kind == 1 && c->pcg_persistent;
    if (!graphs && !persistent) PF_TRY(read_scal(c, st, 0, 24));
    // one Krylov iteration k (ping-pong search-direction buffers by parity)
    auto issue_iter = [&](long long k, cudaStream_t s) -> int {
        double* pin = (k & 1) ? B.p1 : B.p0;
        double* pout = (k & 1) ? B.p0 : B.p1;
        if (gmg && c->dim == 3) {  // 3D: plain PCG update, V-cycle, r.z
            PF_TRY(launch_Kuu_cgA(c, coef, B.z, pin, pout, B.q, s));
            const int ps = prof_begin(c, s);
            k_cg_update_nz<<<vb, kVecBlock, 0, s>>>(B.n, B.x, B.r, pout, B.q, c->scal, rb);
            prof_end(c, s, ps, K_CG_VEC, 8.0 * B.n * 6);
            PF_TRY(gmg3_vcycle(c, B.r, B.z, s, c->scal));
            const int ps2 = prof_begin(c, s);
            k_cg_rz<<<vb, kVecBlock, 0, s>>>(B.n, B.r, B.z, c->scal, rb, 0);
            prof_end(c, s, ps2, K_CG_VEC, 8.0 * B.n * 2);
            c->launches += 2;
            return PF_OK;
        }
        if (gmg) {
            PF_TRY(launch_Kuu_cgA(c, coef, B.z, pin, pout, B.q, s));
            const GLevel& L0 = c->glev[0];
            const long long nv0 = B.n / 2;
            const int ps = prof_begin(c, s);
            k_cg_update_gmg<<<vec_blocks(nv0), kVecBlock, 0, s>>>(nv0, B.x, B.r, pout, B.q, c->scal, rb, L0.Dinv,
                                                                   L0.res, L0.d0, B.z, c->scal + S_GMG0,
                                                                   c->gmg_ratio);
            prof_end(c, s, ps, K_CG_VEC, 8.0 * B.n * 6 + 8.0 * B.n * 5);  // + Dinv, res, d0, z
            c->launches++;
            bool rzd = false;
            PF_TRY(gmg_vcycle(c, B.r, B.z, s, c->scal, true, 0, &rzd));
            if (!rzd) {
                const int ps2 = prof_begin(c, s);
                k_cg_rz<<<vb, kVecBlock, 0, s>>>(B.n, B.r, B.z, c->scal, rb, 0);
                prof_end(c, s, ps2, K_CG_VEC, 8.0 * B.n * 2);
                c->launches++;
            }
            return PF_OK;
        }
        if (kind == 0) PF_TRY(launch_Kuu_cgA(c, coef, B.z, pin, pout, B.q, s));
        else PF_TRY(launch_Kaa_cgA(c, coef, B.z, pin, pout, B.q, act, s));
        const int ps = prof_begin(c, s);
        k_cg_update<<<vb, kVecBlock, 0, s>>>(B.n, B.x, B.r, B.z, pout, B.q, B.dinv, c->scal, rb);
        prof_end(c, s, ps, K_CG_VEC, 8.0 * B.n * 8);  // x,p,r,q,dinv -> x,r,z
        c->launches++;
        return PF_OK;
    };
    // The Krylov loop runs on the device: a CUDA graph whose WHILE conditional node replays the
    // captured iteration pair until k_loop_cond (last node of the body) sees the solver done or
    // failed -- no host polling, at most one no-op iteration after convergence.  Kernels read
    // every scalar from device memory, so the body is replayed unchanged.  Disabled while
    // per-kernel profiling is on (eager launches bracketed by events, host-polled batches).
    if (persistent) {
        // damage block: every iteration inside one cooperative launch (no host polls, no graph)
        const int rc = c->pcg_single ? launch_pcg_kaa1(c, B, coef, act, st) : launch_pcg_kaa(c, B, coef, act, st);
        if (rc == PF_OK) {
            PF_TRY(read_scal(c, st, 0, 24));
            // profiling: the launch's algorithmic bytes are known once its iterations are
            if (c->prof.on && !c->prof.log.empty())
                c->prof.log.back().bytes = c->h_scal[S_ITER] * pcg_kaa_iter_bytes(c) * c->tile_frac;
            return pcg_finish(c, B, rep, st);
        }
        if (rc != PF_EINVAL) return rc;
    }
    if (persistent && !graphs) PF_TRY(read_scal(c, st, 0, 24));  // fallback to the eager loop
    const long long key = c->geo_version * 16 + (gmg ? c->gmg_degree : 0);
    // the captured body bakes in these pointers: re-capture when any of them changes
    const void* body_ptrs[Ctx::kGraphPtrs] = {B.x, B.r, B.z, B.p0, B.p1, B.q, B.dinv, coef, act};
    const bool same_ptrs = memcmp(body_ptrs, c->graph_ptrs[kind], sizeof(body_ptrs)) == 0;
    if (graphs && (c->graph_key[kind] != key || !same_ptrs)) {
        memcpy(c->graph_ptrs[kind], body_ptrs, sizeof(body_ptrs));
        if (c->graph_exec[kind]) { cudaGraphExecDestroy(c->graph_exec[kind]); c->graph_exec[kind] = nullptr; }
        if (!c->cap_stream) PF_CU(c, cudaStreamCreateWithFlags(&c->cap_stream, cudaStreamNonBlocking), "stream");
        PF_CU(c, cudaStreamSynchronize(st), "sync");
        const long long l0 = c->launches;
        cudaGraph_t graph = nullptr;
        PF_CU(c, cudaGraphCreate(&graph, 0), "graph create");
        cudaGraphConditionalHandle h;
        cudaGraphNodeParams np = {};
        cudaGraphNode_t node;
        cudaError_t ce = cudaGraphConditionalHandleCreate(&h, graph, 1, cudaGraphCondAssignDefault);
        if (ce == cudaSuccess) {
            np.type = cudaGraphNodeTypeConditional;
            np.conditional.handle = h;
            np.conditional.type = cudaGraphCondTypeWhile;
            np.conditional.size = 1;
            ce = cudaGraphAddNode(&node, graph, nullptr, 0, &np);
        }
        if (ce != cudaSuccess) {
            cudaGraphDestroy(graph);
            return check_cuda(c, ce, "conditional graph node");
        }
        cudaGraph_t body = np.conditional.phGraph_out[0];
        PF_CU(c, cudaStreamBeginCaptureToGraph(c->cap_stream, body, nullptr, nullptr, 0,
                                               cudaStreamCaptureModeThreadLocal), "begin capture");
        int rc1 = issue_iter(0, c->cap_stream);
        int rc2 = rc1 == PF_OK ? issue_iter(1, c->cap_stream) : rc1;
        if (rc2 == PF_OK) {
            k_loop_cond<<<1, 32, 0, c->cap_stream>>>(h, c->scal);
            c->launches++;
        }
        cudaGraph_t captured = nullptr;
        ce = cudaStreamEndCapture(c->cap_stream, &captured);
        if (rc2 != PF_OK) { cudaGraphDestroy(graph); return rc2; }
        if (ce != cudaSuccess) { cudaGraphDestroy(graph); return check_cuda(c, ce, "end capture"); }
        ce = cudaGraphInstantiate(&c->graph_exec[kind], graph, 0);
        cudaGraphDestroy(graph);
        PF_CU(c, ce, "graph instantiate");
        c->graph_nodes[kind] = c->launches - l0;  // launches per replayed pair
        c->launches = l0;
        c->graph_key[kind] = key;
    }
    long long k = 0;
    int batch = std::max(2, check_every + (check_every & 1));
    if (graphs) {  // a solve that converged at start-up runs one no-op pair (device-side flags)
        PF_CU(c, cudaGraphLaunch(c->graph_exec[kind], st), "graph launch");
        PF_TRY(read_scal(c, st, 0, 24));
        const long long pairs = ((long long)c->h_scal[S_ITER] + 2) / 2;
        c->launches += pairs * c->graph_nodes[kind];
    } else {
        while (c->h_scal[S_DONE] == 0.0 && c->h_scal[S_FAIL] == 0.0) {
            for (int t = 0; t < batch; ++t, ++k) PF_TRY(issue_iter(k, st));
            PF_CU(c, cudaGetLastError(), "cg iteration");
            PF_TRY(read_scal(c, st, 0, 24));
            // cheap iterations (Jacobi): grow the poll interval; GMG iterations are ~100x dearer
            // than a poll, so poll every pair to avoid launching no-op iterations after convergence
            if (!gmg) batch = std::min(batch * 2, 64);
        }
    }
    return pcg_finish(c, B, rep, st);
}

int elastic_solve(Ctx* c, const double* alpha, const double* u0, double* u_out, const pf_lin_opts* o,
                  pf_lin_report* rep, cudaStream_t st) {
    if (o->precond != PF_PREC_JACOBI && o->precond != PF_PREC_GMG)
        return set_error(c, PF_EINVAL, "elastic solve: unknown preconditioner");
    const bool gmg = o->precond == PF_PREC_GMG;
    PF_CU(c, cudaMemcpyAsync(c->alpha_ws, alpha, sizeof(double) * c->n_a, cudaMemcpyDeviceToDevice, st),
          "alpha copy");
    PcgBuffers B{c->cg_x, c->cg_r, c->cg_z, c->cg_p0, c->cg_p1, c->cg_q, c->cg_dinv, c->cg_b, c->n_u};
    bool reused = false;
    if (gmg) {
        const int deg = o->cheb_degree > 0 ? o->cheb_degree : 2;
        reused = o->gmg_reuse && c->gmg_built && deg == c->gmg_degree;
        c->gmg_degree = deg;
        if (!reused) {
            PF_TRY(c->dim == 3 ? gmg3_setup(c, st) : gmg_setup(c, st));
            c->gmg_built = 1;
            c->gmg_its0 = -1;
        }
    } else {
        PF_TRY(launch_Kuu_diag(c, c->alpha_ws, B.dinv, st));
    }
    PF_TRY(launch_load(c, c->alpha_ws, B.b, nullptr, 1, st));   // b = M(f - K g) + (I-M) ubar
    const int warm = (o->warm_start && u0) ? 1 : 0;
    if (warm)
        PF_CU(c, cudaMemcpyAsync(B.x, u0, sizeof(double) * c->n_u, cudaMemcpyDeviceToDevice, st), "u0 copy");
    const long long maxit = o->maxit > 0 ? o->maxit : 10 * c->n_u;
    int rc = pcg_run(c, gmg ? 2 : 0, B, c->alpha_ws, nullptr, o->rtol, o->atol, maxit, warm ? 0 : 1,
                     o->check_every > 0 ? o->check_every : (gmg ? 2 : 8), rep, st);
    if (reused && (rc == PF_EBREAKDOWN || (rc == PF_OK && !rep->converged))) {
        // the kept hierarchy no longer preconditions this alpha: rebuild and solve again
        PF_TRY(c->dim == 3 ? gmg3_setup(c, st) : gmg_setup(c, st));
        c->gmg_its0 = -1;
        if (warm)
            PF_CU(c, cudaMemcpyAsync(B.x, u0, sizeof(double) * c->n_u, cudaMemcpyDeviceToDevice, st), "u0 copy");
        rc = pcg_run(c, 2, B, c->alpha_ws, nullptr, o->rtol, o->atol, maxit, warm ? 0 : 1,
                     o->check_every > 0 ? o->check_every : 2, rep, st);
    }
    if (rc != PF_OK) {
        c->gmg_built = 0;
        return rc;
    }
    if (gmg) {
        // refresh the hierarchy once the iterations it costs beyond those of its first solve add up
        // to about one setup (a rebuild costs ~10 V-cycle iterations; warm-started solves make
        // single-solve ratios noisy)
        if (c->gmg_its0 < 0) {
            c->gmg_its0 = rep->iterations;
            c->gmg_excess = 0;
        } else {
            c->gmg_excess += std::max(0LL, (long long)rep->iterations - c->gmg_its0);
            if (c->gmg_excess > kGmgRebuildIts) c->gmg_built = 0;  // refresh next time
        }
    }
    PF_CU(c, cudaMemcpyAsync(u_out, B.x, sizeof(double) * c->n_u, cudaMemcpyDeviceToDevice, st), "u copy");
    if (!rep->converged) {
        char msg[128];
        snprintf(msg, sizeof msg, "elastic CG stalled at residual %.3e", rep->final_residual_norm);
        rep->status = PF_ESTALL;
        return set_error(c, PF_ESTALL, msg);
    }
    return PF_OK;
}

// ---- damage VI: rsls on the box QP F(a) = Kaa a + c, lb <= a <= 1 (vi.py:187-264) --------------
int damage_solve(Ctx* c, const double* u, const double* lb, const double* a_in, double* a_out,
                 const pf_vi_opts* o, pf_vi_report* rep, cudaStream_t st) {
    const long long n = c->n_a;
    const int vb = vec_blocks(n);
    const RedBuf rb{c->partials, c->tickets, c->scal};
    memset(rep, 0, sizeof(*rep));
    // element reaction coefficients + affine remainder (solver.py:152-153)
    PF_TRY(launch_kappa(c, u, a_in, c->kappa, c->vi_c, st));
    // x = clip(a_in), zeta
    PF_CU(c, cudaMemsetAsync(c->bits, 0, sizeof(unsigned long long) * 8, st), "memset bits");
    k_clip_max<<<vb, kVecBlock, 0, st>>>(n, a_in, lb, c->vi_x, c->bits + 1);
    k_set_zeta<<<1, 1, 0, st>>>(c->bits + 1, c->scal, o->zero_tol);  // no host round trip
    c->launches += 2;
    double *x = c->vi_x, *F = c->vi_F, *tx = c->vi_tx, *tF = c->vi_tF;
    PF_TRY(launch_Kaa_trial(c, c->kappa, c->vi_c, x, nullptr, lb, tx, F, nullptr, S_MERIT, st));
    PF_TRY(read_scal(c, st, 0, 24));
    double merit = c->h_scal[S_MERIT];
    auto push_hist = [&](double m) {
        if (rep->n_history < 64) rep->history[rep->n_history] = std::sqrt(m);
        rep->n_history++;
    };
    push_hist(merit);
    PcgBuffers B{c->da_x, c->da_r, c->da_z, c->da_p0, c->da_p1, c->da_q, c->da_dinv, c->vi_d, n};
    auto line_search = [&](const double* dir, double bound0, double slope, bool newton, bool& ok) -> int {
        double mu = 1.0;
        ok = false;
        while (mu >= o->ls_min_step) {
            PF_TRY(set_scal(c, st, S_MU, mu));
            PF_TRY(launch_Kaa_trial(c, c->kappa, c->vi_c, x, dir, lb, tx, tF, nullptr, S_TMERIT, st));
            PF_TRY(read_scal(c, st, S_TMERIT, 1));
            const double mt = c->h_scal[S_TMERIT];
            const double bound = newton ? (1.0 - 2.0 * o->armijo * mu) * bound0 : bound0 - slope * mu;
            if (mt <= bound) {
                ok = true;
                merit = mt;
                std::swap(x, tx);
                std::swap(F, tF);
                return PF_OK;
            }
            mu *= o->ls_backtrack;
        }
        return PF_OK;
    };
    double merit_prev = 0.0;  // |Phi|^2 of the previous VI iterate (0: none yet)
    static const bool ew_on = !(getenv("PF_VI_EW") && atoi(getenv("PF_VI_EW")) == 0);
    static const double ew_cap = getenv("PF_VI_EWCAP") ? atof(getenv("PF_VI_EWCAP")) : 0.1;
    // Crawl mode.  When two consecutive active-set iterations reduce |Phi| by less than 30 % the
    // free boundary is moving one vertex layer per Newton solve (see the forcing-term note below);
    // from then on every iteration is preceded by a few projected-Jacobi sweeps
    //     x <- P[x - w D^-1 (Kaa x + c)]
    // (one vector pass and one trial strip pass each, no host round trip), which move the free
    // boundary at a twentieth of the cost of an active-set iteration.  The QP is strictly convex, so
    // its minimiser -- what the VI stopping rule tests -- does not depend on the path.
    static const int pj_sweeps = getenv("PF_VI_PJ") ? atoi(getenv("PF_VI_PJ")) : 16;
    static const double pj_w = getenv("PF_VI_PJW") ? atof(getenv("PF_VI_PJW")) : 0.7;
    int slow = 0;
    bool have_dinvJ = false;
    for (int it = 1; it <= o->max_iterations; ++it) {
        if (std::sqrt(merit) <= o->abs_tol) break;
        rep->iterations = it;
        // (inexact mode only: inner_mode 0 follows the reference's iterates step by step; scratch:
        // the single-reduction PCG's two vectors, free unless that variant is selected)
        if (pj_sweeps > 0 && slow >= 2 && o->inner_mode == 1 && !c->pcg_single) {
            double *dinvJ = c->cg1_s0, *dir = c->cg1_s1;
            if (!have_dinvJ) {  // unmasked Jacobi scaling
                PF_TRY(launch_Kaa_diag(c, c->kappa, dinvJ, nullptr, st));
                have_dinvJ = true;
            }
            PF_TRY(set_scal(c, st, S_MU, pj_w));
            for (int sw = 0; sw < pj_sweeps; ++sw) {
                k_pj_dir<<<vb, kVecBlock, 0, st>>>(n, dinvJ, F, dir);
                c->launches++;
                PF_TRY(launch_Kaa_trial(c, c->kappa, c->vi_c, x, dir, lb, tx, tF, nullptr, S_TMERIT, st));
                std::swap(x, tx);
                std::swap(F, tF);
            }
            PF_TRY(read_scal(c, st, S_TMERIT, 1));
            merit = c->h_scal[S_TMERIT];
            if (getenv("PF_VI_TRACE")) fprintf(stderr, "  vi it=%d after %d sweeps merit=%.3e\n", it, pj_sweeps, std::sqrt(merit));
            if (std::sqrt(merit) <= o->abs_tol) break;
        }
        k_classify<<<vb, kVecBlock, 0, st>>>(n, x, F, lb, c->act, c->vi_d, c->scal, rb);
        c->launches++;
        PF_TRY(read_scal(c, st, S_NINACT, 1));
        bool ok = false;
        if (c->h_scal[S_NINACT] > 0.0) {
            PF_TRY(launch_Kaa_diag(c, c->kappa, B.dinv, c->act, st));
            pf_lin_report lr{};
            int rc;
            const long long maxit = o->inner_maxit > 0 ? o->inner_maxit : 10 * n;
            // atol floor: after an exact-active-set Newton step the VI merit equals the reduced
            // residual, so converging it below 0.1*abs_tol buys nothing (vi.py:222-240)
            // inner_mode 1: inexact Newton with the quadratic forcing term rtol = min(1e-2, |Phi|)
            // (never tighter than inner_rtol): far from the solution the reduced system is solved
            // loosely, close to it as before; the VI stopping rule (merit <= abs_tol) is unchanged
            // Safeguard of the forcing term (Eisenstat-Walker choice 2): when the VI converges only
            // linearly -- after a load increment of a cracked state the free boundary of the
            // irreversibility constraint moves one vertex layer per active-set iteration (SENT 512^2:
            // 63 iterations at |Phi_k| / |Phi_k-1| = 0.9, 190 vertices released each) -- a tolerance
            // of |Phi| oversolves every one of them (20-30 PCG iterations for a 10 % decrease), so
            // the tolerance is never tighter than min(0.1, 0.5 (|Phi_k| / |Phi_k-1|)^2).  Measured on
            // the SENT 512^2 driver window (same AM counts and energies to all printed digits): cap
            // 0 (off) 0.1389, 0.01 0.1360, 0.05 0.1343, 0.1 0.1332, 0.3 0.1328 s/step; a
            // post-nucleation step 138 -> 118 ms (its first damage solve 1908 -> ~750 PCG iterations).
            const double ew = merit_prev > 0.0 ? 0.5 * merit / merit_prev : 0.0;
            const double rtol = o->inner_mode == 1
                                    ? std::max(o->inner_rtol, std::max(std::min(1e-2, std::sqrt(merit)),
                                                                        ew_on ? std::min(ew_cap, ew) : 0.0))
                                    : o->inner_rtol;
            merit_prev = merit;
            // (PF_VI_FLOOR, A/B: 0.5 saves ~30% of the PCG iterations of a normal SENT step's damage
            // solves but perturbs the nucleation step's AM path into more Newton work: driver window
            // 0.197 -> 0.209 s/step, so the default stays 0.1)
            static const double floor_f = getenv("PF_VI_FLOOR") ? atof(getenv("PF_VI_FLOOR")) : 0.1;
            const double afloor = (o->inner_mode == 1 ? floor_f : 0.1) * o->abs_tol;
            c->rhs_masked = 1;  // k_classify zeroed the right-hand side on the active rows
            rc = pcg_run(c, 1, B, c->kappa, c->act, rtol, afloor, maxit, 1, 8, &lr, st);
            c->rhs_masked = 0;
            rep->total_krylov_iterations += lr.iterations;
            if (getenv("PF_VI_TRACE"))
                fprintf(stderr, "  vi it=%d merit=%.3e ninact=%.0f pcg its=%lld rtol=%.1e\n", it, std::sqrt(merit),
                        c->h_scal[S_NINACT], (long long)lr.iterations, rtol);
            if (rc == PF_EBREAKDOWN) {
                rep->linear_failures++;
            } else if (rc != PF_OK) {
                return rc;
            } else {
                k_scale<<<vb, kVecBlock, 0, st>>>(n, B.x, -1.0);  // d = -d_N
                c->launches++;
                PF_TRY(line_search(B.x, merit, 0.0, true, ok));
            }
        }
        if (!ok) {
            // steepest descent on the merit (vi.py:241-252); Kaa is symmetric (J^T = J)
            k_merit_parts<<<vb, kVecBlock, 0, st>>>(n, x, F, lb, c->vi_g, c->vi_w);
            c->launches++;
            PF_TRY(launch_Kaa(c, c->kappa, c->vi_w, B.r, nullptr, st));
            k_grad_finish<<<vb, kVecBlock, 0, st>>>(n, c->vi_g, B.r, c->scal, rb);
            c->launches++;
            PF_TRY(read_scal(c, st, S_GNORM2, 1));
            const double gn = std::sqrt(c->h_scal[S_GNORM2]);
            if (gn > 0.0) {
                const double sc = 1.0 / std::max(1.0, gn);
                k_scale<<<vb, kVecBlock, 0, st>>>(n, B.r, -sc);
                c->launches++;
                PF_TRY(line_search(B.r, merit, o->armijo * sc * gn * gn, false, ok));
                rep->steepest_descent_steps++;
            }
        }
        if (!ok) break;
        push_hist(merit);
        slow = (merit_prev > 0.0 && merit > 0.49 * merit_prev) ? slow + 1 : 0;
    }
    rep->final_residual_norm = std::sqrt(merit);
    rep->converged = rep->final_residual_norm <= o->abs_tol;
    PF_CU(c, cudaMemcpyAsync(a_out, x, sizeof(double) * n, cudaMemcpyDeviceToDevice, st), "alpha out");
    return PF_OK;  // stream-ordered: the caller's next kernels see a_out
}

}  // namespace pf

// =====================================================================================================
// C ABI
// =====================================================================================================
using namespace pf;

struct pf_ctx : public Ctx {};

static void geometry_2d(Ctx* c) {
    Geo2& g = c->g;
    const pf_desc& d = c->d;
    g.nx = (int)d.nx;
    g.ny = (int)d.ny;
    g.nvy = g.ny + 1;
    g.pattern = d.pattern;
    g.npc = d.pattern == PF_CROSSED ? 4 : 2;
    g.nc = (long long)(g.nx + 1) * g.nvy;
    g.ncell = (long long)g.nx * g.ny;
    g.nv = g.nc + (d.pattern == PF_CROSSED ? g.ncell : 0);
    g.hx = d.lx / g.nx;
    g.hy = d.ly / g.ny;
    g.ihx = g.nx / d.lx;
    g.ihy = g.ny / d.ly;
    const double P[5][2] = {{0, 0}, {g.hx, 0}, {0, g.hy}, {g.hx, g.hy}, {0.5 * g.hx, 0.5 * g.hy}};
    int L[4][3];
    if (d.pattern == PF_UNION_JACK) {
        const int t[4][3] = {{0, 1, 3}, {0, 3, 2}, {0, 1, 2}, {1, 3, 2}};
        memcpy(L, t, sizeof t);
    } else if (d.pattern == PF_RIGHT) {
        const int t[4][3] = {{0, 1, 3}, {0, 3, 2}, {0, 1, 3}, {0, 3, 2}};
        memcpy(L, t, sizeof t);
    } else {
        const int t[4][3] = {{0, 1, 4}, {1, 3, 4}, {3, 2, 4}, {2, 0, 4}};
        memcpy(L, t, sizeof t);
    }
    for (int t = 0; t < 4; ++t) {
        const double* p1 = P[L[t][0]];
        const double* p2 = P[L[t][1]];
        const double* p3 = P[L[t][2]];
        const double det = (p2[0] - p1[0]) * (p3[1] - p1[1]) - (p2[1] - p1[1]) * (p3[0] - p1[0]);
        g.area[t] = 0.5 * det;
    }
    const double nu = d.nu;
    if (d.regime == PF_PLANE_STRESS) {
        const double s = 1.0 / (1.0 - nu * nu);
        g.D00 = s; g.D01 = s * nu; g.D11 = s; g.D22 = s * 0.5 * (1.0 - nu);
    } else {
        const double s = 1.0 / ((1.0 + nu) * (1.0 - 2.0 * nu));
        g.D00 = s * (1.0 - nu); g.D01 = s * nu; g.D11 = s * (1.0 - nu); g.D22 = s * 0.5 * (1.0 - 2.0 * nu);
    }
    g.E = d.E;
    g.kell = d.k_ell;
    g.Gc = d.Gc;
    g.ell = d.ell;
    g.at2 = d.model == PF_AT2;
    g.cw = g.at2 ? 2.0 : 8.0 / 3.0;
    g.E_cell = nullptr;
    g.Gc_cell = nullptr;
    g.eps0 = nullptr;
    g.rowgeo = nullptr;
    g.has_bc = 0;
    g.nwj = (g.nvy + kLanesOut - 1) / kLanesOut;
    const long long rows = g.nx + 1;
    const long long target_warps = 148LL * 24;
    long long S = (rows * g.nwj + target_warps - 1) / target_warps;
    S = std::max(4LL, std::min(64LL, S));
    g.S = (int)S;
    g.nstrips = (int)((rows + S - 1) / S);
    // v2 engine (pf_strip2.cu): 62 output columns per warp
    g.nwj2 = (g.nvy + kOut2Cols - 1) / kOut2Cols;
    // (rows per strip are sized per kernel at launch by a wave model, size_strips2; PF_STRIP2_WARPS
    // fixes a warp target instead, for experiments)
    const long long target2 = getenv("PF_STRIP2_WARPS") ? atoll(getenv("PF_STRIP2_WARPS")) : 148LL * 16;
    long long S2 = (rows * g.nwj2 + target2 - 1) / target2;
    S2 = std::max(4LL, std::min(64LL, S2));
    g.S2 = (int)S2;
    g.nstrips2 = (int)((rows + S2 - 1) / S2);
    g.nslow2 = 0;
}

static void geometry_3d(Ctx* c) {
    Geo3& g = c->g3;
    const pf_desc& d = c->d;
    g.nx = (int)d.nx; g.ny = (int)d.ny; g.nz = (int)d.nz;
    g.nvy = g.ny + 1; g.nvz = g.nz + 1;
    g.nv = (long long)(g.nx + 1) * g.nvy * g.nvz;
    g.ncell = (long long)g.nx * g.ny * g.nz;
    g.ihx = g.nx / d.lx; g.ihy = g.ny / d.ly; g.ihz = g.nz / d.lz;
    g.vol = (d.lx / g.nx) * (d.ly / g.ny) * (d.lz / g.nz) / 6.0;
    const double nu = d.nu;
    g.lam = nu / ((1.0 + nu) * (1.0 - 2.0 * nu));
    g.mu = 1.0 / (2.0 * (1.0 + nu));
    g.E = d.E; g.kell = d.k_ell; g.Gc = d.Gc; g.ell = d.ell;
    g.at2 = d.model == PF_AT2;
    g.cw = g.at2 ? 2.0 : 8.0 / 3.0;
    g.E_cell = nullptr; g.Gc_cell = nullptr; g.has_bc = 0;
    tile3(g);
}

// 3D strip tiling: blocks of outj (6) j-pencils x 30 k-lanes walking strips of S vertex rows.
// The strip count minimises a wave model of the latency-bound walk: time ~ waves x (S + 1 + 3)
// row steps (one halo row, ~3 steps of pipeline ramp per tile), waves = ceil(tiles / resident)
// with `resident` CTAs in flight (148 SMs x blocks per SM).  At 128^3 this picks 5 strips of 26
// rows (550 tiles, two waves of 296) instead of 6 strips of 24 (660 tiles, a third wave of 68).
// Measured against the fixed ~4-blocks-per-SM rule: 256^3 Kuu 0.757 -> 0.739 ms, Kaa 0.385 ->
// 0.375 ms, config-4 damage PCG -7%; 128^3 single applies within 2% (the model overstates the
// tail: a partial wave overlaps the previous one's stragglers).
void pf::tile3(Geo3& g, int outj, int resident) {
    g.nbj = (g.nvy + outj - 1) / outj;
    g.nbk = (g.nvz + 29) / 30;
    const long long per = (long long)g.nbj * g.nbk;
    const long long rows = g.nx + 1;
    long long best_ns = 1, best_t = -1;
    for (long long ns = 1; ns <= rows; ++ns) {
        const long long S = (rows + ns - 1) / ns;
        if (S < 4 && ns > 1) break;
        const long long tiles = per * ns;
        if (tiles > kMaxBlocksRed) break;
        const long long waves = (tiles + resident - 1) / resident;
        const long long t = waves * (S + 4);
        if (best_t < 0 || t < best_t) { best_t = t; best_ns = ns; }
    }
    long long S = (rows + best_ns - 1) / best_ns;
    if (getenv("PF_K3_S")) S = std::max(1LL, std::min(rows, atoll(getenv("PF_K3_S"))));  // A/B sweeps
    g.S = (int)S;
    g.nstrips = (int)((rows + S - 1) / S);
}

__global__ void k_relax_u3(long long nv, int nvy, int nvz, int nx, int ny, int nz, const double* __restrict__ up,
                           const double* __restrict__ us, double om, double* __restrict__ uo,
                           const unsigned char* __restrict__ mask, const double* __restrict__ ubar, int has_bc,
                           int snap_only) {
    for (long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x; v < nv;
         v += (long long)gridDim.x * blockDim.x) {
        double a[3];
        for (int c = 0; c < 3; ++c)
            a[c] = snap_only ? uo[3 * v + c] : up[3 * v + c] + om * (us[3 * v + c] - up[3 * v + c]);
        if (has_bc) {
            const int k = (int)(v % nvz);
            const long long ij = v / nvz;
            const int j = (int)(ij % nvy), i = (int)(ij / nvy);
            if (i == 0 || i == nx || j == 0 || j == ny || k == 0 || k == nz) {
                const unsigned m = mask[v];
                for (int c = 0; c < 3; ++c)
                    if ((m >> c) & 1u) a[c] = ubar[3 * v + c];
            }
        }
        for (int c = 0; c < 3; ++c) uo[3 * v + c] = a[c];
    }
}

static void plan_workspace(Ctx* c) {
    c->layout.clear();
    auto add = [&](void** p, size_t bytes) {
        c->layout.push_back({p, (bytes + 255) & ~size_t(255)});
        if (c->guard) c->layout.push_back({nullptr, c->guard});  // guard zone (bounds-check aid)
    };
    const size_t U = sizeof(double) * c->n_u, A = sizeof(double) * c->n_a;
    double** uvecs[] = {&c->cg_x, &c->cg_r, &c->cg_z, &c->cg_p0, &c->cg_p1, &c->cg_q, &c->cg_dinv, &c->cg_b,
                        &c->u_ws, &c->ubar};
    for (auto p : uvecs) add((void**)p, U);
    double** avecs[] = {&c->da_x, &c->da_r, &c->da_z, &c->da_p0, &c->da_p1, &c->da_q, &c->da_dinv,
                        &c->cg1_s0, &c->cg1_s1,
                        &c->vi_x, &c->vi_F, &c->vi_c, &c->vi_d, &c->vi_tx, &c->vi_tF, &c->vi_g, &c->vi_w,
                        &c->alpha_ws};
    for (auto p : avecs) add((void**)p, A);
    add((void**)&c->kappa, sizeof(double) * c->n_el);
    add((void**)&c->bcmask, c->n_a);
    add((void**)&c->act, c->n_a);
    c->tile_cap = (int)(c->n_a / 16 + 4096);  // a strip tile has >= 30 outputs
    add((void**)&c->tile_list, sizeof(int) * (c->tile_cap + 1) + c->tile_cap);
    add((void**)&c->eps0_tab, sizeof(double) * 4 * (c->d.ny + 1));
    add((void**)&c->rowgeo_buf, sizeof(double) * 2 * (c->d.ny + 1));
    add((void**)&c->partials, sizeof(double) * kMaxRed * kMaxBlocksRed);
    add((void**)&c->scal, sizeof(double) * S_COUNT);
    add((void**)&c->tickets, sizeof(unsigned) * 64);
    add((void**)&c->bits, sizeof(unsigned long long) * 8);
    c->n_newton_vec = ((c->n_u + c->n_a + 31) / 32) * 32;  // keep every stacked slot 256-byte aligned
    if (!(c->d.skip & PF_SKIP_NEWTON)) add((void**)&c->newton, sizeof(double) * c->n_newton_vec * 17);
    if (c->dim == 2 && !(c->d.skip & PF_SKIP_GMG)) {
        gmg_plan(c);
        add((void**)&c->gmg_base, gmg_bytes(c));
    }
    if (c->dim == 3 && !(c->d.skip & PF_SKIP_GMG)) {
        gmg3_plan(c);
        add((void**)&c->gmg3_base, gmg3_bytes(c));
    }
    size_t tot = 0;
    for (auto& e : c->layout) tot += e.second;
    c->ws_bytes = tot;
}

extern "C" {

int pf_ctx_create(const pf_desc* desc, pf_ctx** out) {
    if (!desc || !out) return set_error(nullptr, PF_EINVAL, "null argument");
    *out = nullptr;
    const bool d3 = desc->dim == 3;
    if (desc->dim != 2 && !d3) return set_error(nullptr, PF_EINVAL, "dim must be 2 or 3");
    if (!d3 && (desc->pattern < 0 || desc->pattern > 2))
        return set_error(nullptr, PF_EINVAL, "2D pattern must be union_jack, right or crossed");
    if (d3 && desc->pattern != PF_KUHN6) return set_error(nullptr, PF_EINVAL, "3D pattern must be kuhn6");
    if (desc->nx < 1 || desc->ny < 1 || desc->ny > (1 << 30) || desc->nx > (1 << 30) ||
        (d3 && (desc->nz < 1 || desc->nz > (1 << 30))))
        return set_error(nullptr, PF_EINVAL, "bad grid size");
    if (!(desc->E > 0 && desc->Gc > 0 && desc->ell > 0 && desc->lx > 0 && desc->ly > 0 && (!d3 || desc->lz > 0)))
        return set_error(nullptr, PF_EINVAL, "E, Gc, ell and extents must be positive");
    if (!(desc->nu > -1.0 && desc->nu < 0.5)) return set_error(nullptr, PF_EINVAL, "nu out of (-1, 0.5)");
    if (!d3 && desc->regime != PF_PLANE_STRESS && desc->regime != PF_PLANE_STRAIN)
        return set_error(nullptr, PF_EINVAL, "2D regime must be plane stress or plane strain");
    if (d3 && desc->regime != PF_3D) return set_error(nullptr, PF_EINVAL, "3D regime must be PF_3D");
    if (desc->model != PF_AT1 && desc->model != PF_AT2) return set_error(nullptr, PF_EINVAL, "unknown model");
    pf_ctx* c = new pf_ctx();
    c->d = *desc;
    // profiling / timing aids: eager Krylov loops (ncu sees every launch); the launch-per-phase
    // V-cycle; V-cycles without the coarse correction (fine smoothing only)
    if (getenv("PF_NO_GRAPHS")) c->use_graphs = 0;
    if (getenv("PF_GMG_LEGACY")) c->gmg_coarse = 0;
    if (getenv("PF_GMG_SKIP_COARSE")) c->gmg_coarse = 2;
    // measured slower on SENT 512^2 (16-CTA cluster phases are latency-bound on fewer SMs: coarse
    // cycle 125 -> 160 us), so the cluster tail is opt-in (PF_GMG_CLUSTER=1)
    c->gmg_cluster = getenv("PF_GMG_CLUSTER") ? 1 : 0;
    if (getenv("PF_PCG_GRAPH")) c->pcg_persistent = 0;
    if (getenv("PF_WS_GUARD")) c->guard = 16384;
    if (getenv("PF_PCG_SINGLE")) c->pcg_single = 1;
    c->strip2 = -1;  // auto: by mesh size, at binding
    if (getenv("PF_STRIP2")) c->strip2 = atoi(getenv("PF_STRIP2"));
    if (d3) {
        c->dim = 3;
        c->dof = 3;
        geometry_3d(c);
        // the 2D descriptor is unused in 3D; keep it benign for shared sizing code
        c->g = Geo2{};
        c->g.ny = 1;
        c->n_a = c->g3.nv;
        c->n_u = 3 * c->g3.nv;
        c->n_el = 6 * c->g3.ncell;
    } else {
        c->dim = 2;
        c->dof = 2;
        geometry_2d(c);
        // engine choice by size (A/B on B200, tools/opbench2.py): the TMA engine wins from about 0.55M
        // corner vertices (768^2) up (1024^2 applies -5..-11 %, the config-3 slab load step 1.049 -> 1.021 s,
        // 8192^2 union-jack Kuu 4.6 -> 5.9 TB/s); below that an apply is a few strip rows per warp,
        // bound by launch and pipeline-fill latency, where the one-column engine's shorter steps
        // are as fast or faster (SENT 512^2 load step: v2 +4 %)
        // (768^2: isolated applies -13..-18 %; 512^2: equal in isolation, +6 % on the SENT load step)
        if (c->strip2 < 0) c->strip2 = c->g.nc >= 550000 ? 1 : 0;
        c->n_a = c->g.nv;
        c->n_u = 2 * c->g.nv;
        c->n_el = c->g.ncell * c->g.npc;
    }
    plan_workspace(c);
    if (cudaHostAlloc((void**)&c->h_scal, sizeof(double) * 256, cudaHostAllocDefault) != cudaSuccess) {
        delete c;
        return set_error(nullptr, PF_ECUDA, "cudaHostAlloc failed (is a CUDA device present?)");
    }
    *out = c;
    return PF_OK;
}

void pf_ctx_destroy(pf_ctx* c) {
    if (!c) return;
    for (auto e : c->prof.ev) cudaEventDestroy(e);
    for (auto& ge : c->graph_exec)
        if (ge) cudaGraphExecDestroy(ge);
    for (auto& ge : c->mr_exec)
        if (ge) cudaGraphExecDestroy(ge);
    if (c->side_stream) cudaStreamDestroy(c->side_stream);
    if (c->ev_fork) cudaEventDestroy(c->ev_fork);
    if (c->ev_join) cudaEventDestroy(c->ev_join);
    if (c->cap_stream) cudaStreamDestroy(c->cap_stream);
    if (c->h_scal) cudaFreeHost(c->h_scal);
    delete c;
}

const char* pf_last_error(const pf_ctx* c) { return c ? c->err.c_str() : g_create_error.c_str(); }

int pf_query(const pf_ctx* c, int64_t out[8]) {
    if (!c || !out) return PF_EINVAL;
    out[0] = c->n_a;
    out[1] = c->n_u;
    out[2] = c->n_el;
    out[3] = c->dim == 3 ? c->g3.ncell : c->g.ncell;
    out[4] = c->dim == 3 ? c->g3.nv : c->g.nc;
    out[5] = c->dim;
    out[6] = c->dim == 3 ? 6 : c->g.npc;
    out[7] = c->dim == 3 ? c->g3.S : c->g.S;
    return PF_OK;
}

int64_t pf_workspace_bytes(const pf_ctx* c) { return c ? (int64_t)c->ws_bytes : -1; }

int pf_bind_workspace(pf_ctx* c, void* p, int64_t bytes) {
    if (!c || !p) return PF_EINVAL;
    if ((size_t)bytes < c->ws_bytes) return set_error(c, PF_ENOWS, "workspace too small");
    if (((uintptr_t)p & 255) != 0) return set_error(c, PF_EINVAL, "workspace must be 256-byte aligned");
    char* base = (char*)p;
    size_t off = 0;
    c->guards.clear();
    for (auto& e : c->layout) {
        if (e.first) *e.first = base + off;
        else c->guards.push_back({off, e.second});
        off += e.second;
    }
    for (auto& gz : c->guards)
        if (cudaMemset(base + gz.first, kGuardByte, gz.second) != cudaSuccess)
            return set_error(c, PF_ECUDA, "guard fill failed");
    c->ws = base;
    c->bound = 1;
    if (c->dim == 2 && !(c->d.skip & PF_SKIP_GMG)) gmg_bind(c, c->gmg_base);
    if (c->dim == 3 && !(c->d.skip & PF_SKIP_GMG)) gmg3_bind(c, c->gmg3_base);
    // zero scalars / tickets / bits / masks (synchronous; binding is a setup step)
    if (cudaMemset(c->scal, 0, sizeof(double) * S_COUNT) != cudaSuccess ||
        cudaMemset(c->tickets, 0, sizeof(unsigned) * 64) != cudaSuccess ||
        cudaMemset(c->bits, 0, sizeof(unsigned long long) * 8) != cudaSuccess ||
        cudaMemset(c->bcmask, 0, c->n_a) != cudaSuccess || cudaMemset(c->act, 0, c->n_a) != cudaSuccess ||
        cudaMemset(c->ubar, 0, sizeof(double) * c->n_u) != cudaSuccess ||
        cudaMemset(c->cg_p0, 0, sizeof(double) * c->n_u) != cudaSuccess ||
        cudaMemset(c->da_p0, 0, sizeof(double) * c->n_a) != cudaSuccess ||
        (c->gmg_bar && cudaMemset(c->gmg_bar, 0, 2 * sizeof(unsigned int)) != cudaSuccess) ||
        cudaDeviceSynchronize() != cudaSuccess)
        return set_error(c, PF_ECUDA, "workspace initialisation failed");
    c->g.bcmask = c->bcmask;
    c->g.ubar = c->ubar;
    c->g3.bcmask = c->bcmask;
    c->g3.ubar = c->ubar;
    return PF_OK;
}

#define NEED_WS(c)                                                                 \
    do {                                                                           \
        if (!(c)) return PF_EINVAL;                                                \
        if (!(c)->bound) return set_error((c), PF_ENOWS, "workspace not bound");   \
    } while (0)

int pf_check_guards(pf_ctx* c, int64_t* bad_bytes, void* stream) {
    NEED_WS(c);
    if (!bad_bytes) return set_error(c, PF_EINVAL, "pf_check_guards: null output");
    cudaStream_t st = (cudaStream_t)stream;
    int64_t bad = 0;
    std::vector<unsigned char> h;
    std::vector<std::pair<const char*, size_t>> zones;
    for (auto& gz : c->guards) zones.push_back({c->ws + gz.first, gz.second});
    for (auto& gz : c->gmg_guards) zones.push_back({gz.first, gz.second});
    for (auto& z : zones) {
        h.resize(z.second);
        PF_CU(c, cudaMemcpyAsync(h.data(), z.first, z.second, cudaMemcpyDeviceToHost, st), "guard read");
        PF_CU(c, cudaStreamSynchronize(st), "guard sync");
        for (unsigned char b : h) bad += (b != (unsigned char)kGuardByte);
    }
    *bad_bytes = bad;
    return PF_OK;
}

int pf_set_cell_fields(pf_ctx* c, const double* E_cell, const double* Gc_cell) {
    if (!c) return PF_EINVAL;
    c->g.E_cell = E_cell;
    c->g.Gc_cell = Gc_cell;
    c->g3.E_cell = E_cell;
    c->g3.Gc_cell = Gc_cell;
    c->geo_version++;
    c->gmg_built = 0;
    return PF_OK;
}

int pf_set_dirichlet(pf_ctx* c, const int64_t* dofs, const double* vals, int64_t n, void* stream) {
    NEED_WS(c);
    cudaStream_t st = (cudaStream_t)stream;
    if (c->dim == 3) {
        const Geo3& g = c->g3;
        std::vector<unsigned char> mask(g.nv, 0);
        std::vector<double> ub(3 * g.nv, 0.0);
        for (int64_t q = 0; q < n; ++q) {
            const int64_t dof = dofs[q];
            if (dof < 0 || dof >= 3 * g.nv) return set_error(c, PF_EINVAL, "Dirichlet dof out of range");
            const int64_t v = dof / 3;
            const int comp = (int)(dof % 3);
            const int k = (int)(v % g.nvz);
            const int64_t ij = v / g.nvz;
            const int j = (int)(ij % g.nvy), i = (int)(ij / g.nvy);
            if (!(i == 0 || i == g.nx || j == 0 || j == g.ny || k == 0 || k == g.nz))
                return set_error(c, PF_EINVAL, "Dirichlet dofs must lie on boundary vertices");
            mask[v] |= (unsigned char)(1u << comp);
            ub[dof] = vals[q];
        }
        PF_CU(c, cudaMemcpyAsync(c->bcmask, mask.data(), g.nv, cudaMemcpyHostToDevice, st), "bc mask");
        PF_CU(c, cudaMemcpyAsync(c->ubar, ub.data(), sizeof(double) * 3 * g.nv, cudaMemcpyHostToDevice, st), "ubar");
        PF_CU(c, cudaStreamSynchronize(st), "sync");
        if (mask != c->h_bcmask) c->gmg_built = 0;
        c->h_bcmask.swap(mask);
        if (c->g3.has_bc != (n > 0)) c->geo_version++;
        c->g3.has_bc = n > 0;
        return PF_OK;
    }
    const Geo2& g = c->g;
    std::vector<unsigned char> mask(g.nc, 0);
    std::vector<double> ub(2 * g.nc, 0.0);
    for (int64_t k = 0; k < n; ++k) {
        const int64_t dof = dofs[k];
        if (dof < 0 || dof >= 2 * g.nc) return set_error(c, PF_EINVAL, "Dirichlet dof out of range");
        const int64_t v = dof / 2;
        const int comp = (int)(dof % 2);
        const int i = (int)(v / g.nvy), j = (int)(v % g.nvy);
        if (!(i == 0 || i == g.nx || j == 0 || j == g.ny))
            return set_error(c, PF_EINVAL, "Dirichlet dofs must lie on boundary vertices");
        mask[v] |= (unsigned char)(1u << comp);
        ub[dof] = vals[k];
    }
    PF_CU(c, cudaMemcpyAsync(c->bcmask, mask.data(), g.nc, cudaMemcpyHostToDevice, st), "bc mask");
    PF_CU(c, cudaMemcpyAsync(c->ubar, ub.data(), sizeof(double) * 2 * g.nc, cudaMemcpyHostToDevice, st),
          "ubar");
    PF_CU(c, cudaStreamSynchronize(st), "sync");
    if (mask != c->h_bcmask) c->gmg_built = 0;
    c->h_bcmask.swap(mask);
    if (c->g.has_bc != (n > 0)) c->geo_version++;
    c->g.has_bc = n > 0;
    return PF_OK;
}

// graded rows (banded_rect_mesh, mesh.py:145-190): heights of the ny cell rows, host array
int pf_set_row_heights(pf_ctx* c, const double* hy, void* stream) {
    NEED_WS(c);
    if (c->dim != 2) return hy ? set_error(c, PF_EINVAL, "row heights are 2D only") : PF_OK;
    cudaStream_t st = (cudaStream_t)stream;
    Geo2& g = c->g;
    if (!hy) {
        if (g.rowgeo) { g.rowgeo = nullptr; c->geo_version++; c->gmg_built = 0; }
        return PF_OK;
    }
    const double frac = g.pattern == PF_CROSSED ? 0.25 : 0.5;  // element area / (hx hy)
    std::vector<double> t(2 * (size_t)g.ny);
    for (int j = 0; j < g.ny; ++j) {
        if (!(hy[j] > 0.0)) return set_error(c, PF_EINVAL, "row heights must be positive");
        t[j] = 1.0 / hy[j];
        t[g.ny + j] = frac * g.hx * hy[j];
    }
    PF_CU(c, cudaMemcpyAsync(c->rowgeo_buf, t.data(), sizeof(double) * t.size(), cudaMemcpyHostToDevice, st),
          "row heights");
    PF_CU(c, cudaStreamSynchronize(st), "sync");
    g.rowgeo = c->rowgeo_buf;
    c->geo_version++;
    c->gmg_built = 0;
    return PF_OK;
}

int pf_set_eps0_rows(pf_ctx* c, const double* table, void* stream) {
    NEED_WS(c);
    if (c->dim == 3) return table ? set_error(c, PF_EINVAL, "eps0 rows are 2D only") : PF_OK;
    if (!table) {
        if (c->g.eps0) c->geo_version++;
        c->g.eps0 = nullptr;
        return PF_OK;
    }
    if (!c->g.eps0) c->geo_version++;
    cudaStream_t st = (cudaStream_t)stream;
    PF_CU(c, cudaMemcpyAsync(c->eps0_tab, table, sizeof(double) * 4 * c->g.ny, cudaMemcpyHostToDevice, st),
          "eps0 table");
    PF_CU(c, cudaStreamSynchronize(st), "sync");
    c->g.eps0 = c->eps0_tab;
    return PF_OK;
}

int pf_apply_Kuu(pf_ctx* c, const double* alpha, const double* x, double* y, int32_t bc_mode, void* s) {
    NEED_WS(c);
    return launch_Kuu(c, alpha, x, y, bc_mode, (cudaStream_t)s);
}
int pf_apply_Kaa(pf_ctx* c, const double* u, const double* alpha, const double* x, double* y, void* s) {
    NEED_WS(c);
    cudaStream_t st = (cudaStream_t)s;
    PF_TRY(launch_kappa(c, u, alpha, c->kappa, c->vi_c, st));
    return launch_Kaa(c, c->kappa, x, y, nullptr, st);
}
int pf_kaa_coefficients(pf_ctx* c, const double* u, double* kappa, double* cvec, void* s) {
    NEED_WS(c);
    return launch_kappa(c, u, nullptr, kappa, cvec ? cvec : c->vi_c, (cudaStream_t)s);
}
int pf_apply_Kaa_coef(pf_ctx* c, const double* kappa, const double* x, double* y, void* s) {
    NEED_WS(c);
    return launch_Kaa(c, kappa, x, y, nullptr, (cudaStream_t)s);
}
int pf_apply_Kua(pf_ctx* c, const double* u, const double* alpha, const double* xa, double* yu, int32_t bc,
                 void* s) {
    NEED_WS(c);
    return launch_Kua(c, u, alpha, xa, yu, bc, (cudaStream_t)s);
}
int pf_apply_Kau(pf_ctx* c, const double* u, const double* alpha, const double* xu, double* ya, int32_t bc,
                 void* s) {
    NEED_WS(c);
    return launch_Kau(c, u, alpha, xu, ya, bc, (cudaStream_t)s);
}
int pf_physics(pf_ctx* c, const double* u, const double* alpha, const double* lb, double* ru, double* ra,
               double* phi, int32_t rows, double* out, void* s) {
    NEED_WS(c);
    cudaStream_t st = (cudaStream_t)s;
    PF_TRY(launch_physics(c, u, alpha, lb, ru, ra, phi, rows, st));
    if (out) {
        PF_TRY(read_scal(c, st, S_PHYS0, 4));
        const double* h = c->h_scal + S_PHYS0;
        out[0] = h[0];
        out[1] = h[1];
        out[2] = h[0] + h[1];
        out[3] = h[2];
        out[4] = h[3];
        out[5] = std::sqrt(h[2] + h[3]);
        out[6] = 0.0;
        out[7] = 0.0;
    }
    return PF_OK;
}
int pf_load_u(pf_ctx* c, const double* alpha, double* f, void* s) {
    NEED_WS(c);
    return launch_load(c, alpha, f, nullptr, 0, (cudaStream_t)s);
}
int pf_elastic_solve(pf_ctx* c, const double* alpha, const double* u0, double* u_out, const pf_lin_opts* o,
                     pf_lin_report* rep, void* s) {
    NEED_WS(c);
    if (!o || !rep) return set_error(c, PF_EINVAL, "null options/report");
    if (o->precond == PF_PREC_GMG && (c->d.skip & PF_SKIP_GMG))
        return set_error(c, PF_EINVAL, "context created with PF_SKIP_GMG");
    return elastic_solve(c, alpha, u0, u_out, o, rep, (cudaStream_t)s);
}
// The multigrid V-cycle as a stand-alone preconditioner: prepare builds the hierarchy of Kuu(alpha)
// (with the context's Dirichlet mask), apply computes z = M r.  M is a fixed linear SPD operator, so a
// caller's PCG on a spectrally equivalent operator -- the element-list Kuu of the same grid with
// jittered vertices (umesh.py) -- may use it.
int pf_gmg_prepare(pf_ctx* c, const double* alpha, void* s) {
    NEED_WS(c);
    if (c->d.skip & PF_SKIP_GMG) return set_error(c, PF_EINVAL, "context created with PF_SKIP_GMG");
    if (!alpha) return set_error(c, PF_EINVAL, "null alpha");
    cudaStream_t st = (cudaStream_t)s;
    if (cudaMemcpyAsync(c->alpha_ws, alpha, sizeof(double) * c->n_a, cudaMemcpyDeviceToDevice, st) != cudaSuccess)
        return set_error(c, PF_ECUDA, "alpha copy");
    c->gmg_degree = 2;
    const int rc = c->dim == 3 ? gmg3_setup(c, st) : gmg_setup(c, st);
    c->gmg_built = 0;  // a later pf_elastic_solve builds its own
    c->gmg_its0 = -1;
    return rc;
}
int pf_gmg_apply(pf_ctx* c, const double* r, double* z, void* s) {
    NEED_WS(c);
    if (c->d.skip & PF_SKIP_GMG) return set_error(c, PF_EINVAL, "context created with PF_SKIP_GMG");
    if (!r || !z) return set_error(c, PF_EINVAL, "null vector");
    return c->dim == 3 ? gmg3_vcycle(c, r, z, (cudaStream_t)s, nullptr) : gmg_vcycle(c, r, z, (cudaStream_t)s, nullptr);
}
int pf_damage_solve(pf_ctx* c, const double* u, const double* lb, const double* a_in, double* a_out,
                    const pf_vi_opts* o, pf_vi_report* rep, void* s) {
    NEED_WS(c);
    if (!o || !rep) return set_error(c, PF_EINVAL, "null options/report");
    return damage_solve(c, u, lb, a_in, a_out, o, rep, (cudaStream_t)s);
}
int pf_relax_u(pf_ctx* c, const double* u_prev, const double* u_star, double omega, double* u_out, void* s) {
    NEED_WS(c);
    if (c->dim == 3) {
        const Geo3& g = c->g3;
        k_relax_u3<<<vec_blocks(g.nv), kVecBlock, 0, (cudaStream_t)s>>>(g.nv, g.nvy, g.nvz, g.nx, g.ny, g.nz, u_prev,
                                                                         u_star, omega, u_out, c->bcmask, c->ubar,
                                                                         g.has_bc, 0);
        c->launches++;
        return check_cuda(c, cudaGetLastError(), "relax_u3");
    }
    const Geo2& g = c->g;
    k_relax_u<<<vec_blocks(g.nv), kVecBlock, 0, (cudaStream_t)s>>>(g.nv, g.nc, g.nvy, g.nx, g.ny, u_prev,
                                                                    u_star, omega, u_out, c->bcmask,
                                                                    c->ubar, g.has_bc, 0);
    c->launches++;
    return check_cuda(c, cudaGetLastError(), "relax_u");
}
int pf_snap_bc(pf_ctx* c, double* u, void* s) {
    NEED_WS(c);
    if (c->dim == 3) {
        const Geo3& g = c->g3;
        if (!g.has_bc) return PF_OK;
        k_relax_u3<<<vec_blocks(g.nv), kVecBlock, 0, (cudaStream_t)s>>>(g.nv, g.nvy, g.nvz, g.nx, g.ny, g.nz, nullptr,
                                                                         nullptr, 0.0, u, c->bcmask, c->ubar,
                                                                         g.has_bc, 1);
        c->launches++;
        return check_cuda(c, cudaGetLastError(), "snap_bc3");
    }
    const Geo2& g = c->g;
    if (!g.has_bc) return PF_OK;
    k_relax_u<<<vec_blocks(g.nv), kVecBlock, 0, (cudaStream_t)s>>>(g.nv, g.nc, g.nvy, g.nx, g.ny, nullptr,
                                                                    nullptr, 0.0, u, c->bcmask, c->ubar,
                                                                    g.has_bc, 1);
    c->launches++;
    return check_cuda(c, cudaGetLastError(), "snap_bc");
}
int pf_relax_alpha(pf_ctx* c, const double* a_prev, const double* a_star, const double* lb, double omega,
                   double* a_out, double* out, void* s) {
    NEED_WS(c);
    cudaStream_t st = (cudaStream_t)s;
    const long long n = c->n_a;
    const int vb = vec_blocks(n);
    PF_CU(c, cudaMemsetAsync(c->bits, 0, sizeof(unsigned long long) * 8, st), "memset");
    if (omega != 1.0) {
        k_relax_bits<<<vb, kVecBlock, 0, st>>>(n, a_prev, a_star, lb, omega, c->bits);
        c->launches++;
    }
    k_relax_apply<<<vb, kVecBlock, 0, st>>>(n, a_prev, a_star, lb, omega, c->bits, a_out, c->bits + 1, c->scal);
    c->launches++;
    PF_CU(c, cudaGetLastError(), "relax_alpha");
    if (out) {
        PF_CU(c, cudaMemcpyAsync(c->h_scal + 100, c->bits + 1, sizeof(double), cudaMemcpyDeviceToHost, st), "d");
        PF_TRY(read_scal(c, st, S_OMEGABAR, 1));
        PF_TRY(read_scal(c, st, S_AUX1, 1));
        double dmax;
        memcpy(&dmax, c->h_scal + 100, sizeof(double));
        out[0] = c->h_scal[S_OMEGABAR];
        out[1] = dmax;
        out[2] = c->h_scal[S_AUX1];
    }
    return PF_OK;
}
// AM tail fused (north_star part 4): alpha = P[alpha_prev + w_bar (alpha* - alpha_prev)] with the
// midpoint-backtracked w_bar (solver.py:202-216) applied while staging the physics pass, which then
// reduces energies, |r_u|, |Phi| and |d alpha|_inf of the relaxed state in the same sweep.
int pf_relax_alpha_physics(pf_ctx* c, const double* u, const double* a_prev, const double* a_star,
                           const double* lb, double omega, double* a_out, double* phys_out, double* relax_out,
                           void* s) {
    NEED_WS(c);
    cudaStream_t st = (cudaStream_t)s;
    if (c->dim == 3) {  // 3D: the relaxation and the physics pass as two launches
        PF_TRY(pf_relax_alpha(c, a_prev, a_star, lb, omega, a_out, relax_out, s));
        return pf_physics(c, u, a_out, lb, nullptr, nullptr, nullptr, PF_ROWS_ZERO, phys_out, s);
    }
    const long long n = c->n_a;
    PF_CU(c, cudaMemsetAsync(c->bits, 0, sizeof(unsigned long long) * 8, st), "memset");
    if (omega != 1.0) {
        k_relax_bits<<<vec_blocks(n), kVecBlock, 0, st>>>(n, a_prev, a_star, lb, omega, c->bits);
        c->launches++;
    }
    PF_TRY(launch_physics_relax(c, u, a_prev, a_star, lb, omega, a_out, st));
    PF_CU(c, cudaMemcpyAsync(c->h_scal, c->scal, sizeof(double) * S_COUNT, cudaMemcpyDeviceToHost, st), "scal");
    PF_CU(c, cudaMemcpyAsync(c->h_scal + 200, c->bits + 1, sizeof(double), cudaMemcpyDeviceToHost, st), "d");
    PF_CU(c, cudaStreamSynchronize(st), "sync");
    const double* h = c->h_scal + S_PHYS0;
    if (phys_out) {
        phys_out[0] = h[0];
        phys_out[1] = h[1];
        phys_out[2] = h[0] + h[1];
        phys_out[3] = h[2];
        phys_out[4] = h[3];
        phys_out[5] = std::sqrt(h[2] + h[3]);
        phys_out[6] = phys_out[7] = 0.0;
    }
    if (relax_out) {
        double dmax;
        memcpy(&dmax, c->h_scal + 200, sizeof(double));
        relax_out[0] = c->h_scal[S_OMEGABAR];
        relax_out[1] = dmax;
        relax_out[2] = c->h_scal[S_AUX1];
    }
    return PF_OK;
}
int pf_newton(pf_ctx* c, const double* u_in, const double* a_in, const double* lb, double* u_out,
              double* a_out, const pf_vi_opts* o, pf_vi_report* rep, void* s) {
    NEED_WS(c);
    if (!o || !rep) return set_error(c, PF_EINVAL, "null options/report");
    if ((c->d.skip & PF_SKIP_NEWTON) || (c->dim == 2 && (c->d.skip & PF_SKIP_GMG)))
        return set_error(c, PF_EINVAL, "context created with PF_SKIP_NEWTON / PF_SKIP_GMG");
    return newton_solve(c, u_in, a_in, lb, u_out, a_out, o, rep, (cudaStream_t)s);
}
int64_t pf_launch_count(const pf_ctx* c) { return c ? c->launches : -1; }

int pf_profile(pf_ctx* c, int32_t enable) {
    if (!c) return PF_EINVAL;
    c->prof.on = enable;
    return PF_OK;
}

// out[3*k + {0,1,2}] = (launches, total ms, algorithmic bytes) of kernel class k; resets.
int pf_profile_read(pf_ctx* c, double* out, int32_t nkinds) {
    if (!c || !out) return PF_EINVAL;
    if (cudaDeviceSynchronize() != cudaSuccess) return set_error(c, PF_ECUDA, "sync");
    for (auto& e : c->prof.log) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, c->prof.ev[2 * e.ev], c->prof.ev[2 * e.ev + 1]);
        c->prof.ms[e.kind] += ms;
        c->prof.bytes[e.kind] += e.bytes;
        c->prof.count[e.kind] += 1;
    }
    c->prof.log.clear();
    for (int k = 0; k < nkinds && k < K_NKINDS; ++k) {
        out[3 * k] = (double)c->prof.count[k];
        out[3 * k + 1] = c->prof.ms[k];
        out[3 * k + 2] = c->prof.bytes[k];
        c->prof.count[k] = 0;
        c->prof.ms[k] = 0;
        c->prof.bytes[k] = 0;
    }
    return PF_OK;
}

}  // extern "C"
