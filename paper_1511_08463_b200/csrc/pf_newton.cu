// pf_newton.cu -- coupled (u, alpha) reduced-space active-set Newton (north-star part 5).
//
// Restates, on the device, rsls_solve (vi.py:187-264) applied to the stacked MCP of
// coupled_mcp (solver.py:274-300): x = [u; alpha], F = [r_u (Dirichlet rows u - ubar); r_alpha],
// J = [[Kuu_bc, Kua_bc], [Kua_bc^T, Kaa]], bounds (-inf, inf) on u and [alpha_lb, 1] on alpha.
// The inactive-block Newton system is solved with preconditioned MINRES (linalg.py:155-219,
// Paige-Saunders recurrence evaluated on the host from device dot products) and the symmetric
// multiplicative field split (linalg.py:398-430):
//     y1 = A^-1 r_u ; z = C^-1 (r_a - B^T y1) ; x_u = y1 - A^-1 B z
// with A^-1 = GMG-PCG and C^-1 = Jacobi-PCG on the inactive damage block, both to a tight
// relative tolerance (the reference's default inner solves are exact LU, linalg.py:438-443).
// Index extraction (extract_submatrix) is replaced by masks: active damage rows/columns are
// identity and every vector is zero there.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <ctime>

#include "pf_internal.cuh"

namespace pf {

constexpr int kNB = 256;
// Chebyshev interval top for the C block: power iteration approaches lambda_max from below, and a
// Chebyshev polynomial preconditioner turns indefinite for eigenvalues much above the interval
// (degree 12: ~5% above already flips its sign) -- so a wider margin than the reference's 1.1
// (measured: 1.1 stalled 3D Newton on config 4).
constexpr double kChebSafety = 1.5;

__global__ void k_ndot(long long n, const double* a, const double* b, double* s, int slot, RedBuf rb) {
    double acc[1] = {0.0};
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        acc[0] += a[i] * b[i];
    grid_reduce<1>(acc, rb, 8, [=](double* t) { s[slot] = t[0]; });
}
__global__ void k_nscale(long long n, double a, const double* x, double* y) {  // y = a x
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        y[i] = a * x[i];
}
__global__ void k_naxpy(long long n, double a, const double* x, double* y) {  // y += a x
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        y[i] += a * x[i];
}
// w = (v - oldeps w1 - delta w2) / gam ; x += phi w
__global__ void k_nminres_w(long long n, const double* v, const double* w1, const double* w2, double* w, double* x,
                            double oldeps, double delta, double gam, double phi) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const double wi = (v[i] - oldeps * w1[i] - delta * w2[i]) / gam;
        w[i] = wi;
        x[i] += phi * wi;
    }
}
// out_a = act ? 0 : (a - b)
__global__ void k_nsubmask(long long n, const double* a, const double* b, const unsigned char* act, double* out) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        out[i] = act[i] ? 0.0 : (a[i] - (b ? b[i] : 0.0));
}
// trial = [u + mu du ; clip(a + mu da, lb, 1)]
__global__ void k_ntrial(long long nu, long long na, const double* x, const double* d, double mu, const double* lb,
                         double* t) {
    const long long n = nu + na;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        double v = x[i] + mu * d[i];
        if (i >= nu) v = fmin(fmax(v, lb[i - nu]), 1.0);
        t[i] = v;
    }
}
// clip alpha into [lb, 1] and max |x| over the stacked vector
__global__ void k_nclip_max(long long nu, long long na, double* x, const double* lb, unsigned long long* xmax) {
    const long long n = nu + na;
    double m = 0.0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        double v = x[i];
        if (i >= nu) { v = fmin(fmax(v, lb[i - nu]), 1.0); x[i] = v; }
        m = fmax(m, fabs(v));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(PF_FULL, m, o));
    if ((threadIdx.x & 31) == 0 && m > 0.0) atomicMax(xmax, (unsigned long long)__double_as_longlong(m));
}
// steepest-descent gradient g = 2 (p phi + J (q phi)): u rows p = 0, q = 1 (free bounds)
__global__ void k_ngrad(long long nu, long long na, const double* pphi_a, const double* Jw, double* g) {
    const long long n = nu + na;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        g[i] = 2.0 * ((i >= nu ? pphi_a[i - nu] : 0.0) + Jw[i]);
}

// ---- fixed linear block preconditioners (inner_mode 1) ----
// y2 = D^-1 y (masked rows of dinv are 1), reduce |y2|^2 into s[slot]
__global__ void k_ndinv_dot(long long n, const double* dinv, const double* y, double* y2, double* s, int slot,
                            RedBuf rb) {
    double acc[1] = {0.0};
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const double v = dinv[i] * y[i];
        y2[i] = v;
        acc[0] += v * v;
    }
    grid_reduce<1>(acc, rb, 8, [=](double* t) { s[slot] = t[0]; });
}
// x = y / sqrt(s[slot])
__global__ void k_nnormalize(long long n, const double* y, double* x, const double* s, int slot) {
    const double inv = s[slot] > 0.0 ? 1.0 / sqrt(s[slot]) : 0.0;  // empty inactive block: x = 0
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        x[i] = y[i] * inv;
}
// power-iteration start: 1 on inactive rows, 0 on active rows
__global__ void k_nones(long long n, const unsigned char* act, double* x) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        x[i] = act[i] ? 0.0 : 1.0;
}
// Chebyshev on D^-1 C: r = b ; d = D^-1 r / theta ; x = d
__global__ void k_ncheb0(long long n, const double* dinv, const double* b, double* r, double* d, double* x,
                         double ith) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const double ri = b[i];
        const double di = dinv[i] * ri * ith;
        r[i] = ri;
        d[i] = di;
        x[i] = di;
    }
}
// r -= C d ; d = a d + b D^-1 r ; x += d
__global__ void k_nchebk(long long n, const double* dinv, const double* Cd, double* r, double* d, double* x,
                         double a, double b) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const double ri = r[i] - Cd[i];
        const double di = a * d[i] + b * dinv[i] * ri;
        r[i] = ri;
        d[i] = di;
        x[i] += di;
    }
}

// ---- device-resident MINRES (fixed block preconditioners, inner_mode 1/2) --------------------
// The Paige-Saunders recurrence of linalg.py:155-219 with every scalar in device memory and every
// vector in a fixed buffer (the host loop rotates buffer pointers; here the rotation is data
// movement fused into the vector passes), so one iteration is a fixed sequence of launches that a
// CUDA graph replays under a WHILE node: no host round trip per iteration.
constexpr int S_MR = 80;  // MINRES state slots
enum {
    MR_BETA = 0, MR_OLDB, MR_DBAR, MR_EPS, MR_PHIBAR, MR_CS, MR_SN, MR_TARGET, MR_IT, MR_MAXIT, MR_DONE,
    MR_FAIL, MR_ALFA, MR_BB, MR_OLDEPS, MR_DELTA, MR_GAM, MR_PHI, MR_TB, MR_TT
};
constexpr int S_CHEB = 100;  // Chebyshev table of the C block: [0] = 1/theta, [2k-1], [2k] = a_k, b_k
constexpr int kMaxChebDeg = 14;

// warm != 0: the target was set from |b|_M (k_mr_target) and the start-up residual is b - J x0
__global__ void k_mr_start(double* s, double rtol, double maxit, int warm) {
    double* m = s + S_MR;
    const double bb = m[MR_BB];
    const double b1 = bb > 0.0 ? sqrt(bb) : 0.0;
    m[MR_BETA] = b1; m[MR_OLDB] = 0.0; m[MR_DBAR] = 0.0; m[MR_EPS] = 0.0; m[MR_PHIBAR] = b1;
    m[MR_CS] = -1.0; m[MR_SN] = 0.0; m[MR_IT] = 0.0; m[MR_MAXIT] = maxit;
    if (!warm) m[MR_TARGET] = rtol * b1;
    m[MR_FAIL] = bb < 0.0 ? 1.0 : 0.0;
    m[MR_DONE] = (bb <= 0.0 || b1 <= m[MR_TARGET]) ? 1.0 : 0.0;
}
__global__ void k_mr_target(double* s, double rtol) {
    const double bb = s[S_MR + MR_BB];
    s[S_MR + MR_TARGET] = rtol * (bb > 0.0 ? sqrt(bb) : 0.0);
}
// x0 = previous solution with the currently active damage rows zeroed; r = b - t (t = J x0)
__global__ void k_mr_x0(long long nu, long long na, const double* __restrict__ dp, const unsigned char* __restrict__ act,
                        double* __restrict__ x) {
    const long long n = nu + na;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        x[i] = (i >= nu && act[i - nu]) ? 0.0 : dp[i];
}
// t.b and t.t for the least-squares scale of the warm start
__global__ void k_mr_dot2(long long n, const double* __restrict__ t, const double* __restrict__ b, double* s, RedBuf rb) {
    double acc[2] = {0.0, 0.0};
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const double ti = t[i];
        acc[0] += ti * b[i];
        acc[1] += ti * ti;
    }
    grid_reduce<2>(acc, rb, 8, [=](double* tt) { s[S_MR + MR_TB] = tt[0]; s[S_MR + MR_TT] = tt[1]; });
}
// x0 = g x ; r1 = r2 = b - g t with g = (t.b)/(t.t) (the best multiple of the previous solution)
__global__ void k_mr_r0(long long n, const double* __restrict__ b, const double* __restrict__ t, double* __restrict__ x,
                        double* __restrict__ r1, double* __restrict__ r2, const double* s) {
    double g = 1.0;  // s == null: x0 as given
    if (s) {
        const double tt = s[S_MR + MR_TT];
        g = tt > 0.0 ? s[S_MR + MR_TB] / tt : 0.0;
    }
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const double v = b[i] - g * t[i];
        x[i] *= g;
        r1[i] = v;
        r2[i] = v;
    }
}
// v = y / beta
__global__ void k_mr_v(long long n, const double* __restrict__ y, double* __restrict__ v, const double* s) {
    const double ib = 1.0 / s[S_MR + MR_BETA];
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        v[i] = y[i] * ib;
}
// t -= (beta / oldb) r1 (not on the first iteration) ; alfa = v . t
__global__ void k_mr_a(long long n, double* __restrict__ t, const double* __restrict__ r1, const double* __restrict__ v,
                       double* s, RedBuf rb) {
    const double* m = s + S_MR;
    const double f = m[MR_IT] >= 1.0 ? m[MR_BETA] / m[MR_OLDB] : 0.0;
    double acc[1] = {0.0};
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const double ti = t[i] - f * r1[i];
        t[i] = ti;
        acc[0] += v[i] * ti;
    }
    grid_reduce<1>(acc, rb, 8, [=](double* tt) { s[S_MR + MR_ALFA] = tt[0]; });
}
// r1 <- r2 ; r2 <- t - (alfa / beta) r2
__global__ void k_mr_b(long long n, const double* __restrict__ t, double* __restrict__ r1, double* __restrict__ r2,
                       const double* s) {
    const double f = s[S_MR + MR_ALFA] / s[S_MR + MR_BETA];
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const double a = r2[i];
        r1[i] = a;
        r2[i] = t[i] - f * a;
    }
}
// bb = r2 . y
__global__ void k_mr_dot(long long n, const double* __restrict__ a, const double* __restrict__ b, double* s,
                         RedBuf rb) {
    double acc[1] = {0.0};
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        acc[0] += a[i] * b[i];
    grid_reduce<1>(acc, rb, 8, [=](double* tt) { s[S_MR + MR_BB] = tt[0]; });
}
// the Givens rotation of one iteration (the host loop's scalar block, minres above)
__global__ void k_mr_rot(double* s) {
    double* m = s + S_MR;
    const double bb = m[MR_BB];
    if (bb < 0.0) { m[MR_FAIL] = 1.0; m[MR_DONE] = 1.0; return; }
    const double alfa = m[MR_ALFA];
    m[MR_OLDB] = m[MR_BETA];
    const double beta = sqrt(bb);
    m[MR_BETA] = beta;
    const double cs = m[MR_CS], sn = m[MR_SN], dbar = m[MR_DBAR];
    m[MR_OLDEPS] = m[MR_EPS];
    m[MR_DELTA] = cs * dbar + sn * alfa;
    const double gbar = sn * dbar - cs * alfa;
    m[MR_EPS] = sn * beta;
    m[MR_DBAR] = -cs * beta;
    const double gam = fmax(hypot(gbar, beta), 2.220446049250313e-16);
    m[MR_GAM] = gam;
    const double csn = gbar / gam, snn = beta / gam;
    m[MR_CS] = csn;
    m[MR_SN] = snn;
    m[MR_PHI] = csn * m[MR_PHIBAR];
    m[MR_PHIBAR] = snn * m[MR_PHIBAR];
    m[MR_IT] += 1.0;
    m[MR_DONE] = (m[MR_PHIBAR] <= m[MR_TARGET] || m[MR_IT] >= m[MR_MAXIT]) ? 1.0 : 0.0;
}
// (w1, w2) <- (w2, w) ; w = (v - oldeps w1 - delta w2) / gam ; x += phi w   [wa = w2, wb = w]
__global__ void k_mr_w(long long n, const double* __restrict__ v, double* __restrict__ wa, double* __restrict__ wb,
                       double* __restrict__ x, const double* s) {
    const double* m = s + S_MR;
    if (m[MR_FAIL] != 0.0) return;
    const double oe = m[MR_OLDEPS], de = m[MR_DELTA], ig = 1.0 / m[MR_GAM], ph = m[MR_PHI];
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const double a = wa[i], b = wb[i];
        const double w = (v[i] - oe * a - de * b) * ig;
        wa[i] = b;
        wb[i] = w;
        x[i] += ph * w;
    }
}
__global__ void k_mr_cond(cudaGraphConditionalHandle h, const double* s) {
    if (threadIdx.x == 0) cudaGraphSetConditional(h, s[S_MR + MR_DONE] == 0.0 ? 1u : 0u);
}
// Chebyshev coefficients of the C block on the device (from |D^-1 C x|^2 in S_AUX1, lambda_C)
__global__ void k_cheb_table(double* s, int deg, double safety) {
    double lmax = sqrt(s[S_AUX1]);
    if (!(lmax > 0.0) || !isfinite(lmax)) lmax = 1.0;
    const double hi = safety * lmax, lo = hi / 30.0;
    const double theta = 0.5 * (hi + lo), delta = 0.5 * (hi - lo), sigma = theta / delta;
    double* t = s + S_CHEB;
    t[0] = 1.0 / theta;
    double rho = 1.0 / sigma;
    for (int k = 1; k < deg; ++k) {
        const double rn = 1.0 / (2.0 * sigma - rho);
        t[2 * k - 1] = rn * rho;
        t[2 * k] = 2.0 * rn / delta;
        rho = rn;
    }
}
__global__ void k_ncheb0_d(long long n, const double* dinv, const double* b, double* r, double* d, double* x,
                           const double* s, const unsigned char* bmask) {
    const double ith = s[S_CHEB];
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const double ri = (bmask && bmask[i]) ? 0.0 : b[i];
        const double di = dinv[i] * ri * ith;
        r[i] = ri;
        d[i] = di;
        x[i] = di;
    }
}
__global__ void k_nchebk_d(long long n, const double* dinv, const double* Cd, double* r, double* d, double* x,
                           const double* s, int k) {
    const double a = s[S_CHEB + 2 * k - 1], b = s[S_CHEB + 2 * k];
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const double ri = r[i] - Cd[i];
        const double di = a * d[i] + b * dinv[i] * ri;
        r[i] = ri;
        d[i] = di;
        x[i] += di;
    }
}

static int nblocks(long long n) { return (int)std::max(1LL, std::min((n + kNB - 1) / kNB, 148LL * 8)); }

#define NTRY(x)                        \
    do {                               \
        int _rc = (x);                 \
        if (_rc != PF_OK) return _rc;  \
    } while (0)
#define NCU(c, x, w)                                                        \
    do {                                                                    \
        cudaError_t _e = (x);                                               \
        if (_e != cudaSuccess) return check_cuda((c), _e, (w));             \
    } while (0)

struct NewtonWs {
    long long nu, na, n;
    double *X, *TX, *FX, *TF, *D, *RHS, *R1, *R2, *Y, *V, *W, *W1, *W2, *TMP, *PP, *G;
    double* DP;        // the previous Newton iteration's MINRES solution (warm start)
    bool dp_valid = false;
};

static int ndot(Ctx* c, long long n, const double* a, const double* b, int slot, double& out, cudaStream_t st) {
    const RedBuf rb{c->partials, c->tickets, c->scal};
    k_ndot<<<nblocks(n), kNB, 0, st>>>(n, a, b, c->scal, slot, rb);
    c->launches++;
    NTRY(read_scal(c, st, slot, 1));
    out = c->h_scal[slot];
    return PF_OK;
}

// physics pass at stacked point x: F (rows VALUE) and merit |Phi|^2 (u rows free)
static int eval_F(Ctx* c, const NewtonWs& w, const double* x, double* F, const double* lb, double& merit,
                  cudaStream_t st) {
    NTRY(launch_physics(c, x, x + w.nu, lb, F, F + w.nu, nullptr, PF_ROWS_VALUE, st));
    NTRY(read_scal(c, st, S_PHYS0, 4));
    merit = c->h_scal[S_PHYS0 + 2] + c->h_scal[S_PHYS0 + 3];
    return PF_OK;
}

// A^-1 b (GMG-PCG, hierarchy already set up for the current alpha) -> out
// inner block solves: to rtol, or (budget > 0) a fixed budget of `budget` PCG iterations at
// rtol 1e-12 (fieldsplit_inner = "cg", inner_cg linalg.py:446-456)
static int solve_A(Ctx* c, const double* b, double* out, double rtol, int budget, long long& its,
                   cudaStream_t st) {
    PcgBuffers B{c->cg_x, c->cg_r, c->cg_z, c->cg_p0, c->cg_p1, c->cg_q, c->cg_dinv, const_cast<double*>(b), c->n_u};
    // pcg_run reads |b|^2 from S_AUX0
    double bb;
    NTRY(ndot(c, c->n_u, b, b, S_AUX0, bb, st));
    pf_lin_report rep{};
    int rc = pcg_run(c, 2, B, c->alpha_ws, nullptr, budget > 0 ? 1e-12 : rtol, 0.0,
                     budget > 0 ? budget : 10 * c->n_u, 1, 2, &rep, st);
    its += rep.iterations;
    if (rc != PF_OK) return set_error(c, PF_EINNER, "inner solve on block 'A' failed: " + c->err);
    NCU(c, cudaMemcpyAsync(out, c->cg_x, sizeof(double) * c->n_u, cudaMemcpyDeviceToDevice, st), "copy");
    return PF_OK;
}
// C^-1 b on the inactive damage block (Jacobi-PCG, kappa / act / dinv ready) -> out
static int solve_C(Ctx* c, const double* b, double* out, double rtol, int budget, long long& its,
                   cudaStream_t st) {
    PcgBuffers B{c->da_x, c->da_r, c->da_z, c->da_p0, c->da_p1, c->da_q, c->da_dinv, const_cast<double*>(b), c->n_a};
    double bb;
    NTRY(ndot(c, c->n_a, b, b, S_AUX0, bb, st));
    pf_lin_report rep{};
    int rc = pcg_run(c, 1, B, c->kappa, c->act, budget > 0 ? 1e-12 : rtol, 0.0,
                     budget > 0 ? budget : 10 * c->n_a, 1, 8, &rep, st);
    its += rep.iterations;
    if (rc != PF_OK) return set_error(c, PF_EINNER, "inner solve on block 'C' failed: " + c->err);
    NCU(c, cudaMemcpyAsync(out, c->da_x, sizeof(double) * c->n_a, cudaMemcpyDeviceToDevice, st), "copy");
    return PF_OK;
}

// lambda_max of D^-1 C on the inactive damage block: 30 power iterations from a deterministic start
// vector (ChebyshevPreconditioner, linalg.py:347-358), normalised on the device (no host polls).
static int lambda_C(Ctx* c, double& lmax, cudaStream_t st) {
    const long long n = c->n_a;
    const int nb = nblocks(n);
    const RedBuf rb{c->partials, c->tickets, c->scal};
    double *x = c->da_x, *y = c->da_q, *y2 = c->da_z;
    k_nones<<<nb, kNB, 0, st>>>(n, c->act, x);
    c->launches++;
    for (int it = 0; it < 30; ++it) {
        NTRY(launch_Kaa(c, c->kappa, x, y, c->act, st));
        k_ndinv_dot<<<nb, kNB, 0, st>>>(n, c->da_dinv, y, y2, c->scal, S_AUX1, rb);
        k_nnormalize<<<nb, kNB, 0, st>>>(n, y2, x, c->scal, S_AUX1);
        c->launches += 2;
    }
    NTRY(read_scal(c, st, S_AUX1, 1));
    lmax = std::sqrt(c->h_scal[S_AUX1]);  // |D^-1 C x| for the unit iterate x
    if (!std::isfinite(lmax)) return set_error(c, PF_EINNER, "field split: damage-block spectrum estimate failed");
    if (lmax == 0.0) lmax = 1.0;  // no inactive damage rows: C^-1 acts on zero vectors only
    return PF_OK;
}
// x = p(D^-1 C) b: `deg` Chebyshev steps on [lmax/30, 1.1 lmax] from x = 0 (a fixed SPD operator)
static int cheb_C(Ctx* c, const double* b, double* x, double lmax, int deg, long long& its, cudaStream_t st) {
    const long long n = c->n_a;
    const int nb = nblocks(n);
    const double hi = kChebSafety * lmax, lo = hi / 30.0;
    const double theta = 0.5 * (hi + lo), delta = 0.5 * (hi - lo), sigma = theta / delta;
    double *r = c->da_r, *d = c->da_p0, *Cd = c->da_q;
    k_ncheb0<<<nb, kNB, 0, st>>>(n, c->da_dinv, b, r, d, x, 1.0 / theta);
    c->launches++;
    double rho = 1.0 / sigma;
    for (int k = 1; k < deg; ++k) {
        const double rn = 1.0 / (2.0 * sigma - rho);
        NTRY(launch_Kaa(c, c->kappa, d, Cd, c->act, st));
        k_nchebk<<<nb, kNB, 0, st>>>(n, c->da_dinv, Cd, r, d, x, rn * rho, 2.0 * rn / delta);
        c->launches++;
        rho = rn;
    }
    its += deg;
    return PF_OK;
}
// the same polynomial with its coefficients read from the device table (graph-capturable); the
// start-up applies the active mask to the raw right-hand side (bmask: rows of b to zero, or null).
// PF_CHEB_FUSED=1 (2D): each step as one strip pass whose epilogue does the update at the owner
// (launch_Kaa_cheb) -- measured slower beside the V-cycle on the side stream (stalled SENT Newton
// phase 0.78 -> 0.82 s): the small separate update kernels interleave with the V-cycle phases.
static int cheb_C_dev(Ctx* c, const double* b, double* x, int deg, long long& its, cudaStream_t st,
                      const unsigned char* bmask = nullptr) {
    const long long n = c->n_a;
    const int nb = nblocks(n);
    double *r = c->da_r, *d = c->da_p0, *Cd = c->da_q;
    k_ncheb0_d<<<nb, kNB, 0, st>>>(n, c->da_dinv, b, r, d, x, c->scal, bmask);
    c->launches++;
    if (c->dim == 2 && getenv("PF_CHEB_FUSED")) {
        double* dn = Cd;
        for (int k = 1; k < deg; ++k) {
            NTRY(launch_Kaa_cheb(c, c->kappa, d, c->act, r, dn, x, c->da_dinv, c->scal + S_CHEB, k, st));
            std::swap(d, dn);
        }
        its += deg;
        return PF_OK;
    }
    for (int k = 1; k < deg; ++k) {
        NTRY(launch_Kaa(c, c->kappa, d, Cd, c->act, st));
        k_nchebk_d<<<nb, kNB, 0, st>>>(n, c->da_dinv, Cd, r, d, x, c->scal, k);
        c->launches++;
    }
    its += deg;
    return PF_OK;
}
// x = one multigrid V-cycle applied to b (hierarchy of the current alpha; a fixed SPD operator)
static int vcycle_A(Ctx* c, const double* b, double* x, long long& its, cudaStream_t st) {
    if (c->dim == 3) NTRY(gmg3_vcycle(c, b, x, st, nullptr));
    else NTRY(gmg_vcycle(c, b, x, st, nullptr, false, -1, nullptr));
    its += 1;
    return PF_OK;
}

// y = P^-1 r (symmetric multiplicative field split, linalg.py:424-430)
struct InnerMg {  // inner_mode 1 (multiplicative) / 2 (additive)
    bool on = false;
    bool additive = false;
    bool dev = false;  // Chebyshev coefficients from the device table (k_cheb_table)
    int deg = 12;
    double lmax = 0.0;
};
static int fieldsplit(Ctx* c, const NewtonWs& w, const double* r, double* y, const double* u, const double* alpha,
                      double inner_rtol, int budget, long long& its, cudaStream_t st, const InnerMg& mg) {
    const long long nu = w.nu, na = w.na;
    double* y1 = y;              // u part of y
    double* z = y + nu;          // alpha part of y
    if (mg.on && mg.additive && mg.dev && !getenv("PF_NEWTON_NO_FORK")) {
        // block-diagonal split, the two blocks concurrently: the Chebyshev polynomial of the C block
        // runs on a side stream beside the V-cycle (whose coarse levels are latency-bound and leave
        // most of the machine idle); fork/join by events, also inside the graph capture
        if (!c->side_stream) {
            NCU(c, cudaStreamCreateWithFlags(&c->side_stream, cudaStreamNonBlocking), "side stream");
            NCU(c, cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming), "event");
            NCU(c, cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming), "event");
        }
        cudaStream_t sd = c->side_stream;
        NCU(c, cudaEventRecord(c->ev_fork, st), "fork");
        NCU(c, cudaStreamWaitEvent(sd, c->ev_fork, 0), "fork wait");
        NTRY(cheb_C_dev(c, r + nu, z, mg.deg, its, sd, c->act));  // (active rows of r zeroed)
        NCU(c, cudaEventRecord(c->ev_join, sd), "join");
        NTRY(vcycle_A(c, r, y1, its, st));
        NCU(c, cudaStreamWaitEvent(st, c->ev_join, 0), "join wait");
        return PF_OK;
    }
    if (mg.on && mg.additive) {  // block-diagonal field split: P^-1 = diag(V-cycle, Chebyshev)
        NTRY(vcycle_A(c, r, y1, its, st));
        k_nsubmask<<<nblocks(na), kNB, 0, st>>>(na, r + nu, nullptr, c->act, w.TMP + nu);
        c->launches++;
        NTRY(mg.dev ? cheb_C_dev(c, w.TMP + nu, z, mg.deg, its, st) : cheb_C(c, w.TMP + nu, z, mg.lmax, mg.deg, its, st));
        return PF_OK;
    }
    if (mg.on) {
        NTRY(vcycle_A(c, r, y1, its, st));
        NTRY(launch_Kau(c, u, alpha, y1, w.TMP + nu, PF_BC_ELIMINATE, st));            // B^T y1
        k_nsubmask<<<nblocks(na), kNB, 0, st>>>(na, r + nu, w.TMP + nu, c->act, w.TMP + nu);
        c->launches++;
        NTRY(mg.dev ? cheb_C_dev(c, w.TMP + nu, z, mg.deg, its, st) : cheb_C(c, w.TMP + nu, z, mg.lmax, mg.deg, its, st));
        NTRY(launch_Kua(c, u, alpha, z, w.TMP, PF_BC_ELIMINATE, st));                   // B z
        NTRY(vcycle_A(c, w.TMP, w.G, its, st));
        k_naxpy<<<nblocks(nu), kNB, 0, st>>>(nu, -1.0, w.G, y1);
        c->launches++;
        return PF_OK;
    }
    NTRY(solve_A(c, r, y1, inner_rtol, budget, its, st));
    NTRY(launch_Kau(c, u, alpha, y1, w.TMP + nu, PF_BC_ELIMINATE, st));            // B^T y1
    k_nsubmask<<<nblocks(na), kNB, 0, st>>>(na, r + nu, w.TMP + nu, c->act, w.TMP + nu);
    c->launches++;
    NTRY(solve_C(c, w.TMP + nu, z, inner_rtol, budget, its, st));
    NTRY(launch_Kua(c, u, alpha, z, w.TMP, PF_BC_ELIMINATE, st));                   // B z
    NTRY(solve_A(c, w.TMP, w.TMP, inner_rtol, budget, its, st));
    k_naxpy<<<nblocks(nu), kNB, 0, st>>>(nu, -1.0, w.TMP, y1);
    c->launches++;
    return PF_OK;
}

// MINRES on the masked inactive block J_NN d = rhs (x0 = 0); returns the iterations.
static int minres(Ctx* c, NewtonWs& w, const double* u, const double* alpha, const double* rhs, double* x,
                  double rtol, long long maxit, double inner_rtol, int budget, long long& kits, bool& converged,
                  cudaStream_t st, const InnerMg& mg) {
    const long long n = w.n, nu = w.nu;
    auto op = [&](const double* v, double* out) {
        return launch_jac(c, u, alpha, v, v + nu, out, out + nu, c->act, st);
    };
    NCU(c, cudaMemsetAsync(x, 0, sizeof(double) * n, st), "memset");
    NCU(c, cudaMemcpyAsync(w.R1, rhs, sizeof(double) * n, cudaMemcpyDeviceToDevice, st), "copy");
    double *r1 = w.R1, *r2 = w.R2, *y = w.Y, *v = w.V, *ww = w.W, *w1 = w.W1, *w2 = w.W2;
    NTRY(fieldsplit(c, w, r1, y, u, alpha, inner_rtol, budget, kits, st, mg));
    double beta1;
    NTRY(ndot(c, n, r1, y, S_AUX1, beta1, st));
    if (beta1 < 0.0) return set_error(c, PF_EBREAKDOWN, "minres: preconditioner not SPD");
    beta1 = std::sqrt(beta1);
    converged = true;
    if (beta1 == 0.0) return PF_OK;
    const double target = rtol * beta1;
    double oldb = 0.0, beta = beta1, dbar = 0.0, epsln = 0.0, phibar = beta1, cs = -1.0, sn = 0.0;
    NCU(c, cudaMemsetAsync(ww, 0, sizeof(double) * n, st), "memset");
    NCU(c, cudaMemsetAsync(w2, 0, sizeof(double) * n, st), "memset");
    NCU(c, cudaMemcpyAsync(r2, r1, sizeof(double) * n, cudaMemcpyDeviceToDevice, st), "copy");
    long long it = 0;
    const int nb = nblocks(n);
    while (it < maxit && phibar > target) {
        ++it;
        k_nscale<<<nb, kNB, 0, st>>>(n, 1.0 / beta, y, v);
        NTRY(op(v, y));
        if (it >= 2) k_naxpy<<<nb, kNB, 0, st>>>(n, -(beta / oldb), r1, y);
        double alfa;
        NTRY(ndot(c, n, v, y, S_AUX1, alfa, st));
        k_naxpy<<<nb, kNB, 0, st>>>(n, -(alfa / beta), r2, y);
        c->launches += 3;
        // r1 <- r2 ; r2 <- y ; y <- M r2 (into the old r1 buffer)
        double* old_r1 = r1;
        r1 = r2;
        r2 = y;
        y = old_r1;
        NTRY(fieldsplit(c, w, r2, y, u, alpha, inner_rtol, budget, kits, st, mg));
        oldb = beta;
        double bb;
        NTRY(ndot(c, n, r2, y, S_AUX1, bb, st));
        if (bb < 0.0) return set_error(c, PF_EBREAKDOWN, "minres: preconditioner not SPD");
        beta = std::sqrt(bb);
        const double oldeps = epsln;
        const double delta = cs * dbar + sn * alfa;
        const double gbar = sn * dbar - cs * alfa;
        epsln = sn * beta;
        dbar = -cs * beta;
        const double gam = std::max(std::hypot(gbar, beta), 2.220446049250313e-16);
        cs = gbar / gam;
        sn = beta / gam;
        const double phi = cs * phibar;
        phibar = sn * phibar;
        // w1 <- w2 ; w2 <- w ; w <- (v - oldeps w1 - delta w2) / gam (into old w1) ; x += phi w
        double* old_w1 = w1;
        w1 = w2;
        w2 = ww;
        ww = old_w1;
        k_nminres_w<<<nb, kNB, 0, st>>>(n, v, w1, w2, ww, x, oldeps, delta, gam, phi);
        c->launches++;
    }
    // keep the rotated buffer roles in the workspace struct consistent for the next call
    converged = phibar <= target;
    kits += it;
    if (getenv("PF_NEWTON_TRACE"))
        fprintf(stderr, "  minres: its=%lld beta1=%.3e phibar=%.3e target=%.3e\n", it, beta1, phibar, target);
    return PF_OK;
}

// MINRES with the state on the device (fixed block preconditioners only): one eager start-up
// (r1 = rhs, y = M r1, beta1) and then a WHILE-node graph over one iteration; one host read at the
// end.  Same recurrence, buffers and counting as minres() above.
static int minres_dev(Ctx* c, NewtonWs& w, const double* u, const double* alpha, const double* rhs, double* x,
                      double rtol, long long maxit, long long& kits, bool& converged, cudaStream_t st,
                      const InnerMg& mg) {
    const long long n = w.n, nu = w.nu;
    const RedBuf rb{c->partials, c->tickets, c->scal};
    const int nb = nblocks(n);
    double *R1 = w.R1, *R2 = w.R2, *Y = w.Y, *V = w.V, *T = w.W, *Wa = w.W1, *Wb = w.W2;
    NCU(c, cudaMemsetAsync(Wa, 0, sizeof(double) * n, st), "memset");
    NCU(c, cudaMemsetAsync(Wb, 0, sizeof(double) * n, st), "memset");
    long long fs_its = 0;
    // warm start (x0 = the previous Newton iteration's solution, active rows zeroed): in a stalled
    // Newton phase consecutive systems barely change.  The stopping target stays rtol |b|_M, the
    // cold start's, so the accepted direction meets the same residual bound; only the iteration
    // count changes.
    bool warm = w.dp_valid && !getenv("PF_MINRES_COLD");
    NTRY(fieldsplit(c, w, rhs, Y, u, alpha, 0.0, 0, fs_its, st, mg));  // y = M b (cold start-up, |b|_M)
    k_mr_dot<<<nb, kNB, 0, st>>>(n, rhs, Y, c->scal, rb);
    k_mr_target<<<1, 1, 0, st>>>(c->scal, rtol);
    c->launches += 2;
    kits += fs_its;
    const long long fs_one = std::max(1LL, fs_its);  // the count of one field-split application
    if (warm) {
        k_mr_x0<<<nb, kNB, 0, st>>>(nu, n - nu, w.DP, c->act, x);
        NTRY(launch_jac(c, u, alpha, x, x + nu, T, T + nu, c->act, st));
        // x0 = the previous solution itself (a least-squares multiple of it was measured worse:
        // SENT 512^2 stalled Newton phase 0.88 s with x0 = d_prev, 1.05 s with the 2-norm-optimal scale)
        k_mr_r0<<<nb, kNB, 0, st>>>(n, rhs, T, x, R1, R2, nullptr);
        NTRY(fieldsplit(c, w, R1, V, u, alpha, 0.0, 0, fs_its, st, mg));  // M r0 (V is free here)
        kits += fs_one;
        k_mr_dot<<<nb, kNB, 0, st>>>(n, R1, V, c->scal, rb);
        c->launches += 4;
        NTRY(read_scal(c, st, S_MR, 20));
        const double bb_r = c->h_scal[S_MR + MR_BB], tgt = c->h_scal[S_MR + MR_TARGET];
        // keep the warm start only when it is closer than the cold one: |b - J x0|_M < |b|_M
        warm = bb_r >= 0.0 && rtol > 0.0 && std::sqrt(bb_r) < tgt / rtol;
        if (warm) NCU(c, cudaMemcpyAsync(Y, V, sizeof(double) * n, cudaMemcpyDeviceToDevice, st), "copy");
    }
    if (!warm) {  // cold: x = 0, r1 = r2 = b, y = M b (computed above), restore |b|_M^2
        NCU(c, cudaMemsetAsync(x, 0, sizeof(double) * n, st), "memset");
        NCU(c, cudaMemcpyAsync(R1, rhs, sizeof(double) * n, cudaMemcpyDeviceToDevice, st), "copy");
        NCU(c, cudaMemcpyAsync(R2, rhs, sizeof(double) * n, cudaMemcpyDeviceToDevice, st), "copy");
        k_mr_dot<<<nb, kNB, 0, st>>>(n, rhs, Y, c->scal, rb);
        c->launches++;
    }
    k_mr_start<<<1, 1, 0, st>>>(c->scal, rtol, (double)maxit, 1);
    c->launches++;
    fs_its = fs_one;
    long long key[Ctx::kMrKey] = {(long long)(uintptr_t)u, (long long)(uintptr_t)alpha, (long long)(uintptr_t)x,
                                 (long long)(uintptr_t)R1, c->geo_version, (long long)c->glev.size(),
                                 c->gmg_degree, mg.deg, mg.additive ? 1 : 0, n, nu, c->dim};
    // one iteration (k_mr_cond ends the graph body; the eager debug loop polls instead)
    auto issue = [&](cudaStream_t s, const cudaGraphConditionalHandle* h) -> int {
        long long dummy = 0;
        k_mr_v<<<nb, kNB, 0, s>>>(n, Y, V, c->scal);
        NTRY(launch_jac(c, u, alpha, V, V + nu, T, T + nu, c->act, s));
        k_mr_a<<<nb, kNB, 0, s>>>(n, T, R1, V, c->scal, rb);
        k_mr_b<<<nb, kNB, 0, s>>>(n, T, R1, R2, c->scal);
        NTRY(fieldsplit(c, w, R2, Y, u, alpha, 0.0, 0, dummy, s, mg));
        k_mr_dot<<<nb, kNB, 0, s>>>(n, R2, Y, c->scal, rb);
        k_mr_rot<<<1, 1, 0, s>>>(c->scal);
        k_mr_w<<<nb, kNB, 0, s>>>(n, V, Wa, Wb, x, c->scal);
        if (h) k_mr_cond<<<1, 32, 0, s>>>(*h, c->scal);
        c->launches += h ? 8 : 7;
        return PF_OK;
    };
    if (getenv("PF_MR_EAGER")) {  // debugging aid: the same launches, host-polled
        NTRY(read_scal(c, st, S_MR, 18));
        while (c->h_scal[S_MR + MR_DONE] == 0.0) {
            NTRY(issue(st, nullptr));
            NTRY(read_scal(c, st, S_MR, 18));
        }
        const double* m = c->h_scal + S_MR;
        if (m[MR_FAIL] != 0.0) return set_error(c, PF_EBREAKDOWN, "minres: preconditioner not SPD");
        const long long it = (long long)m[MR_IT];
        kits += it + it * fs_its;
        converged = m[MR_PHIBAR] <= m[MR_TARGET];
        if (getenv("PF_NEWTON_TRACE"))
            fprintf(stderr, "  minres(eager dev): its=%lld phibar=%.3e target=%.3e\n", it, m[MR_PHIBAR], m[MR_TARGET]);
        return PF_OK;
    }
    int slot = -1;
    for (int q = 0; q < 2; ++q)
        if (c->mr_exec[q] && memcmp(c->mr_key[q], key, sizeof key) == 0) slot = q;
    if (slot < 0) {  // capture one iteration under a WHILE node (replace the older slot)
        // the slot last used with this iterate buffer (stale after a geometry change), else the other
        const long long up = (long long)(uintptr_t)u;
        slot = c->mr_key[0][0] == up ? 0 : (c->mr_key[1][0] == up ? 1 : (c->mr_exec[0] ? 1 : 0));
        if (c->mr_exec[slot]) { cudaGraphExecDestroy(c->mr_exec[slot]); c->mr_exec[slot] = nullptr; }
        if (!c->cap_stream) NCU(c, cudaStreamCreateWithFlags(&c->cap_stream, cudaStreamNonBlocking), "stream");
        NCU(c, cudaStreamSynchronize(st), "sync");
        const long long l0 = c->launches;
        cudaGraph_t graph = nullptr;
        NCU(c, cudaGraphCreate(&graph, 0), "graph create");
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
            return check_cuda(c, ce, "minres conditional node");
        }
        cudaStream_t s = c->cap_stream;
        NCU(c, cudaStreamBeginCaptureToGraph(s, np.conditional.phGraph_out[0], nullptr, nullptr, 0,
                                             cudaStreamCaptureModeThreadLocal), "begin capture");
        const int rc = issue(s, &h);
        cudaGraph_t captured = nullptr;
        ce = cudaStreamEndCapture(s, &captured);
        if (rc != PF_OK) { cudaGraphDestroy(graph); return rc; }
        if (ce != cudaSuccess) { cudaGraphDestroy(graph); return check_cuda(c, ce, "minres end capture"); }
        ce = cudaGraphInstantiate(&c->mr_exec[slot], graph, 0);
        cudaGraphDestroy(graph);
        NCU(c, ce, "minres graph instantiate");
        c->mr_nodes[slot] = c->launches - l0;
        c->launches = l0;
        memcpy(c->mr_key[slot], key, sizeof key);
    }
    NTRY(read_scal(c, st, S_MR, 18));
    const double* m = c->h_scal + S_MR;
    if (m[MR_FAIL] != 0.0) return set_error(c, PF_EBREAKDOWN, "minres: preconditioner not SPD");
    if (m[MR_DONE] == 0.0) {
        NCU(c, cudaGraphLaunch(c->mr_exec[slot], st), "minres graph launch");
        NTRY(read_scal(c, st, S_MR, 18));
    }
    if (m[MR_FAIL] != 0.0) return set_error(c, PF_EBREAKDOWN, "minres: preconditioner not SPD");
    const long long it = (long long)m[MR_IT];
    c->launches += it * c->mr_nodes[slot];
    kits += it + it * fs_its;  // fs_its: the count of one field-split application (start-up call)
    converged = m[MR_PHIBAR] <= m[MR_TARGET];
    if (getenv("PF_NEWTON_TRACE"))
        fprintf(stderr, "  minres(dev): its=%lld beta1=%.3e phibar=%.3e target=%.3e\n", it,
                m[MR_TARGET] / rtol, m[MR_PHIBAR], m[MR_TARGET]);
    return PF_OK;
}

int newton_solve(Ctx* c, const double* u_in, const double* a_in, const double* lb, double* u_out, double* a_out,
                 const pf_vi_opts* o, pf_vi_report* rep, cudaStream_t st) {
    memset(rep, 0, sizeof(*rep));
    NewtonWs w;
    w.nu = c->n_u;
    w.na = c->n_a;
    w.n = w.nu + w.na;
    double** slots[] = {&w.X, &w.TX, &w.FX, &w.TF, &w.D, &w.RHS, &w.R1, &w.R2, &w.Y, &w.V, &w.W, &w.W1, &w.W2,
                        &w.TMP, &w.PP, &w.G};
    for (int k = 0; k < 16; ++k) *slots[k] = c->newton + (size_t)k * c->n_newton_vec;
    w.DP = c->newton + (size_t)16 * c->n_newton_vec;
    const long long nu = w.nu, na = w.na, n = w.n;
    NCU(c, cudaMemcpyAsync(w.X, u_in, sizeof(double) * nu, cudaMemcpyDeviceToDevice, st), "copy");
    NCU(c, cudaMemcpyAsync(w.X + nu, a_in, sizeof(double) * na, cudaMemcpyDeviceToDevice, st), "copy");
    // clip, zeta = 1e-10 (1 + |x0|_inf) (vi.py:197-201)
    NCU(c, cudaMemsetAsync(c->bits, 0, sizeof(unsigned long long) * 8, st), "memset");
    k_nclip_max<<<nblocks(n), kNB, 0, st>>>(nu, na, w.X, lb, c->bits + 1);
    c->launches++;
    NCU(c, cudaMemcpyAsync(c->h_scal + 100, c->bits + 1, sizeof(double), cudaMemcpyDeviceToHost, st), "xmax");
    NCU(c, cudaStreamSynchronize(st), "sync");
    double xmax;
    memcpy(&xmax, c->h_scal + 100, sizeof(double));
    const double zeta = o->zero_tol > 0.0 ? o->zero_tol : 1e-10 * (1.0 + xmax);
    NTRY(set_scal(c, st, S_ZETA, zeta));
    double merit;
    NTRY(eval_F(c, w, w.X, w.FX, lb, merit, st));
    auto push_hist = [&](double m) {
        if (rep->n_history < 64) rep->history[rep->n_history] = std::sqrt(m);
        rep->n_history++;
    };
    push_hist(merit);
    const double fs_rtol = o->fieldsplit_rtol > 0.0 ? o->fieldsplit_rtol : 1e-6;
    // inner block solves (the reference's LU, linalg.py:424-430) run to the MINRES tolerance:
    // tighter inner solves leave the MINRES history unchanged (measured on SENT 512^2 down to
    // 1e-10) at 1.5-2x the cost
    const double inner_rtol = o->inner_rtol > 0.0 ? o->inner_rtol : fs_rtol;
    // inner_mode bit 4: inexact Newton, MINRES rtol_k = max(fieldsplit_rtol, min(1e-2, |Phi_k|)) (the
    // quadratic forcing term, as the damage VI's inner solves): never tighter than the reference's
    // fieldsplit_rtol, loose far from the solution and in stalled phases, where |Phi| stays large
    const int imode = o->inner_mode & 3;
    const bool forcing = (o->inner_mode & 4) != 0;
    double last_mu = 1.0;      // accepted step length of the previous iteration
    double last_lmax = -1.0;   // C-block spectrum estimate of the previous iteration
    auto line_search = [&](const double* dir, double slope, bool newton, bool& ok) -> int {
        double mu = 1.0;
        ok = false;
        while (mu >= o->ls_min_step) {
            k_ntrial<<<nblocks(n), kNB, 0, st>>>(nu, na, w.X, dir, mu, lb, w.TX);
            c->launches++;
            double mt;
            NTRY(eval_F(c, w, w.TX, w.TF, lb, mt, st));
            const double bound = newton ? (1.0 - 2.0 * o->armijo * mu) * merit : merit - slope * mu;
            if (getenv("PF_NEWTON_TRACE")) fprintf(stderr, "  ls: mu=%.3e merit=%.6e bound=%.6e\n", mu, mt, bound);
            if (mt <= bound) {
                ok = true;
                merit = mt;
                last_mu = mu;
                std::swap(w.X, w.TX);
                std::swap(w.FX, w.TF);
                return PF_OK;
            }
            mu *= o->ls_backtrack;
        }
        return PF_OK;
    };
    static const bool tmg = getenv("PF_NEWTON_TIMING") != nullptr;  // (diagnostic: synchronised phases)
    double tmark = 0.0;
    auto tick = [&](const char* what) {
        if (!tmg) return;
        cudaStreamSynchronize(st);
        timespec ts;
        clock_gettime(CLOCK_MONOTONIC, &ts);
        const double now = ts.tv_sec + 1e-9 * ts.tv_nsec;
        if (what) fprintf(stderr, "  newton %-8s %8.3f ms\n", what, 1e3 * (now - tmark));
        tmark = now;
    };
    for (int it = 1; it <= o->max_iterations; ++it) {
        if (std::sqrt(merit) <= o->abs_tol) break;
        rep->iterations = it;
        tick(nullptr);
        const double* u = w.X;
        const double* alpha = w.X + nu;
        // active set on the damage rows; u rows are always inactive (free bounds)
        classify(c, na, alpha, w.FX + nu, lb, c->act, w.RHS + nu, st);
        NCU(c, cudaMemcpyAsync(w.RHS, w.FX, sizeof(double) * nu, cudaMemcpyDeviceToDevice, st), "copy");
        // Jacobian-dependent setup: GMG hierarchy of Kuu(alpha), kappa(u) and masked diag(Kaa)
        NCU(c, cudaMemcpyAsync(c->alpha_ws, alpha, sizeof(double) * na, cudaMemcpyDeviceToDevice, st), "copy");
        // inner_mode 1 (the V-cycle is only a preconditioner): the first Newton iteration keeps the
        // hierarchy of the last AM elastic solve (alpha one damage update older; damage only grows,
        // so the old smoother bounds stay above the spectrum) -- one setup (~2.5 ms) saved per phase
        // 2D only: the 3D re-discretised hierarchy with a stale alpha preconditioned config-4 Newton
        // badly (~160 instead of ~20 MINRES iterations, measured)
        // A stalled Newton phase (the previous accepted step was at most 1/64 of its direction) barely
        // moves the iterate: keep the hierarchy (2.5 ms of setup per iteration at 512^2) and the
        // C-block spectrum estimate of the previous iteration; a breakdown rebuilds and retries.
        const bool fixed_pc = imode == 1 || imode == 2;
        const bool stalled = fixed_pc && it > 1 && last_mu <= 1.0 / 64.0 && !getenv("PF_NEWTON_NO_STALL_KEEP");
        const bool keep = c->dim == 2 && fixed_pc && c->gmg_built &&
                          ((it == 1 && !getenv("PF_NEWTON_NO_KEEP")) || stalled);  // (NO_KEEP: calls
                                                         // independent of the prior hierarchy)
        if (!keep) {
            NTRY(c->dim == 3 ? gmg3_setup(c, st) : gmg_setup(c, st));
            c->gmg_built = 1;  // an elastic solve that follows may keep it (gmg_reuse)
            c->gmg_its0 = -1;
        }
        tick("setup");
        NTRY(launch_kappa(c, u, alpha, c->kappa, c->vi_c, st));
        NTRY(launch_Kaa_diag(c, c->kappa, c->da_dinv, c->act, st));
        InnerMg mg;
        if (imode == 1 || imode == 2) {
            mg.on = true;
            mg.additive = imode == 2;
            mg.deg = o->inner_cycles > 0 ? o->inner_cycles : 12;
            if (stalled && keep && last_lmax > 0.0) {
                mg.lmax = last_lmax;  // S_AUX1 still holds its |D^-1 C x|^2 unless MINRES ran on the host
                NTRY(set_scal(c, st, S_AUX1, last_lmax * last_lmax));
            } else {
                NTRY(lambda_C(c, mg.lmax, st));
            }
            last_lmax = mg.lmax;
            // device-resident MINRES (graph) unless profiling (eager, bracketed launches) or disabled
            mg.dev = c->use_graphs && !c->prof.on && !getenv("PF_NEWTON_HOST_MINRES") && mg.deg <= kMaxChebDeg;
            if (mg.dev) {
                k_cheb_table<<<1, 1, 0, st>>>(c->scal, mg.deg, kChebSafety);
                c->launches++;
            }
        }
        tick("kappa+C");
        bool ok = false;
        long long kits = 0;
        bool lin_ok = false;
        const long long mr_maxit = o->inner_maxit > 0 ? o->inner_maxit : 10 * n;
        const double rtol_it = forcing ? std::max(fs_rtol, std::min(1e-2, std::sqrt(merit))) : fs_rtol;
        auto run_minres = [&]() {
            return mg.dev ? minres_dev(c, w, u, alpha, w.RHS, w.D, rtol_it, mr_maxit, kits, lin_ok, st, mg)
                          : minres(c, w, u, alpha, w.RHS, w.D, rtol_it, mr_maxit, inner_rtol,
                                   mg.on ? 0 : std::max(0, o->inner_cycles), kits, lin_ok, st, mg);
        };
        int rc = run_minres();
        if (rc == PF_EBREAKDOWN && keep) {
            // the kept AM hierarchy gave an indefinite V-cycle: rebuild it for this iterate and retry
            // (as the elastic PCG does on breakdown) instead of spending the iteration on a
            // steepest-descent step
            NTRY(gmg_setup(c, st));
            c->gmg_built = 1;
            c->gmg_its0 = -1;
            rc = run_minres();
        }
        rep->total_krylov_iterations += kits;
        tick("minres");
        if (rc == PF_OK && lin_ok && mg.dev) {  // the next iteration's MINRES starts from it
            NCU(c, cudaMemcpyAsync(w.DP, w.D, sizeof(double) * n, cudaMemcpyDeviceToDevice, st), "copy");
            w.dp_valid = true;
        }
        if (rc == PF_OK && lin_ok) {
            k_nscale<<<nblocks(n), kNB, 0, st>>>(n, -1.0, w.D, w.D);  // d = -d_N (zero on active)
            c->launches++;
            NTRY(line_search(w.D, 0.0, true, ok));
        } else if (rc == PF_OK || rc == PF_EBREAKDOWN || rc == PF_EINNER) {
            rep->linear_failures++;  // solver.py:266-268 raises, rsls catches (vi.py:241-242)
        } else {
            return rc;
        }
        if (!ok) {
            // steepest descent on the merit (vi.py:244-252); J is symmetric (BlockJacobian.matvec)
            merit_parts(c, na, alpha, w.FX + nu, lb, w.PP + nu, w.TMP + nu, st);
            NCU(c, cudaMemcpyAsync(w.TMP, w.FX, sizeof(double) * nu, cudaMemcpyDeviceToDevice, st), "copy");
            NTRY(launch_jac(c, u, alpha, w.TMP, w.TMP + nu, w.G, w.G + nu, nullptr, st));
            k_ngrad<<<nblocks(n), kNB, 0, st>>>(nu, na, w.PP + nu, w.G, w.G);
            c->launches++;
            double gg;
            NTRY(ndot(c, n, w.G, w.G, S_AUX1, gg, st));
            const double gn = std::sqrt(gg);
            if (gn > 0.0) {
                const double sc = 1.0 / std::max(1.0, gn);
                k_nscale<<<nblocks(n), kNB, 0, st>>>(n, -sc, w.G, w.G);
                c->launches++;
                NTRY(line_search(w.G, o->armijo * sc * gn * gn, false, ok));
                rep->steepest_descent_steps++;
            }
        }
        tick("search");
        if (!ok) break;
        push_hist(merit);
    }
    rep->final_residual_norm = std::sqrt(merit);
    rep->converged = rep->final_residual_norm <= o->abs_tol;
    NCU(c, cudaMemcpyAsync(u_out, w.X, sizeof(double) * nu, cudaMemcpyDeviceToDevice, st), "copy");
    NCU(c, cudaMemcpyAsync(a_out, w.X + nu, sizeof(double) * na, cudaMemcpyDeviceToDevice, st), "copy");
    NCU(c, cudaStreamSynchronize(st), "sync");
    return PF_OK;
}

}  // namespace pf
