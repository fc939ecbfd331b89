// pf_gmg3.cu -- geometric multigrid preconditioner for the 3D (Kuhn-tetrahedra) degraded
// elasticity operator (BASELINE config 4: "multigrid-preconditioned CG").
//
// The reference solves the elastic half-step with SuperLU or stationary-preconditioned CG
// (linalg.py:250-262, 294-378).  Here PCG is preconditioned by a V-cycle on the structured 3D
// hierarchy, re-discretised on every level so that each level is applied by the same matrix-free
// Kuhn strip kernel as the fine operator (pf_ops3d.cu):
//   level l+1 : 2:1 coarsening per axis with the ceil rule (the last odd fine vertex is injected),
//               coarse alpha = a^-1 of the P^T-weighted mean of the fine degradation a(alpha),
//               per-cell E averaged over the covered fine cells, Dirichlet bits injected;
//   smoother  : Chebyshev-Jacobi of degree deg on [ratio*lam, lam], lam = 1.25 x the Rayleigh
//               estimate of lambda_max(D^-1 K_l) after 16 power iterations (device-side);
//   transfers : trilinear P (tensor product of the 1D 2:1 ceil-rule weights), P has zero rows on
//               constrained fine dofs and zero columns on constrained coarse dofs;
//   coarsest  : Chebyshev-Jacobi of degree kCoarseDeg3 from zero (a fixed polynomial).
// Every piece is linear and symmetric positive definite, so the V-cycle is a valid fixed PCG
// preconditioner.  Not a Galerkin hierarchy: on cracked states the coarse operators are the
// coefficient-averaged re-discretisation, which costs iterations, never correctness.
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "pf_internal.cuh"

namespace pf {

constexpr int kG3B = 256;
constexpr int kCoarseDeg3 = 6;  // 128^3: same PCG iterations as 12, 3% less time (4: +1 iteration)
constexpr double kCoarseRatio3 = 0.02;
constexpr int kPowIts3 = 16;
constexpr double kPowSafety3 = 1.25;
constexpr int kPowSlot3 = 20;  // grid_reduce ticket slot

__device__ __forceinline__ bool live3(const double* s) {
    return s == nullptr || (s[S_DONE] == 0.0 && s[S_FAIL] == 0.0);
}
__device__ __forceinline__ int p1d3(int f, int nf, int (&c)[2], double (&w)[2]) {
    if ((f & 1) == 0) { c[0] = f >> 1; w[0] = 1.0; return 1; }
    if (f == nf) { c[0] = (f + 1) >> 1; w[0] = 1.0; return 1; }
    c[0] = (f - 1) >> 1; c[1] = (f + 1) >> 1; w[0] = w[1] = 0.5; return 2;
}
__device__ __forceinline__ int finj3(int C, int nf) { return (2 * C <= nf) ? 2 * C : nf; }
__device__ __forceinline__ double wof(int f, int nf, int C) {  // weight of coarse C at fine f
    int c[2];
    double w[2];
    const int n = p1d3(f, nf, c, w);
    for (int a = 0; a < n; ++a)
        if (c[a] == C) return w[a];
    return 0.0;
}
__device__ __forceinline__ long long vid3g(const Geo3& g, int i, int j, int k) {
    return ((long long)i * g.nvy + j) * g.nvz + k;
}

// ---- level construction --------------------------------------------------------------------------
// coarse alpha from the P^T-weighted arithmetic mean of the fine degradation a = (1-alpha)^2 + k_ell
// (the coefficient, not alpha, is averaged: a thin crack softens the coarse level only in
// proportion to the fine cells it covers), mapped back through a^-1
__global__ void k3_coarsen_alpha(Geo3 F, Geo3 C, const double* af, double* ac) {
    for (long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x; v < C.nv;
         v += (long long)gridDim.x * blockDim.x) {
        const int K = (int)(v % C.nvz);
        const long long t = v / C.nvz;
        const int J = (int)(t % C.nvy), I = (int)(t / C.nvy);
        double sa = 0.0, sw = 0.0;
        for (int fi = max(2 * I - 1, 0); fi <= min(2 * I + 1, F.nx); ++fi) {
            const double wx = wof(fi, F.nx, I);
            if (wx == 0.0) continue;
            for (int fj = max(2 * J - 1, 0); fj <= min(2 * J + 1, F.ny); ++fj) {
                const double wy = wof(fj, F.ny, J);
                if (wy == 0.0) continue;
                for (int fk = max(2 * K - 1, 0); fk <= min(2 * K + 1, F.nz); ++fk) {
                    const double wz = wof(fk, F.nz, K);
                    if (wz == 0.0) continue;
                    const double om = 1.0 - __ldg(af + vid3g(F, fi, fj, fk));
                    const double w = wx * wy * wz;
                    sa += w * (om * om + F.kell);
                    sw += w;
                }
            }
        }
        ac[v] = 1.0 - sqrt(fmax(sa / sw - F.kell, 0.0));
    }
}
__global__ void k3_coarsen_E(Geo3 F, Geo3 C, const double* Ef, double* Ec) {
    for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < C.ncell;
         c += (long long)gridDim.x * blockDim.x) {
        const int K = (int)(c % C.nz);
        const long long t = c / C.nz;
        const int J = (int)(t % C.ny), I = (int)(t / C.ny);
        double s = 0.0;
        int n = 0;
        for (int a = 2 * I; a <= min(2 * I + 1, F.nx - 1); ++a)
            for (int b = 2 * J; b <= min(2 * J + 1, F.ny - 1); ++b)
                for (int q = 2 * K; q <= min(2 * K + 1, F.nz - 1); ++q) {
                    s += __ldg(Ef + ((long long)a * F.ny + b) * F.nz + q);
                    ++n;
                }
        Ec[c] = s / n;
    }
}
__global__ void k3_coarsen_mask(Geo3 F, Geo3 C, const unsigned char* mf, unsigned char* mc) {
    for (long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x; v < C.nv;
         v += (long long)gridDim.x * blockDim.x) {
        const int K = (int)(v % C.nvz);
        const long long t = v / C.nvz;
        const int J = (int)(t % C.nvy), I = (int)(t / C.nvy);
        mc[v] = mf[vid3g(F, finj3(I, F.nx), finj3(J, F.ny), finj3(K, F.nz))];
    }
}

// ---- lambda_max(D^-1 K) by power iteration -------------------------------------------------------
__global__ void k3_pow_init(long long n, double* x) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        x[i] = 1.0 + 0.5 * sin(0.7 * (double)i) + 0.25 * cos(1.3 * (double)(i / 3));
}
// z = dinv y ; xy = x.y ; xdx = x.(x / dinv) ; zz = z.z  -> last: lam = safety * xy / xdx, else S_AUX0 = 1/|z|
__global__ void k3_pow_dots(long long n, const double* x, const double* y, const double* dinv, double* z, double* s,
                            RedBuf rb, double* lam, int last) {
    double acc[3] = {0.0, 0.0, 0.0};
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const double xi = x[i], yi = y[i], di = dinv[i];
        const double zi = di * yi;
        z[i] = zi;
        acc[0] += xi * yi;
        acc[1] += xi * xi / di;
        acc[2] += zi * zi;
    }
    grid_reduce<3>(acc, rb, kPowSlot3, [=](double* t) {
        if (last) *lam = kPowSafety3 * t[0] / t[1];
        else s[S_AUX0] = t[2] > 0.0 ? 1.0 / sqrt(t[2]) : 0.0;
    });
}
__global__ void k3_pow_scale(long long n, const double* z, double* x, const double* s) {
    const double f = s[S_AUX0];
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        x[i] = f * z[i];
}

// ---- Chebyshev-Jacobi pieces (scalar dinv, dof-indexed) -----------------------------------------
// res = dinv src ; d = res / theta ; x (=|+=) d
__global__ void k3_cheb0(long long n, const double* dinv, const double* src, double* res, double* d, double* x,
                         int accumulate, const double* lam, double ratio, const double* live) {
    if (!live3(live)) return;
    const Cheb c = cheb_of(lam, ratio);
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const double r = dinv[i] * src[i];
        const double dd = r / c.theta;
        res[i] = r;
        d[i] = dd;
        x[i] = accumulate ? x[i] + dd : dd;
    }
}
// res -= dinv w ; dnext = a d + b res ; x += dnext      (w = K d)
__global__ void k3_cheb_step(long long n, const double* w, const double* d, double* dnext, double* res, double* x,
                             const double* dinv, int k, const double* lam, double ratio, const double* live) {
    if (!live3(live)) return;
    const Cheb c = cheb_of(lam, ratio);
    double a, b;
    cheb_ab(c, k, a, b);
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const double r = res[i] - dinv[i] * w[i];
        const double dn = a * d[i] + b * r;
        res[i] = r;
        dnext[i] = dn;
        x[i] += dn;
    }
}
// r = b - w      (w = K x)
__global__ void k3_resid(long long n, const double* w, const double* b, double* r, const double* live) {
    if (!live3(live)) return;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        r[i] = b[i] - w[i];
}
// post-smoother entry: res = dinv (b - w) ; d0 = res / theta ; x += d0      (w = K x)
__global__ void k3_resid_cheb0(long long n, const double* w, const double* b, const double* dinv, double* res,
                               double* d0, double* x, const double* lam, double ratio, const double* live) {
    if (!live3(live)) return;
    const Cheb c = cheb_of(lam, ratio);
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const double r = dinv[i] * (b[i] - w[i]);
        const double dd = r / c.theta;
        res[i] = r;
        d0[i] = dd;
        x[i] += dd;
    }
}

// ---- trilinear transfers (2:1, ceil rule, masks) ---------------------------------------------------
// b_c = P^T r_f : one thread per coarse vertex
__global__ void k3_restrict(Geo3 F, Geo3 C, const unsigned char* mf, const unsigned char* mc, const double* r,
                            double* bc, const double* live) {
    if (!live3(live)) return;
    for (long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x; v < C.nv;
         v += (long long)gridDim.x * blockDim.x) {
        const int K = (int)(v % C.nvz);
        const long long t = v / C.nvz;
        const int J = (int)(t % C.nvy), I = (int)(t / C.nvy);
        double s[3] = {0.0, 0.0, 0.0};
        for (int fi = max(2 * I - 1, 0); fi <= min(2 * I + 1, F.nx); ++fi) {
            const double wx = wof(fi, F.nx, I);
            if (wx == 0.0) continue;
            for (int fj = max(2 * J - 1, 0); fj <= min(2 * J + 1, F.ny); ++fj) {
                const double wy = wof(fj, F.ny, J);
                if (wy == 0.0) continue;
                for (int fk = max(2 * K - 1, 0); fk <= min(2 * K + 1, F.nz); ++fk) {
                    const double wz = wof(fk, F.nz, K);
                    if (wz == 0.0) continue;
                    const long long f = vid3g(F, fi, fj, fk);
                    const unsigned m = (F.has_bc && mf) ? mf[f] : 0u;
                    const double wt = wx * wy * wz;
#pragma unroll
                    for (int c = 0; c < 3; ++c)
                        if (!((m >> c) & 1u)) s[c] += wt * __ldcg(r + 3 * f + c);
                }
            }
        }
        const unsigned mC = (C.has_bc && mc) ? mc[v] : 0u;
#pragma unroll
        for (int c = 0; c < 3; ++c) bc[3 * v + c] = ((mC >> c) & 1u) ? 0.0 : s[c];
    }
}
// x_f += P x_c : one thread per fine vertex
__global__ void k3_prolong(Geo3 F, Geo3 C, const unsigned char* mf, const unsigned char* mc, const double* xc,
                           double* xf, const double* live) {
    if (!live3(live)) return;
    for (long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x; v < F.nv;
         v += (long long)gridDim.x * blockDim.x) {
        const int fk = (int)(v % F.nvz);
        const long long t = v / F.nvz;
        const int fj = (int)(t % F.nvy), fi = (int)(t / F.nvy);
        int ci[2], cj[2], ck[2];
        double wi[2], wj[2], wk[2];
        const int ni = p1d3(fi, F.nx, ci, wi), nj = p1d3(fj, F.ny, cj, wj), nk = p1d3(fk, F.nz, ck, wk);
        double s[3] = {0.0, 0.0, 0.0};
        for (int a = 0; a < ni; ++a)
            for (int b = 0; b < nj; ++b)
                for (int q = 0; q < nk; ++q) {
                    const long long cv = vid3g(C, ci[a], cj[b], ck[q]);
                    const unsigned mC = (C.has_bc && mc) ? mc[cv] : 0u;
                    const double wt = wi[a] * wj[b] * wk[q];
#pragma unroll
                    for (int c = 0; c < 3; ++c)
                        if (!((mC >> c) & 1u)) s[c] += wt * __ldcg(xc + 3 * cv + c);
                }
        const unsigned m = (F.has_bc && mf) ? mf[v] : 0u;
#pragma unroll
        for (int c = 0; c < 3; ++c)
            if (!((m >> c) & 1u)) xf[3 * v + c] += s[c];
    }
}

// ---- host side -------------------------------------------------------------------------------------
static int gb3(long long n) { return (int)std::max(1LL, std::min((n + kG3B - 1) / kG3B, 148LL * 16)); }

#define G3K(c, bytes, expr)                                     \
    do {                                                        \
        const int _ps = prof_begin((c), st);                    \
        expr;                                                   \
        prof_end((c), st, _ps, K_GMG, (double)(bytes));         \
        (c)->launches++;                                        \
    } while (0)
#define G3S(c, bytes, expr)                                     \
    do {                                                        \
        const int _ps = prof_begin((c), st);                    \
        expr;                                                   \
        prof_end((c), st, _ps, K_GMGSET, (double)(bytes));      \
        (c)->launches++;                                        \
    } while (0)

void gmg3_plan(Ctx* c) {
    c->g3lev.clear();
    G3Level L0;
    L0.g = c->g3;
    c->g3lev.push_back(L0);
    while (c->g3lev.size() < 16) {
        const Geo3& f = c->g3lev.back().g;
        if (std::max(f.nx, std::max(f.ny, f.nz)) <= 2) break;
        G3Level L;
        Geo3 g = f;
        g.nx = (f.nx + 1) / 2;
        g.ny = (f.ny + 1) / 2;
        g.nz = (f.nz + 1) / 2;
        g.nvy = g.ny + 1;
        g.nvz = g.nz + 1;
        g.nv = (long long)(g.nx + 1) * g.nvy * g.nvz;
        g.ncell = (long long)g.nx * g.ny * g.nz;
        g.ihx = g.nx / c->d.lx;
        g.ihy = g.ny / c->d.ly;
        g.ihz = g.nz / c->d.lz;
        g.vol = (c->d.lx / g.nx) * (c->d.ly / g.ny) * (c->d.lz / g.nz) / 6.0;
        tile3(g);
        L.g = g;
        c->g3lev.push_back(L);
    }
}

size_t gmg3_bytes(const Ctx* c) {
    auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
    size_t tot = 0;
    for (size_t l = 0; l < c->g3lev.size(); ++l) {
        const Geo3& g = c->g3lev[l].g;
        const size_t V = (size_t)g.nv;
        if (l > 0) tot += al(8 * V) + al(8 * (size_t)g.ncell) + al(V);  // alpha, E, mask
        tot += 8 * al(8 * 3 * V);                                       // dinv x b r d0 d1 res w
    }
    return tot + 4096;
}

void gmg3_bind(Ctx* c, char* base) {
    size_t off = 0;
    auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
    auto take = [&](size_t b) { char* p = base + off; off += al(b); return p; };
    for (size_t l = 0; l < c->g3lev.size(); ++l) {
        G3Level& L = c->g3lev[l];
        const size_t V = (size_t)L.g.nv;
        if (l > 0) {
            L.alpha = (double*)take(8 * V);
            L.E = (double*)take(8 * (size_t)L.g.ncell);
            L.mask = (unsigned char*)take(V);
        }
        double** vecs[] = {&L.dinv, &L.x, &L.b, &L.r, &L.d0, &L.d1, &L.res, &L.w};
        for (auto p : vecs) *p = (double*)take(8 * 3 * V);
    }
}

// refresh the per-level geometry from the (possibly changed) fine descriptor
static void sync_levels(Ctx* c) {
    std::vector<G3Level>& Ls = c->g3lev;
    Ls[0].g = c->g3;
    Ls[0].alpha = c->alpha_ws;
    Ls[0].mask = c->bcmask;
    for (size_t l = 1; l < Ls.size(); ++l) {
        Geo3& g = Ls[l].g;
        g.has_bc = c->g3.has_bc;
        g.bcmask = Ls[l].mask;
        g.E_cell = c->g3.E_cell ? Ls[l].E : nullptr;
        g.E = c->g3.E;
        g.ubar = nullptr;
    }
}

static int lambda_max(Ctx* c, int l, cudaStream_t st) {
    G3Level& L = c->g3lev[l];
    const long long n = 3 * L.g.nv;
    const RedBuf rb{c->partials, c->tickets, c->scal};
    double* lam = c->scal + S_GMG0 + l;
    G3S(c, 8.0 * n, (k3_pow_init<<<gb3(n), kG3B, 0, st>>>(n, L.x)));
    for (int t = 0; t < kPowIts3; ++t) {
        PF_TRY_GMG(launch3_Kuu_on(c, L.g, L.alpha, L.x, L.w, PF_BC_ELIMINATE, st, K_GMGSET));
        const int last = t == kPowIts3 - 1;
        G3S(c, 32.0 * n, (k3_pow_dots<<<gb3(n), kG3B, 0, st>>>(n, L.x, L.w, L.dinv, L.d0, c->scal, rb, lam, last)));
        if (!last) G3S(c, 16.0 * n, (k3_pow_scale<<<gb3(n), kG3B, 0, st>>>(n, L.d0, L.x, c->scal)));
    }
    return PF_OK;
}

int gmg3_setup(Ctx* c, cudaStream_t st) {
    if (c->g3lev.empty()) return set_error(c, PF_EINVAL, "3D multigrid not planned (PF_SKIP_GMG)");
    sync_levels(c);
    std::vector<G3Level>& Ls = c->g3lev;
    for (size_t l = 1; l < Ls.size(); ++l) {
        const Geo3& F = Ls[l - 1].g;
        const Geo3& C = Ls[l].g;
        G3S(c, 8.0 * F.nv + 8.0 * C.nv, (k3_coarsen_alpha<<<gb3(C.nv), kG3B, 0, st>>>(F, C, Ls[l - 1].alpha, Ls[l].alpha)));
        if (c->g3.E_cell)
            G3S(c, 8.0 * F.ncell + 8.0 * C.ncell, (k3_coarsen_E<<<gb3(C.ncell), kG3B, 0, st>>>(F, C, l == 1 ? c->g3.E_cell : Ls[l - 1].E, Ls[l].E)));
        if (c->g3.has_bc)
            G3S(c, 2.0 * C.nv, (k3_coarsen_mask<<<gb3(C.nv), kG3B, 0, st>>>(F, C, Ls[l - 1].mask, Ls[l].mask)));
    }
    for (size_t l = 0; l < Ls.size(); ++l) {
        PF_TRY_GMG(launch3_Kuu_diag_on(c, Ls[l].g, Ls[l].alpha, Ls[l].dinv, st, K_GMGSET));
        PF_TRY_GMG(lambda_max(c, (int)l, st));
    }
    return check_cuda(c, cudaGetLastError(), "3D multigrid setup");
}

// fused smoother steps (launch3_Kuu_sm); PF_GMG3_UNFUSED=1 keeps one vector pass per step
static bool fused3(int deg) {
    static const bool off = getenv("PF_GMG3_UNFUSED") != nullptr;
    return deg >= 2 && !off;
}
static Sm3Args sm_args(G3Level& L, int l, const double* xin, const double* b, double* res, double* dnext, double* xs,
                       int k, int pending, double ratio, const double* live, Ctx* c) {
    return Sm3Args{L.alpha, xin, b, L.dinv, res, dnext, xs, live, c->scal + S_GMG0 + l, ratio, k, pending};
}

// Chebyshev-Jacobi of degree deg on level l from x = 0 (pre-smoother / coarsest solve)
static int smooth_from_zero(Ctx* c, int l, const double* b, double* x, int deg, double ratio, cudaStream_t st,
                            const double* live) {
    G3Level& L = c->g3lev[l];
    const long long n = 3 * L.g.nv;
    const double* lam = c->scal + S_GMG0 + l;
    double *d = L.d0, *dn = L.d1;
    if (fused3(deg)) {
        // step 1 forms d0 = D b / theta inside the apply; x = d0 + dn
        PF_TRY_GMG(launch3_Kuu_sm(c, L.g, E3_CHEB_B, sm_args(L, l, nullptr, b, L.res, dn, x, 1, 0, ratio, live, c), st, K_GMG));
        std::swap(d, dn);
        for (int k = 2; k < deg; ++k) {
            PF_TRY_GMG(launch3_Kuu_sm(c, L.g, E3_CHEB, sm_args(L, l, d, b, L.res, dn, x, k, 0, ratio, live, c), st, K_GMG));
            std::swap(d, dn);
        }
        return PF_OK;
    }
    G3K(c, 40.0 * n, (k3_cheb0<<<gb3(n), kG3B, 0, st>>>(n, L.dinv, b, L.res, L.d0, x, 0, lam, ratio, live)));
    for (int k = 1; k < deg; ++k) {
        PF_TRY_GMG(launch3_Kuu_on(c, L.g, L.alpha, d, L.w, PF_BC_ELIMINATE, st, K_GMG));
        G3K(c, 64.0 * n, (k3_cheb_step<<<gb3(n), kG3B, 0, st>>>(n, L.w, d, dn, L.res, x, L.dinv, k, lam, ratio, live)));
        std::swap(d, dn);
    }
    return PF_OK;
}

int gmg3_vcycle(Ctx* c, const double* r_in, double* z_out, cudaStream_t st, const double* live) {
    std::vector<G3Level>& Ls = c->g3lev;
    const int nl = (int)Ls.size();
    const int deg = std::max(1, c->gmg_degree);
    const double ratio = c->gmg_ratio;
    const bool fz = fused3(deg);
    for (int l = 0; l < nl - 1; ++l) {
        G3Level& L = Ls[l];
        const long long n = 3 * L.g.nv;
        const double* b = l == 0 ? r_in : L.b;
        double* x = l == 0 ? z_out : L.x;
        PF_TRY_GMG(smooth_from_zero(c, l, b, x, deg, ratio, st, live));
        if (fz) {
            PF_TRY_GMG(launch3_Kuu_sm(c, L.g, E3_RESID, sm_args(L, l, x, b, L.r, nullptr, nullptr, 0, 0, ratio, live, c), st, K_GMG));
        } else {
            PF_TRY_GMG(launch3_Kuu_on(c, L.g, L.alpha, x, L.w, PF_BC_ELIMINATE, st, K_GMG));
            G3K(c, 24.0 * n, (k3_resid<<<gb3(n), kG3B, 0, st>>>(n, L.w, b, L.r, live)));
        }
        G3Level& C = Ls[l + 1];
        G3K(c, 24.0 * n + 24.0 * 3 * C.g.nv, (k3_restrict<<<gb3(C.g.nv), kG3B, 0, st>>>(L.g, C.g, L.mask, C.mask, L.r, C.b, live)));
    }
    {
        G3Level& L = Ls[nl - 1];
        PF_TRY_GMG(smooth_from_zero(c, nl - 1, nl == 1 ? r_in : L.b, nl == 1 ? z_out : L.x, kCoarseDeg3, kCoarseRatio3,
                                st, live));
    }
    for (int l = nl - 2; l >= 0; --l) {
        G3Level& L = Ls[l];
        G3Level& C = Ls[l + 1];
        const long long n = 3 * L.g.nv;
        const double* b = l == 0 ? r_in : L.b;
        double* x = l == 0 ? z_out : L.x;
        const double* lam = c->scal + S_GMG0 + l;
        G3K(c, 48.0 * n + 24.0 * C.g.nv, (k3_prolong<<<gb3(L.g.nv), kG3B, 0, st>>>(L.g, C.g, L.mask, C.mask, C.x, x, live)));
        double *d = L.d0, *dn = L.d1;
        if (fz) {
            // x += d0 is deferred into the first Chebyshev step (the apply reads x)
            PF_TRY_GMG(launch3_Kuu_sm(c, L.g, E3_RESID_CHEB0, sm_args(L, l, x, b, L.res, d, nullptr, 0, 0, ratio, live, c), st, K_GMG));
            for (int k = 1; k < deg; ++k) {
                PF_TRY_GMG(launch3_Kuu_sm(c, L.g, E3_CHEB, sm_args(L, l, d, b, L.res, dn, x, k, k == 1, ratio, live, c), st, K_GMG));
                std::swap(d, dn);
            }
            continue;
        }
        PF_TRY_GMG(launch3_Kuu_on(c, L.g, L.alpha, x, L.w, PF_BC_ELIMINATE, st, K_GMG));
        G3K(c, 64.0 * n, (k3_resid_cheb0<<<gb3(n), kG3B, 0, st>>>(n, L.w, b, L.dinv, L.res, L.d0, x, lam, ratio, live)));
        for (int k = 1; k < deg; ++k) {
            PF_TRY_GMG(launch3_Kuu_on(c, L.g, L.alpha, d, L.w, PF_BC_ELIMINATE, st, K_GMG));
            G3K(c, 64.0 * n, (k3_cheb_step<<<gb3(n), kG3B, 0, st>>>(n, L.w, d, dn, L.res, x, L.dinv, k, lam, ratio, live)));
            std::swap(d, dn);
        }
    }
    return check_cuda(c, cudaGetLastError(), "3D multigrid V-cycle");
}

}  // namespace pf
