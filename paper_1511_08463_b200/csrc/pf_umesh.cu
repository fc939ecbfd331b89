// pf_umesh.cu -- element-list (unstructured / jittered) P1 operator applies, 2D triangles and
// 3D tetrahedra (first step).
//
// The structured engines (pf_ops2d.cu, pf_ops3d.cu) keep the geometry implicit.  A mesh whose
// vertices move (the reference's jittered rect_mesh, mesh.py:134-141, used by the thermal-shock
// case, cases.py:195-234) or whose connectivity is arbitrary needs element lists.  This file
// applies the same centroid-quadrature P1 operators (fem.py:221-276; oracle/p1.py Kuu, Kaa) on
// such a mesh:
//
//   Kuu x   = sum_e A(ab_e) |T_e| E_e  B_e^T D1 B_e x_e                          (bc: eliminate)
//   Kaa x   = sum_e [ (A''(ab) q_e/2 + Gc_e w''(ab)/(c_w ell)) |T_e|/npe^2 11^T
//                     + 2 Gc_e ell/c_w |T_e| G_e^T G_e ] x_e,   q_e = E_e eps(u)^T D1 eps(u)
//
// Design (B200, fp64, HBM-bound):
//  * one thread per VERTEX gathers over its incident elements (vertex->element CSR built on the
//    host, element index ascending): no atomics, bitwise-reproducible sums, every row written
//    once with one coalesced store;
//  * per element one 64 B (2D) / 128 B (3D) record {gradients, |T| E_e, |T| Gc_e}, precomputed
//    at bind time in fp64 (the vertex coordinates are not needed on the device afterwards);
//  * connectivity as int4 (16 B), vertex-sorted mesh => the three/four gathers of an element
//    by its vertices' threads hit L2; compulsory HBM traffic per vertex is the roofline
//    (x, y, alpha, (u), element records, connectivity, CSR).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/phasefrac_b200.h"

struct pf_umesh {
    int dim = 2, regime = 0, model = 0;
    int64_t nv = 0, nt = 0, nadj = 0;
    double E = 1, nu = 0.3, Gc = 1, ell = 0.1, k_ell = 1e-6;
    std::string err;
    // host staging until bind
    std::vector<double> h_rec;
    std::vector<int32_t> h_conn, h_rowptr, h_adj;
    // device (inside the bound workspace)
    double* rec = nullptr;
    int32_t* conn = nullptr;
    int32_t* rowptr = nullptr;
    int32_t* adj = nullptr;
    uint8_t* vmask = nullptr;  // per vertex: bit c = Dirichlet on component c
    // Jacobi-PCG work vectors (d*nv each) + per-block partials + scalars
    double *r = nullptr, *z = nullptr, *p = nullptr, *q = nullptr, *dinv = nullptr, *part = nullptr,
           *scal = nullptr;
    const double* eps0 = nullptr;  // caller-owned inelastic strain per element (T x 3 / T x 6), or null
    unsigned* bar = nullptr;       // software grid barrier of the persistent PCG
    int pcg_blocks[4] = {0, 0, 0, 0};  // resident-block capacity per persistent-PCG variant
    bool bound = false, has_bc = false;
    int64_t launches = 0;
};

namespace {

thread_local std::string g_create_err;  // creation errors have no mesh object to carry them

constexpr int REC2 = 8, REC3 = 16;  // doubles per element record

inline int64_t align256(int64_t b) { return (b + 255) & ~int64_t(255); }

struct UParams {
    double d11, d12, d33;  // 2D unit stiffness
    double lam, mu;        // 3D unit stiffness
    double k_ell, inv_cw, ell, inv_ell;
    int at2;
    const double* eps0;  // inelastic strain (Voigt) per element or null: strains of u are B u - eps0
};

UParams make_params(const pf_umesh* m) {
    UParams p{};
    const double nu = m->nu;
    if (m->regime == PF_PLANE_STRESS) {
        const double s = 1.0 / (1.0 - nu * nu);
        p.d11 = s; p.d12 = s * nu; p.d33 = s * 0.5 * (1.0 - nu);
    } else {
        const double s = 1.0 / ((1.0 + nu) * (1.0 - 2.0 * nu));
        p.d11 = s * (1.0 - nu); p.d12 = s * nu; p.d33 = s * 0.5 * (1.0 - 2.0 * nu);
    }
    p.lam = nu / ((1.0 + nu) * (1.0 - 2.0 * nu));
    p.mu = 1.0 / (2.0 * (1.0 + nu));
    p.k_ell = m->k_ell;
    p.inv_cw = m->model == PF_AT1 ? 3.0 / 8.0 : 0.5;
    p.ell = m->ell;
    p.inv_ell = 1.0 / m->ell;
    p.at2 = m->model == PF_AT2;
    p.eps0 = m->eps0;
    return p;
}
// strain of u minus the element's inelastic strain (fem.py:125-131 with eps0, oracle/p1.py strain)
template <int NVOIGT>
__device__ __forceinline__ void sub_eps0(const UParams& p, int64_t e, double (&eps)[NVOIGT]) {
    if (!p.eps0) return;
#pragma unroll
    for (int i = 0; i < NVOIGT; ++i) eps[i] -= __ldg(p.eps0 + NVOIGT * e + i);
}

// ---- 2D ------------------------------------------------------------------------------------
struct Rec2 { double gx[3], gy[3], volE, volGc; };

__device__ __forceinline__ Rec2 load_rec2(const double* __restrict__ rec, int e) {
    const double2* r = reinterpret_cast<const double2*>(rec + (size_t)e * REC2);
    double2 a = __ldg(r), b = __ldg(r + 1), c = __ldg(r + 2), d = __ldg(r + 3);
    Rec2 o;
    o.gx[0] = a.x; o.gx[1] = a.y; o.gx[2] = b.x;
    o.gy[0] = b.y; o.gy[1] = c.x; o.gy[2] = c.y;
    o.volE = d.x; o.volGc = d.y;
    return o;
}

__device__ __forceinline__ void strain2(const Rec2& r, const double2 (&x)[3], double (&eps)[3]) {
    eps[0] = r.gx[0] * x[0].x + r.gx[1] * x[1].x + r.gx[2] * x[2].x;
    eps[1] = r.gy[0] * x[0].y + r.gy[1] * x[1].y + r.gy[2] * x[2].y;
    eps[2] = r.gy[0] * x[0].x + r.gy[1] * x[1].x + r.gy[2] * x[2].x
           + r.gx[0] * x[0].y + r.gx[1] * x[1].y + r.gx[2] * x[2].y;
}

// Fixed-order block sum of one value per thread (256 threads) -> part[blockIdx.x].
__device__ __forceinline__ void block_partial(double v, double* __restrict__ part) {
    __shared__ double sh[8];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
#pragma unroll
        for (int w = 0; w < 8; ++w) t += sh[w];
        part[blockIdx.x] = t;
    }
    __syncthreads();  // sh is reused by the next call in the same kernel
}

// one row (vertex v) of the (Dirichlet-eliminated when vmask) Kuu apply: gather over the incident
// elements (fem.py:233-244); Dirichlet rows return x (identity)
__device__ __forceinline__ double2 kuu2_row(const double* __restrict__ rec, const int4* __restrict__ conn,
                                           const int32_t* __restrict__ rowptr, const int32_t* __restrict__ adj,
                                           const uint8_t* __restrict__ vmask, const double* __restrict__ alpha,
                                           const double2* __restrict__ x, int64_t v, const UParams& p) {
    const uint8_t mv = vmask ? vmask[v] : 0;
    double y0 = 0.0, y1 = 0.0;
    const int k0 = rowptr[v], k1 = rowptr[v + 1];
    for (int k = k0; k < k1; ++k) {
        const int ent = __ldg(adj + k);
        const int e = ent >> 2, li = ent & 3;
        const int4 c = __ldg(conn + e);
        const int vs[3] = {c.x, c.y, c.z};
        const Rec2 r = load_rec2(rec, e);
        double2 xe[3];
        double ab = 0.0;
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            xe[j] = __ldcg(x + vs[j]);
            ab += __ldg(alpha + vs[j]);
            if (vmask) {
                const uint8_t mj = __ldg(vmask + vs[j]);
                if (mj & 1) xe[j].x = 0.0;
                if (mj & 2) xe[j].y = 0.0;
            }
        }
        ab *= (1.0 / 3.0);
        const double om = 1.0 - ab;
        const double w = (om * om + p.k_ell) * r.volE;
        double eps[3];
        strain2(r, xe, eps);
        const double s0 = w * (p.d11 * eps[0] + p.d12 * eps[1]);
        const double s1 = w * (p.d12 * eps[0] + p.d11 * eps[1]);
        const double s2 = w * (p.d33 * eps[2]);
        const double gxi = li == 0 ? r.gx[0] : (li == 1 ? r.gx[1] : r.gx[2]);
        const double gyi = li == 0 ? r.gy[0] : (li == 1 ? r.gy[1] : r.gy[2]);
        y0 += gxi * s0 + gyi * s2;
        y1 += gyi * s1 + gxi * s2;
    }
    if (mv) {
        const double2 xv = __ldcg(x + v);
        if (mv & 1) y0 = xv.x;
        if (mv & 2) y1 = xv.y;
    }
    return make_double2(y0, y1);
}

template <bool DOT>
__global__ void __launch_bounds__(256) k_umesh_Kuu2(
    const double* __restrict__ rec, const int4* __restrict__ conn, const int32_t* __restrict__ rowptr,
    const int32_t* __restrict__ adj, const uint8_t* __restrict__ vmask, const double* __restrict__ alpha,
    const double2* __restrict__ x, double2* __restrict__ y, int64_t nv, UParams p,
    double* __restrict__ part) {
    // no early exit: every lane reaches the block reduction's full-mask shuffles (a lane past nv
    // recomputes the last vertex and writes nothing)
    const int64_t v0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool live = v0 < nv;
    const int64_t v = live ? v0 : nv - 1;
    const double2 yv = kuu2_row(rec, conn, rowptr, adj, vmask, alpha, x, v, p);
    if (live) y[v] = yv;
    if (DOT) {
        const double2 xv = x[v];
        block_partial(live ? xv.x * yv.x + xv.y * yv.y : 0.0, part);
    }
}

// MODE: KAA_APPLY y = Kaa x; KAA_PCG y = Kaa x on rows with dinv != 0 (the inactive set of the
// damage VI; x is zero on the active rows) else 0, plus block partials of x.y; KAA_DIAG y = diag(Kaa)
// (x unused).
enum { KAA_APPLY = 0, KAA_PCG = 1, KAA_DIAG = 2 };

template <int MODE>
__device__ __forceinline__ void kaa_store(bool live, int64_t v, double acc, const double* __restrict__ x,
                                          double* __restrict__ y, const double* __restrict__ dinv,
                                          double* __restrict__ part) {
    if (MODE == KAA_PCG) {
        if (dinv[v] == 0.0) acc = 0.0;
        if (live) y[v] = acc;
        block_partial(live ? x[v] * acc : 0.0, part);
    } else if (live) {
        y[v] = acc;
    }
}

// one row of the Kaa apply (fem.py:266-282; KAA_DIAG: the diagonal, x unused)
template <int MODE>
__device__ __forceinline__ double kaa2_row(const double* __restrict__ rec, const int4* __restrict__ conn,
                                          const int32_t* __restrict__ rowptr, const int32_t* __restrict__ adj,
                                          const double2* __restrict__ u, const double* __restrict__ x, int64_t v,
                                          const UParams& p) {
    double acc = 0.0;
    const int k0 = rowptr[v], k1 = rowptr[v + 1];
    for (int k = k0; k < k1; ++k) {
        const int ent = __ldg(adj + k);
        const int e = ent >> 2, li = ent & 3;
        const int4 c = __ldg(conn + e);
        const int vs[3] = {c.x, c.y, c.z};
        const Rec2 r = load_rec2(rec, e);
        double2 ue[3];
        double sx = 0.0, gxa = 0.0, gya = 0.0;  // A''(ab) = 2 and w''(ab) are constants
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            ue[j] = __ldg(u + vs[j]);
            const double xj = MODE == KAA_DIAG ? (j == li ? 1.0 : 0.0) : __ldcg(x + vs[j]);
            sx += xj;
            gxa += r.gx[j] * xj;
            gya += r.gy[j] * xj;
        }
        double eps[3];
        strain2(r, ue, eps);
        sub_eps0<3>(p, e, eps);
        const double q = eps[0] * (p.d11 * eps[0] + p.d12 * eps[1])
                       + eps[1] * (p.d12 * eps[0] + p.d11 * eps[1]) + p.d33 * eps[2] * eps[2];
        const double wpp = p.at2 ? 2.0 : 0.0;
        const double kc = r.volGc * p.inv_cw;  // |T| Gc_e / c_w
        const double react = (q * r.volE + kc * wpp * p.inv_ell) * (1.0 / 9.0);  // A''/2 = 1
        const double gxi = li == 0 ? r.gx[0] : (li == 1 ? r.gx[1] : r.gx[2]);
        const double gyi = li == 0 ? r.gy[0] : (li == 1 ? r.gy[1] : r.gy[2]);
        acc += react * sx + 2.0 * kc * p.ell * (gxi * gxa + gyi * gya);
    }
    return acc;
}

template <int MODE>
__global__ void __launch_bounds__(256) k_umesh_Kaa2(
    const double* __restrict__ rec, const int4* __restrict__ conn, const int32_t* __restrict__ rowptr,
    const int32_t* __restrict__ adj, const double2* __restrict__ u,
    const double* __restrict__ x, double* __restrict__ y, int64_t nv, UParams p,
    const double* __restrict__ dinv = nullptr, double* __restrict__ part = nullptr) {
    // no early exit: every lane reaches the block reduction's full-mask shuffles (a lane past nv
    // recomputes the last vertex and writes nothing)
    const int64_t v0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool live = v0 < nv;
    const int64_t v = live ? v0 : nv - 1;
    const double acc = kaa2_row<MODE>(rec, conn, rowptr, adj, u, x, v, p);
    kaa_store<MODE>(live, v, acc, x, y, dinv, part);
}

// ---- 3D ------------------------------------------------------------------------------------
struct Rec3 { double g[3][4]; double volE, volGc; };

__device__ __forceinline__ Rec3 load_rec3(const double* __restrict__ rec, int e) {
    const double2* r = reinterpret_cast<const double2*>(rec + (size_t)e * REC3);
    Rec3 o;
    double t[14];
#pragma unroll
    for (int i = 0; i < 7; ++i) {
        const double2 a = __ldg(r + i);
        t[2 * i] = a.x;
        t[2 * i + 1] = a.y;
    }
#pragma unroll
    for (int d = 0; d < 3; ++d)
#pragma unroll
        for (int j = 0; j < 4; ++j) o.g[d][j] = t[4 * d + j];
    o.volE = t[12];
    o.volGc = t[13];
    return o;
}

// Voigt (e11, e22, e33, g23, g13, g12), engineering shears (oracle/p1.py voigt_B)
__device__ __forceinline__ void strain3(const Rec3& r, const double (&x)[4][3], double (&eps)[6]) {
#pragma unroll
    for (int i = 0; i < 6; ++i) eps[i] = 0.0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const double gx = r.g[0][j], gy = r.g[1][j], gz = r.g[2][j];
        eps[0] += gx * x[j][0];
        eps[1] += gy * x[j][1];
        eps[2] += gz * x[j][2];
        eps[3] += gz * x[j][1] + gy * x[j][2];
        eps[4] += gz * x[j][0] + gx * x[j][2];
        eps[5] += gy * x[j][0] + gx * x[j][1];
    }
}

__device__ __forceinline__ void stress3(const UParams& p, const double (&e)[6], double (&s)[6]) {
    const double tr = p.lam * (e[0] + e[1] + e[2]);
    s[0] = tr + 2.0 * p.mu * e[0];
    s[1] = tr + 2.0 * p.mu * e[1];
    s[2] = tr + 2.0 * p.mu * e[2];
    s[3] = p.mu * e[3];
    s[4] = p.mu * e[4];
    s[5] = p.mu * e[5];
}

__device__ __forceinline__ double pick4(const double (&a)[4], int i) {
    return i == 0 ? a[0] : (i == 1 ? a[1] : (i == 2 ? a[2] : a[3]));
}

__device__ __forceinline__ void kuu3_row(const double* __restrict__ rec, const int4* __restrict__ conn,
                                         const int32_t* __restrict__ rowptr, const int32_t* __restrict__ adj,
                                         const uint8_t* __restrict__ vmask, const double* __restrict__ alpha,
                                         const double* __restrict__ x, int64_t v, const UParams& p,
                                         double (&y)[3]) {
    double y0 = 0.0, y1 = 0.0, y2 = 0.0;
    const int k0 = rowptr[v], k1 = rowptr[v + 1];
    for (int k = k0; k < k1; ++k) {
        const int ent = __ldg(adj + k);
        const int e = ent >> 2, li = ent & 3;
        const int4 c = __ldg(conn + e);
        const int vs[4] = {c.x, c.y, c.z, c.w};
        const Rec3 r = load_rec3(rec, e);
        double xe[4][3];
        double ab = 0.0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const uint8_t mj = vmask ? __ldg(vmask + vs[j]) : 0;
#pragma unroll
            for (int d = 0; d < 3; ++d) xe[j][d] = (mj >> d) & 1 ? 0.0 : __ldcg(x + 3 * (int64_t)vs[j] + d);
            ab += __ldg(alpha + vs[j]);
        }
        ab *= 0.25;
        const double om = 1.0 - ab;
        const double w = (om * om + p.k_ell) * r.volE;
        double eps[6], st[6];
        strain3(r, xe, eps);
        stress3(p, eps, st);
        const double gx = pick4(r.g[0], li), gy = pick4(r.g[1], li), gz = pick4(r.g[2], li);
        y0 += w * (gx * st[0] + gz * st[4] + gy * st[5]);
        y1 += w * (gy * st[1] + gz * st[3] + gx * st[5]);
        y2 += w * (gz * st[2] + gy * st[3] + gx * st[4]);
    }
    const uint8_t mv = vmask ? vmask[v] : 0;
    if (mv & 1) y0 = __ldcg(x + 3 * v);
    if (mv & 2) y1 = __ldcg(x + 3 * v + 1);
    if (mv & 4) y2 = __ldcg(x + 3 * v + 2);
    y[0] = y0; y[1] = y1; y[2] = y2;
}

template <bool DOT>
__global__ void __launch_bounds__(256) k_umesh_Kuu3(
    const double* __restrict__ rec, const int4* __restrict__ conn, const int32_t* __restrict__ rowptr,
    const int32_t* __restrict__ adj, const uint8_t* __restrict__ vmask, const double* __restrict__ alpha,
    const double* __restrict__ x, double* __restrict__ y, int64_t nv, UParams p, double* __restrict__ part) {
    // no early exit: every lane reaches the block reduction's full-mask shuffles (a lane past nv
    // recomputes the last vertex and writes nothing)
    const int64_t v0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool live = v0 < nv;
    const int64_t v = live ? v0 : nv - 1;
    double yv[3];
    kuu3_row(rec, conn, rowptr, adj, vmask, alpha, x, v, p, yv);
    if (live) {
        y[3 * v] = yv[0];
        y[3 * v + 1] = yv[1];
        y[3 * v + 2] = yv[2];
    }
    if (DOT) block_partial(live ? x[3 * v] * yv[0] + x[3 * v + 1] * yv[1] + x[3 * v + 2] * yv[2] : 0.0, part);
}

template <int MODE>
__device__ __forceinline__ double kaa3_row(const double* __restrict__ rec, const int4* __restrict__ conn,
                                          const int32_t* __restrict__ rowptr, const int32_t* __restrict__ adj,
                                          const double* __restrict__ u, const double* __restrict__ x, int64_t v,
                                          const UParams& p) {
    double acc = 0.0;
    const int k0 = rowptr[v], k1 = rowptr[v + 1];
    for (int k = k0; k < k1; ++k) {
        const int ent = __ldg(adj + k);
        const int e = ent >> 2, li = ent & 3;
        const int4 c = __ldg(conn + e);
        const int vs[4] = {c.x, c.y, c.z, c.w};
        const Rec3 r = load_rec3(rec, e);
        double ue[4][3];
        double sx = 0.0, ga[3] = {0.0, 0.0, 0.0};  // A'' = 2 and w'' are constants
#pragma unroll
        for (int j = 0; j < 4; ++j) {
#pragma unroll
            for (int d = 0; d < 3; ++d) ue[j][d] = __ldg(u + 3 * (int64_t)vs[j] + d);
            const double xj = MODE == KAA_DIAG ? (j == li ? 1.0 : 0.0) : __ldcg(x + vs[j]);
            sx += xj;
#pragma unroll
            for (int d = 0; d < 3; ++d) ga[d] += r.g[d][j] * xj;
        }
        double eps[6], st[6];
        strain3(r, ue, eps);
        sub_eps0<6>(p, e, eps);
        stress3(p, eps, st);
        double q = 0.0;
#pragma unroll
        for (int i = 0; i < 6; ++i) q += eps[i] * st[i];
        const double wpp = p.at2 ? 2.0 : 0.0;
        const double kc = r.volGc * p.inv_cw;
        const double react = (q * r.volE + kc * wpp * p.inv_ell) * (1.0 / 16.0);
        const double gi0 = pick4(r.g[0], li), gi1 = pick4(r.g[1], li), gi2 = pick4(r.g[2], li);
        acc += react * sx + 2.0 * kc * p.ell * (gi0 * ga[0] + gi1 * ga[1] + gi2 * ga[2]);
    }
    return acc;
}

template <int MODE>
__global__ void __launch_bounds__(256) k_umesh_Kaa3(
    const double* __restrict__ rec, const int4* __restrict__ conn, const int32_t* __restrict__ rowptr,
    const int32_t* __restrict__ adj, const double* __restrict__ u,
    const double* __restrict__ x, double* __restrict__ y, int64_t nv, UParams p,
    const double* __restrict__ dinv = nullptr, double* __restrict__ part = nullptr) {
    // no early exit: every lane reaches the block reduction's full-mask shuffles (a lane past nv
    // recomputes the last vertex and writes nothing)
    const int64_t v0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool live = v0 < nv;
    const int64_t v = live ? v0 : nv - 1;
    const double acc = kaa3_row<MODE>(rec, conn, rowptr, adj, u, x, v, p);
    kaa_store<MODE>(live, v, acc, x, y, dinv, part);
}

// ---- Jacobi PCG (cg_solve, linalg.py:106-152) ---------------------------------------------
// Diagonal of the eliminated Kuu (Dirichlet dofs -> 1), inverted.
__global__ void __launch_bounds__(256) k_umesh_dinv(
    const double* __restrict__ rec, const int4* __restrict__ conn, const int32_t* __restrict__ rowptr,
    const int32_t* __restrict__ adj, const uint8_t* __restrict__ vmask, const double* __restrict__ alpha,
    double* __restrict__ dinv, int64_t nv, int dim, UParams p) {
    const int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= nv) return;
    double dg[3] = {0.0, 0.0, 0.0};
    const int npe = dim + 1;
    for (int k = rowptr[v]; k < rowptr[v + 1]; ++k) {
        const int ent = __ldg(adj + k);
        const int e = ent >> 2, li = ent & 3;
        const int4 c = __ldg(conn + e);
        const double ab = (__ldg(alpha + c.x) + __ldg(alpha + c.y) + __ldg(alpha + c.z)
                           + (dim == 3 ? __ldg(alpha + c.w) : 0.0)) / npe;
        const double om = 1.0 - ab;
        if (dim == 2) {
            const Rec2 r = load_rec2(rec, e);
            const double w = (om * om + p.k_ell) * r.volE;
            const double gx = r.gx[li], gy = r.gy[li];
            dg[0] += w * (p.d11 * gx * gx + p.d33 * gy * gy);
            dg[1] += w * (p.d11 * gy * gy + p.d33 * gx * gx);
        } else {
            const Rec3 r = load_rec3(rec, e);
            const double w = (om * om + p.k_ell) * r.volE;
            const double g[3] = {r.g[0][li], r.g[1][li], r.g[2][li]};
            const double gg = g[0] * g[0] + g[1] * g[1] + g[2] * g[2];
#pragma unroll
            for (int d = 0; d < 3; ++d) dg[d] += w * ((p.lam + p.mu) * g[d] * g[d] + p.mu * gg);
        }
    }
    const uint8_t mv = vmask[v];
    for (int d = 0; d < dim; ++d) dinv[dim * v + d] = (mv >> d) & 1 ? 1.0 : 1.0 / dg[d];
}

// x = 0, r = b, z = Dinv r, p = z; partials of r.z and r.r
__global__ void __launch_bounds__(256) k_umesh_pcg_init(
    const double* __restrict__ b, double* __restrict__ x, double* __restrict__ r, double* __restrict__ z,
    double* __restrict__ pv, const double* __restrict__ dinv, double* __restrict__ part, int64_t n, int nb) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    double rz = 0.0, rr = 0.0;
    if (i < n) {
        const double ri = b[i], zi = dinv[i] * ri;
        x[i] = 0.0; r[i] = ri; z[i] = zi; pv[i] = zi;
        rz = ri * zi; rr = ri * ri;
    }
    block_partial(rz, part);
    block_partial(rr, part + nb);
}

// one block: fixed-order sums of the partial arrays -> scal[o0], scal[o1]
__global__ void __launch_bounds__(1024) k_umesh_reduce(const double* __restrict__ part, int nb, int npart,
                                                       double* __restrict__ scal, int o0, int o1) {
    __shared__ double sh[32];
    for (int a = 0; a < npart; ++a) {
        double t = 0.0;
        for (int i = threadIdx.x; i < nb; i += 1024) t += part[a * nb + i];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) t += __shfl_down_sync(0xffffffffu, t, o);
        if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = t;
        __syncthreads();
        if (threadIdx.x == 0) {
            double u = 0.0;
            for (int w = 0; w < 32; ++w) u += sh[w];
            scal[a == 0 ? o0 : o1] = u;
        }
        __syncthreads();
    }
}

// scal layout: [0,1] r.z ring, [2] p.q, [3] r.r, [4] breakdown flag
// x += a p, r -= a q, z = Dinv r (a = rz_k / pq); partials of the new r.z and r.r
__global__ void __launch_bounds__(256) k_umesh_pcg_update(
    double* __restrict__ x, double* __restrict__ r, double* __restrict__ z, const double* __restrict__ pv,
    const double* __restrict__ q, const double* __restrict__ dinv, double* __restrict__ scal,
    double* __restrict__ part, int64_t n, int nb, int slot) {
    const double pq = scal[2];
    const double a = pq > 0.0 ? scal[slot] / pq : 0.0;
    // breakdown only for a nonzero residual: r = 0 exactly (a converged solve that is still being
    // iterated between host polls) gives p = 0 and p.q = 0 legitimately
    if (!(pq > 0.0) && scal[slot] != 0.0 && blockIdx.x == 0 && threadIdx.x == 0) scal[4] = 1.0;
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    double rz = 0.0, rr = 0.0;
    if (i < n) {
        x[i] += a * pv[i];
        const double ri = r[i] - a * q[i], zi = dinv[i] * ri;
        r[i] = ri; z[i] = zi;
        rz = ri * zi; rr = ri * ri;
    }
    block_partial(rz, part);
    block_partial(rr, part + nb);
}

// p = z + (rz_{k+1} / rz_k) p
__global__ void __launch_bounds__(256) k_umesh_pcg_dir(double* __restrict__ pv, const double* __restrict__ z,
                                                       const double* __restrict__ scal, int64_t n, int slot) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const double rzo = scal[slot], rzn = scal[slot ^ 1];
    const double beta = rzo != 0.0 ? rzn / rzo : 0.0;
    if (i < n) pv[i] = z[i] + beta * pv[i];
}

// ---- physics: energy parts and gradients (fem.py:162-218; oracle/p1.py energy, residual_*) ----
__device__ __forceinline__ void ab_terms(const UParams& p, double ab, double& A, double& Ap, double& w,
                                         double& wp) {
    const double om = 1.0 - ab;
    A = om * om + p.k_ell;
    Ap = -2.0 * om;
    w = p.at2 ? ab * ab : ab;
    wp = p.at2 ? 2.0 * ab : 1.0;
}

// per element: elastic 1/2 A q |T| E, surface |T| Gc/c_w (w/ell + ell |grad alpha|^2)
__global__ void __launch_bounds__(256) k_umesh_energy(
    const double* __restrict__ rec, const int4* __restrict__ conn, const double* __restrict__ u,
    const double* __restrict__ alpha, double* __restrict__ part, int64_t nt, int nbe, int dim, UParams p) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    double el = 0.0, ds = 0.0;
    if (e < nt) {
        const int4 c = __ldg(conn + e);
        const int vs[4] = {c.x, c.y, c.z, c.w};
        double A, Ap, w, wp, q, volE, volGc, gg = 0.0;
        if (dim == 2) {
            const Rec2 r = load_rec2(rec, (int)e);
            double2 ue[3];
            double ab = 0.0, ga[2] = {0.0, 0.0};
#pragma unroll
            for (int j = 0; j < 3; ++j) {
                ue[j] = __ldg(reinterpret_cast<const double2*>(u) + vs[j]);
                const double aj = __ldg(alpha + vs[j]);
                ab += aj; ga[0] += r.gx[j] * aj; ga[1] += r.gy[j] * aj;
            }
            ab_terms(p, ab * (1.0 / 3.0), A, Ap, w, wp);
            double eps[3];
            strain2(r, ue, eps);
            sub_eps0<3>(p, e, eps);
            q = eps[0] * (p.d11 * eps[0] + p.d12 * eps[1]) + eps[1] * (p.d12 * eps[0] + p.d11 * eps[1])
              + p.d33 * eps[2] * eps[2];
            gg = ga[0] * ga[0] + ga[1] * ga[1];
            volE = r.volE; volGc = r.volGc;
        } else {
            const Rec3 r = load_rec3(rec, (int)e);
            double ue[4][3];
            double ab = 0.0, ga[3] = {0.0, 0.0, 0.0};
#pragma unroll
            for (int j = 0; j < 4; ++j) {
#pragma unroll
                for (int d = 0; d < 3; ++d) ue[j][d] = __ldg(u + 3 * (int64_t)vs[j] + d);
                const double aj = __ldg(alpha + vs[j]);
                ab += aj;
#pragma unroll
                for (int d = 0; d < 3; ++d) ga[d] += r.g[d][j] * aj;
            }
            ab_terms(p, ab * 0.25, A, Ap, w, wp);
            double eps[6], sg[6];
            strain3(r, ue, eps);
            sub_eps0<6>(p, e, eps);
            stress3(p, eps, sg);
            q = 0.0;
#pragma unroll
            for (int i = 0; i < 6; ++i) q += eps[i] * sg[i];
            gg = ga[0] * ga[0] + ga[1] * ga[1] + ga[2] * ga[2];
            volE = r.volE; volGc = r.volGc;
        }
        el = 0.5 * A * q * volE;
        ds = volGc * p.inv_cw * (w * p.inv_ell + p.ell * gg);
    }
    block_partial(el, part);
    block_partial(ds, part + nbe);
}

// per vertex: r_u = dE/du (raw rows) and r_alpha = dE/dalpha
template <int D>
__global__ void __launch_bounds__(256) k_umesh_grad(
    const double* __restrict__ rec, const int4* __restrict__ conn, const int32_t* __restrict__ rowptr,
    const int32_t* __restrict__ adj, const double* __restrict__ u, const double* __restrict__ alpha,
    double* __restrict__ ru, double* __restrict__ ra, int64_t nv, UParams p) {
    const int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= nv) return;
    constexpr int NPE = D + 1;
    double yu[D] = {}, ya = 0.0;
    for (int k = rowptr[v]; k < rowptr[v + 1]; ++k) {
        const int ent = __ldg(adj + k);
        const int e = ent >> 2, li = ent & 3;
        const int4 c = __ldg(conn + e);
        const int vs[4] = {c.x, c.y, c.z, c.w};
        double g[3][4], volE, volGc;
        if (D == 2) {
            const Rec2 r = load_rec2(rec, e);
#pragma unroll
            for (int j = 0; j < 3; ++j) { g[0][j] = r.gx[j]; g[1][j] = r.gy[j]; g[2][j] = 0.0; }
            g[0][3] = g[1][3] = g[2][3] = 0.0;
            volE = r.volE; volGc = r.volGc;
        } else {
            const Rec3 r = load_rec3(rec, e);
#pragma unroll
            for (int d = 0; d < 3; ++d)
#pragma unroll
                for (int j = 0; j < 4; ++j) g[d][j] = r.g[d][j];
            volE = r.volE; volGc = r.volGc;
        }
        double ue[4][3] = {}, ab = 0.0, ga[3] = {0.0, 0.0, 0.0};
#pragma unroll
        for (int j = 0; j < NPE; ++j) {
#pragma unroll
            for (int d = 0; d < D; ++d) ue[j][d] = __ldg(u + D * (int64_t)vs[j] + d);
            const double aj = __ldg(alpha + vs[j]);
            ab += aj;
#pragma unroll
            for (int d = 0; d < D; ++d) ga[d] += g[d][j] * aj;
        }
        double A, Ap, w, wp;
        ab_terms(p, ab / NPE, A, Ap, w, wp);
        double gi[3];
#pragma unroll
        for (int d = 0; d < 3; ++d) gi[d] = li == 0 ? g[d][0] : (li == 1 ? g[d][1] : (li == 2 ? g[d][2] : g[d][3]));
        double q;
        if (D == 2) {
            double e0 = 0.0, e1 = 0.0, e2 = 0.0;
#pragma unroll
            for (int j = 0; j < 3; ++j) {
                e0 += g[0][j] * ue[j][0];
                e1 += g[1][j] * ue[j][1];
                e2 += g[1][j] * ue[j][0] + g[0][j] * ue[j][1];
            }
            if (p.eps0) {
                e0 -= __ldg(p.eps0 + 3 * (int64_t)e);
                e1 -= __ldg(p.eps0 + 3 * (int64_t)e + 1);
                e2 -= __ldg(p.eps0 + 3 * (int64_t)e + 2);
            }
            const double s0 = p.d11 * e0 + p.d12 * e1, s1 = p.d12 * e0 + p.d11 * e1, s2 = p.d33 * e2;
            q = e0 * s0 + e1 * s1 + e2 * s2;
            const double wA = A * volE;
            yu[0] += wA * (gi[0] * s0 + gi[1] * s2);
            yu[1] += wA * (gi[1] * s1 + gi[0] * s2);
        } else {
            Rec3 r;
#pragma unroll
            for (int d = 0; d < 3; ++d)
#pragma unroll
                for (int j = 0; j < 4; ++j) r.g[d][j] = g[d][j];
            double eps[6], sg[6];
            strain3(r, ue, eps);
            sub_eps0<6>(p, e, eps);
            stress3(p, eps, sg);
            q = 0.0;
#pragma unroll
            for (int i = 0; i < 6; ++i) q += eps[i] * sg[i];
            const double wA = A * volE;
            yu[0] += wA * (gi[0] * sg[0] + gi[2] * sg[4] + gi[1] * sg[5]);
            yu[1 % D] += wA * (gi[1] * sg[1] + gi[2] * sg[3] + gi[0] * sg[5]);
            yu[2 % D] += wA * (gi[2] * sg[2] + gi[1] * sg[3] + gi[0] * sg[4]);
        }
        const double kc = volGc * p.inv_cw;
        ya += (0.5 * Ap * q * volE + kc * wp * p.inv_ell) / NPE
            + 2.0 * kc * p.ell * (gi[0] * ga[0] + gi[1] * ga[1] + gi[2] * ga[2]);
    }
    if (ru) {
#pragma unroll
        for (int d = 0; d < D; ++d) ru[D * v + d] = yu[d];
    }
    if (ra) ra[v] = ya;
}

// ---- damage box QP (damage_half_step: rsls on Kaa(u) a + c, vi.py:187-264; oracle/mcp.py rsls) ----
__device__ __forceinline__ double fbf(double a, double b) { return hypot(a, b) - a - b; }

// Phi(a) for lb <= a <= 1 (fb_box, vi.py:95-115), its square into block partials, the reduced-space
// active set (active_sets, zeta) as dinv = 0, dinv = 1/diag on the inactive rows and the Newton
// right-hand side rhs = -g on the inactive rows.
__global__ void __launch_bounds__(256) k_umesh_vi_prep(
    const double* __restrict__ a, const double* __restrict__ g, const double* __restrict__ lb,
    const double* __restrict__ diag, double* __restrict__ dinv, double* __restrict__ rhs,
    double* __restrict__ part, int64_t nv, double zeta) {
    const int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    double ph2 = 0.0;
    if (v < nv) {
        const double av = a[v], gv = g[v], lo = lb[v];
        const double ph = fbf(av - lo, fbf(1.0 - av, -gv));
        ph2 = ph * ph;
        const bool la = (av - lo <= zeta) && (gv > 0.0);
        const bool ua = !la && (1.0 - av <= zeta) && (gv < 0.0);
        const bool act = la || ua;
        dinv[v] = act ? 0.0 : 1.0 / diag[v];
        rhs[v] = act ? 0.0 : -gv;
    }
    block_partial(ph2, part);
}

// out = clip(a + t d, lb, 1) (d may be NULL: a projection of a onto the box)
__global__ void __launch_bounds__(256) k_umesh_vi_cand(
    const double* __restrict__ a, const double* __restrict__ d, const double* __restrict__ lb, double t,
    double* __restrict__ out, int64_t nv) {
    const int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= nv) return;
    const double c = a[v] + (d ? t * d[v] : 0.0);
    out[v] = fmin(fmax(c, lb[v]), 1.0);
}

// ---- persistent Jacobi PCG (whole Krylov loop in one cooperative launch) -------------------------
// The loop of pf_umesh_elastic_solve / the damage VI's inner solve (cg_solve, linalg.py:106-152)
// with every iteration inside one launch: per iteration the apply + p.q (one vertex per thread,
// strided), the x / r / z update + r.z, r.r, and p = z + beta p, separated by a software grid
// barrier.  Every block sums the per-block partials in the same fixed order, so all blocks take the
// same decisions (deterministic).  It replaces 5 launches and a host poll every few iterations; the
// element-list path is launch-bound at the sizes of the reference's thermal-shock case.
__device__ __forceinline__ void ugrid_sync(unsigned int* bar) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned int inc = blockIdx.x == 0 ? 0x80000000u - (gridDim.x - 1) : 1u;
        __threadfence();
        const unsigned int old = atomicAdd(bar, inc);
        unsigned int cur;
        do {
            asm volatile("ld.acquire.gpu.u32 %0, [%1];\n" : "=r"(cur) : "l"(bar) : "memory");
        } while (((old ^ cur) & 0x80000000u) == 0);
    }
    __syncthreads();
}
// sum of rows [0, nb) of part (and [nb, 2 nb) when two): the same fixed order in every block
__device__ __forceinline__ double2 ugrid_total(const double* part, int nb, bool two) {
    __shared__ double2 tot;
    if (threadIdx.x < 32) {
        double a = 0.0, b = 0.0;
        for (int i = threadIdx.x; i < nb; i += 32) {
            a += __ldcg(part + i);
            if (two) b += __ldcg(part + nb + i);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            a += __shfl_xor_sync(0xffffffffu, a, o);
            b += __shfl_xor_sync(0xffffffffu, b, o);
        }
        if (threadIdx.x == 0) tot = make_double2(a, b);
    }
    __syncthreads();
    const double2 r = tot;
    __syncthreads();
    return r;
}
struct UPcg {
    const double* rec;
    const int4* conn;
    const int32_t *rowptr, *adj;
    const uint8_t* vmask;
    const double* alpha;  // Kuu
    const double* u;      // Kaa
    const double* dinv;   // Jacobi (Kaa: 0 on the active rows, masked out)
    double *x, *r, *z, *p, *q, *part, *scal;
    unsigned* bar;
    int64_t nv;
    double tol2;
    int64_t maxit;
    UParams prm;
};
// OP: 0 Kuu 2D, 1 Kuu 3D, 2 masked Kaa 2D, 3 masked Kaa 3D.  Start: scal[0] = r.z, scal[3] = r.r
// (k_umesh_pcg_init); end: scal[5] = iterations, scal[3] = r.r, scal[4] = breakdown flag.
template <int OP>
__global__ void __launch_bounds__(256) k_umesh_pcg_persistent(UPcg a) {
    constexpr int D = (OP == 0) ? 2 : (OP == 1 ? 3 : 1);  // dofs per vertex
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, nth = (int64_t)gridDim.x * blockDim.x;
    const int nb = gridDim.x;
    double rz = a.scal[0], rr = a.scal[3], brk = 0.0;
    int64_t it = 0;
    while (rr > a.tol2 && it < a.maxit) {
        double acc = 0.0;
        for (int64_t v = tid; v < a.nv; v += nth) {
            if constexpr (OP == 0) {
                const double2 y = kuu2_row(a.rec, a.conn, a.rowptr, a.adj, a.vmask, a.alpha,
                                           reinterpret_cast<const double2*>(a.p), v, a.prm);
                reinterpret_cast<double2*>(a.q)[v] = y;
                const double2 pv = reinterpret_cast<const double2*>(a.p)[v];
                acc += pv.x * y.x + pv.y * y.y;
            } else if constexpr (OP == 1) {
                double y[3];
                kuu3_row(a.rec, a.conn, a.rowptr, a.adj, a.vmask, a.alpha, a.p, v, a.prm, y);
#pragma unroll
                for (int d = 0; d < 3; ++d) {
                    a.q[3 * v + d] = y[d];
                    acc += a.p[3 * v + d] * y[d];
                }
            } else {
                double y = OP == 2 ? kaa2_row<KAA_APPLY>(a.rec, a.conn, a.rowptr, a.adj,
                                                         reinterpret_cast<const double2*>(a.u), a.p, v, a.prm)
                                   : kaa3_row<KAA_APPLY>(a.rec, a.conn, a.rowptr, a.adj, a.u, a.p, v, a.prm);
                if (a.dinv[v] == 0.0) y = 0.0;  // active row (KAA_PCG)
                a.q[v] = y;
                acc += a.p[v] * y;
            }
        }
        block_partial(acc, a.part);
        ugrid_sync(a.bar);
        const double pq = ugrid_total(a.part, nb, false).x;
        if (!(pq > 0.0)) {
            if (rz != 0.0) brk = 1.0;
            break;
        }
        const double al = rz / pq;
        double arz = 0.0, arr = 0.0;
        for (int64_t v = tid; v < a.nv; v += nth) {
#pragma unroll
            for (int d = 0; d < D; ++d) {
                const int64_t i = D * v + d;
                a.x[i] += al * a.p[i];
                const double ri = a.r[i] - al * a.q[i], zi = a.dinv[i] * ri;
                a.r[i] = ri;
                a.z[i] = zi;
                arz += ri * zi;
                arr += ri * ri;
            }
        }
        // r.z / r.r partials in rows [nb, 3 nb): no barrier needed against the readers of the p.q
        // partials in [0, nb) (the workspace holds >= 2 x the vertex blocks of partials)
        block_partial(arz, a.part + nb);
        block_partial(arr, a.part + 2 * nb);
        ugrid_sync(a.bar);
        const double2 t = ugrid_total(a.part + nb, nb, true);
        ++it;
        rr = t.y;
        const double rzo = rz;
        rz = t.x;
        if (rr <= a.tol2) break;
        const double be = rzo != 0.0 ? rz / rzo : 0.0;
        for (int64_t v = tid; v < a.nv; v += nth) {
#pragma unroll
            for (int d = 0; d < D; ++d) {
                const int64_t i = D * v + d;
                a.p[i] = a.z[i] + be * a.p[i];
            }
        }
        ugrid_sync(a.bar);  // p complete (and the r.z / r.r partials read) before the next apply
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        a.scal[5] = (double)it;
        a.scal[3] = rr;
        a.scal[4] = brk;
        a.scal[0] = rz;
    }
}

// Merit-gradient ingredients on the box [lb, 1] (vi.py:144-178, the structured k_merit_parts):
// pphi = p * phi and w = q * phi; the gradient of |Phi|^2 is 2 (pphi + Kaa w) (Kaa symmetric).
__device__ __forceinline__ void fb_part_u(double a, double b, double& pa, double& pb) {
    const double rho = hypot(a, b);
    if (rho > 0.0) { pa = a / rho - 1.0; pb = b / rho - 1.0; }
    else { pa = 0.70710678118654752440 - 1.0; pb = pa; }
}
__global__ void __launch_bounds__(256) k_umesh_merit_parts(
    const double* __restrict__ a, const double* __restrict__ g, const double* __restrict__ lb,
    double* __restrict__ pphi, double* __restrict__ w, int64_t nv) {
    const int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= nv) return;
    const double xv = a[v], Fv = g[v], sl = 1.0 - xv, lo = lb[v];
    const double inner = fbf(sl, -Fv);
    double pao, pbo, pai, pbi;
    fb_part_u(xv - lo, inner, pao, pbo);
    fb_part_u(sl, -Fv, pai, pbi);
    const double ph = fbf(xv - lo, inner);
    pphi[v] = (pao - pbo * pai) * ph;
    w[v] = -pbo * pbi * ph;
}
__global__ void __launch_bounds__(256) k_scale_u(double* __restrict__ x, double a, int64_t n) {
    const int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (v < n) x[v] *= a;
}
// gm = 2 (pphi + kw) (in place into kw) and block partials of |gm|^2
__global__ void __launch_bounds__(256) k_umesh_grad_finish(const double* __restrict__ pphi,
                                                           double* __restrict__ kw, double* __restrict__ part,
                                                           int64_t nv) {
    const int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    double g2 = 0.0;
    if (v < nv) {
        const double gv = 2.0 * (pphi[v] + kw[v]);
        kw[v] = gv;
        g2 = gv * gv;
    }
    block_partial(g2, part);
}


// launch the persistent PCG of variant OP over the vertices (cooperative: the blocks must be
// co-resident); returns cudaErrorNotSupported when the variant cannot be made resident
template <int OP>
cudaError_t launch_upcg(pf_umesh* m, const UPcg& a, cudaStream_t s) {
    int& cap = m->pcg_blocks[OP];
    if (cap == 0) {
        int dev = 0, nsm = 0, per = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_umesh_pcg_persistent<OP>, 256, 0);
        if (e != cudaSuccess) return e;
        cap = std::max(0, nsm * per);
    }
    if (cap <= 0) return cudaErrorNotSupported;
    const int64_t n = (OP <= 1 ? m->dim : 1) * m->nv;
    const int64_t nbmax = std::max((n + 255) / 256, (m->nt + 255) / 256);
    // three rows of per-block partials (p.q | r.z | r.r) must fit the 2 * nbmax of the workspace
    const int grid = (int)std::min<int64_t>(std::min<int64_t>(cap, (a.nv + 255) / 256), (2 * nbmax) / 3);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(std::max(grid, 1));
    cfg.blockDim = dim3(256);
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, k_umesh_pcg_persistent<OP>, a);
}

int fail(pf_umesh* m, int code, const std::string& msg) {
    if (m) m->err = msg;
    return code;
}

int cuda_fail(pf_umesh* m, cudaError_t e) {
    return fail(m, PF_ECUDA, std::string("CUDA: ") + cudaGetErrorString(e));
}

// element geometry: |T| and the P1 basis gradients (fem.py:107-123; oracle/p1.py
// simplex_gradients).  Returns false on a non-positive orientation.
bool geom2(const double* P, const int64_t* el, double* out, double E, double Gc) {
    const double* p1 = P + 2 * el[0];
    const double* p2 = P + 2 * el[1];
    const double* p3 = P + 2 * el[2];
    const double det = (p2[0] - p1[0]) * (p3[1] - p1[1]) - (p2[1] - p1[1]) * (p3[0] - p1[0]);
    if (!(det > 0.0)) return false;
    out[0] = (p2[1] - p3[1]) / det;
    out[1] = (p3[1] - p1[1]) / det;
    out[2] = (p1[1] - p2[1]) / det;
    out[3] = (p3[0] - p2[0]) / det;
    out[4] = (p1[0] - p3[0]) / det;
    out[5] = (p2[0] - p1[0]) / det;
    out[6] = 0.5 * det * E;
    out[7] = 0.5 * det * Gc;
    return true;
}

bool geom3(const double* P, const int64_t* el, double* out, double E, double Gc) {
    const double* p0 = P + 3 * el[0];
    double J[3][3];  // columns p_{c+1} - p0
    for (int c = 0; c < 3; ++c)
        for (int r = 0; r < 3; ++r) J[r][c] = P[3 * el[c + 1] + r] - p0[r];
    const double det = J[0][0] * (J[1][1] * J[2][2] - J[1][2] * J[2][1])
                     - J[0][1] * (J[1][0] * J[2][2] - J[1][2] * J[2][0])
                     + J[0][2] * (J[1][0] * J[2][1] - J[1][1] * J[2][0]);
    if (!(det > 0.0)) return false;
    // inv(J) by cofactors; row r of inv(J) = grad lambda_{r+1}
    double inv[3][3];
    inv[0][0] = (J[1][1] * J[2][2] - J[1][2] * J[2][1]) / det;
    inv[0][1] = (J[0][2] * J[2][1] - J[0][1] * J[2][2]) / det;
    inv[0][2] = (J[0][1] * J[1][2] - J[0][2] * J[1][1]) / det;
    inv[1][0] = (J[1][2] * J[2][0] - J[1][0] * J[2][2]) / det;
    inv[1][1] = (J[0][0] * J[2][2] - J[0][2] * J[2][0]) / det;
    inv[1][2] = (J[0][2] * J[1][0] - J[0][0] * J[1][2]) / det;
    inv[2][0] = (J[1][0] * J[2][1] - J[1][1] * J[2][0]) / det;
    inv[2][1] = (J[0][1] * J[2][0] - J[0][0] * J[2][1]) / det;
    inv[2][2] = (J[0][0] * J[1][1] - J[0][1] * J[1][0]) / det;
    for (int d = 0; d < 3; ++d) {
        double s = 0.0;
        for (int j = 1; j < 4; ++j) {
            out[4 * d + j] = inv[j - 1][d];
            s += inv[j - 1][d];
        }
        out[4 * d] = -s;
    }
    out[12] = det / 6.0 * E;
    out[13] = det / 6.0 * Gc;
    out[14] = out[15] = 0.0;
    return true;
}

}  // namespace

extern "C" {

int pf_umesh_create(const pf_umesh_desc* d, pf_umesh** out) {
    if (!out) return PF_EINVAL;
    *out = nullptr;
    auto bad = [](const std::string& msg) { g_create_err = msg; return PF_EINVAL; };
    if (!d) return bad("pf_umesh_create: NULL descriptor");
    if (d->dim != 2 && d->dim != 3) return bad("pf_umesh_create: dim must be 2 or 3");
    if ((d->dim == 3) != (d->regime == PF_3D) || d->regime < 0 || d->regime > 2)
        return bad("pf_umesh_create: regime does not match dim");
    if (d->model != PF_AT1 && d->model != PF_AT2) return bad("pf_umesh_create: model must be AT1 or AT2");
    if (d->n_vertices < 1 || d->n_elements < 1 || !d->vertices || !d->elements)
        return bad("pf_umesh_create: empty mesh");
    if (d->n_vertices >= (int64_t(1) << 31) / 3 || d->n_elements >= (int64_t(1) << 29))
        return bad("pf_umesh_create: mesh too large for 32-bit element lists");
    if (!(d->E > 0) || !(d->Gc > 0) || !(d->ell > 0) || !(d->nu > -1.0 && d->nu < 0.5))
        return bad("pf_umesh_create: invalid material");
    const int dim = d->dim, npe = dim + 1, R = dim == 2 ? REC2 : REC3;
    const int64_t nv = d->n_vertices, nt = d->n_elements;
    auto* m = new pf_umesh();
    m->dim = dim; m->regime = d->regime; m->model = d->model;
    m->nv = nv; m->nt = nt;
    m->E = d->E; m->nu = d->nu; m->Gc = d->Gc; m->ell = d->ell; m->k_ell = d->k_ell;
    m->h_rec.assign((size_t)nt * R, 0.0);
    m->h_conn.assign((size_t)nt * 4, 0);
    m->h_rowptr.assign((size_t)nv + 1, 0);
    for (int64_t e = 0; e < nt; ++e) {
        const int64_t* el = d->elements + e * npe;
        for (int j = 0; j < npe; ++j) {
            if (el[j] < 0 || el[j] >= nv) {
                delete m;
                return bad("pf_umesh_create: element vertex index out of range");
            }
            m->h_conn[4 * e + j] = (int32_t)el[j];
            m->h_rowptr[el[j] + 1]++;
        }
        const double Ee = d->E_elem ? d->E_elem[e] : d->E;
        const double Ge = d->Gc_elem ? d->Gc_elem[e] : d->Gc;
        const bool ok = dim == 2 ? geom2(d->vertices, el, &m->h_rec[e * R], Ee, Ge)
                                 : geom3(d->vertices, el, &m->h_rec[e * R], Ee, Ge);
        if (!ok) {
            delete m;
            return bad(dim == 2 ? "mesh contains non-CCW or degenerate triangles"
                                : "mesh contains inverted or degenerate tetrahedra");
        }
    }
    for (int64_t v = 0; v < nv; ++v) m->h_rowptr[v + 1] += m->h_rowptr[v];
    m->nadj = m->h_rowptr[nv];
    m->h_adj.assign((size_t)m->nadj, 0);
    std::vector<int32_t> fill(m->h_rowptr.begin(), m->h_rowptr.end() - 1);
    for (int64_t e = 0; e < nt; ++e)  // element index ascending within each vertex row
        for (int j = 0; j < npe; ++j) m->h_adj[fill[m->h_conn[4 * e + j]]++] = (int32_t)((e << 2) | j);
    *out = m;
    return PF_OK;
}

void pf_umesh_destroy(pf_umesh* m) { delete m; }

const char* pf_umesh_last_error(const pf_umesh* m) { return m ? m->err.c_str() : g_create_err.c_str(); }

int64_t pf_umesh_workspace_bytes(const pf_umesh* m) {
    if (!m) return -1;
    const int R = m->dim == 2 ? REC2 : REC3;
    const int64_t n = m->dim * m->nv, nb = std::max((n + 255) / 256, (m->nt + 255) / 256);
    return align256(m->nt * R * 8) + align256(m->nt * 16) + align256((m->nv + 1) * 4)
         + align256(m->nadj * 4) + align256(m->nv) + 5 * align256(n * 8) + align256(2 * nb * 8) + 256 + 256;
}

int pf_umesh_bind_workspace(pf_umesh* m, void* dev, int64_t bytes, void* stream) {
    if (!m) return PF_EINVAL;
    if (m->bound) return fail(m, PF_EINVAL, "pf_umesh_bind_workspace: already bound");
    if (!dev || bytes < pf_umesh_workspace_bytes(m))
        return fail(m, PF_ENOWS, "pf_umesh_bind_workspace: workspace too small");
    if (reinterpret_cast<uintptr_t>(dev) % 256)
        return fail(m, PF_EINVAL, "pf_umesh_bind_workspace: workspace must be 256-byte aligned");
    const int R = m->dim == 2 ? REC2 : REC3;
    char* p = static_cast<char*>(dev);
    m->rec = reinterpret_cast<double*>(p); p += align256(m->nt * R * 8);
    m->conn = reinterpret_cast<int32_t*>(p); p += align256(m->nt * 16);
    m->rowptr = reinterpret_cast<int32_t*>(p); p += align256((m->nv + 1) * 4);
    m->adj = reinterpret_cast<int32_t*>(p); p += align256(m->nadj * 4);
    m->vmask = reinterpret_cast<uint8_t*>(p); p += align256(m->nv);
    {
        const int64_t n = m->dim * m->nv, nb = std::max((n + 255) / 256, (m->nt + 255) / 256);
        double** vecs[5] = {&m->r, &m->z, &m->p, &m->q, &m->dinv};
        for (auto v : vecs) { *v = reinterpret_cast<double*>(p); p += align256(n * 8); }
        m->part = reinterpret_cast<double*>(p); p += align256(2 * nb * 8);
        m->scal = reinterpret_cast<double*>(p); p += 256;
        m->bar = reinterpret_cast<unsigned*>(p);
    }
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    cudaError_t e = cudaMemcpyAsync(m->rec, m->h_rec.data(), m->nt * R * 8, cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(m->conn, m->h_conn.data(), m->nt * 16, cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(m->rowptr, m->h_rowptr.data(), (m->nv + 1) * 4, cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(m->adj, m->h_adj.data(), m->nadj * 4, cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) e = cudaMemsetAsync(m->vmask, 0, m->nv, s);
    if (e == cudaSuccess) e = cudaMemsetAsync(m->bar, 0, 256, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return cuda_fail(m, e);
    std::vector<double>().swap(m->h_rec);
    std::vector<int32_t>().swap(m->h_conn);
    std::vector<int32_t>().swap(m->h_rowptr);
    std::vector<int32_t>().swap(m->h_adj);
    m->bound = true;
    return PF_OK;
}

int pf_umesh_set_dirichlet(pf_umesh* m, const int64_t* dofs, int64_t n, void* stream) {
    if (!m) return PF_EINVAL;
    if (!m->bound) return fail(m, PF_ENOWS, "pf_umesh_set_dirichlet: no workspace bound");
    if (n < 0 || (n > 0 && !dofs)) return fail(m, PF_EINVAL, "pf_umesh_set_dirichlet: bad dof list");
    std::vector<uint8_t> mask((size_t)m->nv, 0);
    for (int64_t i = 0; i < n; ++i) {
        if (dofs[i] < 0 || dofs[i] >= m->dim * m->nv)
            return fail(m, PF_EINVAL, "pf_umesh_set_dirichlet: dof out of range");
        mask[dofs[i] / m->dim] |= uint8_t(1u << (dofs[i] % m->dim));
    }
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    cudaError_t e = cudaMemcpyAsync(m->vmask, mask.data(), m->nv, cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);  // host staging dies with this call
    if (e != cudaSuccess) return cuda_fail(m, e);
    m->has_bc = n > 0;
    return PF_OK;
}

int pf_umesh_set_eps0(pf_umesh* m, const double* eps0, void* stream) {
    (void)stream;
    if (!m) return PF_EINVAL;
    m->eps0 = eps0;  // device pointer, T x (3 | 6) Voigt per element; NULL clears
    return PF_OK;
}

int pf_umesh_apply_Kuu(pf_umesh* m, const double* alpha, const double* x, double* y, int32_t bc_mode,
                       void* stream) {
    if (!m) return PF_EINVAL;
    if (!m->bound) return fail(m, PF_ENOWS, "pf_umesh_apply_Kuu: no workspace bound");
    if (!alpha || !x || !y || x == y) return fail(m, PF_EINVAL, "pf_umesh_apply_Kuu: bad pointers");
    const UParams p = make_params(m);
    const uint8_t* mask = (bc_mode == PF_BC_ELIMINATE && m->has_bc) ? m->vmask : nullptr;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const unsigned grid = (unsigned)((m->nv + 255) / 256);
    if (m->dim == 2)
        k_umesh_Kuu2<false><<<grid, 256, 0, s>>>(m->rec, reinterpret_cast<const int4*>(m->conn), m->rowptr,
                                                 m->adj, mask, alpha, reinterpret_cast<const double2*>(x),
                                                 reinterpret_cast<double2*>(y), m->nv, p, nullptr);
    else
        k_umesh_Kuu3<false><<<grid, 256, 0, s>>>(m->rec, reinterpret_cast<const int4*>(m->conn), m->rowptr,
                                                 m->adj, mask, alpha, x, y, m->nv, p, nullptr);
    m->launches++;
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? PF_OK : cuda_fail(m, e);
}

int pf_umesh_apply_Kaa(pf_umesh* m, const double* u, const double* alpha, const double* x, double* y,
                       void* stream) {
    if (!m) return PF_EINVAL;
    if (!m->bound) return fail(m, PF_ENOWS, "pf_umesh_apply_Kaa: no workspace bound");
    if (!u || !alpha || !x || !y || x == y) return fail(m, PF_EINVAL, "pf_umesh_apply_Kaa: bad pointers");
    const UParams p = make_params(m);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const unsigned grid = (unsigned)((m->nv + 255) / 256);
    if (m->dim == 2)
        k_umesh_Kaa2<KAA_APPLY><<<grid, 256, 0, s>>>(m->rec, reinterpret_cast<const int4*>(m->conn), m->rowptr, m->adj,
                                          reinterpret_cast<const double2*>(u), x, y, m->nv, p);
    else
        k_umesh_Kaa3<KAA_APPLY><<<grid, 256, 0, s>>>(m->rec, reinterpret_cast<const int4*>(m->conn), m->rowptr, m->adj,
                                          u, x, y, m->nv, p);
    m->launches++;
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? PF_OK : cuda_fail(m, e);
}

int pf_umesh_elastic_solve(pf_umesh* m, const double* alpha, const double* b, double* x, const pf_lin_opts* o,
                           pf_lin_report* rep, void* stream) {
    if (!m) return PF_EINVAL;
    if (!m->bound) return fail(m, PF_ENOWS, "pf_umesh_elastic_solve: no workspace bound");
    if (!alpha || !b || !x || !o || x == b) return fail(m, PF_EINVAL, "pf_umesh_elastic_solve: bad pointers");
    if (o->precond != PF_PREC_JACOBI)
        return fail(m, PF_EINVAL, "pf_umesh_elastic_solve: element-list meshes take precond = jacobi");
    const UParams p = make_params(m);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int64_t n = m->dim * m->nv;
    const int nb = (int)((n + 255) / 256);
    const unsigned gv = (unsigned)((m->nv + 255) / 256);
    const int64_t maxit = o->maxit > 0 ? o->maxit : 10 * n;
    const int every = o->check_every > 0 ? o->check_every : 10;
    const int4* conn = reinterpret_cast<const int4*>(m->conn);
    double h[5];
    auto poll = [&]() -> cudaError_t {
        cudaError_t e = cudaMemcpyAsync(h, m->scal, sizeof h, cudaMemcpyDeviceToHost, s);
        return e == cudaSuccess ? cudaStreamSynchronize(s) : e;
    };
    if (!rep) return fail(m, PF_EINVAL, "pf_umesh_elastic_solve: NULL report");
    cudaMemsetAsync(m->scal, 0, 8 * sizeof(double), s);
    k_umesh_dinv<<<gv, 256, 0, s>>>(m->rec, conn, m->rowptr, m->adj, m->vmask, alpha, m->dinv, m->nv, m->dim, p);
    k_umesh_pcg_init<<<nb, 256, 0, s>>>(b, x, m->r, m->z, m->p, m->dinv, m->part, n, nb);
    k_umesh_reduce<<<1, 1024, 0, s>>>(m->part, nb, 2, m->scal, 0, 3);
    m->launches += 3;
    cudaError_t e = poll();
    if (e != cudaSuccess) return cuda_fail(m, e);
    const double bnorm = std::sqrt(h[3]);
    const double tol = std::max(o->rtol * bnorm, o->atol);
    rep->b_norm = bnorm;
    rep->iterations = 0;
    rep->final_residual_norm = bnorm;
    rep->converged = bnorm <= tol;
    rep->status = PF_OK;
    // the partial arrays of the Kuu apply (one per vertex block) reuse part[0..gv)
    int64_t it = 0;
    if (!rep->converged && !getenv("PF_UMESH_EAGER")) {  // the whole loop in one persistent launch
        UPcg a{m->rec, conn, m->rowptr, m->adj, m->vmask, alpha, nullptr, m->dinv, x, m->r, m->z, m->p, m->q,
               m->part, m->scal, m->bar, m->nv, tol * tol, maxit, p};
        e = m->dim == 2 ? launch_upcg<0>(m, a, s) : launch_upcg<1>(m, a, s);
        if (e == cudaSuccess) {
            m->launches++;
            double h6[6];
            if ((e = cudaMemcpyAsync(h6, m->scal, sizeof h6, cudaMemcpyDeviceToHost, s)) != cudaSuccess ||
                (e = cudaStreamSynchronize(s)) != cudaSuccess)
                return cuda_fail(m, e);
            rep->iterations = (int64_t)h6[5];
            rep->final_residual_norm = std::sqrt(h6[3]);
            if (h6[4] != 0.0) {
                rep->status = PF_EBREAKDOWN;
                return fail(m, PF_EBREAKDOWN, "CG breakdown: p^T A p <= 0 (operator not SPD)");
            }
            rep->converged = rep->final_residual_norm <= tol;
            return PF_OK;
        }
        cudaGetLastError();  // not co-resident: the launch-per-kernel loop below
    }
    while (!rep->converged && it < maxit) {
        const int slot = (int)(it & 1);
        if (m->dim == 2)
            k_umesh_Kuu2<true><<<gv, 256, 0, s>>>(m->rec, conn, m->rowptr, m->adj, m->vmask, alpha,
                                                  reinterpret_cast<const double2*>(m->p),
                                                  reinterpret_cast<double2*>(m->q), m->nv, p, m->part);
        else
            k_umesh_Kuu3<true><<<gv, 256, 0, s>>>(m->rec, conn, m->rowptr, m->adj, m->vmask, alpha, m->p, m->q,
                                                  m->nv, p, m->part);
        k_umesh_reduce<<<1, 1024, 0, s>>>(m->part, (int)gv, 1, m->scal, 2, 2);
        k_umesh_pcg_update<<<nb, 256, 0, s>>>(x, m->r, m->z, m->p, m->q, m->dinv, m->scal, m->part, n, nb, slot);
        k_umesh_reduce<<<1, 1024, 0, s>>>(m->part, nb, 2, m->scal, slot ^ 1, 3);
        k_umesh_pcg_dir<<<nb, 256, 0, s>>>(m->p, m->z, m->scal, n, slot);
        m->launches += 5;
        ++it;
        if (it % every == 0 || it == maxit) {
            if ((e = poll()) != cudaSuccess) return cuda_fail(m, e);
            rep->iterations = it;
            rep->final_residual_norm = std::sqrt(h[3]);
            if (h[4] != 0.0) {
                rep->status = PF_EBREAKDOWN;
                return fail(m, PF_EBREAKDOWN, "CG breakdown: p^T A p <= 0 (operator not SPD)");
            }
            rep->converged = rep->final_residual_norm <= tol;
        }
    }
    if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(m, e);
    return PF_OK;
}

int pf_umesh_physics(pf_umesh* m, const double* u, const double* alpha, double* r_u, double* r_alpha,
                     double* energy, void* stream) {
    if (!m) return PF_EINVAL;
    if (!m->bound) return fail(m, PF_ENOWS, "pf_umesh_physics: no workspace bound");
    if (!u || !alpha) return fail(m, PF_EINVAL, "pf_umesh_physics: bad pointers");
    const UParams p = make_params(m);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int4* conn = reinterpret_cast<const int4*>(m->conn);
    const unsigned gv = (unsigned)((m->nv + 255) / 256);
    if (r_u || r_alpha) {
        if (m->dim == 2)
            k_umesh_grad<2><<<gv, 256, 0, s>>>(m->rec, conn, m->rowptr, m->adj, u, alpha, r_u, r_alpha, m->nv, p);
        else
            k_umesh_grad<3><<<gv, 256, 0, s>>>(m->rec, conn, m->rowptr, m->adj, u, alpha, r_u, r_alpha, m->nv, p);
        m->launches++;
    }
    if (energy) {
        const int nbe = (int)((m->nt + 255) / 256);
        k_umesh_energy<<<nbe, 256, 0, s>>>(m->rec, conn, u, alpha, m->part, m->nt, nbe, m->dim, p);
        k_umesh_reduce<<<1, 1024, 0, s>>>(m->part, nbe, 2, m->scal, 5, 6);
        m->launches += 2;
        double h[2];
        cudaError_t e = cudaMemcpyAsync(h, m->scal + 5, sizeof h, cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        if (e != cudaSuccess) return cuda_fail(m, e);
        energy[0] = h[0];
        energy[1] = h[1];
        energy[2] = h[0] + h[1];
    }
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? PF_OK : cuda_fail(m, e);
}

int pf_umesh_damage_solve(pf_umesh* m, const double* u, const double* alpha_lb, const double* alpha_in,
                          double* alpha_out, const pf_vi_opts* o, pf_vi_report* rep, void* stream) {
    if (!m) return PF_EINVAL;
    if (!m->bound) return fail(m, PF_ENOWS, "pf_umesh_damage_solve: no workspace bound");
    if (!u || !alpha_lb || !alpha_in || !alpha_out || !o || !rep)
        return fail(m, PF_EINVAL, "pf_umesh_damage_solve: bad pointers");
    if (alpha_out == alpha_lb) return fail(m, PF_EINVAL, "pf_umesh_damage_solve: alpha_out aliases alpha_lb");
    const UParams p = make_params(m);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int64_t nv = m->nv;
    const int nb = (int)((nv + 255) / 256);
    const unsigned gv = (unsigned)nb;
    const int4* conn = reinterpret_cast<const int4*>(m->conn);
    // scratch: every workspace vector holds dim*nv >= 2 nv doubles
    double *r = m->r, *g = m->r + nv, *z = m->z, *d = m->z + nv, *pv = m->p, *cand = m->p + nv;
    double *q = m->q, *dinv = m->dinv, *diag = m->dinv + nv;
    double* a = alpha_out;
    double h[8];
    auto poll = [&]() -> cudaError_t {
        cudaError_t e = cudaMemcpyAsync(h, m->scal, sizeof h, cudaMemcpyDeviceToHost, s);
        return e == cudaSuccess ? cudaStreamSynchronize(s) : e;
    };
    auto grad = [&](const double* x) {
        if (m->dim == 2)
            k_umesh_grad<2><<<gv, 256, 0, s>>>(m->rec, conn, m->rowptr, m->adj, u, x, nullptr, g, nv, p);
        else
            k_umesh_grad<3><<<gv, 256, 0, s>>>(m->rec, conn, m->rowptr, m->adj, u, x, nullptr, g, nv, p);
    };
    *rep = pf_vi_report{};
    cudaMemsetAsync(m->scal, 0, 8 * sizeof(double), s);
    // zeta from the initial iterate (rsls: 1e-10 (1 + |x0|_inf)); the box keeps |a| <= 1
    double zeta = o->zero_tol;
    k_umesh_vi_cand<<<gv, 256, 0, s>>>(alpha_in, nullptr, alpha_lb, 0.0, a, nv);
    if (m->dim == 2)
        k_umesh_Kaa2<KAA_DIAG><<<gv, 256, 0, s>>>(m->rec, conn, m->rowptr, m->adj,
                                                  reinterpret_cast<const double2*>(u), nullptr, diag, nv, p);
    else
        k_umesh_Kaa3<KAA_DIAG><<<gv, 256, 0, s>>>(m->rec, conn, m->rowptr, m->adj, u, nullptr, diag, nv, p);
    grad(a);
    m->launches += 3;
    if (!(zeta > 0.0)) {
        std::vector<double> a0(nv);
        cudaError_t e = cudaMemcpyAsync(a0.data(), alpha_in, nv * 8, cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        if (e != cudaSuccess) return cuda_fail(m, e);
        double mx = 0.0;
        for (double x : a0) mx = std::max(mx, std::fabs(x));
        zeta = 1e-10 * (1.0 + mx);
    }
    k_umesh_vi_prep<<<gv, 256, 0, s>>>(a, g, alpha_lb, diag, dinv, q, m->part, nv, zeta);
    k_umesh_reduce<<<1, 1024, 0, s>>>(m->part, nb, 1, m->scal, 7, 7);
    m->launches += 2;
    cudaError_t e = poll();
    if (e != cudaSuccess) return cuda_fail(m, e);
    double merit = h[7];
    const int maxit = o->max_iterations > 0 ? o->max_iterations : 100;
    const double bt = o->ls_backtrack > 0.0 && o->ls_backtrack < 1.0 ? o->ls_backtrack : 0.5;
    const double tmin = o->ls_min_step > 0.0 ? o->ls_min_step : 1e-10;
    const double irtol = o->inner_rtol > 0.0 ? o->inner_rtol : 1e-10;
    const int64_t imaxit = o->inner_maxit > 0 ? o->inner_maxit : 10 * nv;
    auto record = [&]() {
        if (rep->n_history < 64) rep->history[rep->n_history++] = std::sqrt(merit);
    };
    record();
    int it = 0;
    while (true) {
        rep->final_residual_norm = std::sqrt(merit);
        if (std::sqrt(merit) <= o->abs_tol) { rep->converged = 1; break; }
        if (it >= maxit) break;
        ++it;
        rep->iterations = it;  // counted at the start of the iteration, as vi.py:219
        // reduced Newton system K_II d_I = -g_I by Jacobi PCG (rhs in q, d = 0 on the active rows)
        cudaMemsetAsync(m->scal, 0, 5 * sizeof(double), s);
        k_umesh_pcg_init<<<nb, 256, 0, s>>>(q, d, r, z, pv, dinv, m->part, nv, nb);
        k_umesh_reduce<<<1, 1024, 0, s>>>(m->part, nb, 2, m->scal, 0, 3);
        m->launches += 2;
        if ((e = poll()) != cudaSuccess) return cuda_fail(m, e);
        const double tol = irtol * std::sqrt(h[3]);
        double rn = std::sqrt(h[3]);
        int64_t k = 0;
        bool eager = true;
        if (rn > tol && !getenv("PF_UMESH_EAGER")) {  // the whole inner PCG in one persistent launch
            UPcg a{m->rec, conn, m->rowptr, m->adj, nullptr, nullptr, u, dinv, d, r, z, pv, q, m->part, m->scal,
                   m->bar, nv, tol * tol, imaxit, p};
            e = m->dim == 2 ? launch_upcg<2>(m, a, s) : launch_upcg<3>(m, a, s);
            if (e == cudaSuccess) {
                eager = false;
                m->launches++;
                if ((e = poll()) != cudaSuccess) return cuda_fail(m, e);
                k = (int64_t)h[5];
                rn = std::sqrt(h[3]);
                if (h[4] != 0.0) rn = tol * 2.0 + 1.0;  // breakdown: counted as a linear failure below
            } else {
                cudaGetLastError();
            }
        }
        while (eager && rn > tol && k < imaxit) {
            const int slot = (int)(k & 1);
            if (m->dim == 2)
                k_umesh_Kaa2<KAA_PCG><<<gv, 256, 0, s>>>(m->rec, conn, m->rowptr, m->adj,
                                                         reinterpret_cast<const double2*>(u), pv, q, nv, p,
                                                         dinv, m->part);
            else
                k_umesh_Kaa3<KAA_PCG><<<gv, 256, 0, s>>>(m->rec, conn, m->rowptr, m->adj, u, pv, q, nv, p,
                                                         dinv, m->part);
            k_umesh_reduce<<<1, 1024, 0, s>>>(m->part, nb, 1, m->scal, 2, 2);
            k_umesh_pcg_update<<<nb, 256, 0, s>>>(d, r, z, pv, q, dinv, m->scal, m->part, nv, nb, slot);
            k_umesh_reduce<<<1, 1024, 0, s>>>(m->part, nb, 2, m->scal, slot ^ 1, 3);
            k_umesh_pcg_dir<<<nb, 256, 0, s>>>(pv, z, m->scal, nv, slot);
            m->launches += 5;
            ++k;
            if (k % 10 == 0 || k == imaxit) {
                if ((e = poll()) != cudaSuccess) return cuda_fail(m, e);
                if (h[4] != 0.0) break;
                rn = std::sqrt(h[3]);
            }
        }
        rep->total_krylov_iterations += k;
        if (rn > tol) rep->linear_failures++;
        // projected Newton step with Armijo backtracking on |Phi|^2 (vi.py:207-240); on failure a
        // steepest-descent step on the merit (vi.py:241-252); no descent along either: stall
        // (vi.py:253-254) -- a trial that fails its test is never accepted
        auto line_search = [&](const double* dir, double slope, bool newton, bool& ok) -> cudaError_t {
            ok = false;
            for (double t = 1.0; t >= tmin; t *= bt) {
                k_umesh_vi_cand<<<gv, 256, 0, s>>>(a, dir, alpha_lb, t, cand, nv);
                grad(cand);
                k_umesh_vi_prep<<<gv, 256, 0, s>>>(cand, g, alpha_lb, diag, dinv, q, m->part, nv, zeta);
                k_umesh_reduce<<<1, 1024, 0, s>>>(m->part, nb, 1, m->scal, 7, 7);
                m->launches += 4;
                cudaError_t le = poll();
                if (le != cudaSuccess) return le;
                const double mt = h[7];
                const double bound = newton ? (1.0 - 2.0 * o->armijo * t) * merit : merit - slope * t;
                if (mt <= bound) {
                    ok = true;
                    merit = mt;
                    return cudaMemcpyAsync(a, cand, nv * 8, cudaMemcpyDeviceToDevice, s);
                }
            }
            return cudaSuccess;
        };
        bool ok = false;
        if ((e = line_search(d, 0.0, true, ok)) != cudaSuccess) return cuda_fail(m, e);
        if (!ok) {
            grad(a);  // g at the current iterate (the trials overwrote it)
            k_umesh_merit_parts<<<gv, 256, 0, s>>>(a, g, alpha_lb, z, r, nv);
            if (m->dim == 2)
                k_umesh_Kaa2<KAA_APPLY><<<gv, 256, 0, s>>>(m->rec, conn, m->rowptr, m->adj,
                                                           reinterpret_cast<const double2*>(u), r, pv, nv, p);
            else
                k_umesh_Kaa3<KAA_APPLY><<<gv, 256, 0, s>>>(m->rec, conn, m->rowptr, m->adj, u, r, pv, nv, p);
            k_umesh_grad_finish<<<gv, 256, 0, s>>>(z, pv, m->part, nv);
            k_umesh_reduce<<<1, 1024, 0, s>>>(m->part, nb, 1, m->scal, 6, 6);
            m->launches += 5;
            if ((e = poll()) != cudaSuccess) return cuda_fail(m, e);
            const double gn = std::sqrt(h[6]);
            if (gn > 0.0) {
                const double sc = 1.0 / std::max(1.0, gn);
                k_scale_u<<<gv, 256, 0, s>>>(pv, -sc, nv);
                m->launches++;
                if ((e = line_search(pv, o->armijo * sc * gn * gn, false, ok)) != cudaSuccess) return cuda_fail(m, e);
                rep->steepest_descent_steps++;
            }
            if (!ok) {  // the prep buffers (dinv, rhs) must describe the current iterate again
                k_umesh_vi_prep<<<gv, 256, 0, s>>>(a, g, alpha_lb, diag, dinv, q, m->part, nv, zeta);
                m->launches++;
            }
        }
        if (!ok) break;
        record();
    }
    rep->final_residual_norm = std::sqrt(merit);
    if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return cuda_fail(m, e);
    rep->status = rep->converged ? PF_OK : PF_ESTALL;
    return PF_OK;
}

int64_t pf_umesh_launch_count(const pf_umesh* m) { return m ? m->launches : -1; }

}  // extern "C"
