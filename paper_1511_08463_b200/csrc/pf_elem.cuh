// pf_elem.cuh -- element-level helpers shared by the strip operators and the GMG setup.
#pragma once
#include "pf_internal.cuh"

namespace pf {

template <int N> struct IC { static constexpr int v = N; };

template <int PAT, class F>
__device__ __forceinline__ void for_each_elem(int /*parity*/, F&& f) {
    // f(shape, slot, nodeA, nodeB, nodeC); union-jack odd cells arrive mirrored (see mirror())
    if constexpr (PAT == PF_UNION_JACK || PAT == PF_RIGHT) {
        f(IC<0>{}, IC<0>{}, IC<0>{}, IC<1>{}, IC<3>{});
        f(IC<1>{}, IC<1>{}, IC<0>{}, IC<3>{}, IC<2>{});
    } else {
        f(IC<0>{}, IC<0>{}, IC<0>{}, IC<1>{}, IC<4>{});
        f(IC<1>{}, IC<1>{}, IC<1>{}, IC<3>{}, IC<4>{});
        f(IC<2>{}, IC<2>{}, IC<3>{}, IC<2>{}, IC<4>{});
        f(IC<3>{}, IC<3>{}, IC<2>{}, IC<0>{}, IC<4>{});
    }
}

__device__ __forceinline__ bool on_boundary(const Geo2& g, int i, int j) {
    return i == 0 || i == g.nx || j == 0 || j == g.ny;
}
__device__ __forceinline__ unsigned bcbits(const Geo2& g, int i, int j, long long v) {
    return (g.has_bc && on_boundary(g, i, j)) ? (unsigned)g.bcmask[v] : 0u;
}
__device__ __forceinline__ double cellE(const Geo2& g, long long cell) {
    return g.E_cell ? __ldg(g.E_cell + cell) : g.E;
}
__device__ __forceinline__ double cellGc(const Geo2& g, long long cell) {
    return g.Gc_cell ? __ldg(g.Gc_cell + cell) : g.Gc;
}
__device__ __forceinline__ double fbphi(double a, double b) { return hypot(a, b) - a - b; }
__device__ __forceinline__ double2 ld2(const double* p, long long v) {
    return __ldg(reinterpret_cast<const double2*>(p) + v);
}
__device__ __forceinline__ void st2(double* p, long long v, double a, double b) {
    reinterpret_cast<double2*>(p)[v] = make_double2(a, b);
}

// per-cell-row geometry: graded meshes (banded_rect_mesh, mesh.py:163-190) carry 1/hy and the
// element area per cell row J; uniform meshes use the descriptor constants (a uniform branch)
// Plain (non-volatile) loads on purpose: __ldg is volatile inline asm, so every call site issued
// its own predicated load even on uniform meshes (rowgeo == null; ncu: 13 LDG + 30 LEA per vertex
// in the crossed Kuu apply); plain loads let the compiler hoist and share them per cell.
__device__ __forceinline__ double ihy_at(const Geo2& g, int cj) { return g.rowgeo ? g.rowgeo[cj] : g.ihy; }
__device__ __forceinline__ double area_at(const Geo2& g, int cj) {
    return g.rowgeo ? g.rowgeo[g.ny + cj] : g.area[0];
}

// ---- element kernels ---------------------------------------------------------------------
// On a uniform grid every P1 gradient coefficient is a small integer times 1/hx (b, x-derivative)
// or 1/hy (c, y-derivative).  Shp<PAT, T> holds those integers per element shape, so zero terms
// vanish at compile time and +-1 / +-2 become adds; only two runtime scalings remain.
// Union-jack odd cells are x-mirrored even cells: their local nodes are permuted (0<->1, 2<->3)
// and 1/hx changes sign, which removes the parity branch (no warp divergence).
template <int PAT, int T> struct Shp;
//                                       b (times 1/hx)         c (times 1/hy)
template <> struct Shp<PF_RIGHT, 0>   { static constexpr int b0 = -1, b1 = 1, b2 = 0,  c0 = 0,  c1 = -1, c2 = 1; };
template <> struct Shp<PF_RIGHT, 1>   { static constexpr int b0 = 0,  b1 = 1, b2 = -1, c0 = -1, c1 = 0,  c2 = 1; };
template <> struct Shp<PF_UNION_JACK, 0> : Shp<PF_RIGHT, 0> {};
template <> struct Shp<PF_UNION_JACK, 1> : Shp<PF_RIGHT, 1> {};
template <> struct Shp<PF_CROSSED, 0> { static constexpr int b0 = -1, b1 = 1,  b2 = 0,  c0 = -1, c1 = -1, c2 = 2; };
template <> struct Shp<PF_CROSSED, 1> { static constexpr int b0 = 1,  b1 = 1,  b2 = -2, c0 = -1, c1 = 1,  c2 = 0; };
template <> struct Shp<PF_CROSSED, 2> { static constexpr int b0 = 1,  b1 = -1, b2 = 0,  c0 = 1,  c1 = 1,  c2 = -2; };
template <> struct Shp<PF_CROSSED, 3> { static constexpr int b0 = -1, b1 = -1, b2 = 2,  c0 = 1,  c1 = -1, c2 = 0; };

template <int K> __device__ __forceinline__ double kterm(double x) {
    if constexpr (K == 1) return x;
    else if constexpr (K == -1) return -x;
    else if constexpr (K == 2) return x + x;
    else if constexpr (K == -2) return -(x + x);
    else return (double)K * x;
}
template <int K> __device__ __forceinline__ double kadd(double acc, double x) {
    if constexpr (K == 0) return acc;
    else if constexpr (K == 1) return acc + x;
    else if constexpr (K == -1) return acc - x;
    else return fma((double)K, x, acc);
}
// K0 x0 + K1 x1 + K2 x2 with compile-time integer weights (zero terms dropped)
template <int K0, int K1, int K2>
__device__ __forceinline__ double idot(double x0, double x1, double x2) {
    if constexpr (K0 != 0) return kadd<K2>(kadd<K1>(kterm<K0>(x0), x1), x2);
    else if constexpr (K1 != 0) return kadd<K2>(kterm<K1>(x1), x2);
    else return kterm<K2>(x2);
}

template <int PAT>
__device__ __forceinline__ void mirror(int par, double (&X)[5]) {
    if constexpr (PAT == PF_UNION_JACK) {
        const double a = par ? X[1] : X[0], b = par ? X[0] : X[1];
        const double c = par ? X[3] : X[2], d = par ? X[2] : X[3];
        X[0] = a; X[1] = b; X[2] = c; X[3] = d;
    }
}

// strain (e11, e22, g12) = B u_e of shape T on nodes A, B, C; hx = +-1/hx, hy = 1/hy
template <int PAT, int T, int A, int B, int C>
__device__ __forceinline__ void strain(double hx, double hy, const double (&U1)[5], const double (&U2)[5],
                                       double& e0, double& e1, double& e2) {
    using S = Shp<PAT, T>;
    e0 = hx * idot<S::b0, S::b1, S::b2>(U1[A], U1[B], U1[C]);
    e1 = hy * idot<S::c0, S::c1, S::c2>(U2[A], U2[B], U2[C]);
    e2 = fma(hy, idot<S::c0, S::c1, S::c2>(U1[A], U1[B], U1[C]),
             hx * idot<S::b0, S::b1, S::b2>(U2[A], U2[B], U2[C]));
}
// Y_m += B_m^T (s0, s1, s2)
template <int PAT, int T, int A, int B, int C>
__device__ __forceinline__ void scatter_BT(double hx, double hy, double s0, double s1, double s2,
                                           double (&Y1)[5], double (&Y2)[5]) {
    using S = Shp<PAT, T>;
    const double x0 = s0 * hx, y2 = s2 * hy, y1 = s1 * hy, x2 = s2 * hx;
    Y1[A] = kadd<S::c0>(kadd<S::b0>(Y1[A], x0), y2);  Y2[A] = kadd<S::b0>(kadd<S::c0>(Y2[A], y1), x2);
    Y1[B] = kadd<S::c1>(kadd<S::b1>(Y1[B], x0), y2);  Y2[B] = kadd<S::b1>(kadd<S::c1>(Y2[B], y1), x2);
    Y1[C] = kadd<S::c2>(kadd<S::b2>(Y1[C], x0), y2);  Y2[C] = kadd<S::b2>(kadd<S::c2>(Y2[C], y1), x2);
}
// scalar P1 gradient of shape T and its transpose-scatter: Y_m += base + b_m gx' + c_m gy'
template <int PAT, int T, int A, int B, int C>
__device__ __forceinline__ void grad(double hx, double hy, const double (&X)[5], double& gx, double& gy) {
    using S = Shp<PAT, T>;
    gx = hx * idot<S::b0, S::b1, S::b2>(X[A], X[B], X[C]);
    gy = hy * idot<S::c0, S::c1, S::c2>(X[A], X[B], X[C]);
}
template <int PAT, int T, int A, int B, int C>
__device__ __forceinline__ void grad_scatter(double hx, double hy, double base, double fx, double fy,
                                             double (&Y)[5]) {
    using S = Shp<PAT, T>;
    const double x = fx * hx, y = fy * hy;
    Y[A] = kadd<S::c0>(kadd<S::b0>(Y[A] + base, x), y);
    Y[B] = kadd<S::c1>(kadd<S::b1>(Y[B] + base, x), y);
    Y[C] = kadd<S::c2>(kadd<S::b2>(Y[C] + base, x), y);
}
__device__ __forceinline__ void unit_stress(const Geo2& g, double e0, double e1, double e2,
                                            double& s0, double& s1, double& s2) {
    s0 = g.D00 * e0 + g.D01 * e1;
    s1 = g.D01 * e0 + g.D11 * e1;
    s2 = g.D22 * e2;
}


}  // namespace pf
