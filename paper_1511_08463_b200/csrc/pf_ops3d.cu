// pf_ops3d.cu -- matrix-free P1 operators on structured 3D Kuhn-tetrahedra meshes (sm_100a, fp64).
//
// Each hex cell (I,J,K) is split into the 6 Kuhn tetrahedra around its v000-v111 diagonal; tet
// s = the s-th permutation (a,b,c) of the axes in itertools order (oracle/meshgen.py:kuhn_paths)
// with nodes v000, v000+e_a, v000+e_a+e_b, v111.  Its barycentric gradients are
// -e_a/h_a, e_a/h_a - e_b/h_b, e_b/h_b - e_c/h_c, e_c/h_c, so every strain is three differences
// along the tet's axis path and every nodal force is a difference of three "axis fluxes".
//
// Engine (k_strip3d): a 512-thread block = 16 warps; warp w owns the vertex pencil
// j = 14*bj - 1 + w, lanes own k = 30*bk - 1 + lane (lanes 1..30 and warps 1..14 produce output),
// and the block walks vertex rows i of its strip.  Per row step:
//   * the pencil row ci+1 (and the cell data of row ci) arrive by cp.async PD steps ahead;
//   * j+1 neighbour values come from warp w+1 through shared memory (barrier A);
//   * k+1 neighbour values come from lane+1 by shuffle;
//   * contributions to k+1 go to lane+1 by shuffle, to j+1 to warp w+1 through shared memory
//     (barrier B), to i+1 are carried in registers.
// Every input is read once from HBM, every output written once, no atomics (deterministic).
// Reference formulas: fem.py:149-276 (dim-generic restatement in oracle/p1.py).
#include <type_traits>

#include "pf_internal.cuh"

namespace pf {

// Block tiling: by default 8-warp blocks, two resident per SM (128 registers).  The two blocks'
// barriers are independent, so one block's fp64 phase overlaps the other's shuffle/barrier phase:
// against one 16-warp block per SM, Kuu 128^3 0.143 -> 0.133 ms, 256^3 0.91 -> 0.82 ms; Kaa
// 128^3 0.076 -> 0.066 ms.  Register-heavy ops (Op::MINB = 1) get one 8-warp block and 255
// registers instead of spilling.  PF_K3W=16 / 8 switches the Kuu / Kaa applies for A/B runs.
constexpr int kW3 = 8;

template <class Op, class = void> struct WarpsOf { static constexpr int v = kW3; };
template <class Op> struct WarpsOf<Op, std::void_t<decltype(Op::W3)>> { static constexpr int v = Op::W3; };
template <class Op, class = void> struct MinBlocksOf { static constexpr int v = 2; };
template <class Op> struct MinBlocksOf<Op, std::void_t<decltype(Op::MINB)>> { static constexpr int v = Op::MINB; };
// an operator re-tiled: W warps per block, MB resident blocks per SM
template <class Base, int W, int MB> struct Tiled3 : Base {
    static constexpr int W3 = W, MINB = MB;
};

template <int N> struct IC3 { static constexpr int v = N; };

// the 6 Kuhn paths, itertools.permutations((0,1,2)) order
template <class F>
__device__ __forceinline__ void for_each_tet(F&& f) {
    f(IC3<0>{}, IC3<0>{}, IC3<1>{}, IC3<2>{});
    f(IC3<1>{}, IC3<0>{}, IC3<2>{}, IC3<1>{});
    f(IC3<2>{}, IC3<1>{}, IC3<0>{}, IC3<2>{});
    f(IC3<3>{}, IC3<1>{}, IC3<2>{}, IC3<0>{});
    f(IC3<4>{}, IC3<2>{}, IC3<0>{}, IC3<1>{});
    f(IC3<5>{}, IC3<2>{}, IC3<1>{}, IC3<0>{});
}
// corner index q = 4*di + 2*dj + dk ; axis bit: i -> 4, j -> 2, k -> 1
template <int AX> struct Bit { static constexpr int v = AX == 0 ? 4 : (AX == 1 ? 2 : 1); };

__device__ __forceinline__ double ihof(const Geo3& g, int ax) { return ax == 0 ? g.ihx : (ax == 1 ? g.ihy : g.ihz); }

// displacement-gradient based strain of tet (A,B,C): G[comp][axis]
template <int A, int B, int C>
__device__ __forceinline__ void tet_grad(const Geo3& g, const double (&U)[3][8], double (&G)[3][3]) {
    constexpr int q1 = Bit<A>::v, q2 = Bit<A>::v | Bit<B>::v;
    const double ha = ihof(g, A), hb = ihof(g, B), hc = ihof(g, C);
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        G[c][A] = (U[c][q1] - U[c][0]) * ha;
        G[c][B] = (U[c][q2] - U[c][q1]) * hb;
        G[c][C] = (U[c][7] - U[c][q2]) * hc;
    }
}
// Voigt strain (e11,e22,e33,g23,g13,g12) from G
__device__ __forceinline__ void voigt(const double (&G)[3][3], double (&e)[6]) {
    e[0] = G[0][0]; e[1] = G[1][1]; e[2] = G[2][2];
    e[3] = G[1][2] + G[2][1]; e[4] = G[0][2] + G[2][0]; e[5] = G[0][1] + G[1][0];
}
// unit-E isotropic stress sigma (Voigt) = D e
__device__ __forceinline__ void stress3(const Geo3& g, const double (&e)[6], double (&s)[6]) {
    const double tr = g.lam * (e[0] + e[1] + e[2]);
    s[0] = tr + 2.0 * g.mu * e[0]; s[1] = tr + 2.0 * g.mu * e[1]; s[2] = tr + 2.0 * g.mu * e[2];
    s[3] = g.mu * e[3]; s[4] = g.mu * e[4]; s[5] = g.mu * e[5];
}
// Y_m += k * B_m^T s  for tet (A,B,C): node forces from the axis fluxes F_ax = k s(:,ax) ih_ax
template <int A, int B, int C>
__device__ __forceinline__ void tet_scatter(const Geo3& g, double k, const double (&s)[6], double (&Y)[3][8]) {
    constexpr int q1 = Bit<A>::v, q2 = Bit<A>::v | Bit<B>::v;
    // sigma as 3x3: [[s0,s5,s4],[s5,s1,s3],[s4,s3,s2]]
    const double S[3][3] = {{s[0], s[5], s[4]}, {s[5], s[1], s[3]}, {s[4], s[3], s[2]}};
    const double ka = k * ihof(g, A), kb = k * ihof(g, B), kc = k * ihof(g, C);
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        const double fa = ka * S[c][A], fb = kb * S[c][B], fc = kc * S[c][C];
        Y[c][0] -= fa;
        Y[c][q1] += fa - fb;
        Y[c][q2] += fb - fc;
        Y[c][7] += fc;
    }
}
// scalar gradient of tet (A,B,C) and its transpose scatter  Y_m += base + del * grad(lam_m).g
template <int A, int B, int C>
__device__ __forceinline__ void tet_sgrad(const Geo3& g, const double (&X)[8], double (&gr)[3]) {
    constexpr int q1 = Bit<A>::v, q2 = Bit<A>::v | Bit<B>::v;
    gr[A] = (X[q1] - X[0]) * ihof(g, A);
    gr[B] = (X[q2] - X[q1]) * ihof(g, B);
    gr[C] = (X[7] - X[q2]) * ihof(g, C);
}
template <int A, int B, int C>
__device__ __forceinline__ void tet_sscatter(const Geo3& g, double base, double del, const double (&gr)[3],
                                             double (&Y)[8]) {
    constexpr int q1 = Bit<A>::v, q2 = Bit<A>::v | Bit<B>::v;
    const double fa = del * gr[A] * ihof(g, A), fb = del * gr[B] * ihof(g, B), fc = del * gr[C] * ihof(g, C);
    Y[0] += base - fa;
    Y[q1] += base + fa - fb;
    Y[q2] += base + fb - fc;
    Y[7] += base + fc;
}
template <int A, int B, int C>
__device__ __forceinline__ double tet_abar(const double (&Al)[8]) {
    constexpr int q1 = Bit<A>::v, q2 = Bit<A>::v | Bit<B>::v;
    return ((Al[0] + Al[q1]) + (Al[q2] + Al[7])) * 0.25;
}

// Degraded stiffness action of one hex, Y += sum_t s_t B_t^T D B_t U, tets grouped by their first
// axis a: the pair (a,b,c), (a,c,b) shares the first path edge (difference D1 and flux F1), the
// second and third edges are per tet.  ISO (hx = hy = hz): both 1/h factors fold into s_t, so no
// per-edge scaling at all (~280 instead of ~450 fp64 ops per hex).
template <int A, int B, int C, bool ISO>
__device__ __forceinline__ void kuu_tet(const Geo3& g, const double (&U)[3][8], const double (&Al)[8], double s07,
                                        double ve, const double (&D1)[3], double (&F1)[3], double (&Y)[3][8]) {
    constexpr int q1 = Bit<A>::v, q2 = Bit<A>::v | Bit<B>::v;
    double D2[3], D3[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        D2[i] = U[i][q2] - U[i][q1];
        D3[i] = U[i][7] - U[i][q2];
        if (!ISO) {
            D2[i] *= ihof(g, B);
            D3[i] *= ihof(g, C);
        }
    }
    const double ab = (s07 + (Al[q1] + Al[q2])) * 0.25;
    const double om = 1.0 - ab;
    const double sk = (om * om + g.kell) * ve;
    // strains in the tet's (A, B, C) axes
    const double eaa = D1[A], ebb = D2[B], ecc = D3[C];
    const double gab = D1[B] + D2[A], gac = D1[C] + D3[A], gbc = D2[C] + D3[B];
    const double lt = (sk * g.lam) * (eaa + ebb + ecc);
    const double m2 = sk * (2.0 * g.mu), m1 = sk * g.mu;
    const double saa = lt + m2 * eaa, sbb = lt + m2 * ebb, scc = lt + m2 * ecc;
    const double sab = m1 * gab, sac = m1 * gac, sbc = m1 * gbc;
    double f1[3], f2[3], f3[3];  // sigma(:, A), sigma(:, B), sigma(:, C) by component
    f1[A] = saa; f1[B] = sab; f1[C] = sac;
    f2[A] = sab; f2[B] = sbb; f2[C] = sbc;
    f3[A] = sac; f3[B] = sbc; f3[C] = scc;
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        if (!ISO) {
            f1[i] *= ihof(g, A);
            f2[i] *= ihof(g, B);
            f3[i] *= ihof(g, C);
        }
        F1[i] += f1[i];
        Y[i][q1] -= f2[i];
        Y[i][q2] += f2[i] - f3[i];
        Y[i][7] += f3[i];
    }
}
template <int A, int B, int C, bool ISO>
__device__ __forceinline__ void kuu_pair(const Geo3& g, const double (&U)[3][8], const double (&Al)[8], double s07,
                                         double ve, double (&Y)[3][8]) {
    constexpr int q1 = Bit<A>::v;
    double D1[3], F1[3] = {0.0, 0.0, 0.0};
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        D1[i] = U[i][q1] - U[i][0];
        if (!ISO) D1[i] *= ihof(g, A);
    }
    kuu_tet<A, B, C, ISO>(g, U, Al, s07, ve, D1, F1, Y);
    kuu_tet<A, C, B, ISO>(g, U, Al, s07, ve, D1, F1, Y);
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        Y[i][0] -= F1[i];
        Y[i][q1] += F1[i];
    }
}
template <bool ISO>
__device__ __forceinline__ void kuu_hex(const Geo3& g, const double (&U)[3][8], const double (&Al)[8], double Ec,
                                        double (&Y)[3][8]) {
    const double s07 = Al[0] + Al[7];
    const double ve = ISO ? g.vol * Ec * (g.ihx * g.ihx) : g.vol * Ec;
    kuu_pair<0, 1, 2, ISO>(g, U, Al, s07, ve, Y);
    kuu_pair<1, 0, 2, ISO>(g, U, Al, s07, ve, Y);
    kuu_pair<2, 0, 1, ISO>(g, U, Al, s07, ve, Y);
}

// Edge-flux form of the same action (used by Op3Kuu).  Every Kuhn path edge is a cube edge: tet
// (A,B,C) walks axis A at corner 0, axis B at corner bit(A), axis C at corner 7 - bit(C).  So the
// 12 cube-edge differences are formed once per hex (36 subtractions instead of 45), each tet adds
// its three axis fluxes to its path edges (the A edge is shared by the pair (A,B,C), (A,C,B); the C
// edge by (A,B,C), (B,A,C)), and each node force is the difference of the fluxes of its three
// edges (66 adds instead of 108).  Y is assigned, not accumulated.
template <bool ISO>
__device__ __forceinline__ void kuu_hex_e(const Geo3& g, const double (&U)[3][8], const double (&Al)[8], double Ec,
                                          double (&Y)[3][8]) {
    double D[3][8][3], F[3][8][3];  // [axis][low corner][component]; corners with the axis bit set unused
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
        const int b = ax == 0 ? 4 : (ax == 1 ? 2 : 1);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            if (q & b) continue;
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                D[ax][q][c] = U[c][q | b] - U[c][q];
                if (!ISO) D[ax][q][c] *= ihof(g, ax);
            }
        }
    }
    const double s07 = Al[0] + Al[7];
    const double ve = ISO ? g.vol * Ec * (g.ihx * g.ihx) : g.vol * Ec;
    for_each_tet([&](auto, auto A_, auto B_, auto C_) {
        constexpr int A = decltype(A_)::v, B = decltype(B_)::v, C = decltype(C_)::v;
        constexpr int q1 = Bit<A>::v, q2 = Bit<A>::v | Bit<B>::v;
        const double (&D1)[3] = D[A][0];
        const double (&D2)[3] = D[B][q1];
        const double (&D3)[3] = D[C][q2];
        const double ab = (s07 + (Al[q1] + Al[q2])) * 0.25;
        const double om = 1.0 - ab;
        const double sk = (om * om + g.kell) * ve;
        const double eaa = D1[A], ebb = D2[B], ecc = D3[C];
        const double gab = D1[B] + D2[A], gac = D1[C] + D3[A], gbc = D2[C] + D3[B];
        const double lt = (sk * g.lam) * (eaa + ebb + ecc);
        const double m2 = sk * (2.0 * g.mu), m1 = sk * g.mu;
        const double saa = lt + m2 * eaa, sbb = lt + m2 * ebb, scc = lt + m2 * ecc;
        const double sab = m1 * gab, sac = m1 * gac, sbc = m1 * gbc;
        double f1[3], f2[3], f3[3];
        f1[A] = saa; f1[B] = sab; f1[C] = sac;
        f2[A] = sab; f2[B] = sbb; f2[C] = sbc;
        f3[A] = sac; f3[B] = sbc; f3[C] = scc;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            if (B < C) F[A][0][c] = f1[c]; else F[A][0][c] += f1[c];
            F[B][q1][c] = f2[c];
            if (A < B) F[C][q2][c] = f3[c]; else F[C][q2][c] += f3[c];
        }
    });
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
        const int b = ax == 0 ? 4 : (ax == 1 ? 2 : 1);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            if (q & b) continue;
#pragma unroll
            for (int c = 0; c < 3; ++c)
                if (!ISO) F[ax][q][c] *= ihof(g, ax);
        }
    }
    // node q: + flux of each edge ending at q, - flux of each edge starting at q
#pragma unroll
    for (int q = 0; q < 8; ++q)
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const double t0 = (q & 4) ? F[0][q ^ 4][c] : -F[0][q][c];
            const double t1 = (q & 2) ? F[1][q ^ 2][c] : -F[1][q][c];
            const double t2 = (q & 1) ? F[2][q ^ 1][c] : -F[2][q][c];
            Y[c][q] = (t0 + t1) + t2;
        }
}

// ---- staging helpers (same conventions as 2D: slot q of lane l at q*256 + 8l) ------------------
__device__ __forceinline__ unsigned smem_addr3(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void cp8(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_addr3(dst)), "l"(src));
}
__device__ __forceinline__ void cp4(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(smem_addr3(dst)), "l"(src));
}
__device__ __forceinline__ void cp_commit3() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait3() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }
struct S3 {
    unsigned char* p;
    int lane;
    __device__ __forceinline__ double* d(int q) const { return reinterpret_cast<double*>(p + q * 256) + lane; }
    __device__ __forceinline__ unsigned* w(int q) const { return reinterpret_cast<unsigned*>(p + q * 256) + lane; }
    __device__ __forceinline__ S3 at(int q) const { return S3{p + q * 256, lane}; }
};
__device__ __forceinline__ void put1_3(const S3& s, int q, const double* b, long long v) { cp8(s.d(q), b + v); }
__device__ __forceinline__ void put3_3(const S3& s, int q, const double* b, long long v) {
    cp8(s.d(q), b + 3 * v); cp8(s.d(q + 1), b + 3 * v + 1); cp8(s.d(q + 2), b + 3 * v + 2);
}
__device__ __forceinline__ void putb_3(const S3& s, int q, const unsigned char* b, long long v) {
    cp4(s.w(q), b + (v & ~3LL));
}
__device__ __forceinline__ double get1_3(const S3& s, int q) { return *s.d(q); }
__device__ __forceinline__ unsigned getb_3(const S3& s, int q, long long v) {
    return (*s.w(q) >> (8 * (unsigned)(v & 3))) & 0xffu;
}

__device__ __forceinline__ long long vid3(const Geo3& g, int i, int j, int k) {
    return ((long long)i * g.nvy + j) * g.nvz + k;
}
__device__ __forceinline__ long long cid3(const Geo3& g, int i, int j, int k) {
    return ((long long)i * g.ny + j) * g.nz + k;
}
__device__ __forceinline__ bool onb3(const Geo3& g, int i, int j, int k) {
    return i == 0 || i == g.nx || j == 0 || j == g.ny || k == 0 || k == g.nz;
}
__device__ __forceinline__ unsigned bc3(const Geo3& g, int i, int j, int k, long long v) {
    return (g.has_bc && onb3(g, i, j, k)) ? (unsigned)g.bcmask[v] : 0u;
}

// ---- the 3D strip engine ----------------------------------------------------------------------
// one tile (j-block bj, k-block bk, strip bs) of the engine; `tile` plays the role of the block index
// (k_strip3d: one tile per CTA; the persistent damage PCG: tiles distributed over resident CTAs).
// One block barrier per row step: step ci computes cell row ci from the vertex rows ci / ci+1 it
// already holds, then fixes vertex row ci+2 (and cell row ci+1) from the stage ring and publishes
// both its j-carry contributions and row ci+2 in one double-buffered exchange.  (The first form
// published row ci+1 and the contributions behind two barriers per step; barrier stalls were
// the largest stall reason of the 256^3 Kuu apply.)
template <class Op, int kW3>
__device__ __forceinline__ void strip3_tile(const Geo3& g, Op& op, unsigned char* smem, int tile) {
    constexpr int kOutJ3 = kW3 - 2;  // output pencils per block
    constexpr int NV = Op::NV, NC = Op::NC, PD = Op::PD, NE = Op::NE, SV = Op::SV, SC = Op::SC;
    constexpr int STAGE = (SV + SC) * 256;
    const int w = __shfl_sync(PF_FULL, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;  // warp-uniform for the compiler
    double* vx = reinterpret_cast<double*>(smem + kW3 * PD * STAGE);   // [2][kW3][NV][32]
    double* cx = vx + 2 * kW3 * NV * 32;                                 // [2][kW3][2][NC][32]
    const int bk = tile % g.nbk;
    const int rest = tile / g.nbk;
    const int bj = rest % g.nbj;
    const int bs = rest / g.nbj;
    const int j = bj * kOutJ3 - 1 + w, k = bk * 30 - 1 + lane;
    const bool vv = j >= 0 && j <= g.ny && k >= 0 && k <= g.nz;
    const bool cv = j >= 0 && j < g.ny && k >= 0 && k < g.nz && w < kW3 - 1 && lane < 31;
    const bool ov = vv && w >= 1 && w <= kOutJ3 && lane >= 1 && lane <= 30;
    // interior tile: pencils bj*kOutJ3-1 .. +kW3-1 and lanes bk*30-1 .. +31 all strictly inside the mesh
    const bool tile_in = bj * kOutJ3 - 1 >= 1 && bj * kOutJ3 - 1 + kW3 - 1 <= g.ny - 1 &&
                         bk * 30 - 1 >= 1 && bk * 30 - 1 + 31 <= g.nz - 1;
    const bool ovf = w >= 1 && w <= kOutJ3 && lane >= 1 && lane <= 30;  // ov on an interior tile
    const int i0 = bs * g.S;
    const int i1 = min(i0 + g.S, g.nx + 1);
    const int vlast = min(i1, g.nx), clast = min(i1 - 1, g.nx - 1);
    unsigned char* wbase = smem + w * (PD * STAGE);
    double vc[NV], rc[NV], vn[NV], rn[NV], ec[NE], carry[NC];
#pragma unroll
    for (int q = 0; q < NC; ++q) carry[q] = 0.0;
    int ci = i0 - 1;
    auto issue = [&](int u, int r, int cr) {
        const S3 s{wbase + u * STAGE, lane};
        if (r <= vlast && vv) op.issue_v(g, r, j, k, s);
        if (cr >= 0 && cr <= clast && cv) op.issue_c(g, cr, j, k, s.at(SV));
        cp_commit3();
    };
    auto xv = [&](int b, int ww, int q) -> double* { return vx + ((b * kW3 + ww) * NV + q) * 32 + lane; };
    auto xc = [&](int b, int ww, int h, int q) -> double* { return cx + (((b * kW3 + ww) * 2 + h) * NC + q) * 32 + lane; };
    // row ci (synchronously through stage 0), then the ring of rows ci+1 .. ci+PD
#pragma unroll
    for (int q = 0; q < NV; ++q) vc[q] = 0.0;
    if (ci >= 0 && vv) {
        const S3 s0{wbase, lane};
        op.issue_v(g, ci, j, k, s0);
        cp_commit3();
        cp_wait3<0>();
        op.fix_v(g, ci, j, k, s0, vc);
    }
#pragma unroll
    for (int q = 0; q < NV; ++q) *xv(0, w, q) = vc[q];
    __syncthreads();
#pragma unroll
    for (int q = 0; q < NV; ++q) rc[q] = (w + 1 < kW3) ? *xv(0, w + 1, q) : 0.0;
    __syncthreads();  // every warp read row ci before stage 0 / buffer 0 are reused
#pragma unroll
    for (int u = 0; u < PD; ++u) issue(u, ci + 1 + u, ci + u);
    // row ci+1 and cell row ci from stage 0 (buffer 1)
    {
        cp_wait3<PD - 1>();
        const S3 s{wbase, lane};
#pragma unroll
        for (int q = 0; q < NV; ++q) vn[q] = 0.0;
#pragma unroll
        for (int q = 0; q < NE; ++q) ec[q] = 0.0;
        if (ci + 1 <= vlast && vv) op.fix_v(g, ci + 1, j, k, s, vn);
        if (ci >= 0 && ci < g.nx && cv) op.fix_c(g, ci, j, k, s.at(SV), ec);
#pragma unroll
        for (int q = 0; q < NV; ++q) *xv(1, w, q) = vn[q];
        __syncthreads();
#pragma unroll
        for (int q = 0; q < NV; ++q) rn[q] = (w + 1 < kW3) ? *xv(1, w + 1, q) : 0.0;
        issue(0, ci + 1 + PD, ci + PD);
    }
    int buf = 0;
    int us = 1 % PD;  // the stage holding vertex row ci+2 / cell row ci+1
    // One row step.  FAST: the tile is interior (every pencil and lane a valid vertex, none on the
    // mesh boundary) and rows ci .. ci+2 are interior rows of the strip, so the validity predicates,
    // the zero fills they guard and the Dirichlet-mask lookups (a descriptor copy with has_bc = 0)
    // drop out at compile time; the general form keeps them.
    Geo3 gi = g;
    gi.has_bc = 0;
    auto step = [&](auto fast_c) {
        constexpr bool FAST = decltype(fast_c)::v != 0;
        const Geo3& gg = FAST ? gi : g;
        const bool cell_ok = FAST ? true : (ci >= 0 && ci < g.nx && cv);
        // corners: q = 4 di + 2 dj + dk
        double X[NV][8];
#pragma unroll
        for (int q = 0; q < NV; ++q) {
            X[q][0] = vc[q]; X[q][2] = rc[q]; X[q][4] = vn[q]; X[q][6] = rn[q];
            X[q][1] = __shfl_down_sync(PF_FULL, vc[q], 1);
            X[q][3] = __shfl_down_sync(PF_FULL, rc[q], 1);
            X[q][5] = __shfl_down_sync(PF_FULL, vn[q], 1);
            X[q][7] = __shfl_down_sync(PF_FULL, rn[q], 1);
        }
        double Y[NC][8];
#pragma unroll
        for (int q = 0; q < NC; ++q)
#pragma unroll
            for (int c = 0; c < 8; ++c) Y[q][c] = 0.0;
        if (cell_ok) op.cell(gg, ci, j, k, X, ec, Y, FAST ? ovf : ((ci >= i0) && ov));
        // k-combine: T_ab = Y[ab0] + shfl_up(Y[ab1])
        double T00[NC], T01[NC], T10[NC], T11[NC];
#pragma unroll
        for (int q = 0; q < NC; ++q) {
            T00[q] = Y[q][0] + __shfl_up_sync(PF_FULL, Y[q][1], 1);
            T01[q] = Y[q][2] + __shfl_up_sync(PF_FULL, Y[q][3], 1);
            T10[q] = Y[q][4] + __shfl_up_sync(PF_FULL, Y[q][5], 1);
            T11[q] = Y[q][6] + __shfl_up_sync(PF_FULL, Y[q][7], 1);
        }
        // next rows from the ring
        cp_wait3<PD - 1>();
        const S3 s{wbase + us * STAGE, lane};
        double vnn[NV], ecn[NE];
#pragma unroll
        for (int q = 0; q < NV; ++q) vnn[q] = 0.0;
#pragma unroll
        for (int q = 0; q < NE; ++q) ecn[q] = 0.0;
        if (FAST || (ci + 2 <= vlast && vv)) op.fix_v(gg, ci + 2, j, k, s, vnn);
        if (FAST || (ci + 1 >= 0 && ci + 1 <= clast && cv)) op.fix_c(gg, ci + 1, j, k, s.at(SV), ecn);
        // one exchange: j-carry contributions of row ci and vertex row ci+2
#pragma unroll
        for (int q = 0; q < NC; ++q) {
            *xc(buf, w, 0, q) = T01[q];
            *xc(buf, w, 1, q) = T11[q];
        }
#pragma unroll
        for (int q = 0; q < NV; ++q) *xv(buf, w, q) = vnn[q];
        __syncthreads();
        double tot[NC];
#pragma unroll
        for (int q = 0; q < NC; ++q) {
            const double l01 = w > 0 ? *xc(buf, w - 1, 0, q) : 0.0;
            const double l11 = w > 0 ? *xc(buf, w - 1, 1, q) : 0.0;
            tot[q] = carry[q] + T00[q] + l01;
            carry[q] = T10[q] + l11;
        }
        double rnn[NV];
#pragma unroll
        for (int q = 0; q < NV; ++q) rnn[q] = (w + 1 < kW3) ? *xv(buf, w + 1, q) : 0.0;
        if (FAST ? ovf : (ci >= i0 && ov)) op.out(gg, ci, j, k, tot, vc);
#pragma unroll
        for (int q = 0; q < NV; ++q) { vc[q] = vn[q]; rc[q] = rn[q]; vn[q] = vnn[q]; rn[q] = rnn[q]; }
#pragma unroll
        for (int q = 0; q < NE; ++q) ec[q] = ecn[q];
        issue(us, ci + 2 + PD, ci + 1 + PD);
        us = us + 1 == PD ? 0 : us + 1;
        buf ^= 1;
        ++ci;
    };
    // fast rounds of three steps (the row registers rotate with period 3: no moves): rows ci .. ci+4
    // interior and owned, i.e. ci >= max(i0, 1) and ci + 4 <= min(vlast, nx - 1), ci + 3 <= clast
    const int flo = max(i0, 1), fhi = min(min(vlast, g.nx - 1) - 4, clast - 3);
    while (ci < i1) {
        if (tile_in && ci >= flo && ci <= fhi) {
            step(IC3<1>{});
            step(IC3<1>{});
            step(IC3<1>{});
        } else {
            step(IC3<0>{});
        }
    }
    cp_wait3<0>();
}

template <class Op, int kW3, int kMinB>
__global__ void __launch_bounds__(kW3 * 32, kMinB) k_strip3d(const Geo3 g, Op op) {
    extern __shared__ __align__(16) unsigned char smem[];
    if (!op.enter()) return;
    strip3_tile<Op, kW3>(g, op, smem, blockIdx.x);
    op.finish();
}

template <class Op, int kW3>
static constexpr int strip3_smem() {
    return kW3 * Op::PD * (Op::SV + Op::SC) * 256 + 2 * (kW3 * Op::NV * 32 * 8 + kW3 * 2 * Op::NC * 32 * 8);
}

struct NoRed3 {
    __device__ bool enter() const { return true; }
    __device__ void finish() {}
};
__device__ __forceinline__ double getE3(const Geo3& g, const S3& s, int q) { return g.E_cell ? get1_3(s, q) : g.E; }
__device__ __forceinline__ double getGc3(const Geo3& g, const S3& s, int q) { return g.Gc_cell ? get1_3(s, q) : g.Gc; }
__device__ __forceinline__ void putE3(const Geo3& g, const S3& s, int q, long long c) { if (g.E_cell) put1_3(s, q, g.E_cell, c); }
__device__ __forceinline__ void putGc3(const Geo3& g, const S3& s, int q, long long c) { if (g.Gc_cell) put1_3(s, q, g.Gc_cell, c); }

// ================================================================================================
// Kuu (plain or fused CG step A).  vertex slots: x|z (3), [p_in (3)], alpha ; cell: E
// ================================================================================================
template <bool FUSED, bool ISO = false>
struct Op3Kuu {
    static constexpr int NV = 4, NC = 3, PD = 3, NE = 1, SV = FUSED ? 7 : 4, SC = 1;
    const double* alpha;
    const double* x;
    const double* pin;
    double* pout;
    double* y;
    int bcmode;
    double* scal;
    RedBuf rb;
    double acc;
    __device__ bool enter() const { return !FUSED || (scal[S_DONE] == 0.0 && scal[S_FAIL] == 0.0); }
    __device__ __forceinline__ double beta() const { return scal[S_ITER] > 0.0 ? scal[S_BETA] : 0.0; }
    __device__ void issue_v(const Geo3& g, int i, int j, int k, const S3& s) const {
        const long long v = vid3(g, i, j, k);
        put3_3(s, 0, x, v);
        if (FUSED) { put3_3(s, 3, pin, v); put1_3(s, 6, alpha, v); }
        else put1_3(s, 3, alpha, v);
    }
    __device__ void fix_v(const Geo3& g, int i, int j, int k, const S3& s, double (&v)[NV]) const {
        const unsigned m = bcmode ? bc3(g, i, j, k, vid3(g, i, j, k)) : 0u;
        const double b = FUSED ? beta() : 0.0;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            double xv = get1_3(s, c);
            if (FUSED) xv += b * get1_3(s, 3 + c);
            v[c] = ((m >> c) & 1u) ? 0.0 : xv;
        }
        v[3] = get1_3(s, FUSED ? 6 : 3);
    }
    __device__ void issue_c(const Geo3& g, int ci, int j, int k, const S3& s) const { putE3(g, s, 0, cid3(g, ci, j, k)); }
    __device__ void fix_c(const Geo3& g, int, int, int, const S3& s, double (&e)[NE]) const { e[0] = getE3(g, s, 0); }
    __device__ void cell(const Geo3& g, int, int, int, const double (&X)[NV][8], const double (&ec)[NE],
                         double (&Y)[NC][8], bool) {
        const double (&U)[3][8] = *reinterpret_cast<const double(*)[3][8]>(&X[0][0]);
        kuu_hex_e<ISO>(g, U, X[3], ec[0], Y);
    }
    __device__ __forceinline__ double xval(const Geo3&, long long v, int c) const {
        double z = __ldg(x + 3 * v + c);
        if (FUSED) z += beta() * __ldg(pin + 3 * v + c);
        return z;
    }
    __device__ void out(const Geo3& g, int i, int j, int k, const double (&t)[NC], const double (&v)[NV]) {
        const long long id = vid3(g, i, j, k);
        const unsigned m = bcmode ? bc3(g, i, j, k, id) : 0u;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            double yy = t[c], p = v[c];
            if ((m >> c) & 1u) { p = xval(g, id, c); yy = p; }
            y[3 * id + c] = yy;
            if (FUSED) { pout[3 * id + c] = p; acc += p * yy; }
        }
    }
    __device__ void finish() {
        if (!FUSED) return;
        double vv[1] = {acc};
        double* s = scal;
        grid_reduce<1>(vv, rb, 0, [s](double* tot) {
            s[S_PAP] = tot[0];
            if (!(tot[0] > 0.0)) s[S_FAIL] = 1.0;
            else s[S_GAMMA] = s[S_RZ] / tot[0];
        });
    }
};

// Kuu with a multigrid-smoother epilogue: pf_gmg3.cu's pointwise Chebyshev / residual steps run
// in the apply's output stage instead of as separate vector passes.  The 3D apply is fp64- and
// latency-bound (~0.15 of HBM), so the epilogue's vector bytes ride along almost for free; the
// V-cycle saves the w = K d round trip and one launch per step.  w below is the apply's output
// (identity rows for eliminated dofs), p its input at the vertex.
//   E3_CHEB        r = res - D w ; dn = a p + b r ; res = r ; dnext = dn ; x += [p +] dn
//   E3_CHEB_B      first step from x = 0: the input p = (D b)/theta is formed on the fly (the
//                  separate k3_cheb0 pass disappears) ; r = D b - D w ; x = p + dn
//   E3_RESID       res = b - w
//   E3_RESID_CHEB0 r = D (b - w) ; res = r ; dnext = r/theta (x += dnext is deferred to the next
//                  E3_CHEB step, "pending": the input x cannot be written while it is read)
template <int EPI, bool ISO>
struct Op3KuuSm : Op3Kuu<false, ISO> {
    using Base = Op3Kuu<false, ISO>;
    static constexpr int SV = EPI == E3_CHEB_B ? 7 : 4;

    const double* b;
    const double* dinv;
    double* res;
    double* dnext;
    double* xs;
    const double* live;
    const double* lam;
    double ratio;
    int k;
    int pending;
    double th, ca, cb;
    __device__ bool enter() {
        if (live && !(live[S_DONE] == 0.0 && live[S_FAIL] == 0.0)) return false;
        const Cheb c = cheb_of(lam, ratio);
        th = c.theta;
        ca = cb = 0.0;
        if (EPI == E3_CHEB || EPI == E3_CHEB_B) cheb_ab(c, k, ca, cb);
        return true;
    }
    __device__ void issue_v(const Geo3& g, int i, int j, int k_, const S3& s) const {
        if (EPI != E3_CHEB_B) { Base::issue_v(g, i, j, k_, s); return; }
        const long long v = vid3(g, i, j, k_);
        put3_3(s, 0, b, v);
        put3_3(s, 3, dinv, v);
        put1_3(s, 6, this->alpha, v);
    }
    __device__ void fix_v(const Geo3& g, int i, int j, int k_, const S3& s, double (&v)[4]) const {
        if (EPI != E3_CHEB_B) { Base::fix_v(g, i, j, k_, s, v); return; }
        const unsigned m = this->bcmode ? bc3(g, i, j, k_, vid3(g, i, j, k_)) : 0u;
#pragma unroll
        for (int c = 0; c < 3; ++c) v[c] = ((m >> c) & 1u) ? 0.0 : (get1_3(s, 3 + c) * get1_3(s, c)) / th;
        v[3] = get1_3(s, 6);
    }
    __device__ void out(const Geo3& g, int i, int j, int k_, const double (&t)[3], const double (&v)[4]) {
        const long long id = vid3(g, i, j, k_);
        const unsigned m = this->bcmode ? bc3(g, i, j, k_, id) : 0u;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const long long q = 3 * id + c;
            double w = t[c], p = v[c];
            if ((m >> c) & 1u) {
                p = EPI == E3_CHEB_B ? (__ldg(dinv + q) * __ldg(b + q)) / th : __ldg(this->x + q);
                w = p;
            }
            if (EPI == E3_RESID) {
                res[q] = __ldg(b + q) - w;
            } else if (EPI == E3_RESID_CHEB0) {
                const double r = __ldg(dinv + q) * (__ldg(b + q) - w);
                res[q] = r;
                dnext[q] = r / th;
            } else {
                const double dq = __ldg(dinv + q);
                const double r = (EPI == E3_CHEB_B ? dq * __ldg(b + q) : res[q]) - dq * w;
                const double dn = ca * p + cb * r;
                res[q] = r;
                dnext[q] = dn;
                if (EPI == E3_CHEB_B) xs[q] = p + dn;
                else xs[q] = pending ? (xs[q] + p) + dn : xs[q] + dn;
            }
        }
    }
};

// diag(Kuu) -> dinv (eliminated rows 1).  vertex: alpha ; cell: E
struct Op3KuuDiag : NoRed3 {
    static constexpr int NV = 1, NC = 3, PD = 3, NE = 1, SV = 1, SC = 1;
    const double* alpha;
    double* dinv;
    __device__ void issue_v(const Geo3& g, int i, int j, int k, const S3& s) const { put1_3(s, 0, alpha, vid3(g, i, j, k)); }
    __device__ void fix_v(const Geo3&, int, int, int, const S3& s, double (&v)[NV]) const { v[0] = get1_3(s, 0); }
    __device__ void issue_c(const Geo3& g, int ci, int j, int k, const S3& s) const { putE3(g, s, 0, cid3(g, ci, j, k)); }
    __device__ void fix_c(const Geo3& g, int, int, int, const S3& s, double (&e)[NE]) const { e[0] = getE3(g, s, 0); }
    __device__ void cell(const Geo3& g, int, int, int, const double (&X)[NV][8], const double (&ec)[NE],
                         double (&Y)[NC][8], bool) {
        for_each_tet([&](auto, auto A, auto B, auto C) {
            const double ab = tet_abar<A.v, B.v, C.v>(X[0]);
            const double om = 1.0 - ab;
            const double s = (om * om + g.kell) * g.vol * ec[0];
            constexpr int q1 = Bit<A.v>::v, q2 = Bit<A.v>::v | Bit<B.v>::v;
            const double ha = ihof(g, A.v), hb = ihof(g, B.v), hc = ihof(g, C.v);
            // grad lambda per node: (axis weights); diag block entry for comp c:
            // |grad|^2 mu + (lam + mu) grad_c^2
            auto add = [&](int q, double ga, double gb, double gc) {
                double gr[3] = {0, 0, 0};
                gr[A.v] = ga; gr[B.v] = gb; gr[C.v] = gc;
                const double n2 = gr[0] * gr[0] + gr[1] * gr[1] + gr[2] * gr[2];
                for (int c = 0; c < 3; ++c) Y[c][q] += s * (g.mu * n2 + (g.lam + g.mu) * gr[c] * gr[c]);
            };
            add(0, -ha, 0.0, 0.0);
            add(q1, ha, -hb, 0.0);
            add(q2, 0.0, hb, -hc);
            add(7, 0.0, 0.0, hc);
        });
    }
    __device__ void out(const Geo3& g, int i, int j, int k, const double (&t)[NC], const double (&)[NV]) {
        const long long id = vid3(g, i, j, k);
        const unsigned m = bc3(g, i, j, k, id);
        for (int c = 0; c < 3; ++c) dinv[3 * id + c] = ((m >> c) & 1u) ? 1.0 : 1.0 / t[c];
    }
};

// ================================================================================================
// Damage block: kappa_e = (q + [AT2] 2 kc/ell) |T| / 16 ; c_v = sum_e |T|/4 (-q + [AT1] kc/ell)
// vertex: u (3) ; cell: E, Gc
// ================================================================================================
struct Op3Kappa : NoRed3 {
    static constexpr int NV = 3, NC = 1, PD = 3, NE = 2, SV = 3, SC = 2;
    const double* u;
    double* kappa;
    double* cvec;
    __device__ void issue_v(const Geo3& g, int i, int j, int k, const S3& s) const { put3_3(s, 0, u, vid3(g, i, j, k)); }
    __device__ void fix_v(const Geo3&, int, int, int, const S3& s, double (&v)[NV]) const {
        v[0] = get1_3(s, 0); v[1] = get1_3(s, 1); v[2] = get1_3(s, 2);
    }
    __device__ void issue_c(const Geo3& g, int ci, int j, int k, const S3& s) const {
        const long long c = cid3(g, ci, j, k);
        putE3(g, s, 0, c);
        putGc3(g, s, 1, c);
    }
    __device__ void fix_c(const Geo3& g, int, int, int, const S3& s, double (&e)[NE]) const {
        e[0] = getE3(g, s, 0);
        e[1] = getGc3(g, s, 1);
    }
    __device__ void cell(const Geo3& g, int ci, int j, int k, const double (&X)[NV][8], const double (&ec)[NE],
                         double (&Y)[NC][8], bool own) {
        const double (&U)[3][8] = *reinterpret_cast<const double(*)[3][8]>(&X[0][0]);
        const long long cell = cid3(g, ci, j, k);
        const double kc = ec[1] / g.cw;
        for_each_tet([&](auto S, auto A, auto B, auto C) {
            double G[3][3], e[6], sg[6];
            tet_grad<A.v, B.v, C.v>(g, U, G);
            voigt(G, e);
            stress3(g, e, sg);
            const double q = ec[0] * (e[0] * sg[0] + e[1] * sg[1] + e[2] * sg[2] + e[3] * sg[3] + e[4] * sg[4] +
                                      e[5] * sg[5]);
            const double kap = (q + (g.at2 ? 2.0 * kc / g.ell : 0.0)) * g.vol * (1.0 / 16.0);
            const double cc = g.vol * 0.25 * (-q + (g.at2 ? 0.0 : kc / g.ell));
            constexpr int q1 = Bit<A.v>::v, q2 = Bit<A.v>::v | Bit<B.v>::v;
            Y[0][0] += cc; Y[0][q1] += cc; Y[0][q2] += cc; Y[0][7] += cc;
            if (own) kappa[(long long)S.v * g.ncell + cell] = kap;
        });
    }
    __device__ void out(const Geo3& g, int i, int j, int k, const double (&t)[NC], const double (&)[NV]) {
        cvec[vid3(g, i, j, k)] = t[0];
    }
};

template <int A, int B, int C>
__device__ __forceinline__ void elem3_kaa(const Geo3& g, double kap, double kc, const double (&X)[8], double (&Y)[8]) {
    constexpr int q1 = Bit<A>::v, q2 = Bit<A>::v | Bit<B>::v;
    const double del = 2.0 * kc * g.ell * g.vol;
    double gr[3];
    tet_sgrad<A, B, C>(g, X, gr);
    tet_sscatter<A, B, C>(g, kap * ((X[0] + X[q1]) + (X[q2] + X[7])), del, gr, Y);
}

// Kaa apply (plain / fused CG / masked).  vertex: x|z, [p_in], [act word] ; cell: Gc, kappa x 6
template <bool FUSED, bool MASKED>
struct Op3Kaa {
    static constexpr int NV = 1, NC = 1, PD = 4, NE = 7;
    static constexpr int SV = 1 + (FUSED ? 1 : 0) + (MASKED ? 1 : 0), SC = 7;
    const double* kappa;
    const double* x;
    const double* pin;
    double* pout;
    double* y;
    const unsigned char* act;
    double* scal;
    RedBuf rb;
    double acc;
    double breg = 0.0;  // persistent PCG (k_pcg_kaa3): beta held in a register instead of scal[S_BETA]
    int use_breg = 0;
    __device__ bool enter() const { return !FUSED || (scal[S_DONE] == 0.0 && scal[S_FAIL] == 0.0); }
    __device__ __forceinline__ double bval() const {
        if (use_breg) return breg;
        return scal[S_ITER] > 0.0 ? scal[S_BETA] : 0.0;
    }
    __device__ void issue_v(const Geo3& g, int i, int j, int k, const S3& s) const {
        const long long v = vid3(g, i, j, k);
        put1_3(s, 0, x, v);
        if (FUSED) put1_3(s, 1, pin, v);
        if (MASKED) putb_3(s, FUSED ? 2 : 1, act, v);
    }
    __device__ void fix_v(const Geo3& g, int i, int j, int k, const S3& s, double (&v)[NV]) const {
        double z = get1_3(s, 0);
        if (FUSED) z += bval() * get1_3(s, 1);
        const bool a = MASKED && getb_3(s, FUSED ? 2 : 1, vid3(g, i, j, k)) != 0u;
        v[0] = a ? 0.0 : z;
    }
    __device__ void issue_c(const Geo3& g, int ci, int j, int k, const S3& s) const {
        const long long c = cid3(g, ci, j, k);
        putGc3(g, s, 0, c);
#pragma unroll
        for (int t = 0; t < 6; ++t) put1_3(s, 1 + t, kappa, (long long)t * g.ncell + c);
    }
    __device__ void fix_c(const Geo3& g, int, int, int, const S3& s, double (&e)[NE]) const {
        e[0] = getGc3(g, s, 0);
#pragma unroll
        for (int t = 0; t < 6; ++t) e[1 + t] = get1_3(s, 1 + t);
    }
    __device__ void cell(const Geo3& g, int, int, int, const double (&X)[NV][8], const double (&ec)[NE],
                         double (&Y)[NC][8], bool) {
        const double kc = ec[0] / g.cw;
        for_each_tet([&](auto S, auto A, auto B, auto C) { elem3_kaa<A.v, B.v, C.v>(g, ec[1 + S.v], kc, X[0], Y[0]); });
    }
    __device__ void out(const Geo3& g, int i, int j, int k, const double (&t)[NC], const double (&v)[NV]) {
        const long long id = vid3(g, i, j, k);
        double yy = t[0], p = v[0];
        if (MASKED && act[id]) {
            p = __ldg(x + id);
            if (FUSED) p += bval() * __ldg(pin + id);
            yy = p;
        }
        y[id] = yy;
        if (FUSED) { pout[id] = p; acc += p * yy; }
    }
    __device__ void finish() {
        if (!FUSED) return;
        double vv[1] = {acc};
        double* s = scal;
        grid_reduce<1>(vv, rb, 0, [s](double* tot) {
            s[S_PAP] = tot[0];
            if (!(tot[0] > 0.0)) s[S_FAIL] = 1.0;
            else s[S_GAMMA] = s[S_RZ] / tot[0];
        });
    }
};

template <bool MASKED>
struct Op3KaaDiag : NoRed3 {
    static constexpr int NV = 1, NC = 1, PD = 3, NE = 7, SV = 0, SC = 7;
    const double* kappa;
    double* dinv;
    const unsigned char* act;
    __device__ void issue_v(const Geo3&, int, int, int, const S3&) const {}
    __device__ void fix_v(const Geo3&, int, int, int, const S3&, double (&v)[NV]) const { v[0] = 0.0; }
    __device__ void issue_c(const Geo3& g, int ci, int j, int k, const S3& s) const {
        const long long c = cid3(g, ci, j, k);
        putGc3(g, s, 0, c);
        for (int t = 0; t < 6; ++t) put1_3(s, 1 + t, kappa, (long long)t * g.ncell + c);
    }
    __device__ void fix_c(const Geo3& g, int, int, int, const S3& s, double (&e)[NE]) const {
        e[0] = getGc3(g, s, 0);
        for (int t = 0; t < 6; ++t) e[1 + t] = get1_3(s, 1 + t);
    }
    __device__ void cell(const Geo3& g, int, int, int, const double (&)[NV][8], const double (&ec)[NE],
                         double (&Y)[NC][8], bool) {
        const double kc = ec[0] / g.cw;
        for_each_tet([&](auto S, auto A, auto B, auto C) {
            constexpr int q1 = Bit<A.v>::v, q2 = Bit<A.v>::v | Bit<B.v>::v;
            const double del = 2.0 * kc * g.ell * g.vol;
            const double ha = ihof(g, A.v), hb = ihof(g, B.v), hc = ihof(g, C.v);
            const double kap = ec[1 + S.v];
            Y[0][0] += kap + del * ha * ha;
            Y[0][q1] += kap + del * (ha * ha + hb * hb);
            Y[0][q2] += kap + del * (hb * hb + hc * hc);
            Y[0][7] += kap + del * hc * hc;
        });
    }
    __device__ void out(const Geo3& g, int i, int j, int k, const double (&t)[NC], const double (&)[NV]) {
        const long long id = vid3(g, i, j, k);
        dinv[id] = (MASKED && act[id]) ? 1.0 : 1.0 / t[0];
    }
};

// VI line-search trial: trial = clip(x + mu d, lb, 1) ; F = Kaa trial + c ; merit
struct Op3KaaTrial {
    static constexpr int NV = 1, NC = 1, PD = 3, NE = 7, SV = 3, SC = 7;
    const double* kappa;
    const double* cvec;
    const double* x;
    const double* d;
    const double* lb;
    double* trial;
    double* F;
    double* scal;
    int merit_slot;
    RedBuf rb;
    double acc_m;
    __device__ bool enter() const { return true; }
    __device__ void issue_v(const Geo3& g, int i, int j, int k, const S3& s) const {
        const long long v = vid3(g, i, j, k);
        put1_3(s, 0, x, v);
        if (d) { put1_3(s, 1, d, v); put1_3(s, 2, lb, v); }
    }
    __device__ void fix_v(const Geo3&, int, int, int, const S3& s, double (&v)[NV]) const {
        const double xv = get1_3(s, 0);
        v[0] = d ? fmin(fmax(xv + scal[S_MU] * get1_3(s, 1), get1_3(s, 2)), 1.0) : xv;
    }
    __device__ void issue_c(const Geo3& g, int ci, int j, int k, const S3& s) const {
        const long long c = cid3(g, ci, j, k);
        putGc3(g, s, 0, c);
        for (int t = 0; t < 6; ++t) put1_3(s, 1 + t, kappa, (long long)t * g.ncell + c);
    }
    __device__ void fix_c(const Geo3& g, int, int, int, const S3& s, double (&e)[NE]) const {
        e[0] = getGc3(g, s, 0);
        for (int t = 0; t < 6; ++t) e[1 + t] = get1_3(s, 1 + t);
    }
    __device__ void cell(const Geo3& g, int, int, int, const double (&X)[NV][8], const double (&ec)[NE],
                         double (&Y)[NC][8], bool) {
        const double kc = ec[0] / g.cw;
        for_each_tet([&](auto S, auto A, auto B, auto C) { elem3_kaa<A.v, B.v, C.v>(g, ec[1 + S.v], kc, X[0], Y[0]); });
    }
    __device__ void out(const Geo3& g, int i, int j, int k, const double (&t)[NC], const double (&v)[NV]) {
        const long long id = vid3(g, i, j, k);
        const double Fv = t[0] + __ldg(cvec + id), tv = v[0], l = __ldg(lb + id);
        trial[id] = tv;
        F[id] = Fv;
        const double ph = (hypot(tv - l, hypot(1.0 - tv, -Fv) - (1.0 - tv) + Fv) - (tv - l) -
                           (hypot(1.0 - tv, -Fv) - (1.0 - tv) + Fv));
        acc_m += ph * ph;
    }
    __device__ void finish() {
        double vv[1] = {acc_m};
        double* s = scal;
        const int ms = merit_slot;
        grid_reduce<1>(vv, rb, 1, [s, ms](double* tot) { s[ms] = tot[0]; });
    }
};

// ================================================================================================
// Physics pass (energies, r_u, r_alpha, Phi, norms).  vertex: u (3), alpha ; cell: E, Gc
// ================================================================================================
template <int ROWS>
struct Op3Phys {
    static constexpr int NV = 4, NC = 4, PD = 2, NE = 2, SV = 4, SC = 2, MINB = 1;
    const double* u;
    const double* alpha;
    const double* lb;
    double* ru;
    double* ra;
    double* phi;
    double* scal;
    RedBuf rb;
    double eel, ed, nru, nphi;
    __device__ bool enter() const { return true; }
    __device__ void issue_v(const Geo3& g, int i, int j, int k, const S3& s) const {
        const long long v = vid3(g, i, j, k);
        put3_3(s, 0, u, v);
        put1_3(s, 3, alpha, v);
    }
    __device__ void fix_v(const Geo3&, int, int, int, const S3& s, double (&v)[NV]) const {
        for (int q = 0; q < 4; ++q) v[q] = get1_3(s, q);
    }
    __device__ void issue_c(const Geo3& g, int ci, int j, int k, const S3& s) const {
        const long long c = cid3(g, ci, j, k);
        putE3(g, s, 0, c);
        putGc3(g, s, 1, c);
    }
    __device__ void fix_c(const Geo3& g, int, int, int, const S3& s, double (&e)[NE]) const {
        e[0] = getE3(g, s, 0);
        e[1] = getGc3(g, s, 1);
    }
    __device__ void cell(const Geo3& g, int, int, int, const double (&X)[NV][8], const double (&ec)[NE],
                         double (&Y)[NC][8], bool own) {
        const double (&U)[3][8] = *reinterpret_cast<const double(*)[3][8]>(&X[0][0]);
        double (&YU)[3][8] = *reinterpret_cast<double(*)[3][8]>(&Y[0][0]);
        // edge-flux form (see kuu_hex_e): the 12 cube-edge differences of u and alpha are formed
        // once per hex; each tet adds its axis fluxes to its three path edges and its nodal source
        // to its four nodes; node forces are edge-flux differences.  Y is assigned.
        const double (&Al)[8] = X[3];
        const double Ec = ec[0], kc = ec[1] / g.cw;
        const double del = 2.0 * kc * g.ell * g.vol;
        double D[3][8][3], Da[3][8], F[3][8][3], Fa[3][8];
#pragma unroll
        for (int ax = 0; ax < 3; ++ax) {
            const int b = ax == 0 ? 4 : (ax == 1 ? 2 : 1);
            const double ih = ihof(g, ax);
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                if (q & b) continue;
#pragma unroll
                for (int c = 0; c < 3; ++c) D[ax][q][c] = (U[c][q | b] - U[c][q]) * ih;
                Da[ax][q] = (Al[q | b] - Al[q]) * ih;
            }
        }
        double n_all = 0.0, n_q1[3], n_q2[3];  // nodal sources: nodes 0 and 7 / single-bit / two-bit
        for_each_tet([&](auto, auto A_, auto B_, auto C_) {
            constexpr int A = decltype(A_)::v, B = decltype(B_)::v, C = decltype(C_)::v;
            constexpr int q1 = Bit<A>::v, q2 = Bit<A>::v | Bit<B>::v;
            const double ab = ((Al[0] + Al[q1]) + (Al[q2] + Al[7])) * 0.25;
            const double om = 1.0 - ab;
            const double a = om * om + g.kell, ap = -2.0 * om;
            const double w = g.at2 ? ab * ab : ab, wp = g.at2 ? 2.0 * ab : 1.0;
            const double (&D1)[3] = D[A][0];
            const double (&D2)[3] = D[B][q1];
            const double (&D3)[3] = D[C][q2];
            const double eaa = D1[A], ebb = D2[B], ecc = D3[C];
            const double gab = D1[B] + D2[A], gac = D1[C] + D3[A], gbc = D2[C] + D3[B];
            const double lt = g.lam * (eaa + ebb + ecc);
            const double saa = lt + 2.0 * g.mu * eaa, sbb = lt + 2.0 * g.mu * ebb, scc = lt + 2.0 * g.mu * ecc;
            const double sab = g.mu * gab, sac = g.mu * gac, sbc = g.mu * gbc;
            const double q = Ec * (eaa * saa + ebb * sbb + ecc * scc + gab * sab + gac * sac + gbc * sbc);
            const double kk = a * g.vol * Ec;
            double f1[3], f2[3], f3[3];
            f1[A] = kk * saa; f1[B] = kk * sab; f1[C] = kk * sac;
            f2[A] = kk * sab; f2[B] = kk * sbb; f2[C] = kk * sbc;
            f3[A] = kk * sac; f3[B] = kk * sbc; f3[C] = kk * scc;
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                if (B < C) F[A][0][c] = f1[c]; else F[A][0][c] += f1[c];
                F[B][q1][c] = f2[c];
                if (A < B) F[C][q2][c] = f3[c]; else F[C][q2][c] += f3[c];
            }
            const double ga = Da[A][0], gb = Da[B][q1], gc = Da[C][q2];
            if (B < C) Fa[A][0] = del * ga; else Fa[A][0] += del * ga;
            Fa[B][q1] = del * gb;
            if (A < B) Fa[C][q2] = del * gc; else Fa[C][q2] += del * gc;
            const double nod = (0.5 * ap * q + kc * wp / g.ell) * g.vol * 0.25;
            if (A == 0 && B == 1) n_all = nod; else n_all += nod;
            if (B < C) n_q1[A] = nod; else n_q1[A] += nod;
            if (A < B) n_q2[C] = nod; else n_q2[C] += nod;
            if (own) {
                eel += 0.5 * g.vol * a * q;
                ed += g.vol * kc * (w / g.ell + g.ell * (ga * ga + gb * gb + gc * gc));
            }
        });
#pragma unroll
        for (int ax = 0; ax < 3; ++ax) {
            const int b = ax == 0 ? 4 : (ax == 1 ? 2 : 1);
            const double ih = ihof(g, ax);
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                if (q & b) continue;
#pragma unroll
                for (int c = 0; c < 3; ++c) F[ax][q][c] *= ih;
                Fa[ax][q] *= ih;
            }
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) {
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                const double t0 = (q & 4) ? F[0][q ^ 4][c] : -F[0][q][c];
                const double t1 = (q & 2) ? F[1][q ^ 2][c] : -F[1][q][c];
                const double t2 = (q & 1) ? F[2][q ^ 1][c] : -F[2][q][c];
                YU[c][q] = (t0 + t1) + t2;
            }
            const double t0 = (q & 4) ? Fa[0][q ^ 4] : -Fa[0][q];
            const double t1 = (q & 2) ? Fa[1][q ^ 2] : -Fa[1][q];
            const double t2 = (q & 1) ? Fa[2][q ^ 1] : -Fa[2][q];
            // nodal source: nodes 0 and 7 in all six tets; node bit(A) in the two tets with first
            // axis A; node 7 - bit(C) in the two tets with last axis C
            const int nb = __popc(q);
            const double src = (nb == 0 || nb == 3) ? n_all
                             : (nb == 1 ? n_q1[q == 4 ? 0 : (q == 2 ? 1 : 2)] : n_q2[q == 3 ? 0 : (q == 5 ? 1 : 2)]);
            Y[3][q] = src + ((t0 + t1) + t2);
        }
    }
    __device__ void out(const Geo3& g, int i, int j, int k, const double (&t)[NC], const double (&v)[NV]) {
        const long long id = vid3(g, i, j, k);
        const unsigned m = bc3(g, i, j, k, id);
        double r[3] = {t[0], t[1], t[2]};
        for (int c = 0; c < 3; ++c) {
            if ((m >> c) & 1u) {
                if (ROWS == PF_ROWS_ZERO) r[c] = 0.0;
                else if (ROWS == PF_ROWS_VALUE) r[c] = __ldg(u + 3 * id + c) - __ldg(g.ubar + 3 * id + c);
            }
            if (ru) ru[3 * id + c] = r[c];
            nru += r[c] * r[c];
        }
        if (ra) ra[id] = t[3];
        if (lb) {
            const double av = v[3], rav = t[3];
            const double inner = hypot(1.0 - av, -rav) - (1.0 - av) + rav;
            const double ph = hypot(av - __ldg(lb + id), inner) - (av - __ldg(lb + id)) - inner;
            if (phi) phi[id] = ph;
            nphi += ph * ph;
        }
    }
    __device__ void finish() {
        double vv[4] = {eel, ed, nru, nphi};
        double* s = scal;
        grid_reduce<4>(vv, rb, 2, [s](double* tot) {
            s[S_PHYS0 + 0] = tot[0]; s[S_PHYS0 + 1] = tot[1]; s[S_PHYS0 + 2] = tot[2]; s[S_PHYS0 + 3] = tot[3];
        });
    }
};

// Elastic right-hand side b = -M r_raw(g) + (I - M) ubar (or the load f).  vertex: alpha ; cell: E
template <bool LOADONLY>
struct Op3Rhs {
    static constexpr int NV = 4, NC = 3, PD = 3, NE = 1, SV = 1, SC = 1;
    const double* alpha;
    double* b;
    double* scal;
    RedBuf rb;
    double acc;
    __device__ bool enter() const { return true; }
    __device__ void issue_v(const Geo3& g, int i, int j, int k, const S3& s) const { put1_3(s, 0, alpha, vid3(g, i, j, k)); }
    __device__ void fix_v(const Geo3& g, int i, int j, int k, const S3& s, double (&v)[NV]) const {
        const long long id = vid3(g, i, j, k);
        v[0] = v[1] = v[2] = 0.0;
        if (!LOADONLY) {
            const unsigned m = bc3(g, i, j, k, id);
            for (int c = 0; c < 3; ++c)
                if ((m >> c) & 1u) v[c] = __ldg(g.ubar + 3 * id + c);
        }
        v[3] = get1_3(s, 0);
    }
    __device__ void issue_c(const Geo3& g, int ci, int j, int k, const S3& s) const { putE3(g, s, 0, cid3(g, ci, j, k)); }
    __device__ void fix_c(const Geo3& g, int, int, int, const S3& s, double (&e)[NE]) const { e[0] = getE3(g, s, 0); }
    __device__ void cell(const Geo3& g, int, int, int, const double (&X)[NV][8], const double (&ec)[NE],
                         double (&Y)[NC][8], bool) {
        const double (&U)[3][8] = *reinterpret_cast<const double(*)[3][8]>(&X[0][0]);
        for_each_tet([&](auto, auto A, auto B, auto C) {
            const double ab = tet_abar<A.v, B.v, C.v>(X[3]);
            const double om = 1.0 - ab;
            const double s = (om * om + g.kell) * g.vol * ec[0];
            double G[3][3], e[6] = {0, 0, 0, 0, 0, 0}, sg[6];
            if (!LOADONLY) {
                tet_grad<A.v, B.v, C.v>(g, U, G);
                voigt(G, e);
            }
            stress3(g, e, sg);
            tet_scatter<A.v, B.v, C.v>(g, s, sg, Y);
        });
    }
    __device__ void out(const Geo3& g, int i, int j, int k, const double (&t)[NC], const double (&v)[NV]) {
        const long long id = vid3(g, i, j, k);
        const unsigned m = LOADONLY ? 0u : bc3(g, i, j, k, id);
        for (int c = 0; c < 3; ++c) {
            const double bv = ((m >> c) & 1u) ? v[c] : -t[c];
            b[3 * id + c] = bv;
            acc += bv * bv;
        }
    }
    __device__ void finish() {
        double vv[1] = {acc};
        double* s = scal;
        grid_reduce<1>(vv, rb, 3, [s](double* tot) { s[S_AUX0] = tot[0]; });
    }
};

// Coupled Jacobian apply [[Kuu_bc, Kua_bc], [Kau_bc, Kaa]] (optionally masked by act), also used
// for Kua (xu = 0) / Kau (xa = 0) alone.  vertex: u, alpha, xu, xa, [act] ; cell: E, Gc
struct Op3Jac : NoRed3 {
    static constexpr int NV = 8, NC = 4, PD = 2, NE = 2, SV = 9, SC = 2, MINB = 1;
    const double* u;
    const double* alpha;
    const double* xu;
    const double* xa;
    double* yu;
    double* ya;
    const unsigned char* act;
    int mode;  // 0 full Jacobian (masked), 1 Kua (yu = Kua xa), 2 Kau (ya = Kau xu)
    int bcmode;
    __device__ void issue_v(const Geo3& g, int i, int j, int k, const S3& s) const {
        const long long v = vid3(g, i, j, k);
        put3_3(s, 0, u, v);
        put1_3(s, 3, alpha, v);
        if (xu) put3_3(s, 4, xu, v);
        if (xa) put1_3(s, 7, xa, v);
        if (act) putb_3(s, 8, act, v);
    }
    __device__ void fix_v(const Geo3& g, int i, int j, int k, const S3& s, double (&v)[NV]) const {
        const long long id = vid3(g, i, j, k);
        const unsigned m = bcmode ? bc3(g, i, j, k, id) : 0u;
        for (int q = 0; q < 4; ++q) v[q] = get1_3(s, q);
        for (int c = 0; c < 3; ++c) v[4 + c] = (xu && !((m >> c) & 1u)) ? get1_3(s, 4 + c) : 0.0;
        const bool a = act && getb_3(s, 8, id) != 0u;
        v[7] = (xa && !a) ? get1_3(s, 7) : 0.0;
    }
    __device__ void issue_c(const Geo3& g, int ci, int j, int k, const S3& s) const {
        const long long c = cid3(g, ci, j, k);
        putE3(g, s, 0, c);
        putGc3(g, s, 1, c);
    }
    __device__ void fix_c(const Geo3& g, int, int, int, const S3& s, double (&e)[NE]) const {
        e[0] = getE3(g, s, 0);
        e[1] = getGc3(g, s, 1);
    }
    __device__ void cell(const Geo3& g, int, int, int, const double (&X)[NV][8], const double (&ec)[NE],
                         double (&Y)[NC][8], bool) {
        const double (&U)[3][8] = *reinterpret_cast<const double(*)[3][8]>(&X[0][0]);
        const double (&XU)[3][8] = *reinterpret_cast<const double(*)[3][8]>(&X[4][0]);
        double (&YU)[3][8] = *reinterpret_cast<double(*)[3][8]>(&Y[0][0]);
        const double Ec = ec[0], kc = ec[1] / g.cw;
        for_each_tet([&](auto, auto A, auto B, auto C) {
            constexpr int q1 = Bit<A.v>::v, q2 = Bit<A.v>::v | Bit<B.v>::v;
            const double ab = tet_abar<A.v, B.v, C.v>(X[3]);
            const double om = 1.0 - ab;
            const double a = om * om + g.kell, ap = -2.0 * om;
            double G[3][3], e[6], sg[6], Gx[3][3], ex[6], tx[6];
            tet_grad<A.v, B.v, C.v>(g, U, G);
            voigt(G, e);
            stress3(g, e, sg);
            const double cpl = ap * g.vol * Ec * 0.25;
            const double sxa = (X[7][0] + X[7][q1]) + (X[7][q2] + X[7][7]);
            if (mode != 2) {
                // u rows: a|T|E B^T D B x_u + cpl * sxa * B^T sigma
                double comb[6];
                if (mode == 0) {
                    tet_grad<A.v, B.v, C.v>(g, XU, Gx);
                    voigt(Gx, ex);
                    stress3(g, ex, tx);
                    for (int t = 0; t < 6; ++t) comb[t] = a * g.vol * Ec * tx[t] + cpl * sxa * sg[t];
                } else {
                    for (int t = 0; t < 6; ++t) comb[t] = cpl * sxa * sg[t];
                }
                tet_scatter<A.v, B.v, C.v>(g, 1.0, comb, YU);
            }
            if (mode != 1) {
                tet_grad<A.v, B.v, C.v>(g, XU, Gx);
                voigt(Gx, ex);
                const double fa = cpl * (ex[0] * sg[0] + ex[1] * sg[1] + ex[2] * sg[2] + ex[3] * sg[3] +
                                         ex[4] * sg[4] + ex[5] * sg[5]);
                Y[3][0] += fa; Y[3][q1] += fa; Y[3][q2] += fa; Y[3][7] += fa;
                if (mode == 0) {
                    const double q = Ec * (e[0] * sg[0] + e[1] * sg[1] + e[2] * sg[2] + e[3] * sg[3] +
                                           e[4] * sg[4] + e[5] * sg[5]);
                    const double kap = (q + (g.at2 ? 2.0 * kc / g.ell : 0.0)) * g.vol * (1.0 / 16.0);
                    elem3_kaa<A.v, B.v, C.v>(g, kap, kc, X[7], Y[3]);
                }
            }
        });
    }
    __device__ void out(const Geo3& g, int i, int j, int k, const double (&t)[NC], const double (&)[NV]) {
        const long long id = vid3(g, i, j, k);
        const unsigned m = bcmode ? bc3(g, i, j, k, id) : 0u;
        if (mode != 2) {
            for (int c = 0; c < 3; ++c) {
                double yv = t[c];
                if ((m >> c) & 1u) yv = (mode == 0) ? __ldg(xu + 3 * id + c) : 0.0;
                yu[3 * id + c] = yv;
            }
        }
        if (mode != 1) ya[id] = (act && act[id]) ? __ldg(xa + id) : t[3];
    }
};

// ---- launch plumbing -----------------------------------------------------------------------------
template <class Op>
static int run3g(Ctx* c, const Geo3& g0, Op op, cudaStream_t st, int kind, double bytes) {
    constexpr int kW3 = WarpsOf<Op>::v;
    Geo3 g = g0;
    if (kW3 != 8 || MinBlocksOf<Op>::v != 2) tile3(g, kW3 - 2, 148 * MinBlocksOf<Op>::v);  // Geo3's own tiling: 8 warps x 2
    constexpr int smem = strip3_smem<Op, kW3>();
    static_assert(smem <= 227 * 1024, "3D stage ring exceeds shared memory");
    static std::atomic<bool> attr[kMaxDev];
    const int dv = cur_dev();
    if (!attr[dv].load()) {
        cudaError_t e = cudaFuncSetAttribute(k_strip3d<Op, kW3, MinBlocksOf<Op>::v>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return check_cuda(c, e, "3D kernel attribute");
        attr[dv] = true;
    }
    const long long nb = (long long)g.nbj * g.nbk * g.nstrips;
    if (nb > kMaxBlocksRed) return set_error(c, PF_EINVAL, "3D grid too large for the reduction buffer");
    const int ps = prof_begin(c, st);
    k_strip3d<Op, kW3, MinBlocksOf<Op>::v><<<(int)nb, kW3 * 32, smem, st>>>(g, op);
    prof_end(c, st, ps, kind, bytes);
    c->launches++;
    return check_cuda(c, cudaGetLastError(), "3D strip kernel launch");
}
template <class Op>
static int run3(Ctx* c, Op op, cudaStream_t st, int kind, double bytes) {
    return run3g(c, c->g3, op, st, kind, bytes);
}
// A/B switch for the tiling of the Kuu / Kaa applies: PF_K3W=16 (one 16-warp block per SM) or 8
// (two 8-warp blocks per SM)
template <class Op>
static int run3w(Ctx* c, const Geo3& g, Op op, cudaStream_t st, int kind, double bytes) {
    static const int w = getenv("PF_K3W") ? atoi(getenv("PF_K3W")) : 0;
    if (w == 16) return run3g(c, g, Tiled3<Op, 16, 1>{op}, st, kind, bytes);
    if (w == 8) return run3g(c, g, Tiled3<Op, 8, 2>{op}, st, kind, bytes);
    return run3g(c, g, op, st, kind, bytes);
}
static RedBuf rb3(Ctx* c) { return RedBuf{c->partials, c->tickets, c->scal}; }

// operators on an explicit (e.g. coarse multigrid level) geometry
static bool iso3(const Geo3& g) { return g.ihx == g.ihy && g.ihx == g.ihz; }
int launch3_Kuu_on(Ctx* c, const Geo3& g, const double* alpha, const double* x, double* y, int bcmode,
                   cudaStream_t st, int kind) {
    if (iso3(g)) {
        Op3Kuu<false, true> op{alpha, x, nullptr, nullptr, y, bcmode, c->scal, rb3(c), 0.0};
        return run3w(c, g, op, st, kind, 56.0 * g.nv);
    }
    Op3Kuu<false, false> op{alpha, x, nullptr, nullptr, y, bcmode, c->scal, rb3(c), 0.0};
    return run3g(c, g, op, st, kind, 56.0 * g.nv);
}
template <int EPI, bool ISO>
static int run3_sm(Ctx* c, const Geo3& g, const Sm3Args& a, cudaStream_t st, int kind) {
    Op3KuuSm<EPI, ISO> op{{a.alpha, a.xin, nullptr, nullptr, nullptr, PF_BC_ELIMINATE, c->scal, rb3(c), 0.0},
                          a.b, a.dinv, a.res, a.dnext, a.xs, a.live, a.lam, a.ratio, a.k, a.pending,
                          0.0, 0.0, 0.0};
    const double vec = EPI == E3_RESID ? 48.0 : (EPI == E3_RESID_CHEB0 ? 96.0 : (EPI == E3_CHEB ? 144.0 : 144.0));
    const double bytes = (EPI == E3_CHEB_B ? 56.0 + 24.0 : 56.0 - 24.0) * g.nv + vec * g.nv;
    // the first step from zero stages 7 vertex slots and spills 76 B at 128 registers (two 8-warp
    // blocks per SM); PF_K3SM_MINB1=1 runs it one block per SM with 212 registers and no spill
    // instead.  Measured on config 4 (128^3, steps 7-11): 0.2668 / 0.1650 / 0.2335 / 0.2287 / 0.2059 s
    // with the spilling two-block tiling, 0.2678 / 0.1658 / 0.2344 / 0.2299 / 0.2067 s without the
    // spill -- the spill costs nothing measurable (one of four smoother steps, L1-resident), the lost
    // occupancy slightly more, so the default stays
    if constexpr (EPI == E3_CHEB_B) {
        static const bool one = getenv("PF_K3SM_MINB1") != nullptr;
        if (one) {
            Tiled3<Op3KuuSm<EPI, ISO>, 8, 1> t;
            static_cast<Op3KuuSm<EPI, ISO>&>(t) = op;
            return run3g(c, g, t, st, kind, bytes);
        }
    }
    return run3g(c, g, op, st, kind, bytes);
}
int launch3_Kuu_sm(Ctx* c, const Geo3& g, int epi, const Sm3Args& a, cudaStream_t st, int kind) {
    const bool iso = iso3(g);
    switch (epi) {
        case E3_CHEB: return iso ? run3_sm<E3_CHEB, true>(c, g, a, st, kind) : run3_sm<E3_CHEB, false>(c, g, a, st, kind);
        case E3_CHEB_B: return iso ? run3_sm<E3_CHEB_B, true>(c, g, a, st, kind) : run3_sm<E3_CHEB_B, false>(c, g, a, st, kind);
        case E3_RESID: return iso ? run3_sm<E3_RESID, true>(c, g, a, st, kind) : run3_sm<E3_RESID, false>(c, g, a, st, kind);
        default: return iso ? run3_sm<E3_RESID_CHEB0, true>(c, g, a, st, kind)
                            : run3_sm<E3_RESID_CHEB0, false>(c, g, a, st, kind);
    }
}
int launch3_Kuu_diag_on(Ctx* c, const Geo3& g, const double* alpha, double* dinv, cudaStream_t st, int kind) {
    Op3KuuDiag op;
    op.alpha = alpha;
    op.dinv = dinv;
    return run3g(c, g, op, st, kind, 32.0 * g.nv);
}

int launch3_Kuu(Ctx* c, const double* alpha, const double* x, double* y, int bcmode, cudaStream_t st) {
    return launch3_Kuu_on(c, c->g3, alpha, x, y, bcmode, st, K_KUU);
}
int launch3_Kuu_cgA(Ctx* c, const double* alpha, const double* z, const double* p_in, double* p_out, double* q,
                    cudaStream_t st) {
    if (iso3(c->g3)) {
        Op3Kuu<true, true> op{alpha, z, p_in, p_out, q, PF_BC_ELIMINATE, c->scal, rb3(c), 0.0};
        return run3(c, op, st, K_KUU_CG, 104.0 * c->g3.nv);
    }
    Op3Kuu<true, false> op{alpha, z, p_in, p_out, q, PF_BC_ELIMINATE, c->scal, rb3(c), 0.0};
    return run3(c, op, st, K_KUU_CG, 104.0 * c->g3.nv);
}
int launch3_Kuu_diag(Ctx* c, const double* alpha, double* dinv, cudaStream_t st) {
    Op3KuuDiag op;
    op.alpha = alpha;
    op.dinv = dinv;
    return run3(c, op, st, K_KUU_DIAG, 32.0 * c->g3.nv);
}
int launch3_kappa(Ctx* c, const double* u, double* kappa, double* cvec, cudaStream_t st) {
    Op3Kappa op;
    op.u = u; op.kappa = kappa; op.cvec = cvec;
    return run3(c, op, st, K_KAPPA, 32.0 * c->g3.nv + 8.0 * c->n_el);
}
int launch3_Kaa(Ctx* c, const double* kappa, const double* x, double* y, const unsigned char* act, cudaStream_t st) {
    const double bytes = 16.0 * c->g3.nv + 8.0 * c->n_el;
    if (act) {
        Op3Kaa<false, true> op{kappa, x, nullptr, nullptr, y, act, c->scal, rb3(c), 0.0};
        return run3w(c, c->g3, op, st, K_KAA, bytes);
    }
    Op3Kaa<false, false> op{kappa, x, nullptr, nullptr, y, nullptr, c->scal, rb3(c), 0.0};
    return run3w(c, c->g3, op, st, K_KAA, bytes);
}
int launch3_Kaa_cgA(Ctx* c, const double* kappa, const double* z, const double* p_in, double* p_out, double* q,
                    const unsigned char* act, cudaStream_t st) {
    const double bytes = 33.0 * c->g3.nv + 8.0 * c->n_el;
    if (act) {
        Op3Kaa<true, true> op{kappa, z, p_in, p_out, q, act, c->scal, rb3(c), 0.0};
        return run3w(c, c->g3, op, st, K_KAA_CG, bytes);
    }
    Op3Kaa<true, false> op{kappa, z, p_in, p_out, q, nullptr, c->scal, rb3(c), 0.0};
    return run3w(c, c->g3, op, st, K_KAA_CG, bytes);
}
// ---- free tiles of the masked damage PCG ---------------------------------------------------------
// On an active row the masked system is the identity with a zero right-hand side, so x, r, z, p and
// q stay 0 there for the whole solve.  A tile whose input box (its output vertices +-1 in every
// direction) holds active vertices only therefore writes zeros and adds 0 to p.q: the persistent
// loop visits just the tiles on this list (ascending, so the sums keep a fixed order), and its
// vector pass skips the active rows.  After localisation the free set of an AT1 damage solve is a
// thin layer around the crack.
__global__ void __launch_bounds__(256) k_tile_flags3(const Geo3 g, const unsigned char* __restrict__ act, int ntile,
                                                     unsigned char* __restrict__ flag) {
    const int t = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    if (t >= ntile) return;
    const int bk = t % g.nbk, rest = t / g.nbk, bj = rest % g.nbj, bs = rest / g.nbj;
    const int k = bk * 30 - 1 + lane;
    const int j0 = max(bj * (kW3 - 2) - 1, 0), j1 = min(bj * (kW3 - 2) + (kW3 - 2), g.ny);
    const int i0 = max(bs * g.S - 1, 0), i1 = min(bs * g.S + g.S, g.nx);
    bool f = false;
    if (k >= 0 && k <= g.nz)
        for (int i = i0; i <= i1; ++i)
            for (int j = j0; j <= j1; ++j) f |= act[vid3(g, i, j, k)] == 0;
    f = __any_sync(PF_FULL, f);
    if (lane == 0) flag[t] = f ? 1 : 0;
}
// list[0] = number of flagged tiles, list[1..] = their indices in ascending order (one block)
__global__ void __launch_bounds__(1024) k_tile_compact(int ntile, const unsigned char* __restrict__ flag,
                                                       int* __restrict__ list) {
    __shared__ int wsum[32];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int per = ((ntile + 31) / 32 + 31) / 32 * 32;  // tiles per warp, a multiple of 32
    const int b0 = w * per, b1 = min(b0 + per, ntile);
    int cnt = 0;
    for (int b = b0; b < b1; b += 32) {
        const int t = b + lane;
        cnt += __popc(__ballot_sync(PF_FULL, t < b1 && flag[t]));
    }
    if (lane == 0) wsum[w] = cnt;
    __syncthreads();
    int off = 0;
    for (int q = 0; q < w; ++q) off += wsum[q];
    for (int b = b0; b < b1; b += 32) {
        const int t = b + lane;
        const bool f = t < b1 && flag[t];
        const unsigned m = __ballot_sync(PF_FULL, f);
        if (f) list[1 + off + __popc(m & ((1u << lane) - 1u))] = t;
        off += __popc(m);
    }
    if (threadIdx.x == 1023) list[0] = off;
}
void launch_tile_compact(int ntile, const unsigned char* flag, int* list, cudaStream_t st) {
    k_tile_compact<<<1, 1024, 0, st>>>(ntile, flag, list);
}

// The whole masked Jacobi-PCG loop on the 3D damage block in one cooperative launch, as the 2D
// k_pcg_kaa (pf_ops2d.cu): per iteration one strip pass over all tiles (p = z + beta p, q = Kaa p,
// p.q) and one vector pass (x += gamma p, r -= gamma q, z = D^-1 r, r.r, r.z), separated by grid
// barriers; the scalar decisions come from fixed-order sums, identical in every CTA.  Replaces two
// launches per iteration (plus the graph's loop node) on a latency-bound 2-17 MB problem.
template <bool MASKED>
__global__ void __launch_bounds__(kW3 * 32, 2) k_pcg_kaa3(const Geo3 g, Op3Kaa<true, MASKED> op, int ntile, long long n,
                                                         double* x, double* r, double* z, double* p0, double* p1,
                                                         double* q, const double* dinv, double* s, double* partials,
                                                         unsigned int* bar, const int* __restrict__ tiles) {
    extern __shared__ __align__(16) unsigned char smem[];
    if (!(s[S_DONE] == 0.0 && s[S_FAIL] == 0.0)) return;  // uniform
    // free tiles only (see k_tile_flags3), when at most half of the tiles are flagged
    const int nfree = tiles ? tiles[0] : ntile;
    const bool sparse = MASKED && tiles && 2 * nfree <= ntile;
    const int nt = sparse ? nfree : ntile;
    const double target = s[S_TARGET], maxit = s[S_MAXIT];
    double rz = s[S_RZ], beta = s[S_BETA], rn = s[S_RNORM], pap = 0.0, gm = 0.0;
    long long it = (long long)s[S_ITER];
    double done = 0.0, fail = 0.0;
    const long long tid = blockIdx.x * (long long)blockDim.x + threadIdx.x, nth = (long long)gridDim.x * blockDim.x;
    for (;;) {
        double* pin = (it & 1) ? p1 : p0;
        double* pout = (it & 1) ? p0 : p1;
        op.x = z;
        op.pin = pin;
        op.pout = pout;
        op.y = q;
        op.acc = 0.0;
        op.use_breg = 1;
        op.breg = it > 0 ? beta : 0.0;
        for (int m = blockIdx.x; m < nt; m += gridDim.x) {
            __syncthreads();  // the previous tile's readers of the exchange buffers are done
            strip3_tile<Op3Kaa<true, MASKED>, kW3>(g, op, smem, sparse ? tiles[1 + m] : m);
        }
        block_partials(&op.acc, 1, partials, 0);
        grid_sync(bar);
        pap = grid_total(partials, 0);
        if (!(pap > 0.0)) { fail = 1.0; break; }
        gm = rz / pap;
        double acc[2] = {0.0, 0.0};
        auto upd = [&](long long i, bool live) {
            const double xi = __ldcg(x + i) + gm * __ldcg(pout + i);
            const double ri = __ldcg(r + i) - gm * __ldcg(q + i);
            const double zi = dinv[i] * ri;
            if (live) {
                x[i] = xi;
                r[i] = ri;
                z[i] = zi;
                acc[0] += ri * ri;
                acc[1] += ri * zi;
            }
        };
        if (sparse) {  // the rows the flagged tiles own (every free row is one of them), spread over
                       // all threads: item = (tile on the list, row of the tile, pencil, lane)
            const int R = g.S * (kW3 - 2) * 32;
            const long long items = (long long)nfree * R;
            for (long long e = tid; e < items; e += nth) {
                const int m = (int)(e / R), rho = (int)(e % R), l = rho & 31;
                if (l >= 30) continue;
                const int t = tiles[1 + m];
                const int bk = t % g.nbk, rest = t / g.nbk, bj = rest % g.nbj, bs = rest / g.nbj;
                const int j = bj * (kW3 - 2) + (rho >> 5) % (kW3 - 2), k = bk * 30 + l;
                const int i = bs * g.S + (rho >> 5) / (kW3 - 2);
                if (i > g.nx || j > g.ny || k > g.nz) continue;
                const long long v = vid3(g, i, j, k);
                if (op.act[v]) continue;  // most rows of a flagged 3D tile are active: skip their loads
                upd(v, true);
            }
        } else {
            for (long long i = tid; i < n; i += nth) upd(i, true);
        }
        block_partials(acc, 2, partials, 1);
        grid_sync(bar);
        const double2 t2 = grid_total2(partials, 1);
        const double rr = t2.x, rzn = t2.y;
        ++it;
        rn = sqrt(rr);
        if (rn <= target) { done = 1.0; break; }
        if (!(rzn > 0.0)) { fail = 2.0; break; }
        beta = rzn / rz;
        rz = rzn;
        if ((double)it >= maxit) { done = 3.0; break; }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        s[S_ITER] = (double)it;
        s[S_RNORM] = rn;
        s[S_PAP] = pap;
        s[S_GAMMA] = gm;
        s[S_RZ] = rz;
        s[S_BETA] = beta;
        s[S_DONE] = done;
        s[S_FAIL] = fail;
    }
}

template <bool MASKED>
static int launch3_pcg_kaa_m(Ctx* c, const PcgBuffers& B, const double* kappa, const unsigned char* act,
                             cudaStream_t st) {
    using Op = Op3Kaa<true, MASKED>;
    constexpr int smem = strip3_smem<Op, kW3>();
    static std::atomic<int> per_dev[kMaxDev];
    const int dvp = cur_dev();
    int per = per_dev[dvp].load();
    if (per <= 0) {
        cudaError_t e = cudaFuncSetAttribute(k_pcg_kaa3<MASKED>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return check_cuda(c, e, "persistent 3D pcg attribute");
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_pcg_kaa3<MASKED>, kW3 * 32, smem);
        if (e != cudaSuccess) return check_cuda(c, e, "persistent 3D pcg occupancy");
        per_dev[dvp] = per;
    }
    int dev = 0, nsm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    const Geo3& g = c->g3;
    const int ntile = g.nbj * g.nbk * g.nstrips;
    const int nb = std::min(ntile, nsm * std::max(per, 1));
    if (per < 1 || nb > kMaxBlocksRed) return PF_EINVAL;  // caller falls back to the graph loop
    Op op{kappa, B.z, B.p0, B.p1, B.q, act, c->scal, rb3(c), 0.0};
    const int* tiles = nullptr;
    c->tile_frac = 1.0;
    static const bool skip_off = getenv("PF_NO_TILE_SKIP") != nullptr;
    if (MASKED && c->rhs_masked && !skip_off && c->tile_list && ntile <= c->tile_cap) {
        unsigned char* flag = reinterpret_cast<unsigned char*>(c->tile_list + c->tile_cap + 1);
        k_tile_flags3<<<(ntile + 7) / 8, 256, 0, st>>>(g, act, ntile, flag);
        launch_tile_compact(ntile, flag, c->tile_list, st);
        c->launches += 2;
        tiles = c->tile_list;
        if (c->prof.on || getenv("PF_TILE_TRACE")) {  // (diagnostics only: one host read)
            int nfree = 0;
            cudaMemcpyAsync(&nfree, c->tile_list, sizeof(int), cudaMemcpyDeviceToHost, st);
            cudaStreamSynchronize(st);
            c->tile_frac = 2LL * nfree <= (long long)ntile ? (double)nfree / (double)ntile : 1.0;
        }
        if (getenv("PF_TILE_TRACE")) {
            int nfree = 0;
            cudaMemcpyAsync(&nfree, c->tile_list, sizeof(int), cudaMemcpyDeviceToHost, st);
            cudaStreamSynchronize(st);
            fprintf(stderr, "  damage pcg: %d of %d tiles hold free vertices\n", nfree, ntile);
        }
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(nb);
    cfg.blockDim = dim3(kW3 * 32);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    const int ps = prof_begin(c, st);
    cudaError_t e = cudaLaunchKernelEx(&cfg, k_pcg_kaa3<MASKED>, g, op, ntile, B.n, B.x, B.r, B.z, B.p0, B.p1, B.q,
                                       (const double*)B.dinv, c->scal, c->partials, c->tickets + 62, tiles);
    prof_end(c, st, ps, K_KAA_CG, 0.0);
    c->launches++;
    return check_cuda(c, e, "persistent 3D pcg launch");
}
int launch3_pcg_kaa(Ctx* c, const PcgBuffers& B, const double* kappa, const unsigned char* act, cudaStream_t st) {
    return act ? launch3_pcg_kaa_m<true>(c, B, kappa, act, st) : launch3_pcg_kaa_m<false>(c, B, kappa, act, st);
}

int launch3_Kaa_diag(Ctx* c, const double* kappa, double* dinv, const unsigned char* act, cudaStream_t st) {
    if (act) {
        Op3KaaDiag<true> op;
        op.kappa = kappa; op.dinv = dinv; op.act = act;
        return run3(c, op, st, K_KAA_DIAG, 8.0 * c->g3.nv + 8.0 * c->n_el);
    }
    Op3KaaDiag<false> op;
    op.kappa = kappa; op.dinv = dinv; op.act = nullptr;
    return run3(c, op, st, K_KAA_DIAG, 8.0 * c->g3.nv + 8.0 * c->n_el);
}
int launch3_Kaa_trial(Ctx* c, const double* kappa, const double* cvec, const double* x, const double* d,
                      const double* lb, double* trial, double* F, int merit_slot, cudaStream_t st) {
    Op3KaaTrial op{kappa, cvec, x, d, lb, trial, F, c->scal, merit_slot, rb3(c), 0.0};
    return run3(c, op, st, K_KAA_TRIAL, 48.0 * c->g3.nv + 8.0 * c->n_el);
}
int launch3_physics(Ctx* c, const double* u, const double* alpha, const double* lb, double* ru, double* ra,
                    double* phi, int rows, cudaStream_t st) {
    const double bytes = c->g3.nv * (32.0 + 8.0 + (ru ? 24.0 : 0.0) + (ra ? 8.0 : 0.0) + (phi ? 8.0 : 0.0));
    if (rows == PF_ROWS_ZERO) {
        Op3Phys<PF_ROWS_ZERO> op{u, alpha, lb, ru, ra, phi, c->scal, rb3(c), 0, 0, 0, 0};
        return run3(c, op, st, K_PHYS, bytes);
    }
    if (rows == PF_ROWS_VALUE) {
        Op3Phys<PF_ROWS_VALUE> op{u, alpha, lb, ru, ra, phi, c->scal, rb3(c), 0, 0, 0, 0};
        return run3(c, op, st, K_PHYS, bytes);
    }
    Op3Phys<PF_ROWS_RAW> op{u, alpha, lb, ru, ra, phi, c->scal, rb3(c), 0, 0, 0, 0};
    return run3(c, op, st, K_PHYS, bytes);
}
int launch3_load(Ctx* c, const double* alpha, double* f, int rows, cudaStream_t st) {
    if (rows == 0) {
        Op3Rhs<true> op{alpha, f, c->scal, rb3(c), 0.0};
        return run3(c, op, st, K_RHS, 32.0 * c->g3.nv);
    }
    Op3Rhs<false> op{alpha, f, c->scal, rb3(c), 0.0};
    return run3(c, op, st, K_RHS, 32.0 * c->g3.nv);
}
int launch3_jac(Ctx* c, const double* u, const double* alpha, const double* xu, const double* xa, double* yu,
                double* ya, const unsigned char* act, int mode, int bcmode, cudaStream_t st) {
    Op3Jac op;
    op.u = u; op.alpha = alpha; op.xu = xu; op.xa = xa; op.yu = yu; op.ya = ya; op.act = act;
    op.mode = mode; op.bcmode = bcmode;
    return run3(c, op, st, mode == 0 ? K_JAC : (mode == 1 ? K_KUA : K_KAU), 96.0 * c->g3.nv);
}

}  // namespace pf
