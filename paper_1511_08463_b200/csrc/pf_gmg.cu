// pf_gmg.cu -- geometric multigrid preconditioner for the degraded elasticity operator.
//
// The reference solves the elastic half-step with SuperLU (linalg.py:250-262; 88 s per
// factorisation at 512^2) or Jacobi/SSOR/Chebyshev-PCG (linalg.py:294-378; ~4000 iterations at
// 512^2).  North-star part (3) replaces it by PCG with a Chebyshev-smoothed geometric multigrid
// V-cycle on the structured hierarchy:
//   level 0 : the fine mesh, matrix-free (strip kernels), block-Jacobi (2x2) Chebyshev smoother;
//   level 1 : crossed pattern -> corner grid with centres condensed (P0: centre = mean of its cell
//             corners); other patterns -> 2:1 coarsening;
//   level l : 9-point 2x2-block stencils, Galerkin A_{l+1} = P^T A_l P with bilinear P and a
//             ceil rule for odd cell counts (the last odd fine vertex is injected);
//   coarsest: dense inverse (n <= 2*kCoarseMaxV dofs, from a banded Cholesky factor), applied as
//             one matvec spread over the whole grid.
// Dirichlet dofs: the fine operator is the eliminated one (fem.py:282-294); P has zero rows on
// constrained fine dofs and zero columns on coarse dofs injected from constrained fine dofs, so
// coarse corrections never touch them and every level stays SPD.  Coefficient jumps (cracks,
// a = k_ell) are seen by the coarse operators because they are Galerkin products.
// Stencil layout: A[(k*4 + e)*nv + v], k = (di+1)*3 + (dj+1) neighbour, e = 2r + c block entry.
#include <algorithm>
#include <type_traits>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "pf_elem.cuh"

namespace pf {

// Layout of a level's 9-point 2x2-block stencil: the four entries of block k of vertex v are
// contiguous, A[(k nv + v) 4 + e], so an apply reads a block with two 16-byte loads.  The level
// phases of the V-cycle are bound by the number of outstanding load requests per SM, not by bytes:
// against the entry-major layout A[(4k + e) nv + v] (four 8-byte loads per block) the persistent
// coarse cycle of SENT 512^2 issues 18 instead of 36 stencil requests per vertex.
__host__ __device__ __forceinline__ size_t aidx(long long nv, int k, int e, long long v) {
    return ((size_t)k * (size_t)nv + (size_t)v) * 4 + (size_t)e;
}

constexpr int kCoarseMaxV = 300;  // coarsest level: at most this many vertices (dense inverse)
constexpr int kBandSmem = 200 * 1024;  // banded factor of the coarsest operator, in shared memory
// half-bandwidth (in dofs) of a level's operator: vertex neighbours differ by <= nvy + 1
__host__ __device__ __forceinline__ int band_of(int ny) { return 2 * (ny + 1) + 3; }
constexpr int kGB = 256;          // block size of the GMG kernels

__device__ __forceinline__ bool gmg_live(const double* s) {
    return s == nullptr || (s[S_DONE] == 0.0 && s[S_FAIL] == 0.0);
}
__device__ __forceinline__ void atomic_max_pos(double* addr, double v) {
    if (v > 0.0) atomicMax(reinterpret_cast<unsigned long long*>(addr), (unsigned long long)__double_as_longlong(v));
}

// ---- element matrix blocks (setup only; runtime gradient values) ----------------------------
// 2x2 block K_e[m][n] = s B_m^T D B_n for P1 triangles with gradients (b, c).
__device__ __forceinline__ void ke_block(const Geo2& g, double s, double bm, double cm, double bn, double cn,
                                         double (&K)[4]) {
    K[0] = s * (bm * bn * g.D00 + cm * cn * g.D22);
    K[1] = s * (bm * cn * g.D01 + cm * bn * g.D22);
    K[2] = s * (cm * bn * g.D01 + bm * cn * g.D22);
    K[3] = s * (cm * cn * g.D11 + bm * bn * g.D22);
}

// Gradients (b, c) of shape T's three local nodes, with the union-jack mirror sign.
template <int PAT, int T>
__device__ __forceinline__ void shape_grads(const Geo2& g, int cj, double hxs, double (&b)[3], double (&c)[3]) {
    using S = Shp<PAT, T>;
    b[0] = S::b0 * hxs; b[1] = S::b1 * hxs; b[2] = S::b2 * hxs;
    const double ihy = ihy_at(g, cj);
    c[0] = S::c0 * ihy; c[1] = S::c1 * ihy; c[2] = S::c2 * ihy;
}

// Cell matrix on the cell's local nodes (0..3 corners, 4 centre): M[(r*5 + s)][4] blocks.
// Union-jack odd cells are handled by mirroring the local node order (see pf_elem.cuh).
template <int PAT>
__device__ void cell_matrix(const Geo2& g, int ci, int cj, const double* alpha, double (&M)[25][4]) {
    const long long cell = (long long)ci * g.ny + cj;
    const double Ec = g.E_cell ? g.E_cell[cell] : g.E;
    double Al[5];
    const long long v00 = (long long)ci * g.nvy + cj;
    Al[0] = alpha[v00];
    Al[1] = alpha[v00 + g.nvy];
    Al[2] = alpha[v00 + 1];
    Al[3] = alpha[v00 + g.nvy + 1];
    Al[4] = PAT == PF_CROSSED ? alpha[g.nc + cell] : 0.0;
    const int par = (PAT == PF_UNION_JACK) ? ((ci + cj) & 1) : 0;
    const double hxs = par ? -g.ihx : g.ihx;
    mirror<PAT>(par, Al);
#pragma unroll
    for (int k = 0; k < 25; ++k) M[k][0] = M[k][1] = M[k][2] = M[k][3] = 0.0;
    // perm maps mirrored local slot -> physical local node
    const int perm[5] = {par ? 1 : 0, par ? 0 : 1, par ? 3 : 2, par ? 2 : 3, 4};
    for_each_elem<PAT>(par, [&](auto T, auto, auto A, auto B, auto C) {
        const int nodes[3] = {A.v, B.v, C.v};
        const double ab = (Al[A.v] + Al[B.v] + Al[C.v]) * (1.0 / 3.0);
        const double om = 1.0 - ab;
        const double s = (om * om + g.kell) * area_at(g, cj) * Ec;
        double b[3], c[3];
        shape_grads<PAT, T.v>(g, cj, hxs, b, c);
        for (int m = 0; m < 3; ++m)
            for (int n = 0; n < 3; ++n) {
                double K[4];
                ke_block(g, s, b[m], c[m], b[n], c[n], K);
                const int r = perm[nodes[m]], q = perm[nodes[n]];
                M[r * 5 + q][0] += K[0]; M[r * 5 + q][1] += K[1];
                M[r * 5 + q][2] += K[2]; M[r * 5 + q][3] += K[3];
            }
    });
}

// local corner slot -> offset of that corner from the cell origin
__device__ __forceinline__ int cdi(int k) { return (k == 1 || k == 3) ? 1 : 0; }
__device__ __forceinline__ int cdj(int k) { return (k >= 2) ? 1 : 0; }

__device__ __forceinline__ unsigned vmask(const unsigned char* mask, long long v) { return mask ? mask[v] : 0u; }

// finalize a stencil row: Dirichlet elimination, block-Jacobi inverse, Gershgorin bound of D^-1 A
__device__ void finish_row(double (&S)[9][4], unsigned mrow, const unsigned* mcol, long long v, long long nv,
                           double* A, double* Dinv, double* lam) {
    for (int k = 0; k < 9; ++k) {
        for (int r = 0; r < 2; ++r)
            for (int c = 0; c < 2; ++c) {
                const bool kill = ((mrow >> r) & 1u) || ((mcol[k] >> c) & 1u);
                if (kill) S[k][2 * r + c] = 0.0;
            }
    }
    if (mrow & 1u) S[4][0] = 1.0;
    if (mrow & 2u) S[4][3] = 1.0;
    // coarse dofs with no coupling at all (fully masked support) become identity
    if (S[4][0] == 0.0 && S[4][1] == 0.0 && S[4][2] == 0.0) S[4][0] = 1.0;
    if (S[4][3] == 0.0 && S[4][1] == 0.0 && S[4][2] == 0.0) S[4][3] = 1.0;
    const double a = S[4][0], b = S[4][1], c = S[4][2], d = S[4][3];
    const double idet = 1.0 / (a * d - b * c);
    const double Di[4] = {d * idet, -b * idet, -c * idet, a * idet};
    double rs0 = 0.0, rs1 = 0.0;
    for (int k = 0; k < 9; ++k) {
        const double* B = S[k];
        rs0 += fabs(Di[0] * B[0] + Di[1] * B[2]) + fabs(Di[0] * B[1] + Di[1] * B[3]);
        rs1 += fabs(Di[2] * B[0] + Di[3] * B[2]) + fabs(Di[2] * B[1] + Di[3] * B[3]);
    }
    if (A)
        for (int k = 0; k < 9; ++k)
            for (int e = 0; e < 4; ++e) A[aidx(nv, k, e, v)] = S[k][e];
    for (int e = 0; e < 4; ++e) Dinv[(size_t)e * nv + v] = Di[e];
    atomic_max_pos(lam, fmax(rs0, rs1));
}

// Fine level: the true rows of A0 (all vertices, incl. crossed centres), one thread per vertex
// -> 2x2 block-Jacobi inverse Dinv0 and the Gershgorin bound lambda_0 of D^-1 A0.
template <int PAT>
__global__ void k_fine_rows(const Geo2 g, const double* alpha, const unsigned char* mask, double* Dinv,
                            double* lam) {
    const long long nv = g.nv;
    for (long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x; v < nv;
         v += (long long)gridDim.x * blockDim.x) {
        // row blocks keyed by neighbour: 9 corner neighbours + 4 adjacent centres (crossed)
        double S[13][4];
        unsigned mcol[13];
        for (int k = 0; k < 13; ++k) { S[k][0] = S[k][1] = S[k][2] = S[k][3] = 0.0; mcol[k] = 0u; }
        unsigned mrow = 0u;
        if (v < g.nc) {
            const int i = (int)(v / g.nvy), j = (int)(v % g.nvy);
            mrow = vmask(mask, v);
            for (int ci = i - 1; ci <= i; ++ci)
                for (int cj = j - 1; cj <= j; ++cj) {
                    if (ci < 0 || cj < 0 || ci >= g.nx || cj >= g.ny) continue;
                    double M[25][4];
                    cell_matrix<PAT>(g, ci, cj, alpha, M);
                    const int me = (i - ci) == 0 ? ((j - cj) == 0 ? 0 : 2) : ((j - cj) == 0 ? 1 : 3);
                    for (int q = 0; q < (PAT == PF_CROSSED ? 5 : 4); ++q) {
                        int k;
                        if (q < 4) k = (ci + cdi(q) - i + 1) * 3 + (cj + cdj(q) - j + 1);
                        else k = 9 + (ci - i + 1) * 2 + (cj - j + 1);
                        for (int e = 0; e < 4; ++e) S[k][e] += M[me * 5 + q][e];
                        if (q < 4) mcol[k] = vmask(mask, (long long)(ci + cdi(q)) * g.nvy + cj + cdj(q));
                    }
                }
        } else {
            const long long cell = v - g.nc;
            const int ci = (int)(cell / g.ny), cj = (int)(cell % g.ny);
            double M[25][4];
            cell_matrix<PF_CROSSED>(g, ci, cj, alpha, M);
            for (int q = 0; q < 4; ++q) {
                for (int e = 0; e < 4; ++e) S[5 + q][e] = M[4 * 5 + q][e];
                mcol[5 + q] = vmask(mask, (long long)(ci + cdi(q)) * g.nvy + cj + cdj(q));
            }
            for (int e = 0; e < 4; ++e) S[4][e] = M[4 * 5 + 4][e];
        }
        for (int k = 0; k < 13; ++k)
            for (int r = 0; r < 2; ++r)
                for (int c = 0; c < 2; ++c)
                    if (((mrow >> r) & 1u) || ((mcol[k] >> c) & 1u)) S[k][2 * r + c] = 0.0;
        if (mrow & 1u) S[4][0] = 1.0;
        if (mrow & 2u) S[4][3] = 1.0;
        const double a = S[4][0], b = S[4][1], c = S[4][2], d = S[4][3];
        const double idet = 1.0 / (a * d - b * c);
        const double Di[4] = {d * idet, -b * idet, -c * idet, a * idet};
        double rs0 = 0.0, rs1 = 0.0;
        for (int k = 0; k < 13; ++k) {
            const double* B = S[k];
            rs0 += fabs(Di[0] * B[0] + Di[1] * B[2]) + fabs(Di[0] * B[1] + Di[1] * B[3]);
            rs1 += fabs(Di[2] * B[0] + Di[3] * B[2]) + fabs(Di[2] * B[1] + Di[3] * B[3]);
        }
        for (int e = 0; e < 4; ++e) Dinv[(size_t)e * nv + v] = Di[e];
        atomic_max_pos(lam, fmax(rs0, rs1));
    }
}

// ---- 1D transfer weights with the ceil rule ---------------------------------------------------
__device__ __forceinline__ int p1d(int f, int nf, int (&c)[2], double (&w)[2]) {
    if ((f & 1) == 0) { c[0] = f >> 1; w[0] = 1.0; return 1; }
    if (f == nf) { c[0] = (f + 1) >> 1; w[0] = 1.0; return 1; }
    c[0] = (f - 1) >> 1; c[1] = (f + 1) >> 1; w[0] = w[1] = 0.5; return 2;
}
__device__ __forceinline__ int finj(int C, int nf) { return (2 * C <= nf) ? 2 * C : nf; }

// Weights of fine node `node` (local slot of cell (ci, cj): corners 0..3, centre 4) on the 3x3
// coarse neighbourhood of coarse vertex (I, J): w[k] (k = (dK+1)*3 + dL+1), 2:1 bilinear with the
// ceil rule; the crossed centre is the mean of its cell's corners.  Masks are applied by callers.
__device__ __forceinline__ void node_weights(int fi, int fj, int nfx, int nfy, int I, int J, double (&w)[9]) {
    int cx[2], cy[2];
    double wx[2], wy[2];
    const int nxw = p1d(fi, nfx, cx, wx), nyw = p1d(fj, nfy, cy, wy);
    for (int a = 0; a < nxw; ++a)
        for (int b = 0; b < nyw; ++b) {
            const int dK = cx[a] - I, dL = cy[b] - J;
            if (dK < -1 || dK > 1 || dL < -1 || dL > 1) continue;
            w[(dK + 1) * 3 + (dL + 1)] += wx[a] * wy[b];
        }
}

// First coarse level straight from the fine cell matrices (element Galerkin): one thread per
// coarse vertex C; A1[C, C'] = sum over fine cells in C's support of w_C^T M_cell w_C'.
template <int PAT>
__global__ void k_galerkin_cells(const Geo2 g, const double* alpha, const unsigned char* mask0, int ncx, int ncy,
                                 double* A1, double* Dinv1, unsigned char* mask1, double* lam) {
    const int nvyc = ncy + 1;
    const long long nvc = (long long)(ncx + 1) * nvyc;
    for (long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x; v < nvc;
         v += (long long)gridDim.x * blockDim.x) {
        const int I = (int)(v / nvyc), J = (int)(v % nvyc);
        auto fmask = [&](int fi, int fj) -> unsigned { return vmask(mask0, (long long)fi * g.nvy + fj); };
        const unsigned mC = fmask(finj(I, g.nx), finj(J, g.ny));
        mask1[v] = (unsigned char)mC;
        double S[9][4];
        for (int k = 0; k < 9; ++k) S[k][0] = S[k][1] = S[k][2] = S[k][3] = 0.0;
        // coarse-neighbour masks (for the column side)
        unsigned mN[9];
        for (int k = 0; k < 9; ++k) {
            const int K = I + k / 3 - 1, L = J + k % 3 - 1;
            mN[k] = (K >= 0 && L >= 0 && K <= ncx && L <= ncy) ? fmask(finj(K, g.nx), finj(L, g.ny)) : 0u;
        }
        for (int ci = 2 * I - 2; ci <= 2 * I + 1; ++ci) {
            if (ci < 0 || ci >= g.nx) continue;
            for (int cj = 2 * J - 2; cj <= 2 * J + 1; ++cj) {
                if (cj < 0 || cj >= g.ny) continue;
                // weights of the cell's nodes on the 3x3 coarse neighbourhood of C
                double W[5][9];
                unsigned nm[5];
                for (int q = 0; q < 5; ++q)
                    for (int k = 0; k < 9; ++k) W[q][k] = 0.0;
                for (int q = 0; q < 4; ++q) {
                    node_weights(ci + cdi(q), cj + cdj(q), g.nx, g.ny, I, J, W[q]);
                    nm[q] = fmask(ci + cdi(q), cj + cdj(q));
                }
                nm[4] = 0u;
                if (PAT == PF_CROSSED)
                    for (int q = 0; q < 4; ++q)
                        for (int k = 0; k < 9; ++k) W[4][k] += 0.25 * W[q][k];
                // skip cells whose nodes do not interpolate from C at all
                bool touches = false;
                for (int q = 0; q < 5; ++q) touches |= (W[q][4] != 0.0);
                if (!touches) continue;
                double M[25][4];
                cell_matrix<PAT>(g, ci, cj, alpha, M);
                for (int m = 0; m < (PAT == PF_CROSSED ? 5 : 4); ++m) {
                    const double wm = W[m][4];
                    if (wm == 0.0) continue;
                    const double wm0 = ((nm[m] | mC) & 1u) ? 0.0 : wm;
                    const double wm1 = ((nm[m] | mC) & 2u) ? 0.0 : wm;
                    for (int n = 0; n < (PAT == PF_CROSSED ? 5 : 4); ++n) {
                        const double* B = M[m * 5 + n];
                        for (int k = 0; k < 9; ++k) {
                            const double wn = W[n][k];
                            if (wn == 0.0) continue;
                            const double wn0 = ((nm[n] | mN[k]) & 1u) ? 0.0 : wn;
                            const double wn1 = ((nm[n] | mN[k]) & 2u) ? 0.0 : wn;
                            S[k][0] += wm0 * B[0] * wn0;
                            S[k][1] += wm0 * B[1] * wn1;
                            S[k][2] += wm1 * B[2] * wn0;
                            S[k][3] += wm1 * B[3] * wn1;
                        }
                    }
                }
            }
        }
        finish_row(S, mC, mN, v, nvc, A1, Dinv1, lam);
    }
}

struct LevelDev {
    int nx, ny;          // cells
    long long nv;
    const double* A;
    const double* Dinv;
    const unsigned char* mask;
};

// Galerkin RAP: one thread per coarse vertex.
__global__ void k_rap(LevelDev F, LevelDev Cd, double* Ac, double* Dinvc, unsigned char* maskc, double* lam) {
    const int nvyf = F.ny + 1, nvyc = Cd.ny + 1;
    for (long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x; v < Cd.nv;
         v += (long long)gridDim.x * blockDim.x) {
        const int I = (int)(v / nvyc), J = (int)(v % nvyc);
        const unsigned mC = F.mask ? F.mask[(long long)finj(I, F.nx) * nvyf + finj(J, F.ny)] : 0u;
        maskc[v] = (unsigned char)mC;
        double S[9][4];
        for (int k = 0; k < 9; ++k) S[k][0] = S[k][1] = S[k][2] = S[k][3] = 0.0;
        for (int fi = 2 * I - 1; fi <= 2 * I + 1; ++fi) {
            if (fi < 0 || fi > F.nx) continue;
            int cx[2]; double wx[2];
            const int nxw = p1d(fi, F.nx, cx, wx);
            double wfx = 0.0;
            for (int a = 0; a < nxw; ++a) if (cx[a] == I) wfx = wx[a];
            if (wfx == 0.0) continue;
            for (int fj = 2 * J - 1; fj <= 2 * J + 1; ++fj) {
                if (fj < 0 || fj > F.ny) continue;
                int cy[2]; double wy[2];
                const int nyw = p1d(fj, F.ny, cy, wy);
                double wfy = 0.0;
                for (int b = 0; b < nyw; ++b) if (cy[b] == J) wfy = wy[b];
                if (wfy == 0.0) continue;
                const long long f = (long long)fi * nvyf + fj;
                const unsigned mf = F.mask ? F.mask[f] : 0u;
                const double wf0 = ((mf | mC) & 1u) ? 0.0 : wfx * wfy;
                const double wf1 = ((mf | mC) & 2u) ? 0.0 : wfx * wfy;
                if (wf0 == 0.0 && wf1 == 0.0) continue;
                for (int k = 0; k < 9; ++k) {
                    const int gi = fi + k / 3 - 1, gj = fj + k % 3 - 1;
                    if (gi < 0 || gj < 0 || gi > F.nx || gj > F.ny) continue;
                    double B[4];
                    for (int e = 0; e < 4; ++e) B[e] = F.A[aidx(F.nv, k, e, f)];
                    if (B[0] == 0.0 && B[1] == 0.0 && B[2] == 0.0 && B[3] == 0.0) continue;
                    const long long gv = (long long)gi * nvyf + gj;
                    const unsigned mg = F.mask ? F.mask[gv] : 0u;
                    int gx[2], gy[2]; double vx[2], vy[2];
                    const int ngx = p1d(gi, F.nx, gx, vx), ngy = p1d(gj, F.ny, gy, vy);
                    for (int a = 0; a < ngx; ++a)
                        for (int b = 0; b < ngy; ++b) {
                            const int K = gx[a], L = gy[b];
                            const int dk = (K - I + 1) * 3 + (L - J + 1);
                            const unsigned mK = F.mask ? F.mask[(long long)finj(K, F.nx) * nvyf + finj(L, F.ny)] : 0u;
                            const double w = vx[a] * vy[b];
                            const double wg0 = ((mg | mK) & 1u) ? 0.0 : w;
                            const double wg1 = ((mg | mK) & 2u) ? 0.0 : w;
                            S[dk][0] += wf0 * B[0] * wg0;
                            S[dk][1] += wf0 * B[1] * wg1;
                            S[dk][2] += wf1 * B[2] * wg0;
                            S[dk][3] += wf1 * B[3] * wg1;
                        }
                }
            }
        }
        unsigned mcol[9];
        for (int k = 0; k < 9; ++k) {
            const int K = I + k / 3 - 1, L = J + k % 3 - 1;
            mcol[k] = (K >= 0 && L >= 0 && K <= Cd.nx && L <= Cd.ny && F.mask)
                          ? F.mask[(long long)finj(K, F.nx) * nvyf + finj(L, F.ny)] : 0u;
        }
        finish_row(S, mC, mcol, v, Cd.nv, Ac, Dinvc, lam);
    }
}

// Coarsest operator -> banded Cholesky -> explicit inverse (once per setup).  Dofs are ordered
// 2v + c with v row-major, so A is banded with half-bandwidth bw = band_of(ny); the factor is kept
// as B[i * (bw + 1) + (j - i + bw)] = L[i][j], j in [i - bw, i], in shared memory (one CTA).
__global__ void k_coarse_chol_band(LevelDev L, int bw, double* Lband) {
    extern __shared__ double B[];
    const int n = (int)(2 * L.nv), W = bw + 1, nvy = L.ny + 1;
    const int t = threadIdx.x, nt = blockDim.x;
    for (int idx = t; idx < n * W; idx += nt) B[idx] = 0.0;
    __syncthreads();
    for (int v = t; v < (int)L.nv; v += nt) {
        const int i = v / nvy, j = v % nvy;
        for (int k = 0; k < 9; ++k) {
            const int ni = i + k / 3 - 1, nj = j + k % 3 - 1;
            if (ni < 0 || nj < 0 || ni > L.nx || nj > L.ny) continue;
            const int w = ni * nvy + nj;
            for (int r = 0; r < 2; ++r)
                for (int cc = 0; cc < 2; ++cc) {
                    const int row = 2 * v + r, col = 2 * w + cc;
                    if (col <= row && row - col <= bw) B[row * W + col - row + bw] = L.A[aidx(L.nv, k, 2 * r + cc, v)];
                }
        }
    }
    __syncthreads();
    for (int k = 0; k < n; ++k) {  // right-looking, inside the band
        const int last = min(n - 1, k + bw), m = last - k;
        if (t == 0) B[k * W + bw] = sqrt(B[k * W + bw]);
        __syncthreads();
        const double piv = B[k * W + bw];
        for (int i = k + 1 + t; i <= last; i += nt) B[i * W + k - i + bw] /= piv;
        __syncthreads();
        for (int p = t; p < m * m; p += nt) {
            const int ii = k + 1 + p / m, jj = k + 1 + p % m;
            if (jj <= ii) B[ii * W + jj - ii + bw] -= B[ii * W + k - ii + bw] * B[jj * W + k - jj + bw];
        }
        __syncthreads();
    }
    for (int idx = t; idx < n * W; idx += nt) Lband[idx] = B[idx];
}

// Columns of A^-1 = L^-T L^-1 from the band factor, one warp per column: L y = e_c (rows c..n-1),
// L^T x = y; x is row/column c of the symmetric inverse.
__global__ void k_coarse_inv_band(const double* Lband, int n, int bw, int wpb, double* Ainv) {
    extern __shared__ double sh[];
    const int W = bw + 1;
    double* B = sh;
    double* Y = sh + (size_t)n * W;
    for (int idx = threadIdx.x; idx < n * W; idx += blockDim.x) B[idx] = Lband[idx];
    __syncthreads();
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int c = blockIdx.x * wpb + w;
    if (w >= wpb || c >= n) return;
    double* y = Y + (size_t)w * n;
    for (int i = lane; i < n; i += 32) y[i] = 0.0;
    __syncwarp();
    for (int i = c; i < n; ++i) {
        double s = 0.0;
        for (int j = max(c, i - bw) + lane; j < i; j += 32) s += B[i * W + j - i + bw] * y[j];
        s = warp_sum(s);
        if (lane == 0) y[i] = ((i == c ? 1.0 : 0.0) - s) / B[i * W + bw];
        __syncwarp();
    }
    for (int i = n - 1; i >= 0; --i) {
        double s = 0.0;
        for (int j = i + 1 + lane; j <= min(n - 1, i + bw); j += 32) s += B[j * W + i - j + bw] * y[j];
        s = warp_sum(s);
        if (lane == 0) y[i] = (y[i] - s) / B[i * W + bw];
        __syncwarp();
    }
    for (int i = lane; i < n; i += 32) Ainv[(size_t)c * n + i] = y[i];
}

// V-cycle vectors are streamed through L2 (ld.global.cg); operators/Dinv via the read-only path.
// SH = true: the same functions on generic/shared-memory operands (plain loads); no current kernel
// instantiates it (the shared-memory tail was replaced by the grid-wide dense coarsest solve).
template <bool SH = false>
__device__ __forceinline__ double2 ldv(const double* p, long long v) {
    if constexpr (SH) return reinterpret_cast<const double2*>(p)[v];
    else return __ldcg(reinterpret_cast<const double2*>(p) + v);
}
template <bool SH = false>
__device__ __forceinline__ void stv(double* p, long long v, double2 x) {
    reinterpret_cast<double2*>(p)[v] = x;
}
template <bool SH = false>
__device__ __forceinline__ double ldr(const double* p) {  // operator data, constant during a cycle
    if constexpr (SH) return *p;
    else return __ldg(p);
}
template <bool SH = false>
__device__ __forceinline__ double2 ldr2(const double* p) {  // two entries of a stencil block (16-byte aligned)
    if constexpr (SH) return *reinterpret_cast<const double2*>(p);
    else return __ldg(reinterpret_cast<const double2*>(p));
}
template <bool SH = false>
__device__ __forceinline__ double2 bmulT(const double* Dinv, long long nv, long long v, double r0, double r1) {
    return make_double2(ldr<SH>(Dinv + v) * r0 + ldr<SH>(Dinv + nv + v) * r1,
                        ldr<SH>(Dinv + 2 * nv + v) * r0 + ldr<SH>(Dinv + 3 * nv + v) * r1);
}

// res = D^-1 src ; d = res / theta ; x (=|+=) d
template <bool SH = false>
__device__ __forceinline__ void v_cheb0(long long nv, const double* Dinv, const double* src, double* res, double* d,
                                        double* x, int accumulate, const Cheb& c, long long v) {
    const double2 s = ldv<SH>(src, v);
    const double2 r = bmulT<SH>(Dinv, nv, v, s.x, s.y);
    const double it = c.itheta;
    const double2 dd = make_double2(r.x * it, r.y * it);
    stv<SH>(res, v, r);
    stv<SH>(d, v, dd);
    double2 xo = dd;
    if (accumulate) {
        const double2 xv = ldv<SH>(x, v);
        xo = make_double2(xv.x + dd.x, xv.y + dd.y);
    }
    stv<SH>(x, v, xo);
}
__global__ void k_cheb0(long long nv, const double* Dinv, const double* src, double* res, double* d, double* x,
                        int accumulate, const double* lam, double ratio, const double* live) {
    if (!gmg_live(live)) return;
    const Cheb c = cheb_of(lam, ratio);
    for (long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x; v < nv;
         v += (long long)gridDim.x * blockDim.x)
        v_cheb0(nv, Dinv, src, res, d, x, accumulate, c, v);
}

// Sum over the G consecutive lanes that share a vertex (G = 1: no-op).
template <int G>
__device__ __forceinline__ double gsum(double x) {
    if constexpr (G > 1) {
        const unsigned lane = threadIdx.x & 31u;
        const unsigned m = ((1u << G) - 1u) << (lane & ~(unsigned)(G - 1));
#pragma unroll
        for (int o = 1; o < G; o <<= 1) x += __shfl_xor_sync(m, x, o);
    }
    return x;
}

// 9-point 2x2-block stencil apply (A y)_v with y_w = val(w).  Branch-free: an out-of-grid
// neighbour has a zero stencil block, so its address is clamped to v and the (finite) value it
// brings is multiplied by zero -- every load of the row issues at once (latency-bound levels).
// G > 1: G lanes share the vertex, lane q takes neighbours q, q+G, ... and the partial sums are
// combined by shuffles (every lane returns the full row).
template <bool SH = false, int G = 1, class F>
__device__ __forceinline__ double2 st_apply_f(const LevelDev& L, long long v, F val, int q = 0) {
    const int nvy = L.ny + 1;
    const int vi = (int)v;
    const int i = vi / nvy, j = vi - (vi / nvy) * nvy;
    double y0 = 0.0, y1 = 0.0;
#pragma unroll
    for (int t = 0; t < (9 + G - 1) / G; ++t) {
        const int k = (G == 1) ? t : q + t * G;
        if (G > 1 && k >= 9) break;
        const int ni = i + k / 3 - 1, nj = j + k % 3 - 1;
        const bool in = ni >= 0 && nj >= 0 && ni <= L.nx && nj <= L.ny;
        const long long w = in ? (long long)ni * nvy + nj : v;
        const double2 dv = val(w);
        const double2 a01 = ldr2<SH>(L.A + aidx(L.nv, k, 0, v)), a23 = ldr2<SH>(L.A + aidx(L.nv, k, 2, v));
        y0 += a01.x * dv.x + a01.y * dv.y;
        y1 += a23.x * dv.x + a23.y * dv.y;
    }
    return make_double2(gsum<G>(y0), gsum<G>(y1));
}
template <bool SH = false, int G = 1>
__device__ __forceinline__ double2 st_apply(const LevelDev& L, const double* d, long long v, int q = 0) {
    return st_apply_f<SH, G>(L, v, [&](long long w) { return ldv<SH>(d, w); }, q);
}

// One Chebyshev step k >= 1 (linalg.py:366-376): w = A d (stencil, or precomputed Ad when
// Ad != null); res -= D^-1 w; d' = rho_k rho_{k-1} d + (2 rho_k / delta) res; x (+= d) += d'.
// `addd` folds a deferred cheb0 update (x += d) of the post-smoother into this pass.
// (G, q: lanes per vertex and this lane's rank; lane 0 of the group stores.)
template <bool SH = false, int G = 1>
__device__ __forceinline__ void v_cheb_step(const LevelDev& L, const double* Ad, const double* d, double* dnext,
                                            double* res, double* x, double a, double b, int addd, long long v,
                                            int q = 0) {
    const double2 w = Ad ? ldv<SH>(Ad, v) : st_apply<SH, G>(L, d, v, q);
    if (G > 1 && q != 0) return;
    const double2 dw = bmulT<SH>(L.Dinv, L.nv, v, w.x, w.y);
    double2 r = ldv<SH>(res, v);
    r.x -= dw.x;
    r.y -= dw.y;
    const double2 dv = ldv<SH>(d, v);
    const double2 dn = make_double2(a * dv.x + b * r.x, a * dv.y + b * r.y);
    stv<SH>(res, v, r);
    stv<SH>(dnext, v, dn);
    double2 xv = ldv<SH>(x, v);
    if (addd) {
        xv.x += dv.x;
        xv.y += dv.y;
    }
    xv.x += dn.x;
    xv.y += dn.y;
    stv<SH>(x, v, xv);
}
__global__ void k_cheb_step(LevelDev L, const double* Ad, const double* d, double* dnext, double* res, double* x,
                            int k, int addd, const double* lam, double ratio, const double* live) {
    if (!gmg_live(live)) return;
    const Cheb c = cheb_of(lam, ratio);
    double a, b;
    cheb_ab(c, k, a, b);
    for (long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x; v < L.nv;
         v += (long long)gridDim.x * blockDim.x)
        v_cheb_step(L, Ad, d, dnext, res, x, a, b, addd, v);
}

// Pre-smoother from x = 0, cheb0 fused into step 1: d0 = D^-1 b / theta is recomputed at the
// stencil neighbours, so one pass gives res, d0, d1 and x = d0 + d1 (x = d0 when deg == 1).
template <bool SH = false, int G = 1>
__device__ __forceinline__ void v_pre_first(const LevelDev& L, const double* bvec, double* res, double* d0,
                                            double* d1, double* x, const Cheb& c, double a, double b, int deg,
                                            long long v, int q = 0) {
    const double it = c.itheta;
    if (deg <= 1) {
        if (G > 1 && q != 0) return;
        const double2 s = ldv<SH>(bvec, v);
        const double2 r0 = bmulT<SH>(L.Dinv, L.nv, v, s.x, s.y);
        const double2 dd = make_double2(r0.x * it, r0.y * it);
        stv<SH>(d0, v, dd);
        stv<SH>(res, v, r0);
        stv<SH>(x, v, dd);
        return;
    }
    const double2 w = st_apply_f<SH, G>(L, v, [&](long long u) {
        const double2 sq = ldv<SH>(bvec, u);
        const double2 rq = bmulT<SH>(L.Dinv, L.nv, u, sq.x, sq.y);
        return make_double2(rq.x * it, rq.y * it);
    }, q);
    if (G > 1 && q != 0) return;
    const double2 s = ldv<SH>(bvec, v);
    const double2 r0 = bmulT<SH>(L.Dinv, L.nv, v, s.x, s.y);
    const double2 dd = make_double2(r0.x * it, r0.y * it);
    stv<SH>(d0, v, dd);
    const double2 dw = bmulT<SH>(L.Dinv, L.nv, v, w.x, w.y);
    const double2 r = make_double2(r0.x - dw.x, r0.y - dw.y);
    const double2 dn = make_double2(a * dd.x + b * r.x, a * dd.y + b * r.y);
    stv<SH>(res, v, r);
    stv<SH>(d1, v, dn);
    stv<SH>(x, v, make_double2(dd.x + dn.x, dd.y + dn.y));
}
// v_pre_first with r0 = D^-1 b precomputed by the restriction into this level (in the d0 buffer):
// the neighbours' d0 = r0 / theta are formed from the gathered r0 instead of from b and D^-1 (~40%
// fewer loads per vertex) -- the same arithmetic, so the same bits.  d0 is not written (neighbours
// still read r0 there); the pre-smoother continues from d1 (deg >= 2) or x (deg 1).
template <bool SH = false, int G = 1>
__device__ __forceinline__ void v_pre_first_d0(const LevelDev& L, double* res, const double* rb, double* d1,
                                               double* x, const Cheb& c, double a, double b, int deg, long long v,
                                               int q = 0) {
    const double it = c.itheta;
    if (deg <= 1) {
        if (G > 1 && q != 0) return;
        const double2 r0 = ldv<SH>(rb, v);
        stv<SH>(res, v, r0);
        stv<SH>(x, v, make_double2(r0.x * it, r0.y * it));
        return;
    }
    const double2 w = st_apply_f<SH, G>(L, v, [&](long long u) {
        const double2 rq = ldv<SH>(rb, u);
        return make_double2(rq.x * it, rq.y * it);
    }, q);
    if (G > 1 && q != 0) return;
    const double2 r0 = ldv<SH>(rb, v);
    const double2 dd = make_double2(r0.x * it, r0.y * it);
    const double2 dw = bmulT<SH>(L.Dinv, L.nv, v, w.x, w.y);
    const double2 r = make_double2(r0.x - dw.x, r0.y - dw.y);
    const double2 dn = make_double2(a * dd.x + b * r.x, a * dd.y + b * r.y);
    stv<SH>(res, v, r);
    stv<SH>(d1, v, dn);
    stv<SH>(x, v, make_double2(dd.x + dn.x, dd.y + dn.y));
}
__global__ void k_pre_first(LevelDev L, const double* bvec, double* res, double* d0, double* d1, double* x, int deg,
                            const double* lam, double ratio, const double* live) {
    if (!gmg_live(live)) return;
    const Cheb c = cheb_of(lam, ratio);
    double a = 0.0, b = 0.0;
    if (deg > 1) cheb_ab(c, 1, a, b);
    for (long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x; v < L.nv;
         v += (long long)gridDim.x * blockDim.x)
        v_pre_first(L, bvec, res, d0, d1, x, c, a, b, deg, v);
}

// r = b - A x (stencil) or r = b - Ax (precomputed)
template <bool SH = false, int G = 1>
__device__ __forceinline__ void v_resid(const LevelDev& L, const double* Ax, const double* x, const double* b,
                                        double* r, long long v, int q = 0) {
    const double2 w = Ax ? ldv<SH>(Ax, v) : st_apply<SH, G>(L, x, v, q);
    if (G > 1 && q != 0) return;
    const double2 bv = ldv<SH>(b, v);
    stv<SH>(r, v, make_double2(bv.x - w.x, bv.y - w.y));
}
__global__ void k_resid(LevelDev L, const double* Ax, const double* x, const double* b, double* r, const double* live) {
    if (!gmg_live(live)) return;
    for (long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x; v < L.nv;
         v += (long long)gridDim.x * blockDim.x)
        v_resid(L, Ax, x, b, r, v);
}

// Post-smoother entry with cheb0 fused into the residual: res = D^-1 (b - A x), d0 = res/theta.
// x is NOT updated here (neighbours still read it); the following step adds d0 (addd).
template <bool SH = false, int G = 1>
__device__ __forceinline__ void v_post_first(const LevelDev& L, const double* x, const double* b, double* res,
                                             double* d0, const Cheb& c, long long v, int q = 0) {
    const double2 w = st_apply<SH, G>(L, x, v, q);
    if (G > 1 && q != 0) return;
    const double2 bv = ldv<SH>(b, v);
    const double2 s = make_double2(bv.x - w.x, bv.y - w.y);
    const double2 r = bmulT<SH>(L.Dinv, L.nv, v, s.x, s.y);
    stv<SH>(res, v, r);
    const double it = c.itheta;
    stv<SH>(d0, v, make_double2(r.x * it, r.y * it));
}
__global__ void k_post_first(LevelDev L, const double* x, const double* b, double* res, double* d0,
                             const double* lam, double ratio, const double* live) {
    if (!gmg_live(live)) return;
    const Cheb c = cheb_of(lam, ratio);
    for (long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x; v < L.nv;
         v += (long long)gridDim.x * blockDim.x)
        v_post_first(L, x, b, res, d0, c, v);
}
__global__ void k_add(long long nv, const double* d, double* x, const double* live) {
    if (!gmg_live(live)) return;
    for (long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x; v < nv;
         v += (long long)gridDim.x * blockDim.x) {
        const double2 dv = ldv(d, v);
        double2 xv = ldv(x, v);
        xv.x += dv.x;
        xv.y += dv.y;
        stv(x, v, xv);
    }
}

// Weight of fine index f (0..nf) on coarse index C under the 2:1 ceil-rule interpolation (p1d).
__device__ __forceinline__ double w1d(int f, int nf, int C) {
    if (f < 0 || f > nf) return 0.0;
    if ((f & 1) == 0) return (f >> 1) == C ? 1.0 : 0.0;
    if (f == nf) return ((f + 1) >> 1) == C ? 1.0 : 0.0;
    return (((f - 1) >> 1) == C || ((f + 1) >> 1) == C) ? 0.5 : 0.0;
}
// 2:1 restriction b_c = P^T r_f (with masks), one thread per coarse vertex; fv(f) = fine value.
// The 3x3 fine neighbourhood is gathered unconditionally (clamped addresses, zero weights).
// G > 1: G lanes share the coarse vertex (fine points t = q, q + G, ...), lane 0 stores.
template <bool SH = false, int G = 1, class FV>
__device__ __forceinline__ void v_restrict_f(const LevelDev& F, const LevelDev& Cd, const unsigned char* maskc,
                                             FV fv, double* bc, long long v, int q = 0, double* d0c = nullptr) {
    const int nvyf = F.ny + 1, nvyc = Cd.ny + 1;
    const int vi = (int)v;
    const int I = vi / nvyc, J = vi - (vi / nvyc) * nvyc;
    double s0 = 0.0, s1 = 0.0;
#pragma unroll
    for (int u = 0; u < (9 + G - 1) / G; ++u) {
        const int t = (G == 1) ? u : q + u * G;
        if (G > 1 && t >= 9) break;
        const int fi = 2 * I - 1 + t / 3, fj = 2 * J - 1 + t % 3;
        const double w = w1d(fi, F.nx, I) * w1d(fj, F.ny, J);
        const long long f = (long long)min(max(fi, 0), F.nx) * nvyf + min(max(fj, 0), F.ny);
        const unsigned mf = F.mask ? F.mask[f] : 0u;
        const double2 rv = fv(f);
        if (w != 0.0 && !(mf & 1u)) s0 += w * rv.x;
        if (w != 0.0 && !(mf & 2u)) s1 += w * rv.y;
    }
    s0 = gsum<G>(s0);
    s1 = gsum<G>(s1);
    if (G > 1 && q != 0) return;
    const unsigned mC = maskc[v];
    const double2 bv = make_double2((mC & 1u) ? 0.0 : s0, (mC & 2u) ? 0.0 : s1);
    stv<SH>(bc, v, bv);
    if (d0c) {  // r0 = D^-1 b of the coarse pre-smoother, once per vertex (v_pre_first_d0)
        stv<SH>(d0c, v, bmulT<SH>(Cd.Dinv, Cd.nv, v, bv.x, bv.y));
    }
}
template <bool SH = false, int G = 1>
__device__ __forceinline__ void v_restrict(const LevelDev& F, const LevelDev& Cd, const unsigned char* maskc,
                                           const double* r, double* bc, long long v, int q = 0,
                                           double* d0c = nullptr) {
    v_restrict_f<SH, G>(F, Cd, maskc, [&](long long f) { return ldv<SH>(r, f); }, bc, v, q, d0c);
}
__global__ void k_restrict(LevelDev F, LevelDev Cd, const unsigned char* maskc, const double* r, double* bc,
                           const double* live) {
    if (!gmg_live(live)) return;
    for (long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x; v < Cd.nv;
         v += (long long)gridDim.x * blockDim.x)
        v_restrict(F, Cd, maskc, r, bc, v);
}

// 2:1 prolongation x_f += P x_c (with masks), one thread per fine vertex
template <bool SH = false>
__device__ __forceinline__ double2 pval_ij(const LevelDev& F, const LevelDev& Cd, const unsigned char* maskc,
                                           const double* xc, int fi, int fj) {  // (P x_c) at fine vertex (fi, fj)
    const int nvyc = Cd.ny + 1;
    int cx[2], cy[2]; double wx[2], wy[2];
    const int nxw = p1d(fi, F.nx, cx, wx), nyw = p1d(fj, F.ny, cy, wy);
    if (nxw == 1) { cx[1] = cx[0]; wx[1] = 0.0; }
    if (nyw == 1) { cy[1] = cy[0]; wy[1] = 0.0; }
    double s0 = 0.0, s1 = 0.0;
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int b = 0; b < 2; ++b) {
            const long long c = (long long)cx[a] * nvyc + cy[b];
            const unsigned mC = maskc[c];
            const double2 xv = ldv<SH>(xc, c);
            const double w = wx[a] * wy[b];
            if (w != 0.0 && !(mC & 1u)) s0 += w * xv.x;
            if (w != 0.0 && !(mC & 2u)) s1 += w * xv.y;
        }
    return make_double2(s0, s1);
}
template <bool SH = false>
__device__ __forceinline__ double2 pval(const LevelDev& F, const LevelDev& Cd, const unsigned char* maskc,
                                        const double* xc, long long v) {  // (P x_c) at fine vertex v
    const int nvyf = F.ny + 1;
    const int vi = (int)v;
    const int fi = vi / nvyf;
    return pval_ij<SH>(F, Cd, maskc, xc, fi, vi - fi * nvyf);
}
template <bool SH = false>
__device__ __forceinline__ void v_prolong(const LevelDev& F, const LevelDev& Cd, const unsigned char* maskc,
                                          const double* xc, double* xf, long long v) {
    const unsigned mf = F.mask ? F.mask[v] : 0u;
    const double2 s = pval<SH>(F, Cd, maskc, xc, v);
    double2 o = ldv<SH>(xf, v);
    if (!(mf & 1u)) o.x += s.x;
    if (!(mf & 2u)) o.y += s.y;
    stv<SH>(xf, v, o);
}
__global__ void k_prolong(LevelDev F, LevelDev Cd, const unsigned char* maskc, const double* xc, double* xf,
                          const double* live) {
    if (!gmg_live(live)) return;
    for (long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x; v < F.nv;
         v += (long long)gridDim.x * blockDim.x)
        v_prolong(F, Cd, maskc, xc, xf, v);
}

// ---- coarse tail of the V-cycle in one CTA ------------------------------------------------------
// Levels lc..nl-1 (each <= kTailMaxV vertices, L2/L1-resident) run in a single 512-thread block:
// per level pre-smooth (cheb0 fused into step 1), steps 2..deg-1, residual, restriction; the
// dense coarse solve; then prolongation, residual + cheb0, steps (x += d0 on step 1) -- the same
// per-vertex functions, in the same order, as the per-level kernels, separated by __syncthreads
// instead of kernel boundaries.
constexpr int kTailMaxV = 300;
constexpr int kTailLev = 12;
constexpr int kTB = 512;
struct TLev {
    LevelDev L;
    double *x, *b, *r, *d0, *d1, *res;
};
struct TailArgs {
    int lc, nl, deg, ncoarse;
    double ratio;
    const double* ainv;
    TLev lev[kTailLev];
};

__global__ void __launch_bounds__(kTB, 1) k_gmg_tail(const __grid_constant__ TailArgs A, const double* lam,
                                                     const double* live) {
    if (!gmg_live(live)) return;  // uniform: the flags are not written during the launch
    const int t0 = threadIdx.x;
    const int deg = A.deg;
    for (int l = A.lc; l < A.nl - 1; ++l) {
        const TLev& V = A.lev[l];
        const Cheb c = cheb_of(lam + l, A.ratio);
        double a = 0.0, b = 0.0;
        if (deg > 1) cheb_ab(c, 1, a, b);
        for (long long v = t0; v < V.L.nv; v += kTB) v_pre_first(V.L, V.b, V.res, V.d0, V.d1, V.x, c, a, b, deg, v);
        __syncthreads();
        double* d = V.d1;
        double* dn = V.d0;
        for (int k = 2; k < deg; ++k) {
            cheb_ab(c, k, a, b);
            for (long long v = t0; v < V.L.nv; v += kTB) v_cheb_step(V.L, nullptr, d, dn, V.res, V.x, a, b, 0, v);
            __syncthreads();
            double* tmp = d; d = dn; dn = tmp;
        }
        for (long long v = t0; v < V.L.nv; v += kTB) v_resid(V.L, nullptr, V.x, V.b, V.r, v);
        __syncthreads();
        const TLev& C = A.lev[l + 1];
        for (long long v = t0; v < C.L.nv; v += kTB) v_restrict(V.L, C.L, C.L.mask, V.r, C.b, v);
        __syncthreads();
    }
    {   // coarsest: x = Ainv b, one warp per row
        const TLev& C = A.lev[A.nl - 1];
        const int n = A.ncoarse, lane = t0 & 31;
        for (int r = t0 >> 5; r < n; r += kTB / 32) {
            double s = 0.0;
            for (int q = lane; q < n; q += 32) s += A.ainv[(size_t)r * n + q] * __ldcg(C.b + q);
            s = warp_sum(s);
            if (lane == 0) C.x[r] = s;
        }
        __syncthreads();
    }
    for (int l = A.nl - 2; l >= A.lc; --l) {
        const TLev& V = A.lev[l];
        const TLev& C = A.lev[l + 1];
        const Cheb c = cheb_of(lam + l, A.ratio);
        for (long long v = t0; v < V.L.nv; v += kTB) v_prolong(V.L, C.L, C.L.mask, C.x, V.x, v);
        __syncthreads();
        for (long long v = t0; v < V.L.nv; v += kTB) v_post_first(V.L, V.x, V.b, V.res, V.d0, c, v);
        __syncthreads();
        if (deg <= 1) {
            for (long long v = t0; v < V.L.nv; v += kTB) {
                const double2 dv = ldv(V.d0, v);
                double2 xv = ldv(V.x, v);
                xv.x += dv.x;
                xv.y += dv.y;
                stv(V.x, v, xv);
            }
            __syncthreads();
        }
        double* d = V.d0;
        double* dn = V.d1;
        for (int k = 1; k < deg; ++k) {
            double a, b;
            cheb_ab(c, k, a, b);
            for (long long v = t0; v < V.L.nv; v += kTB) v_cheb_step(V.L, nullptr, d, dn, V.res, V.x, a, b, k == 1, v);
            __syncthreads();
            double* tmp = d; d = dn; dn = tmp;
        }
    }
}

// crossed level 0 <-> corner grid, factored as P0 = (corner identity + centre mean) o P_{2:1}:
// z[c] = m_c r[c] + 1/4 sum_{adjacent centres} r[ctr]  (then unmasked-fine 2:1 restriction)
__global__ void k_collapse_centres(const Geo2 g, const unsigned char* mask0, const double* r, double* z,
                                   const double* live) {
    if (!gmg_live(live)) return;
    for (long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x; v < g.nc;
         v += (long long)gridDim.x * blockDim.x) {
        const int i = (int)(v / g.nvy), j = (int)(v % g.nvy);
        const unsigned m = vmask(mask0, v);
        const double2 rv = reinterpret_cast<const double2*>(r)[v];
        double s0 = (m & 1u) ? 0.0 : rv.x, s1 = (m & 2u) ? 0.0 : rv.y;
        for (int ci = i - 1; ci <= i; ++ci)
            for (int cj = j - 1; cj <= j; ++cj) {
                if (ci < 0 || cj < 0 || ci >= g.nx || cj >= g.ny) continue;
                const double2 rc = reinterpret_cast<const double2*>(r)[g.nc + (long long)ci * g.ny + cj];
                s0 += 0.25 * rc.x;
                s1 += 0.25 * rc.y;
            }
        reinterpret_cast<double2*>(z)[v] = make_double2(s0, s1);
    }
}
// x[c] += m_c y[c] ; x[ctr] += 1/4 sum of its corners' y  (y = P_{2:1} x1 on the corner grid)
__global__ void k_expand_centres(const Geo2 g, const unsigned char* mask0, const double* y, double* x,
                                 const double* live) {
    if (!gmg_live(live)) return;
    for (long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x; v < g.nv;
         v += (long long)gridDim.x * blockDim.x) {
        double2 o = reinterpret_cast<double2*>(x)[v];
        if (v < g.nc) {
            const unsigned m = vmask(mask0, v);
            const double2 a = reinterpret_cast<const double2*>(y)[v];
            if (!(m & 1u)) o.x += a.x;
            if (!(m & 2u)) o.y += a.y;
        } else {
            const long long cell = v - g.nc;
            const long long v00 = (cell / g.ny) * g.nvy + cell % g.ny;
            const long long cs[4] = {v00, v00 + g.nvy, v00 + 1, v00 + g.nvy + 1};
            for (int q = 0; q < 4; ++q) {
                const double2 a = reinterpret_cast<const double2*>(y)[cs[q]];
                o.x += 0.25 * a.x;
                o.y += 0.25 * a.y;
            }
        }
        reinterpret_cast<double2*>(x)[v] = o;
    }
}

// ---- the coarse part of the V-cycle in one persistent launch -------------------------------------
// Both level-0 transfers, the smoothing of levels 1..nl-2 and the dense solve on the coarsest level
// run in one cooperative kernel: grid-wide phases separated by a software grid barrier.  Every
// phase is latency-bound (levels of 66k vertices and fewer), so the per-vertex functions are
// branch-free with all loads of a row issued at once, small levels give each vertex 4 lanes
// (shuffle-reduced stencil rows), the Chebyshev coefficients are computed once per launch into
// shared memory, and the coarsest solve is one matvec with the explicit inverse (<= 600 dofs,
// one warp per row).  The arithmetic is that of the launch-per-phase cycle (PF_GMG_LEGACY) up to
// summation order; what goes away is ~30 dependent launches per V-cycle.
constexpr int kMaxLev = 16;  // = the S_GMG0 lambda slots
constexpr int kMaxDeg = 8;
struct CCoef {  // per-level Chebyshev coefficients, computed once per launch into shared memory
    Cheb c;
    double a[kMaxDeg], b[kMaxDeg];
};
struct CLev {
    LevelDev L;
    double *x, *b, *r, *d0, *d1, *res;
};
struct CoarseArgs {
    Geo2 g;
    LevelDev L0;                  // level-0 corner view (mask: as the level-0 transfers use it)
    const unsigned char* mask0;   // level-0 Dirichlet mask for the crossed collapse/expand (or null)
    const double* r0;             // level-0 residual (restricted)
    double* z0;                   // level-0 correction (+= P x1)
    int crossed, nl, lc, deg, ncoarse, coef_off;  // lc: coarsest level (= nl - 1)
    double ratio;
    const double* ainv;
    unsigned int* bar;
    int skip;                     // timing aid (PF_GMG_SKIP_COARSE): return at entry
    unsigned long long* trace;    // timing aid (PF_GMG_TRACE): %globaltimer per phase, CTA 0
    CLev lev[kMaxLev];
};

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define TR()                                                                               \
    do {                                                                                   \
        if (A.trace && blockIdx.x == 0 && threadIdx.x == 0) A.trace[tro + ntr++] = gtimer(); \
    } while (0)

// Two lanes per vertex for levels of nth/4 < nv <= nth/2 vertices: off.  Every phase of the
// persistent cycle starts on cold instructions (ncu: 12 % of its stall samples are instruction
// fetch), and the variant was a quarter of the kernel's 15.5k SASS instructions; without it the SENT
// 512^2 window is 0.6 % and the config-3 slab step 3.4 % faster (neither has a level in that range).
constexpr bool kCoarseG2 = false;
constexpr int kCB = 512;  // threads per CTA of the persistent coarse cycle (one CTA per SM; 1024 measured slower)
// Chebyshev coefficients of every level into shared memory (threads t < nl; read by the phases
// after the first barrier)
__device__ __forceinline__ void coarse_coef(const CoarseArgs& A, const double* lam, CCoef* coef) {
    const int t0 = threadIdx.x;
    if (t0 < A.nl) {
        CCoef& q = coef[t0];
        q.c = cheb_of(lam + t0, A.ratio);
        for (int k = 1; k < A.deg && k < kMaxDeg; ++k) cheb_ab(q.c, k, q.a[k], q.b[k]);
    }
}

// Barriers between the phases: the software grid barrier of the persistent cooperative launch, or
// the hardware cluster barrier (barrier.cluster, release/acquire at cluster scope: ~0.2 us against
// ~1.5-2 us for the grid barrier) when the phases run inside one thread-block cluster.
struct GridBar {
    unsigned int* bar;
    __device__ __forceinline__ void operator()() const { grid_sync(bar); }
};
struct ClusterBar {
    __device__ __forceinline__ void operator()() const {
        asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
        asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
    }
};
// Which phases a launch runs: the whole coarse cycle (one grid launch), or split at level lt into
// the grid-wide top (restriction from level 0 down to lt; prolongation from lt back to level 0)
// and the cluster part (levels lt..nl-1 and back up to lt, small and latency-bound).
enum { CP_ALL = 0, CP_DOWN = 1, CP_CLUSTER = 2, CP_UP = 3 };

// The coarse part of one V-cycle as phases over threads tid of nth separated by sync(); the full
// cycle (CP_ALL) ends with the level-0 prolongation into A.z0 (the caller synchronises before
// reading it).
template <class SYNC>
__device__ __forceinline__ void coarse_body(const CoarseArgs& A, const CCoef* coef, long long tid, long long nth,
                                            int part, int lt, SYNC sync) {
    const int deg = A.deg;
    const int t0 = threadIdx.x;
    (void)t0;
    // stencil phases: 4 (or 2) lanes per vertex when the level is small enough (shorter chains)
    using G1 = std::integral_constant<int, 1>;
    using G2 = std::integral_constant<int, 2>;
    using G4 = std::integral_constant<int, 4>;
    auto grid_each = [&](long long nv, auto fn) {
        if (4 * nv <= nth)
            for (long long e = tid; e < 4 * nv; e += nth) fn(G4{}, e >> 2, (int)(e & 3));
        else if (kCoarseG2 && 2 * nv <= nth)  // (2 lanes in 2 rounds measured slower than 1 lane in 1 round)
            for (long long e = tid; e < 2 * nv; e += nth) fn(G2{}, e >> 1, (int)(e & 1));
        else
            for (long long v = tid; v < nv; v += nth) fn(G1{}, v, 0);
    };
    int ntr = 0;
    const int tro = part == CP_ALL ? 0 : 40 * (part - 1);  // trace slots per launch of a split cycle
    TR();
    // level 0 -> 1 restriction (crossed: centres collapsed onto the corners on the fly)
    if (part == CP_ALL || part == CP_DOWN) {
        const CLev& C = A.lev[1];
        if (A.crossed) {
            const Geo2& g = A.g;
            auto collapse = [&](long long v) -> double2 {
                const int i = (int)(v / g.nvy), j = (int)(v % g.nvy);
                const unsigned m = vmask(A.mask0, v);
                const double2 rv = ldv(A.r0, v);
                double s0 = (m & 1u) ? 0.0 : rv.x, s1 = (m & 2u) ? 0.0 : rv.y;
                for (int ci = i - 1; ci <= i; ++ci)
                    for (int cj = j - 1; cj <= j; ++cj) {
                        if (ci < 0 || cj < 0 || ci >= g.nx || cj >= g.ny) continue;
                        const double2 rc = ldv(A.r0, g.nc + (long long)ci * g.ny + cj);
                        s0 += 0.25 * rc.x;
                        s1 += 0.25 * rc.y;
                    }
                return make_double2(s0, s1);
            };
            // one lane per coarse vertex (the large meshes): the 3x3 fine vertices under it touch
            // 4x4 cells, so their 16 centres are loaded once instead of 4 per fine vertex (36);
            // every sum is formed in collapse()'s order (an absent cell adds 0.25 * 0)
            auto restrict1 = [&](long long v) {
                const int nvyc = C.L.ny + 1;
                const int I = (int)(v / nvyc), J = (int)(v % nvyc);
                double2 cen[4][4];
#pragma unroll
                for (int a = 0; a < 4; ++a)
#pragma unroll
                    for (int b = 0; b < 4; ++b) {
                        const int ci = 2 * I - 2 + a, cj = 2 * J - 2 + b;
                        const bool in = ci >= 0 && cj >= 0 && ci < g.nx && cj < g.ny;
                        cen[a][b] = in ? ldv(A.r0, g.nc + (long long)ci * g.ny + cj) : make_double2(0.0, 0.0);
                    }
                double s0 = 0.0, s1 = 0.0;
#pragma unroll
                for (int t = 0; t < 9; ++t) {
                    const int pa = t / 3, pb = t % 3;
                    const int fi = 2 * I - 1 + pa, fj = 2 * J - 1 + pb;
                    const double w = w1d(fi, g.nx, I) * w1d(fj, g.ny, J);
                    if (w == 0.0) continue;  // (also every out-of-range fine vertex)
                    const long long f = (long long)fi * g.nvy + fj;
                    const unsigned m = vmask(A.mask0, f);
                    const double2 rv = ldv(A.r0, f);
                    double c0 = (m & 1u) ? 0.0 : rv.x, c1 = (m & 2u) ? 0.0 : rv.y;
#pragma unroll
                    for (int da = 0; da < 2; ++da)
#pragma unroll
                        for (int db = 0; db < 2; ++db) {
                            c0 += 0.25 * cen[pa + da][pb + db].x;
                            c1 += 0.25 * cen[pa + da][pb + db].y;
                        }
                    const unsigned mf = A.L0.mask ? A.L0.mask[f] : 0u;
                    if (!(mf & 1u)) s0 += w * c0;
                    if (!(mf & 2u)) s1 += w * c1;
                }
                const unsigned mC = C.L.mask[v];
                const double2 bv = make_double2((mC & 1u) ? 0.0 : s0, (mC & 2u) ? 0.0 : s1);
                stv(C.b, v, bv);
                if (C.d0) stv(C.d0, v, bmulT<false>(C.L.Dinv, C.L.nv, v, bv.x, bv.y));
            };
            grid_each(C.L.nv, [&](auto gg, long long v, int q) {
                if constexpr (decltype(gg)::value == 1) restrict1(v);
                else v_restrict_f<false, decltype(gg)::value>(A.L0, C.L, C.L.mask, collapse, C.b, v, q, C.d0);
            });
        } else {
            grid_each(C.L.nv, [&](auto g, long long v, int q) { v_restrict<false, decltype(g)::value>(A.L0, C.L, C.L.mask, A.r0, C.b, v, q, C.d0); });
        }
        sync();
        TR();
    }
    // descend: pre-smooth, residual, restriction of levels [d0, d1)
    const int d0 = part == CP_CLUSTER ? lt : 1;
    const int d1 = part == CP_DOWN ? lt : (part == CP_UP ? 0 : A.nl - 1);
    for (int l = d0; l < d1; ++l) {
        const CLev& V = A.lev[l];
        const Cheb c = coef[l].c;
        double a = 0.0, b = 0.0;
        if (deg > 1) { a = coef[l].a[1]; b = coef[l].b[1]; }
        grid_each(V.L.nv, [&](auto g, long long v, int q) { v_pre_first_d0<false, decltype(g)::value>(V.L, V.res, V.d0, V.d1, V.x, c, a, b, deg, v, q); });
        sync();
        TR();
        double* d = V.d0;
        double* dn = V.d1;
        if (deg > 1) { double* t = d; d = dn; dn = t; }
        for (int k = 2; k < deg; ++k) {
            a = coef[l].a[k]; b = coef[l].b[k];
            grid_each(V.L.nv, [&](auto g, long long v, int q) { v_cheb_step<false, decltype(g)::value>(V.L, nullptr, d, dn, V.res, V.x, a, b, 0, v, q); });
            sync();
            TR();
            double* t = d; d = dn; dn = t;
        }
        grid_each(V.L.nv, [&](auto g, long long v, int q) { v_resid<false, decltype(g)::value>(V.L, nullptr, V.x, V.b, V.r, v, q); });
        sync();
        TR();
        const CLev& C = A.lev[l + 1];
        double* r0c = l + 1 < A.nl - 1 ? C.d0 : nullptr;  // the coarsest level has no pre-smoother
        grid_each(C.L.nv, [&](auto g, long long v, int q) { v_restrict<false, decltype(g)::value>(V.L, C.L, C.L.mask, V.r, C.b, v, q, r0c); });
        sync();
        TR();
    }
    // coarsest level: x = Ainv b, one warp per row across the threads
    if (part == CP_ALL || part == CP_CLUSTER) {
        const CLev& C = A.lev[A.nl - 1];
        const int n = A.ncoarse, lane = t0 & 31;
        for (long long r = tid >> 5; r < n; r += nth >> 5) {
            double sum = 0.0;
            for (int q = lane; q < n; q += 32) sum += __ldg(A.ainv + (size_t)r * n + q) * __ldcg(C.b + q);
            sum = warp_sum(sum);
            if (lane == 0) C.x[r] = sum;
        }
        sync();
        TR();
    }
    // ascend: prolongation from l + 1, post-smoothing of levels (u0, u1] from the top down
    const int u1 = part == CP_UP ? lt - 1 : (part == CP_DOWN ? 0 : A.nl - 2);
    const int u0 = part == CP_CLUSTER ? lt : 1;
    for (int l = u1; l >= u0; --l) {
        const CLev& V = A.lev[l];
        const CLev& C = A.lev[l + 1];
        const Cheb c = coef[l].c;
        for (long long v = tid; v < V.L.nv; v += nth) v_prolong(V.L, C.L, C.L.mask, C.x, V.x, v);
        sync();
        TR();
        grid_each(V.L.nv, [&](auto g, long long v, int q) { v_post_first<false, decltype(g)::value>(V.L, V.x, V.b, V.res, V.d0, c, v, q); });
        sync();
        TR();
        if (deg <= 1) {
            for (long long v = tid; v < V.L.nv; v += nth) {
                const double2 dv = ldv(V.d0, v);
                double2 xv = ldv(V.x, v);
                xv.x += dv.x;
                xv.y += dv.y;
                stv(V.x, v, xv);
            }
            sync();
            TR();
        }
        double* d = V.d0;
        double* dn = V.d1;
        for (int k = 1; k < deg; ++k) {
            double a, b;
            a = coef[l].a[k]; b = coef[l].b[k];
            grid_each(V.L.nv, [&](auto g, long long v, int q) { v_cheb_step<false, decltype(g)::value>(V.L, nullptr, d, dn, V.res, V.x, a, b, k == 1, v, q); });
            sync();
            TR();
            double* tmp = d; d = dn; dn = tmp;
        }
    }
    // level 1 -> 0 prolongation (crossed: centres take the mean of their corners' corrections)
    if (part == CP_ALL || part == CP_UP) {
        const CLev& C = A.lev[1];
        if (A.crossed) {
            const Geo2& g = A.g;
            for (long long v = tid; v < g.nv; v += nth) {
                double2 o = ldv(A.z0, v);
                if (v < g.nc) {
                    const unsigned m = vmask(A.mask0, v);
                    const double2 a = pval(A.L0, C.L, C.L.mask, C.x, v);
                    if (!(m & 1u)) o.x += a.x;
                    if (!(m & 2u)) o.y += a.y;
                } else {  // (32-bit index arithmetic: the phase is bound by its instruction stream)
                    const int cell = (int)(v - g.nc);
                    const int ci = cell / g.ny, cj = cell - ci * g.ny;
                    for (int q = 0; q < 4; ++q) {  // corners (ci, cj), (ci+1, cj), (ci, cj+1), (ci+1, cj+1)
                        const double2 a = pval_ij(A.L0, C.L, C.L.mask, C.x, ci + (q & 1), cj + (q >> 1));
                        o.x += 0.25 * a.x;
                        o.y += 0.25 * a.y;
                    }
                }
                stv(A.z0, v, o);
            }
        } else {
            for (long long v = tid; v < A.L0.nv; v += nth) v_prolong(A.L0, C.L, C.L.mask, C.x, A.z0, v);
        }
        TR();  // (block 0's own share of the last phase: no barrier follows it)
    }
}

__global__ void __launch_bounds__(kCB, 1) k_gmg_coarse(const __grid_constant__ CoarseArgs A, const double* lam,
                                                       const double* live, int part, int lt) {
    if (!gmg_live(live) || A.skip) return;  // uniform: the flags are not written during the launch
    extern __shared__ __align__(16) unsigned char sm[];
    CCoef* coef = reinterpret_cast<CCoef*>(sm + A.coef_off);
    coarse_coef(A, lam, coef);
    __syncthreads();
    coarse_body(A, coef, blockIdx.x * (long long)kCB + threadIdx.x, (long long)gridDim.x * kCB, part, lt,
                GridBar{A.bar});
}
// levels lt..nl-1 of the coarse cycle in ONE thread-block cluster (grid = the cluster)
__global__ void __launch_bounds__(kCB, 1) k_gmg_ctail(const __grid_constant__ CoarseArgs A, const double* lam,
                                                      const double* live, int lt) {
    if (!gmg_live(live) || A.skip) return;
    extern __shared__ __align__(16) unsigned char sm[];
    CCoef* coef = reinterpret_cast<CCoef*>(sm + A.coef_off);
    coarse_coef(A, lam, coef);
    __syncthreads();
    coarse_body(A, coef, blockIdx.x * (long long)kCB + threadIdx.x, (long long)gridDim.x * kCB, CP_CLUSTER, lt,
                ClusterBar{});
}

// z_f = 0 helper + level-0 vector ops
__global__ void k_fill0(long long n, double* x) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        x[i] = 0.0;
}

// ---- host side ----------------------------------------------------------------------------------
static int gblocks(long long n) {
    long long b = (n + kGB - 1) / kGB;
    return (int)std::max(1LL, std::min(b, (long long)148 * 16));
}

void gmg_plan(Ctx* c) {
    c->glev.clear();
    const Geo2& g = c->g;
    GLevel L0;
    L0.nx = g.nx;
    L0.ny = g.ny;
    L0.nv = g.nv;  // incl. centres (crossed); matrix-free, no stencil
    c->glev.push_back(L0);
    int nx = g.nx, ny = g.ny;
    do {  // level 1 always exists (element Galerkin); then 2:1 while above the dense size
        nx = (nx + 1) / 2;
        ny = (ny + 1) / 2;
        GLevel L;
        L.nx = nx; L.ny = ny; L.nv = (long long)(nx + 1) * (ny + 1);
        c->glev.push_back(L);
    } while ((c->glev.back().nv > kCoarseMaxV ||
              8LL * 2 * c->glev.back().nv * (band_of(c->glev.back().ny) + 1) > kBandSmem) &&
             (nx > 1 || ny > 1));
}

size_t gmg_bytes(const Ctx* c) {
    size_t tot = 0;
    auto al = [&](size_t b) { return ((b + 255) & ~size_t(255)) + c->guard; };  // + guard zone (PF_WS_GUARD)
    for (size_t l = 0; l < c->glev.size(); ++l) {
        const GLevel& L = c->glev[l];
        const long long nvc = (l == 0) ? c->g.nc : L.nv;
        if (l > 0) tot += al(sizeof(double) * 36 * L.nv);
        tot += al(sizeof(double) * 4 * L.nv);          // Dinv
        tot += al(nvc);                                 // mask
        tot += 7 * al(sizeof(double) * 2 * L.nv);      // x b r d0 d1 res w
    }
    const long long nco = 2 * c->glev.back().nv;
    tot += 2 * al(sizeof(double) * nco * nco);
    tot += al(2 * sizeof(unsigned int));  // grid barrier
    return tot + 4096;
}

void gmg_bind(Ctx* c, char* base) {
    size_t off = 0;
    c->gmg_guards.clear();
    auto take = [&](size_t b) {
        char* p = base + off;
        off += (b + 255) & ~size_t(255);
        if (c->guard) {
            c->gmg_guards.push_back({base + off, c->guard});
            cudaMemset(base + off, kGuardByte, c->guard);
            off += c->guard;
        }
        return p;
    };
    for (size_t l = 0; l < c->glev.size(); ++l) {
        GLevel& L = c->glev[l];
        const long long nvc = (l == 0) ? c->g.nc : L.nv;
        L.A = (l > 0) ? (double*)take(sizeof(double) * 36 * L.nv) : nullptr;
        L.Dinv = (double*)take(sizeof(double) * 4 * L.nv);
        L.mask = (unsigned char*)take(nvc);
        L.x = (double*)take(sizeof(double) * 2 * L.nv);
        L.b = (double*)take(sizeof(double) * 2 * L.nv);
        L.r = (double*)take(sizeof(double) * 2 * L.nv);
        L.d0 = (double*)take(sizeof(double) * 2 * L.nv);
        L.d1 = (double*)take(sizeof(double) * 2 * L.nv);
        L.res = (double*)take(sizeof(double) * 2 * L.nv);
        L.w = (double*)take(sizeof(double) * 2 * L.nv);
    }
    const long long nco = 2 * c->glev.back().nv;
    c->gmg_dense = (double*)take(sizeof(double) * nco * nco);
    c->gmg_ainv = (double*)take(sizeof(double) * nco * nco);
    c->gmg_bar = (unsigned int*)take(2 * sizeof(unsigned int));
}

static LevelDev ldev(const Ctx* c, int l) {
    const GLevel& L = c->glev[l];
    LevelDev d;
    d.nx = L.nx;
    d.ny = L.ny;
    d.nv = (l == 0) ? c->g.nc : L.nv;  // stencil / transfer view of level 0 = corners
    d.A = L.A;
    d.Dinv = L.Dinv;
    d.mask = L.mask;
    return d;
}

// launch + profiling bracket; `bytes` = algorithmic bytes of the launch (inputs read once,
// outputs written once), `kind` = K_GMG (cycle) or K_GMGSET (hierarchy setup)
#define GKB(c, kind, bytes, expr)                               \
    do {                                                        \
        const int _ps = prof_begin((c), st);                    \
        expr;                                                   \
        prof_end((c), st, _ps, (kind), (double)(bytes));        \
        (c)->launches++;                                        \
    } while (0)
#define GK(c, expr) GKB(c, K_GMG, 0.0, expr)

// Build the hierarchy for the current alpha (c->alpha_ws) and Dirichlet mask.
int gmg_setup(Ctx* c, cudaStream_t st) {
    const Geo2& g = c->g;
    const int nl = (int)c->glev.size();
    double* lam = c->scal + S_GMG0;
    if (cudaMemsetAsync(lam, 0, sizeof(double) * 16, st) != cudaSuccess) return set_error(c, PF_ECUDA, "memset");
    // level-0 mask = Dirichlet mask of the corners (centres never constrained)
    if (cudaMemcpyAsync(c->glev[0].mask, c->bcmask, g.nc, cudaMemcpyDeviceToDevice, st) != cudaSuccess)
        return set_error(c, PF_ECUDA, "mask copy");
    const unsigned char* m0 = g.has_bc ? c->glev[0].mask : nullptr;
    if (!g.has_bc) cudaMemsetAsync(c->glev[0].mask, 0, g.nc, st);
    {
        GLevel& L1 = c->glev[1];
        const long long nv1 = L1.nv;
        switch (g.pattern) {
            case PF_UNION_JACK:
                GKB(c, K_GMGSET, 40.0 * g.nv, (k_fine_rows<PF_UNION_JACK><<<gblocks(g.nv), kGB, 0, st>>>(g, c->alpha_ws, m0, c->glev[0].Dinv, lam)));
                GKB(c, K_GMGSET, 8.0 * g.nv + 329.0 * nv1, (k_galerkin_cells<PF_UNION_JACK><<<gblocks(nv1), kGB, 0, st>>>(
                          g, c->alpha_ws, m0, L1.nx, L1.ny, L1.A, L1.Dinv, L1.mask, lam + 1)));
                break;
            case PF_RIGHT:
                GKB(c, K_GMGSET, 40.0 * g.nv, (k_fine_rows<PF_RIGHT><<<gblocks(g.nv), kGB, 0, st>>>(g, c->alpha_ws, m0, c->glev[0].Dinv, lam)));
                GKB(c, K_GMGSET, 8.0 * g.nv + 329.0 * nv1, (k_galerkin_cells<PF_RIGHT><<<gblocks(nv1), kGB, 0, st>>>(
                          g, c->alpha_ws, m0, L1.nx, L1.ny, L1.A, L1.Dinv, L1.mask, lam + 1)));
                break;
            default:
                GKB(c, K_GMGSET, 40.0 * g.nv, (k_fine_rows<PF_CROSSED><<<gblocks(g.nv), kGB, 0, st>>>(g, c->alpha_ws, m0, c->glev[0].Dinv, lam)));
                GKB(c, K_GMGSET, 8.0 * g.nv + 329.0 * nv1, (k_galerkin_cells<PF_CROSSED><<<gblocks(nv1), kGB, 0, st>>>(
                          g, c->alpha_ws, m0, L1.nx, L1.ny, L1.A, L1.Dinv, L1.mask, lam + 1)));
                break;
        }
    }
    for (int l = 1; l + 1 < nl; ++l) {
        LevelDev F = ldev(c, l), Cd = ldev(c, l + 1);
        GKB(c, K_GMGSET, 289.0 * F.nv + 329.0 * Cd.nv, (k_rap<<<gblocks(Cd.nv), kGB, 0, st>>>(F, Cd, c->glev[l + 1].A, c->glev[l + 1].Dinv,
                                                      c->glev[l + 1].mask, lam + l + 1)));
    }
    {
        const GLevel& Lc = c->glev[nl - 1];
        const int n = (int)(2 * Lc.nv), bw = band_of(Lc.ny), W = bw + 1;
        const int smem = (int)sizeof(double) * n * W;
        int wpb = 8;
        while (wpb > 1 && smem + (int)sizeof(double) * wpb * n > 225 * 1024) --wpb;
        const int smem2 = smem + (int)sizeof(double) * wpb * n;
        static std::atomic<bool> attr[kMaxDev];
        const int dv = cur_dev();
        if (!attr[dv].load()) {
            cudaFuncSetAttribute(k_coarse_chol_band, cudaFuncAttributeMaxDynamicSharedMemorySize, 225 * 1024);
            cudaFuncSetAttribute(k_coarse_inv_band, cudaFuncAttributeMaxDynamicSharedMemorySize, 225 * 1024);
            attr[dv] = true;
        }
        GKB(c, K_GMGSET, 2.0 * 8.0 * n * W, (k_coarse_chol_band<<<1, 1024, smem, st>>>(ldev(c, nl - 1), bw, c->gmg_dense)));
        GKB(c, K_GMGSET, 8.0 * n * W + 8.0 * n * n, (k_coarse_inv_band<<<(n + wpb - 1) / wpb, 32 * wpb, smem2, st>>>(
                                                      c->gmg_dense, n, bw, wpb, c->gmg_ainv)));
    }
    return check_cuda(c, cudaGetLastError(), "gmg setup");
}

static GmgEpi epi0(Ctx* c, const double* live) {
    GLevel& L = c->glev[0];
    GmgEpi e{};
    e.Dinv = L.Dinv;
    e.nvD = L.nv;
    e.res = L.res;
    e.lam = c->scal + S_GMG0;
    e.ratio = c->gmg_ratio;
    e.k = 1;
    e.live = live;
    e.rz_first = -1;
    return e;
}

// first level of the single-CTA tail (>= 1; nl - 1 = the dense solve only)
static int tail_level(const Ctx* c) {
    const int nl = (int)c->glev.size();
    int lc = nl - 1;
    while (lc > 1 && c->glev[lc - 1].nv <= kTailMaxV && nl - (lc - 1) <= kTailLev) --lc;
    return lc;
}

static int launch_tail(Ctx* c, int lc, cudaStream_t st, const double* live) {
    const int nl = (int)c->glev.size();
    TailArgs a;
    memset(&a, 0, sizeof(a));
    a.lc = lc;
    a.nl = nl;
    a.deg = std::max(1, c->gmg_degree);
    a.ratio = c->gmg_ratio;
    a.ainv = c->gmg_ainv;
    a.ncoarse = (int)(2 * c->glev[nl - 1].nv);
    double bytes = 8.0 * a.ncoarse * a.ncoarse + 32.0 * a.ncoarse;
    for (int l = lc; l < nl; ++l) {
        GLevel& L = c->glev[l];
        a.lev[l].L = ldev(c, l);
        a.lev[l].x = L.x; a.lev[l].b = L.b; a.lev[l].r = L.r;
        a.lev[l].d0 = L.d0; a.lev[l].d1 = L.d1; a.lev[l].res = L.res;
        if (l + 1 < nl)  // the same algorithmic bytes as the per-level kernels it replaces
            bytes += (416.0 + 336.0 + 16.0 + 32.0 + 400.0 + 416.0) * L.nv + 34.0 * c->glev[l + 1].nv;
    }
    GKB(c, K_GMG, bytes, (k_gmg_tail<<<1, kTB, 0, st>>>(a, c->scal + S_GMG0, live)));
    return PF_OK;
}

// Level-0 pre-smoother from z = 0 with the matrix-free fine operator (fused epilogues); leaves the
// fine residual r - A z in L0.r.
static int fine_pre(Ctx* c, const double* b, double* x, cudaStream_t st, const double* live, bool cheb0_done) {
    GLevel& L = c->glev[0];
    const long long nv = L.nv;
    const int deg = std::max(1, c->gmg_degree);
    double* d = L.d0;
    double* dn = L.d1;
    if (!cheb0_done)
        GKB(c, K_GMG, 96.0 * nv, (k_cheb0<<<gblocks(nv), kGB, 0, st>>>(nv, L.Dinv, b, L.res, L.d0, x, 0, c->scal + S_GMG0, c->gmg_ratio, live)));
    for (int k = 1; k < deg; ++k) {
        GmgEpi e = epi0(c, live);
        e.dnext = dn;
        e.xs = x;
        e.k = k;
        PF_TRY_GMG(launch_Kuu_smooth(c, EPI_CHEB, c->alpha_ws, d, e, st));
        std::swap(d, dn);
    }
    GmgEpi e = epi0(c, live);
    e.bvec = b;
    e.rout = L.r;
    return launch_Kuu_smooth(c, EPI_RESID, c->alpha_ws, x, e, st);
}

// Level-0 post-smoother: res = D^-1 (b - A x), d0 = res/theta ; steps (x += d0 on step 1); the PCG
// r.z rides on the last step when rz_first >= 0.
static int fine_post(Ctx* c, const double* b, double* x, cudaStream_t st, const double* live, int rz_first,
                     bool* rz_done) {
    GLevel& L = c->glev[0];
    const long long nv = L.nv;
    const int deg = std::max(1, c->gmg_degree);
    double* d = L.d0;
    double* dn = L.d1;
    GmgEpi e = epi0(c, live);
    e.bvec = b;
    e.dnext = L.d0;
    PF_TRY_GMG(launch_Kuu_smooth(c, EPI_RESID_CHEB0, c->alpha_ws, x, e, st));
    if (deg <= 1) GKB(c, K_GMG, 48.0 * nv, (k_add<<<gblocks(nv), kGB, 0, st>>>(nv, L.d0, x, live)));
    for (int k = 1; k < deg; ++k) {
        GmgEpi es = epi0(c, live);
        es.dnext = dn;
        es.xs = x;
        es.k = k;
        if (k == deg - 1 && rz_first >= 0) {
            es.rcg = b;
            es.rz_first = rz_first;
            if (rz_done) *rz_done = true;
        }
        PF_TRY_GMG(launch_Kuu_smooth(c, k == 1 ? EPI_CHEB_ADDD : EPI_CHEB, c->alpha_ws, d, es, st));
        std::swap(d, dn);
    }
    return PF_OK;
}

#define GCU(c, x, where) PF_TRY_GMG(check_cuda((c), (x), (where)))

// Shared memory of the persistent coarse cycle: the per-level Chebyshev coefficient table.
static int coarse_plan(const Ctx* c, CoarseArgs& a) {
    const int nl = (int)c->glev.size();
    if (nl > kMaxLev) return -1;
    a.lc = nl - 1;
    a.coef_off = 0;
    return (int)sizeof(CCoef) * nl;
}

// Arguments of the coarse cycle for fine residual r0 and correction z0; returns the shared memory
// bytes (coefficient table) or -1 when the hierarchy does not fit the persistent cycle.
static int make_coarse_args(Ctx* c, const double* r0, double* z0, CoarseArgs& a) {
    const Geo2& g = c->g;
    const int nl = (int)c->glev.size();
    memset(&a, 0, sizeof(a));
    const int smem = coarse_plan(c, a);
    if (smem < 0) return -1;
    a.g = g;
    a.crossed = g.pattern == PF_CROSSED;
    a.mask0 = g.has_bc ? c->glev[0].mask : nullptr;
    a.L0 = ldev(c, 0);
    a.L0.mask = a.crossed ? nullptr : a.mask0;  // crossed: the collapse/expand apply the fine mask
    a.r0 = r0;
    a.z0 = z0;
    a.nl = nl;
    a.deg = std::max(1, c->gmg_degree);
    a.ratio = c->gmg_ratio;
    a.ainv = c->gmg_ainv;
    a.ncoarse = (int)(2 * c->glev[nl - 1].nv);
    a.bar = c->gmg_bar;
    a.skip = c->gmg_coarse == 2;
    for (int l = 1; l < nl; ++l) {
        GLevel& L = c->glev[l];
        a.lev[l].L = ldev(c, l);
        a.lev[l].x = L.x; a.lev[l].b = L.b; a.lev[l].r = L.r;
        a.lev[l].d0 = L.d0; a.lev[l].d1 = L.d1; a.lev[l].res = L.res;
    }
    return smem;
}

// The small coarse levels (<= kClusterMaxV vertices) run inside one thread-block cluster of
// kClusterCTAs CTAs (cluster barriers instead of grid barriers); the levels above stay grid-wide.
constexpr long long kClusterMaxV = 20000;
static int cluster_level(const Ctx* c) {
    const int nl = (int)c->glev.size();
    int lt = nl - 1;
    while (lt > 1 && c->glev[lt - 1].nv <= kClusterMaxV) --lt;
    return lt;
}
// algorithmic bytes of the per-phase launches the persistent phases of levels [la, lb) replace
static double coarse_level_bytes(const Ctx* c, int la, int lb, int deg, int ncoarse) {
    const int nl = (int)c->glev.size();
    double bytes = 0.0;
    for (int l = std::max(1, la); l < lb && l < nl; ++l) {
        const double nv = (double)c->glev[l].nv;
        if (l == nl - 1) { bytes += 8.0 * ncoarse * ncoarse + 32.0 * ncoarse; break; }
        const double nvc = (double)c->glev[l + 1].nv;
        bytes += (deg > 1 ? 416.0 : 96.0) * nv + 416.0 * std::max(0, deg - 2) * nv + 336.0 * nv + 16.0 * nv + 17.0 * nvc;
        bytes += 32.0 * nv + 17.0 * nvc + 400.0 * nv + (deg <= 1 ? 48.0 : 416.0 * (deg - 1)) * nv;
    }
    return bytes;
}

static int launch_coarse(Ctx* c, const double* r0, double* z0, cudaStream_t st, const double* live) {
    const Geo2& g = c->g;
    const int nl = (int)c->glev.size();
    CoarseArgs a;
    const int smem = make_coarse_args(c, r0, z0, a);
    if (smem < 0) return set_error(c, PF_EINVAL, "gmg: hierarchy too deep for the persistent coarse cycle");
    static unsigned long long* trace = nullptr;
    static int ntrace_calls = 0;
    if (getenv("PF_GMG_TRACE") && !trace) cudaMalloc(&trace, 128 * sizeof(unsigned long long));
    a.trace = trace;
    static int nb_cache_d[kMaxDev], nb_smem_d[kMaxDev], ncl_d[kMaxDev];
    static std::atomic<bool> nb_ok[kMaxDev];
    const int dvc = cur_dev();
    int& nb_cache = nb_cache_d[dvc];
    int& nb_smem = nb_smem_d[dvc];
    int& ncl = ncl_d[dvc];  // CTAs of the cluster part (0: no cluster launch possible)
    if (!nb_ok[dvc].load() || nb_smem != smem) {
        int dev = 0, nsm = 0, per = 0;
        GCU(c, cudaGetDevice(&dev), "device");
        GCU(c, cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev), "sm count");
        GCU(c, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_gmg_coarse, kCB, smem), "occupancy");
        if (per < 1) return set_error(c, PF_ECUDA, "gmg: coarse-cycle kernel cannot be resident");
        nb_cache = nsm * per;
        nb_smem = smem;
        // the largest cluster (16 non-portable, else 8) this kernel can be launched with
        ncl = 0;
        cudaFuncSetAttribute(k_gmg_ctail, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        for (int cs : {16, 8}) {
            cudaLaunchConfig_t q = {};
            q.gridDim = dim3(cs);
            q.blockDim = dim3(kCB);
            q.dynamicSmemBytes = smem;
            cudaLaunchAttribute qa[1];
            qa[0].id = cudaLaunchAttributeClusterDimension;
            qa[0].val.clusterDim.x = cs; qa[0].val.clusterDim.y = 1; qa[0].val.clusterDim.z = 1;
            q.attrs = qa;
            q.numAttrs = 1;
            int nclusters = 0;
            if (cudaOccupancyMaxActiveClusters(&nclusters, k_gmg_ctail, &q) == cudaSuccess && nclusters >= 1) {
                ncl = cs;
                break;
            }
            cudaGetLastError();
        }
        nb_ok[dvc] = true;
    }
    const int deg = a.deg;
    const GLevel& L1 = c->glev[1];
    const double top = a.crossed ? 48.0 * g.nc + 16.0 * g.nc + 17.0 * L1.nv + 32.0 * g.nc + 17.0 * L1.nv + 48.0 * g.nv
                                 : 16.0 * g.nc + 17.0 * L1.nv + 32.0 * g.nc + 17.0 * L1.nv;
    const double* lam = c->scal + S_GMG0;
    cudaError_t le = cudaSuccess;
    if (trace) cudaMemsetAsync(trace, 0, 128 * sizeof(unsigned long long), st);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(nb_cache);
    cfg.blockDim = dim3(kCB);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    const int lt = cluster_level(c);
    const bool split = ncl > 0 && c->gmg_cluster && lt < nl;
    if (!split) {
        const double bytes = top + coarse_level_bytes(c, 1, nl, deg, a.ncoarse);
        GKB(c, K_GMG, bytes, (le = cudaLaunchKernelEx(&cfg, k_gmg_coarse, a, lam, live, (int)CP_ALL, lt)));
    } else {
        const double b_top = coarse_level_bytes(c, 1, lt, deg, a.ncoarse);
        GKB(c, K_GMG, 0.5 * (top + b_top), (le = cudaLaunchKernelEx(&cfg, k_gmg_coarse, a, lam, live, (int)CP_DOWN, lt)));
        if (le == cudaSuccess) {
            cudaLaunchConfig_t q = {};
            q.gridDim = dim3(ncl);
            q.blockDim = dim3(kCB);
            q.dynamicSmemBytes = smem;
            q.stream = st;
            cudaLaunchAttribute qa[1];
            qa[0].id = cudaLaunchAttributeClusterDimension;
            qa[0].val.clusterDim.x = ncl; qa[0].val.clusterDim.y = 1; qa[0].val.clusterDim.z = 1;
            q.attrs = qa;
            q.numAttrs = 1;
            GKB(c, K_GMG, coarse_level_bytes(c, lt, nl, deg, a.ncoarse), (le = cudaLaunchKernelEx(&q, k_gmg_ctail, a, lam, live, lt)));
        }
        if (le == cudaSuccess)
            GKB(c, K_GMG, 0.5 * (top + b_top), (le = cudaLaunchKernelEx(&cfg, k_gmg_coarse, a, lam, live, (int)CP_UP, lt)));
    }
    if (trace && ++ntrace_calls % 8 == 5) {  // eager mode only (PF_NO_GRAPHS): print one cycle's phases
        unsigned long long h[128];
        cudaMemcpyAsync(h, trace, sizeof h, cudaMemcpyDeviceToHost, st);
        cudaStreamSynchronize(st);
        fprintf(stderr, "coarse cycle nb=%d cluster=%d lt=%d nl=%d smem=%d phases(us):", nb_cache, split ? ncl : 0, lt,
                nl, smem);
        for (int seg = 0; seg < 3; ++seg) {
            fprintf(stderr, seg ? " |" : "");
            for (int q = 40 * seg + 1; q < 40 * seg + 40 && h[q]; ++q) fprintf(stderr, " %.2f", 1e-3 * (double)(h[q] - h[q - 1]));
        }
        fprintf(stderr, "\n");
    }
    return check_cuda(c, le, "coarse-cycle launch");
}

// z = M r : one V-cycle, level 0 vectors are the PCG r (input) and z (output).
// cheb0_done: the caller already wrote the level-0 cheb0 (res = D^-1 r, d0 = z = res / theta;
// k_cg_update_gmg).  rz_first >= 0: fuse the PCG r . z into the last fine smoother step
// (*rz_done reports whether it was fused; with degree 1 it is not).
int gmg_vcycle(Ctx* c, const double* r_in, double* z_out, cudaStream_t st, const double* live, bool cheb0_done,
               int rz_first, bool* rz_done) {
    if (rz_done) *rz_done = false;
    const Geo2& g = c->g;
    const int nl = (int)c->glev.size();
    const int deg = std::max(1, c->gmg_degree);
    const double ratio = c->gmg_ratio;
    double* lam = c->scal + S_GMG0;
    if (c->gmg_coarse && nl <= kMaxLev && deg < kMaxDeg) {  // fine smoothing + one persistent launch for everything coarser
        PF_TRY_GMG(fine_pre(c, r_in, z_out, st, live, cheb0_done));
        PF_TRY_GMG(launch_coarse(c, c->glev[0].r, z_out, st, live));
        PF_TRY_GMG(fine_post(c, r_in, z_out, st, live, rz_first, rz_done));
        return check_cuda(c, cudaGetLastError(), "gmg vcycle");
    }
    const int lc = tail_level(c);  // per-level kernels down to level lc, then the one-CTA tail
    // descend through the per-level kernels
    for (int l = 0; l < lc; ++l) {
        GLevel& L = c->glev[l];
        const long long nv = L.nv;
        const double* b = (l == 0) ? r_in : L.b;
        double* x = (l == 0) ? z_out : L.x;
        LevelDev Ld = ldev(c, l);
        Ld.nv = nv;
        double* d = L.d0;
        double* dn = L.d1;
        if (l == 0) {
            PF_TRY_GMG(fine_pre(c, b, x, st, live, cheb0_done));
        } else {
            GKB(c, K_GMG, (deg > 1 ? 416.0 : 96.0) * nv, (k_pre_first<<<gblocks(nv), kGB, 0, st>>>(Ld, b, L.res, L.d0, L.d1, x, deg, lam + l, ratio, live)));
            if (deg > 1) std::swap(d, dn);
            for (int k = 2; k < deg; ++k) {
                GKB(c, K_GMG, 416.0 * nv, (k_cheb_step<<<gblocks(nv), kGB, 0, st>>>(Ld, nullptr, d, dn, L.res, x, k, 0, lam + l, ratio, live)));
                std::swap(d, dn);
            }
            GKB(c, K_GMG, 336.0 * nv, (k_resid<<<gblocks(nv), kGB, 0, st>>>(Ld, nullptr, x, b, L.r, live)));
        }
        // restrict
        GLevel& C = c->glev[l + 1];
        if (l == 0 && g.pattern == PF_CROSSED) {
            LevelDev F = ldev(c, 0), Cd = ldev(c, 1);
            F.mask = nullptr;  // fine masks were applied by the collapse
            GKB(c, K_GMG, 48.0 * g.nc, (k_collapse_centres<<<gblocks(g.nc), kGB, 0, st>>>(
                                           g, g.has_bc ? c->glev[0].mask : nullptr, L.r, L.w, live)));
            GKB(c, K_GMG, 16.0 * F.nv + 17.0 * Cd.nv, (k_restrict<<<gblocks(Cd.nv), kGB, 0, st>>>(
                                                         F, Cd, C.mask, L.w, C.b, live)));
        } else if (l == 0) {
            LevelDev F = ldev(c, 0), Cd = ldev(c, 1);
            F.mask = g.has_bc ? c->glev[0].mask : nullptr;
            GKB(c, K_GMG, 16.0 * F.nv + 17.0 * Cd.nv, (k_restrict<<<gblocks(Cd.nv), kGB, 0, st>>>(
                                                         F, Cd, C.mask, L.r, C.b, live)));
        } else {
            LevelDev F = ldev(c, l), Cd = ldev(c, l + 1);
            GKB(c, K_GMG, 16.0 * F.nv + 17.0 * Cd.nv, (k_restrict<<<gblocks(Cd.nv), kGB, 0, st>>>(F, Cd, C.mask, L.r, C.b, live)));
        }
    }
    PF_TRY_GMG(launch_tail(c, lc, st, live));  // levels lc..nl-1 incl. the dense coarse solve
    // ascend
    for (int l = lc - 1; l >= 0; --l) {
        GLevel& L = c->glev[l];
        GLevel& C = c->glev[l + 1];
        const long long nv = L.nv;
        const double* b = (l == 0) ? r_in : L.b;
        double* x = (l == 0) ? z_out : L.x;
        LevelDev Ld = ldev(c, l);
        Ld.nv = nv;
        if (l == 0 && g.pattern == PF_CROSSED) {
            LevelDev F = ldev(c, 0), Cd = ldev(c, 1);
            F.mask = nullptr;
            GK(c, (k_fill0<<<gblocks(2 * g.nc), kGB, 0, st>>>(2 * g.nc, L.w)));
            GKB(c, K_GMG, 32.0 * F.nv + 17.0 * Cd.nv, (k_prolong<<<gblocks(F.nv), kGB, 0, st>>>(
                                                         F, Cd, C.mask, C.x, L.w, live)));
            GKB(c, K_GMG, 48.0 * g.nv, (k_expand_centres<<<gblocks(g.nv), kGB, 0, st>>>(
                                           g, g.has_bc ? c->glev[0].mask : nullptr, L.w, x, live)));
        } else if (l == 0) {
            LevelDev F = ldev(c, 0), Cd = ldev(c, 1);
            F.mask = g.has_bc ? c->glev[0].mask : nullptr;
            GKB(c, K_GMG, 32.0 * F.nv + 17.0 * Cd.nv, (k_prolong<<<gblocks(F.nv), kGB, 0, st>>>(
                                                         F, Cd, C.mask, C.x, x, live)));
        } else {
            LevelDev F = ldev(c, l), Cd = ldev(c, l + 1);
            GKB(c, K_GMG, 32.0 * F.nv + 17.0 * Cd.nv, (k_prolong<<<gblocks(F.nv), kGB, 0, st>>>(F, Cd, C.mask, C.x, x, live)));
        }
        double* d = L.d0;
        double* dn = L.d1;
        if (l == 0) {
            PF_TRY_GMG(fine_post(c, b, x, st, live, rz_first, rz_done));
        } else {  // residual + cheb0 in one pass; the x += d0 rides on step 1
            GKB(c, K_GMG, 400.0 * nv, (k_post_first<<<gblocks(nv), kGB, 0, st>>>(Ld, x, b, L.res, L.d0, lam + l, ratio, live)));
            if (deg <= 1) GKB(c, K_GMG, 48.0 * nv, (k_add<<<gblocks(nv), kGB, 0, st>>>(nv, L.d0, x, live)));
            for (int k = 1; k < deg; ++k) {
                GKB(c, K_GMG, 416.0 * nv, (k_cheb_step<<<gblocks(nv), kGB, 0, st>>>(Ld, nullptr, d, dn, L.res, x, k, k == 1, lam + l, ratio, live)));
                std::swap(d, dn);
            }
        }
    }
    return check_cuda(c, cudaGetLastError(), "gmg vcycle");
}

}  // namespace pf
