// pf_internal.cuh -- shared internals of the sm_100a phase-field load-step library.
//
// Design: structured P1 meshes with implicit geometry.  Every operator is a
// matrix-free "strip" kernel: a warp owns 30 vertex columns (j, the contiguous index) plus a
// one-column halo and walks a strip of S vertex rows (i); vertex data of row i+1 is loaded
// once (coalesced along j), the right neighbour column comes from the next lane by shuffle,
// and element contributions to the next row / next column are carried in registers /
// shuffled left->right, so every vertex value is read once from HBM and every output is
// written once, with no atomics (deterministic).  Reductions are per-block partials summed by
// the last block in a fixed order (bitwise reproducible run to run).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <string>
#include <utility>
#include <vector>

#include "../../include/phasefrac_b200.h"

#define PF_FULL 0xffffffffu

namespace pf {

// Per-device one-time launch setup (the >48 KB shared-memory opt-in and occupancy queries are
// properties of a device context): slot of the current device in a static per-kernel table.
constexpr int kMaxDev = 64;
constexpr int kGuardByte = 0xA5;  // workspace guard zones (PF_WS_GUARD)
inline int cur_dev() {
    int d = 0;
    cudaGetDevice(&d);
    return d & (kMaxDev - 1);
}

constexpr int kGmgRebuildIts = 12;  // excess PCG iterations that trigger a multigrid rebuild
constexpr int kBlock = 256;        // threads per block for strip kernels
constexpr int kLanesOut = 30;      // output columns per warp
constexpr int kOut2Cols = 62;      // output columns per warp of the v2 engine (two columns per lane)
constexpr int kMaxRed = 8;         // max values per fused reduction
constexpr int kMaxBlocksRed = 8192;  // partials capacity per reduction value

// ---- geometry / material descriptor passed by value to every 2D kernel ------------------
struct Geo2 {
    int nx, ny, nvy;          // cells, ny+1
    int pattern, npc;         // PF_*, elements per cell
    long long nc, ncell, nv;  // corner vertices, cells, all vertices
    double hx, hy, ihx, ihy;
    // element types (local nodes 0=v00 1=v10 2=v01 3=v11 4=centre)
    double area[4];
    // unit-E stiffness (Voigt e11, e22, g12)
    double D00, D01, D11, D22;
    double E, kell, Gc, ell, cw;
    int at2;
    const double* E_cell;     // nullable, per cell (I*ny + J)
    const double* Gc_cell;    // nullable
    const double* eps0;       // nullable, isotropic strain per (type, J): t*ny + J
    const double* rowgeo;     // nullable (uniform rows): graded rows, [1/hy (ny) | element area (ny)] per cell row J
    const unsigned char* bcmask;  // per corner vertex, bit c = component c constrained
    const double* ubar;       // n_u (values on constrained dofs)
    int has_bc;
    // strip decomposition
    int nwj, S, nstrips;
    // strip decomposition of the v2 engine (62 output columns per warp, pf_strip2.cu)
    int nwj2, S2, nstrips2;
    int nslow2;   // boundary windows whose strips are split between two warps (0: none)
};

// ---- 3D (Kuhn tetrahedra) descriptor ------------------------------------------------------------
struct Geo3 {
    int nx, ny, nz, nvy, nvz;     // cells; ny+1, nz+1
    long long nv, ncell;
    double ihx, ihy, ihz, vol;    // 1/h per axis, tet volume hx hy hz / 6
    double lam, mu;               // unit-E Lame constants
    double E, kell, Gc, ell, cw;
    int at2;
    const double* E_cell;
    const double* Gc_cell;
    const unsigned char* bcmask;  // per vertex, bit c = component c constrained
    const double* ubar;           // 3 nv
    int has_bc;
    int nbj, nbk, S, nstrips;     // block tiling
};

// ---- reductions --------------------------------------------------------------------------
struct RedBuf {
    double* partials;      // [kMaxRed][kMaxBlocksRed]
    unsigned int* ticket;  // one counter per reduction site
    double* out;           // result slots
};

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(PF_FULL, v, o);
    return v;
}

// software grid barrier (all CTAs co-resident: cooperative launch).  One arrival word: CTA 0 adds
// 2^31 - (nb - 1), the others 1, so the top bit flips exactly when the last CTA arrives.
__device__ __forceinline__ void grid_sync(unsigned int* bar) {
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

// Block-reduce NV values, store per-block partials, and let the last block sum them in a
// fixed order; `fin(vals)` runs on thread 0 of the last block with the grid totals.
template <int NV, class Fin>
__device__ __forceinline__ void grid_reduce(double (&v)[NV], const RedBuf& rb, int slot, Fin fin) {
    __shared__ double sm[NV][32];
    __shared__ bool s_last;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int nb = gridDim.x;
#pragma unroll
    for (int k = 0; k < NV; ++k) {
        double t = warp_sum(v[k]);
        if (lane == 0) sm[k][warp] = t;
    }
    __syncthreads();
    if (warp == 0) {
#pragma unroll
        for (int k = 0; k < NV; ++k) {
            double t = lane < nw ? sm[k][lane] : 0.0;
            t = warp_sum(t);
            if (lane == 0) rb.partials[(size_t)k * kMaxBlocksRed + blockIdx.x] = t;
        }
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned int t = atomicAdd(rb.ticket + slot, 1u);
        s_last = (t == (unsigned)nb - 1u);
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    if (warp == 0) {
        double tot[NV];
#pragma unroll
        for (int k = 0; k < NV; ++k) {
            double t = 0.0;
            for (int b = lane; b < nb; b += 32) t += __ldcg(rb.partials + (size_t)k * kMaxBlocksRed + b);
            tot[k] = warp_sum(t);
        }
        if (lane == 0) {
            fin(tot);
            rb.ticket[slot] = 0u;
        }
    }
}

// ---- device scalar block (solver state kept on device) -----------------------------------
enum ScalarSlot {
    S_RZ = 0, S_PAP, S_GAMMA, S_BETA, S_RR, S_BNORM, S_TARGET, S_RNORM,
    S_ITER, S_DONE, S_FAIL, S_MAXIT, S_RZNEW, S_MU, S_MERIT, S_TMERIT,
    S_ZETA, S_NINACT, S_XMAX, S_GNORM2, S_DALPHA, S_OMEGABAR, S_AUX0, S_AUX1,
    S_PHYS0 = 32,  // 8 slots of physics-pass outputs
    S_CGVEC0 = 48,
    S_GMG0 = 64,   // 16 slots: per-level lambda_max bounds
    S_COUNT = 128
};

// ---- per-kernel-class profiling (CUDA events around launches; read after the timed region) --
enum KernelKind {
    K_KUU = 0, K_KUU_CG, K_KUU_DIAG, K_KAPPA, K_KAA, K_KAA_CG, K_KAA_DIAG, K_KAA_TRIAL, K_PHYS,
    K_RHS, K_KUA, K_KAU, K_JAC, K_CG_VEC, K_VEC, K_GMG, K_GMGSET, K_NKINDS
};
struct ProfEntry { int kind; int ev; double bytes; };
struct Prof {
    int on = 0;
    std::vector<cudaEvent_t> ev;   // pairs (start, stop)
    std::vector<ProfEntry> log;
    double ms[K_NKINDS] = {0};
    double bytes[K_NKINDS] = {0};
    long long count[K_NKINDS] = {0};
};

// ---- Chebyshev smoother scalars (linalg.py:366-376) -------------------------------------------
// Shared by the GMG level kernels (pf_gmg.cu) and the fused fine-level strip epilogues (pf_ops2d.cu)
// so both evaluate the same expressions.
struct Cheb {
    double theta, delta, sigma, itheta;
};
__device__ __forceinline__ Cheb cheb_of(const double* lam, double ratio) {
    const double hi = *lam, lo = hi * ratio;
    Cheb c;
    c.theta = 0.5 * (hi + lo);
    c.delta = 0.5 * (hi - lo);
    c.sigma = c.theta / c.delta;
    c.itheta = 1.0 / c.theta;
    return c;
}
__device__ __forceinline__ double cheb_rho(const Cheb& c, int k) {  // rho_k, rho_0 = 1/sigma
    double rho = 1.0 / c.sigma;
    for (int t = 1; t <= k; ++t) rho = 1.0 / (2.0 * c.sigma - rho);
    return rho;
}
__device__ __forceinline__ void cheb_ab(const Cheb& c, int k, double& a, double& b) {
    const double rp = cheb_rho(c, k - 1), rn = cheb_rho(c, k);
    a = rn * rp;
    b = 2.0 * rn / c.delta;
}
// 2x2 block-Jacobi inverse applied at vertex v: Dinv[(2r + c) * nv + v]
__device__ __forceinline__ double2 bmul(const double* Dinv, long long nv, long long v, double r0, double r1) {
    return make_double2(__ldg(Dinv + v) * r0 + __ldg(Dinv + nv + v) * r1,
                        __ldg(Dinv + 2 * nv + v) * r0 + __ldg(Dinv + 3 * nv + v) * r1);
}

// ---- over-relaxation: first feasible midpoint candidate (solver.py:202-216) ---------------------
__device__ __forceinline__ void choose_omega(double omega, unsigned long long bits, double& wb, int& kk,
                                             bool& use_star) {
    // first feasible k in 0..59 with (k == 0 or w_k != 1); else the unrelaxed update
    double w = omega;
    use_star = true;
    wb = 1.0;
    kk = 60;
    if (omega == 1.0) { kk = 0; return; }
    for (int k = 0; k < 60; ++k) {
        if (k > 0 && w == 1.0) { kk = k; return; }
        if (!((bits >> k) & 1ull)) { wb = w; kk = k; use_star = false; return; }
        w = 0.5 * (1.0 + w);
    }
}

// ---- GMG fine-level smoother epilogues fused into the Kuu strip kernel (pf_ops2d.cu) -----------
enum {
    EPI_NONE = 0,
    EPI_CHEB,         // Chebyshev step k on input d:  res -= D^-1 K d ; dnext = a d + b res ; x += dnext
    EPI_CHEB_ADDD,    // the same, plus the post-smoother's deferred x += d  (first post step)
    EPI_RESID,        // rout = b - K x
    EPI_RESID_CHEB0,  // res = D^-1 (b - K x) ; dnext = res / theta  (post-smoother entry)
};
struct GmgEpi {
    const double* Dinv;   // level-0 2x2 block-Jacobi inverse [4][nvD]
    long long nvD;
    double* res;
    double* dnext;
    double* xs;           // smoother iterate
    const double* bvec;   // right-hand side (resid modes)
    double* rout;         // residual out (EPI_RESID)
    const double* lam;    // level-0 lambda_max bound (device)
    double ratio;
    int k;                // Chebyshev step index (>= 1)
    const double* live;   // solver scalars (null: always live)
    const double* rcg;    // PCG residual for the fused r . z (rz_first >= 0)
    int rz_first;         // -1: no r . z ; 1: first (S_RZ only) ; 0: also S_BETA
};

// ---- multigrid level (pf_gmg.cu) -------------------------------------------------------------
struct GLevel {
    int nx = 0, ny = 0;        // cells
    long long nv = 0;          // vertices (level 0: incl. crossed centres)
    double* A = nullptr;       // 9-point 2x2-block stencil [36][nv_corner] (null on crossed level 0)
    double* Dinv = nullptr;    // 2x2 block-Jacobi inverse [4][nv]
    unsigned char* mask = nullptr;  // Dirichlet component bits per corner vertex
    double *x = nullptr, *b = nullptr, *r = nullptr, *d0 = nullptr, *d1 = nullptr, *res = nullptr, *w = nullptr;
};

// ---- 3D multigrid level (pf_gmg3.cu) ---------------------------------------------------------
struct G3Level {
    Geo3 g;                          // level geometry (coarse: 2:1 with the ceil rule)
    double* alpha = nullptr;         // level damage (coarse: max-pooled)
    double* E = nullptr;             // per-cell E (coarse: averaged), when the fine level has one
    unsigned char* mask = nullptr;   // Dirichlet bits (coarse: injected)
    double* dinv = nullptr;          // 1 / diag(K_l) (3 nv)
    double *x = nullptr, *b = nullptr, *r = nullptr, *d0 = nullptr, *d1 = nullptr, *res = nullptr, *w = nullptr;
};

// ---- context -------------------------------------------------------------------------
struct Ctx {
    pf_desc d;
    Geo2 g;
    Geo3 g3;
    std::string err;
    long long n_u = 0, n_a = 0, n_el = 0;
    int dim = 2, dof = 2;
    // workspace
    size_t ws_bytes = 0;
    char* ws = nullptr;
    std::vector<std::pair<void**, size_t>> layout;
    // bounds-check aid (PF_WS_GUARD=1 at creation): a guard zone after every workspace buffer,
    // filled with kGuardByte at binding; pf_check_guards counts the bytes kernels overwrote
    size_t guard = 0;
    std::vector<std::pair<size_t, size_t>> guards;  // (offset, bytes) in the workspace
    std::vector<std::pair<char*, size_t>> gmg_guards;  // guard zones between the hierarchy buffers
    // named buffers (device)
    double *cg_x, *cg_r, *cg_z, *cg_p0, *cg_p1, *cg_q, *cg_dinv, *cg_b;     // n_u
    double *da_x, *da_r, *da_z, *da_p0, *da_p1, *da_q, *da_dinv;             // n_a (damage CG)
    double *cg1_s0, *cg1_s1;                                                 // n_a (single-reduction CG)
    double *vi_x, *vi_F, *vi_c, *vi_d, *vi_tx, *vi_tF, *vi_g, *vi_w;          // n_a
    double *kappa;                                                           // n_el
    double *alpha_ws, *u_ws;                                                 // n_a, n_u
    double *ubar;                                                            // n_u
    unsigned char *bcmask, *act;                                             // n_a
    int* tile_list = nullptr;  // free tiles of the masked damage PCG: [0] count, [1..] tiles, then tile_cap flag bytes
    int tile_cap = 0;
    double tile_frac = 1.0;    // share of the tiles the last persistent damage PCG visited (profiling)
    int rhs_masked = 0;        // the running masked PCG has b = 0 on its active rows (pf_damage_solve; not the
                               // Newton field split's C block, whose identity rows carry b): the list applies
    double *eps0_tab;                                                        // 4*ny
    double *rowgeo_buf;                                                      // 2*ny (graded rows)
    double *partials, *scal;
    unsigned int* tickets;
    unsigned long long* bits;                                                // 8 words
    double* newton;                                                          // Newton block vectors
    long long n_newton_vec = 0;
    // host pinned mirror of scalars
    double* h_scal = nullptr;
    long long launches = 0;
    cudaStream_t cur = nullptr;
    int has_eps0 = 0;
    int bound = 0;
    int blocks_per_strip_grid = 0;
    Prof prof;
    // multigrid
    std::vector<GLevel> glev;
    std::vector<G3Level> g3lev;
    char* gmg3_base = nullptr;
    char* gmg_base = nullptr;
    double* gmg_dense = nullptr;
    double* gmg_ainv = nullptr;
    unsigned int* gmg_bar = nullptr;   // grid barrier of the persistent coarse-cycle kernel (2 words)
    int pcg_persistent = 1;         // damage PCG in one cooperative launch (PF_PCG_GRAPH=1: graph loop)
    int pcg_single = 0;             // ... in the single-reduction form (PF_PCG_SINGLE=1; measured slower)
    int gmg_coarse = 1;             // persistent coarse cycle (0: one launch per phase, PF_GMG_LEGACY)
    int gmg_cluster = 0;            // small coarse levels in one thread-block cluster (PF_GMG_CLUSTER=1: on)
    int gmg_degree = 2;
    int strip2 = 1;                 // v2 strip engine (TMA row tiles, two columns per lane): auto by mesh size; PF_STRIP2=0/1 forces
    int gmg_built = 0;              // hierarchy valid for reuse (pf_lin_opts.gmg_reuse)
    long long gmg_its0 = -1;        // iterations of the first elastic solve on it (-1: none yet)
    long long gmg_excess = 0;       // iterations beyond gmg_its0 accumulated by the later solves on it
    std::vector<unsigned char> h_bcmask;  // last Dirichlet mask (detects mask changes)
    double gmg_ratio = 0.1;
    // device-side Krylov loop graphs per solver kind (0 Kuu-Jacobi, 1 Kaa-masked, 2 Kuu-GMG):
    // a WHILE node over a captured iteration pair
    static constexpr int kGraphPtrs = 9;
    int use_graphs = 1;
    cudaStream_t cap_stream = nullptr;
    cudaGraphExec_t graph_exec[3] = {nullptr, nullptr, nullptr};
    long long graph_nodes[3] = {0, 0, 0};
    long long graph_key[3] = {-1, -1, -1};
    const void* graph_ptrs[3][kGraphPtrs] = {};
    long long geo_version = 0;   // bumped whenever Geo2 fields baked into kernels change
    // device-resident MINRES of the Newton phase (pf_newton.cu): one graph per Newton-iterate
    // buffer (the line search ping-pongs two), keyed on the pointers and sizes it bakes in
    static constexpr int kMrKey = 12;
    cudaStream_t side_stream = nullptr;  // the C block of the block-diagonal split, beside the V-cycle
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    cudaGraphExec_t mr_exec[2] = {nullptr, nullptr};
    long long mr_nodes[2] = {0, 0};
    long long mr_key[2][kMrKey] = {};
};

#define PF_TRY_GMG(x)                   \
    do {                                \
        int _rc = (x);                  \
        if (_rc != PF_OK) return _rc;   \
    } while (0)

// profiling brackets (no-ops unless enabled)
int prof_begin(Ctx* c, cudaStream_t st);
void prof_end(Ctx* c, cudaStream_t st, int slot, int kind, double bytes);

int set_error(Ctx* c, int code, const std::string& msg);
int check_cuda(Ctx* c, cudaError_t e, const char* where);

// strip grid
inline int strip_blocks(const Geo2& g) {
    long long warps = (long long)g.nwj * g.nstrips;
    return (int)((warps * 32 + kBlock - 1) / kBlock);
}

// ---- 2D operator launchers (pf_ops2d.cu) -------------------------------------------------
struct CgScal {  // pointers into the scalar block used by fused CG kernels
    double* s;
};

// y = K x (mode: PF_BC_*) ; if fused: p_out = z + beta p_in (beta from scal, 0 at iter 0),
// y = K p_out and pAp reduced into scal (CG step A).
int launch_Kuu(Ctx* c, const double* alpha, const double* x, double* y, int bcmode,
               cudaStream_t st);
void tile3(Geo3& g, int outj = 6, int resident = 296);  // outj = output pencils per block (warps - 2)
int launch3_Kuu_on(Ctx* c, const Geo3& g, const double* alpha, const double* x, double* y, int bcmode,
                   cudaStream_t st, int kind);
// Kuu apply with a fused multigrid-smoother epilogue (pf_ops3d.cu, Op3KuuSm)
enum { E3_CHEB = 1, E3_CHEB_B = 2, E3_RESID = 3, E3_RESID_CHEB0 = 4 };
struct Sm3Args {
    const double* alpha;
    const double* xin;
    const double* b;
    const double* dinv;
    double* res;
    double* dnext;
    double* xs;
    const double* live;
    const double* lam;
    double ratio;
    int k, pending;
};
int launch3_Kuu_sm(Ctx* c, const Geo3& g, int epi, const Sm3Args& a, cudaStream_t st, int kind);
int launch3_Kuu_diag_on(Ctx* c, const Geo3& g, const double* alpha, double* dinv, cudaStream_t st, int kind);
int launch_physics_relax(Ctx* c, const double* u, const double* a_prev, const double* a_star, const double* lb,
                         double omega, double* a_out, cudaStream_t st);
int launch_Kuu_smooth(Ctx* c, int epi, const double* alpha, const double* d, const GmgEpi& e, cudaStream_t st);
int launch_Kuu_cgA(Ctx* c, const double* alpha, const double* z, const double* p_in,
                   double* p_out, double* q, cudaStream_t st);
int launch_Kuu_diag(Ctx* c, const double* alpha, double* dinv, cudaStream_t st);
int launch_kappa(Ctx* c, const double* u, const double* alpha, double* kappa, double* cvec,
                 cudaStream_t st);
int launch_Kaa(Ctx* c, const double* kappa, const double* x, double* y, const unsigned char* act,
               cudaStream_t st);
int launch_Kaa_cheb(Ctx* c, const double* kappa, const double* d, const unsigned char* act, double* r,
                    double* dnext, double* x, const double* dinv, const double* tab, int k, cudaStream_t st);
int launch_Kaa_cgA(Ctx* c, const double* kappa, const double* z, const double* p_in,
                   double* p_out, double* q, const unsigned char* act, cudaStream_t st);
int launch_Kaa_diag(Ctx* c, const double* kappa, double* dinv, const unsigned char* act,
                    cudaStream_t st);
// F = Kaa trial + c with trial = clip(x + mu d, lb, 1) (mu from scal S_MU, or d == null ->
// trial = x); writes trial, F, the activity mask (classification with zeta) and reduces
// merit = |Phi|^2 into scal[slot_merit].
int launch_Kaa_trial(Ctx* c, const double* kappa, const double* cvec, const double* x,
                     const double* d, const double* lb, double* trial, double* F,
                     unsigned char* act, int merit_slot, cudaStream_t st);
int launch_physics(Ctx* c, const double* u, const double* alpha, const double* lb, double* ru,
                   double* ra, double* phi, int rows, cudaStream_t st);
int launch_load(Ctx* c, const double* alpha, double* f, const double* u_or_null,
                int rows, cudaStream_t st);
int launch_Kua(Ctx* c, const double* u, const double* alpha, const double* xa, double* yu,
               int bcmode, cudaStream_t st);
int launch_Kau(Ctx* c, const double* u, const double* alpha, const double* xu, double* ya,
               int bcmode, cudaStream_t st);
// Newton: reduced coupled Jacobian apply [Kuu_bc Kua_bc; Kau Kaa] on inactive set
int launch_jac(Ctx* c, const double* u, const double* alpha, const double* xu, const double* xa,
               double* yu, double* ya, const unsigned char* act, cudaStream_t st);

// ---- 3D operator launchers (pf_ops3d.cu) --------------------------------------------------------
int launch3_Kuu(Ctx* c, const double* alpha, const double* x, double* y, int bcmode, cudaStream_t st);
int launch3_Kuu_cgA(Ctx* c, const double* alpha, const double* z, const double* p_in, double* p_out, double* q,
                    cudaStream_t st);
int launch3_Kuu_diag(Ctx* c, const double* alpha, double* dinv, cudaStream_t st);
int launch3_kappa(Ctx* c, const double* u, double* kappa, double* cvec, cudaStream_t st);
int launch3_Kaa(Ctx* c, const double* kappa, const double* x, double* y, const unsigned char* act, cudaStream_t st);
int launch3_Kaa_cgA(Ctx* c, const double* kappa, const double* z, const double* p_in, double* p_out, double* q,
                    const unsigned char* act, cudaStream_t st);
int launch3_Kaa_diag(Ctx* c, const double* kappa, double* dinv, const unsigned char* act, cudaStream_t st);
int launch3_Kaa_trial(Ctx* c, const double* kappa, const double* cvec, const double* x, const double* d,
                      const double* lb, double* trial, double* F, int merit_slot, cudaStream_t st);
int launch3_physics(Ctx* c, const double* u, const double* alpha, const double* lb, double* ru, double* ra,
                    double* phi, int rows, cudaStream_t st);
int launch3_load(Ctx* c, const double* alpha, double* f, int rows, cudaStream_t st);
int launch3_jac(Ctx* c, const double* u, const double* alpha, const double* xu, const double* xa, double* yu,
                double* ya, const unsigned char* act, int mode, int bcmode, cudaStream_t st);

// ---- vector kernels + solvers (pf_core.cu) ---------------------------------------------
// ---- persistent-kernel reductions (fixed order: every CTA computes identical totals) -----------
__device__ __forceinline__ void block_partials(const double* v, int nv, double* partials, int row0) {
    __shared__ double sm[4][32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int k = 0; k < nv; ++k) {
        const double t = warp_sum(v[k]);
        if (lane == 0) sm[k][warp] = t;
    }
    __syncthreads();
    if (warp == 0)
        for (int k = 0; k < nv; ++k) {
            double t = lane < nw ? sm[k][lane] : 0.0;
            t = warp_sum(t);
            if (lane == 0) partials[(size_t)(row0 + k) * kMaxBlocksRed + blockIdx.x] = t;
        }
}
// after a grid barrier: the grid total of partial row `row` (fixed order; identical in every CTA)
__device__ __forceinline__ double grid_total(const double* partials, int row) {
    __shared__ double tot;
    if (threadIdx.x < 32) {
        double t = 0.0;
        for (int b = threadIdx.x; b < (int)gridDim.x; b += 32) t += __ldcg(partials + (size_t)row * kMaxBlocksRed + b);
        t = warp_sum(t);
        if (threadIdx.x == 0) tot = t;
    }
    __syncthreads();
    const double r = tot;
    __syncthreads();
    return r;
}

// the totals of partial rows `row` and `row + 1` in one pass
__device__ __forceinline__ double2 grid_total2(const double* partials, int row) {
    __shared__ double2 tot2;
    if (threadIdx.x < 32) {
        double a = 0.0, b = 0.0;
        for (int k = threadIdx.x; k < (int)gridDim.x; k += 32) {
            a += __ldcg(partials + (size_t)row * kMaxBlocksRed + k);
            b += __ldcg(partials + (size_t)(row + 1) * kMaxBlocksRed + k);
        }
        a = warp_sum(a);
        b = warp_sum(b);
        if (threadIdx.x == 0) tot2 = make_double2(a, b);
    }
    __syncthreads();
    const double2 r = tot2;
    __syncthreads();
    return r;
}

struct PcgBuffers {
    double *x, *r, *z, *p0, *p1, *q, *dinv, *b;
    long long n;
};
// the whole Kaa Jacobi-PCG loop in one cooperative launch (2D): two-phase standard PCG (kaa) or the
// single-reduction Chronopoulos-Gear form (kaa1); PF_EINVAL: not resident -> graph loop
int launch_pcg_kaa1(Ctx* c, const PcgBuffers& B, const double* kappa, const unsigned char* act, cudaStream_t st);
double pcg_kaa_iter_bytes(const Ctx* c);
int launch_pcg_kaa(Ctx* c, const PcgBuffers& B, const double* kappa, const unsigned char* act, cudaStream_t st);
int launch3_pcg_kaa(Ctx* c, const PcgBuffers& B, const double* kappa, const unsigned char* act, cudaStream_t st);
void launch_tile_compact(int ntile, const unsigned char* flag, int* list, cudaStream_t st);
// kind: 0 = Kuu Jacobi (coef = alpha), 1 = Kaa masked by act (coef = kappa), 2 = Kuu GMG
int pcg_run(Ctx* c, int kind, const PcgBuffers& B, const double* coef, const unsigned char* act,
            double rtol, double atol, long long maxit, int zero_x0, int check_every,
            pf_lin_report* rep, cudaStream_t st);
int read_scal(Ctx* c, cudaStream_t st, int first, int count);
int set_scal(Ctx* c, cudaStream_t st, int slot, double v);
int vec_blocks_n(long long n);
void classify(Ctx* c, long long n, const double* x, const double* F, const double* lb, unsigned char* act,
              double* rhs, cudaStream_t st);
void merit_parts(Ctx* c, long long n, const double* x, const double* F, const double* lb, double* pphi,
                 double* w, cudaStream_t st);
int elastic_solve(Ctx* c, const double* alpha, const double* u0, double* u_out,
                  const pf_lin_opts* o, pf_lin_report* rep, cudaStream_t st);
int damage_solve(Ctx* c, const double* u, const double* lb, const double* a_in, double* a_out,
                 const pf_vi_opts* o, pf_vi_report* rep, cudaStream_t st);
void gmg_plan(Ctx* c);
size_t gmg_bytes(const Ctx* c);
void gmg_bind(Ctx* c, char* base);
int gmg_setup(Ctx* c, cudaStream_t st);
void gmg3_plan(Ctx* c);
size_t gmg3_bytes(const Ctx* c);
void gmg3_bind(Ctx* c, char* base);
int gmg3_setup(Ctx* c, cudaStream_t st);
int gmg3_vcycle(Ctx* c, const double* r_in, double* z_out, cudaStream_t st, const double* live);
int gmg_vcycle(Ctx* c, const double* r_in, double* z_out, cudaStream_t st, const double* live,
               bool cheb0_done = false, int rz_first = -1, bool* rz_done = nullptr);
int newton_solve(Ctx* c, const double* u_in, const double* a_in, const double* lb, double* u_out,
                 double* a_out, const pf_vi_opts* o, pf_vi_report* rep, cudaStream_t st);

}  // namespace pf
