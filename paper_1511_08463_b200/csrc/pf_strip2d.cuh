// pf_strip2d.cuh -- the 2D strip engine and its operator structs (shared by pf_ops2d.cu and pf_strip2.cu).
//
// One "strip" engine (k_strip2d) drives every operator.  A warp owns vertex columns
// j = 30w-1 .. 30w+30 (lanes 0..31; lanes 1..30 produce output) and walks vertex rows
// i0-1 .. i1 of its strip.  At row step ci it holds vertex rows ci (vc) and ci+1 (vn) of its
// column in registers, gets column j+1 from lane+1 (rc, rn) by shuffle, computes the elements
// of cell (ci, j) and scatters their nodal contributions:
//     c00 -> (ci, j)      own lane, this step       c01 -> (ci, j+1)   lane+1 (shfl_up)
//     c10 -> (ci+1, j)    own lane, next step       c11 -> (ci+1, j+1) lane+1, next step
// so vertex (ci, j) is final once cell row ci is done.  Loads: 1 vertex per lane per step,
// coalesced along j; halo re-reads (1/30 columns, 1/S rows) hit L2.  No atomics: all
// outputs and reductions are deterministic.
//
// Reference formulas: fem.py:149-276 (element kinematics, energy, residuals, Hessian blocks),
// model.py:49-76 (stiffness, damage pair).  Element types per pattern (local nodes
// 0=v00 1=v10 2=v01 3=v11 4=centre), in the reference's storage order (mesh.py:95-99):
//   union-jack even cell: (0,1,3) (0,3,2);  odd cell: (0,1,2) (1,3,2)
//   right:                (0,1,3) (0,3,2)
//   crossed:              (0,1,4) (1,3,4) (3,2,4) (2,0,4)
#pragma once
#include <type_traits>

#include "pf_elem.cuh"

namespace pf {

// ---- cp.async staging ----------------------------------------------------------------------
// Every warp owns a ring of PD shared-memory stages.  A stage holds, per lane, the raw bytes of
// one vertex row (SV 8-byte slots) and one cell row (SC slots), laid out slot-major
// (slot q of lane l at q*256 + 8l; 16-byte items span two slots at q*256 + 16l) so that warp
// accesses are conflict-free.  Copies are issued PD row-steps ahead with cp.async (LDGSTS) and
// nothing touches the data until the step that consumes it: no register ring, no early
// scoreboard dependency on the loads.
__device__ __forceinline__ unsigned smem_addr(const void* p) {
    return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void cpa16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_addr(dst)), "l"(src));
}
__device__ __forceinline__ void cpa8(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_addr(dst)), "l"(src));
}
__device__ __forceinline__ void cpa4(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(smem_addr(dst)), "l"(src));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

struct Slots {
    unsigned char* p;
    int lane;          // column position inside the warp window (v1: the lane; v2: 2 lane + c)
    int pitch = 256;   // bytes per 8-byte slot row (v1: 32 columns; v2: kPitch2)
    int direct = 0;    // v2 (TMA rows): rows start at the 16-byte aligned item at or below the window's
    int idx0 = 0;      //   first item idx0, so 8-byte items sit (idx0 & 1) and bytes (idx0 & 15) further in
    __device__ __forceinline__ double* d(int q) const {
        return reinterpret_cast<double*>(p + q * pitch) + lane + (direct ? (idx0 & 1) : 0);
    }
    __device__ __forceinline__ double2* d2(int q) const {
        return reinterpret_cast<double2*>(p + q * pitch) + lane;
    }
    __device__ __forceinline__ unsigned* w(int q) const {
        return reinterpret_cast<unsigned*>(p + q * pitch) + lane;
    }
    __device__ __forceinline__ Slots at(int q) const { return Slots{p + q * pitch, lane, pitch, direct, idx0}; }
    // the same columns of an array indexed `delta` items further (crossed centres: nc, kappa slot k: k ncell)
    __device__ __forceinline__ Slots sh(long long delta) const {
        return Slots{p, lane, pitch, direct, direct ? idx0 + (int)delta : 0};
    }
};
// stage helpers for common items
__device__ __forceinline__ void put2(const Slots& s, int q, const double* base, long long v) {
    cpa16(s.d2(q), base + 2 * v);
}
__device__ __forceinline__ void put1(const Slots& s, int q, const double* base, long long v) {
    cpa8(s.d(q), base + v);
}
__device__ __forceinline__ void putb(const Slots& s, int q, const unsigned char* base, long long v) {
    cpa4(s.w(q), base + (v & ~3LL));  // the aligned word holding byte v
}
__device__ __forceinline__ double2 get2(const Slots& s, int q) { return *s.d2(q); }
__device__ __forceinline__ double get1(const Slots& s, int q) { return *s.d(q); }
__device__ __forceinline__ unsigned getb(const Slots& s, int q, long long v) {
    if (s.direct) return (unsigned)*(s.p + q * s.pitch + s.lane + (s.idx0 & 15));
    return (*s.w(q) >> (8 * (unsigned)(v & 3))) & 0xffu;
}

// ---- TMA row staging (strip engine v2) -----------------------------------------------------
// The v2 engine stages whole row tiles with the tensor memory accelerator instead of per-lane
// cp.async: every staged array is a rank-1 tensor map (cuTensorMapEncodeTiled on the host, passed
// as a __grid_constant__ kernel parameter) whose box is one warp window of 64 columns, and one
// elected lane issues cp.async.bulk.tensor.1d per item per row step (SASS UTMALDG) completing on
// the stage's mbarrier.  Rank-1 coordinates are in elements, so the window may start at any
// vertex (the reference layout's row pitch ny+1 is usually odd: rows of 8-byte items are not
// 16-byte aligned and 2D maps / plain bulk copies would not apply); out-of-range columns are
// zero-filled by the hardware and never read.
struct alignas(64) TmaMap { unsigned long long opaque[16]; };  // CUtensorMap (128 B)
constexpr int kTmaMaps = 8;
struct TmaSet { TmaMap m[kTmaMaps]; };
constexpr int kCols2 = 64;    // window columns per warp (2 per lane)
constexpr int kOut2 = kOut2Cols;  // output columns per warp
constexpr int kPitch2 = 640;  // bytes per 8-byte slot row (66 items: the aligned start may sit one item early)

__device__ __forceinline__ void mbar_init(unsigned bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_fence_init() {
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "PF_MBAR_WAIT:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@p bra PF_MBAR_DONE;\n"
        "bra PF_MBAR_WAIT;\n"
        "PF_MBAR_DONE:\n"
        "}\n" ::"r"(bar), "r"(parity) : "memory");
}
__device__ __forceinline__ void tma_row(unsigned dst, const TmaMap* map, int c0, unsigned bar) {
    asm volatile(
        "cp.async.bulk.tensor.1d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2}], [%3];\n" ::"r"(dst),
        "l"(reinterpret_cast<unsigned long long>(map)), "r"(c0), "r"(bar)
        : "memory");
}
// one stage refill, run by the elected lane: the op's tissue_* calls put*() per staged item
struct TmaIssue {
    unsigned dst;        // shared address of the stage (or of a slot inside it, after at())
    unsigned bar;        // shared address of the stage's mbarrier
    const TmaMap* maps;
    unsigned* bytes;     // running transaction byte count of this refill
    // The TMA wants 16-byte aligned global addresses: 8-byte and byte rows start at the aligned item
    // at or below v (boxes of 66 doubles / 80 bytes) and the readers skip the difference (Slots::idx0).
    __device__ __forceinline__ void put2(int q, int m, long long v) const {  // 16-byte items (slots q, q+1)
        tma_row(dst + q * kPitch2, maps + m, (int)(2 * v), bar);
        *bytes += kCols2 * 16;
    }
    __device__ __forceinline__ void put1(int q, int m, long long v) const {  // 8-byte items
        tma_row(dst + q * kPitch2, maps + m, (int)(v & ~1LL), bar);
        *bytes += (kCols2 + 2) * 8;
    }
    __device__ __forceinline__ void putb(int q, int m, long long v) const {  // byte items
        tma_row(dst + q * kPitch2, maps + m, (int)(v & ~15LL), bar);
        *bytes += kCols2 + 16;
    }
    __device__ __forceinline__ TmaIssue at(int q) const { return TmaIssue{dst + q * kPitch2, bar, maps, bytes}; }
};

// host side of the v2 engine (pf_strip2.cu): the op lists its staged arrays in maps(), run_strip2
// encodes them and launches; -1 = not applicable (array not 16-byte aligned / too long / no driver
// entry point), the caller then runs the v1 engine
struct MapBuilder {
    TmaSet set{};
    bool ok = true;
    void f1(int m, const double* p, long long n);         // 8-byte items
    void f2(int m, const double* p, long long n);         // 16-byte items (n pairs)
    void u8(int m, const unsigned char* p, long long n);  // byte items
};
template <class Op>
int run_strip2(Ctx* c, const Op& op, cudaStream_t st, int kind, double bytes);
template <class T, class = void> struct is_v2 : std::false_type {};
template <class T> struct is_v2<T, std::void_t<decltype(T::V2)>> : std::true_type {};

// ---- the strip engine ----------------------------------------------------------------------
// One pass of the engine for global warp index gw (= one strip of vertex rows x 30 columns).
template <class Op, int PAT>
__device__ __forceinline__ void strip_pass(const Geo2& g, Op& op, unsigned char* smem, int gw) {
    constexpr int NV = Op::NV, NC = Op::NC, PD = Op::pd(PAT);
    constexpr int NE = Op::ne(PAT) > 0 ? Op::ne(PAT) : 1;
    constexpr int SV = Op::sv(PAT), SC = Op::sc(PAT) > 0 ? Op::sc(PAT) : 0;
    constexpr int STAGE = (SV + SC) * 256;
    const int lane = threadIdx.x & 31;
    const int wj = gw % g.nwj, wi = gw / g.nwj;
    if (wi < g.nstrips) {
        unsigned char* wbase = smem + (threadIdx.x >> 5) * (PD * STAGE);
        const int j = wj * kLanesOut - 1 + lane;
        const bool jv = (j >= 0) && (j <= g.ny);
        const bool jc = (j >= 0) && (j < g.ny) && (lane < 31);
        const bool jo = jv && lane >= 1 && lane <= kLanesOut;
        const int i0 = wi * g.S;
        const int i1 = min(i0 + g.S, g.nx + 1);
        const int vlast = min(i1, g.nx);          // last vertex row this strip reads
        const int clast = min(i1 - 1, g.nx - 1);  // last cell row this strip computes
        double vc[NV], rc[NV], carry[NC];
#pragma unroll
        for (int k = 0; k < NC; ++k) carry[k] = 0.0;
        int ci = i0 - 1;
        auto issue = [&](int u, int r, int cr) {
            const Slots sv{wbase + u * STAGE, lane};
            if (r <= vlast && jv) op.issue_v(g, r, j, sv);
            if constexpr (SC > 0) {
                if (cr >= 0 && cr <= clast && jc) op.template issue_c<PAT>(g, cr, j, sv.at(SV));
            }
            cp_commit();
        };
#pragma unroll
        for (int k = 0; k < NV; ++k) vc[k] = 0.0;
        if (ci >= 0 && jv) {  // first row of the strip: stage through slot 0 synchronously
            const Slots s0{wbase, lane};
            op.issue_v(g, ci, j, s0);
            cp_commit();
            cp_wait<0>();
            op.fix_v(g, ci, j, s0, vc);
        }
#pragma unroll
        for (int u = 0; u < PD; ++u) issue(u, ci + 1 + u, ci + u);
#pragma unroll
        for (int k = 0; k < NV; ++k) rc[k] = __shfl_down_sync(PF_FULL, vc[k], 1);
        while (ci < i1) {
#pragma unroll
            for (int u = 0; u < PD; ++u) {
                if (ci < i1) {
                    cp_wait<PD - 1>();
                    const Slots sv{wbase + u * STAGE, lane};
                    double vn[NV], rn[NV], ec[NE];
#pragma unroll
                    for (int k = 0; k < NV; ++k) vn[k] = 0.0;
#pragma unroll
                    for (int k = 0; k < NE; ++k) ec[k] = 0.0;
                    const bool cvalid = ci >= 0 && ci < g.nx && jc;
                    if (ci + 1 <= vlast && jv) op.fix_v(g, ci + 1, j, sv, vn);
                    if (cvalid) op.template fix_c<PAT>(g, ci, j, sv.at(SV), ec);
#pragma unroll
                    for (int k = 0; k < NV; ++k) rn[k] = __shfl_down_sync(PF_FULL, vn[k], 1);
                    double c00[NC], c10[NC], c01[NC], c11[NC];
#pragma unroll
                    for (int k = 0; k < NC; ++k) { c00[k] = c10[k] = c01[k] = c11[k] = 0.0; }
                    if (cvalid)
                        op.template cell<PAT>(g, ci, j, vc, vn, rc, rn, ec, c00, c10, c01, c11,
                                              (ci >= i0) && jo);
#pragma unroll
                    for (int k = 0; k < NC; ++k) {
                        const double l01 = __shfl_up_sync(PF_FULL, c01[k], 1);
                        const double l11 = __shfl_up_sync(PF_FULL, c11[k], 1);
                        c00[k] += carry[k] + l01;
                        carry[k] = c10[k] + l11;
                    }
                    if (ci >= i0 && jo) op.out(g, ci, j, c00, vc);
#pragma unroll
                    for (int k = 0; k < NV; ++k) { vc[k] = vn[k]; rc[k] = rn[k]; }
                    // refill this stage for step ci + PD (its old contents are consumed)
                    issue(u, ci + 1 + PD, ci + PD);
                    ++ci;
                }
            }
        }
        cp_wait<0>();
    }
}

template <class Op, int PAT>
__global__ void __launch_bounds__(kBlock, Op::MINB) k_strip2d(const Geo2 g, Op op) {
    extern __shared__ __align__(16) unsigned char smem[];
    if (!op.enter()) return;  // device-side early exit (solver converged): uniform
    strip_pass<Op, PAT>(g, op, smem, blockIdx.x * (kBlock / 32) + (threadIdx.x >> 5));
    op.finish();
}

// vertex id helpers
__device__ __forceinline__ long long vid(const Geo2& g, int i, int j) { return (long long)i * g.nvy + j; }
__device__ __forceinline__ long long cid(const Geo2& g, int ci, int j) { return (long long)ci * g.ny + j; }
__device__ __forceinline__ long long ctr(const Geo2& g, int ci, int j) { return g.nc + cid(g, ci, j); }
__host__ __device__ __forceinline__ constexpr int npc_of(int pat) { return pat == PF_CROSSED ? 4 : 2; }
__host__ __device__ __forceinline__ constexpr int crossed(int pat) { return pat == PF_CROSSED ? 1 : 0; }

// ---- the strip engine, v2: two columns per lane, TMA row tiles -----------------------------------
// A warp owns a window of 64 vertex columns j0 .. j0+63 (j0 = 62 wj - 1); lane l holds columns
// A = 2l and B = 2l+1 of the window and computes the cells A (columns A, B: no exchange) and B
// (columns B and the next lane's A: one shuffle).  Window columns 1..62 are outputs.  Per vertex
// this halves the shuffles, the loop control, the stage waits and the boundary predicates of the
// one-column engine, and the union-jack parity of a cell is lane-independent ((ci + j0 + c) & 1).
// Stages are filled by TMA (TmaIssue above): nothing per lane is spent on addresses.  The sums are
// formed in the order of the one-column engine (c00 + (carry + left c01)).
//
// Two forms of the row step.  The general one predicates every vertex and cell on the mesh and
// strip edges.  The fast one runs when the window and the two vertex rows of the step are interior
// (no mesh boundary, every column valid, row owned by the strip): no validity predicates, no
// Dirichlet-mask lookups (fix_v<false> / out<false>), the cell parity a compile-time constant, and
// it is unrolled in pairs so the row registers rotate by renaming.  Lane 31's cell B and lane 0's
// column A are computed on don't-care data and never stored.
// Op interface: the v1 methods with fix_v<BND>, out<BND>, cell<PAT, NE, PARH> (PARH: the cell's
// union-jack parity when known at compile time, else -1) plus
//   static pd2(pat); tissue_v(g, i, j0, t); tissue_c<PAT>(g, ci, j0, t)   (elected lane only).
template <class Op, int PAT>
__device__ __forceinline__ void strip_pass2(const Geo2& g, Op& op, const TmaMap* maps, unsigned char* smem,
                                            int gw, int wib, int nwb) {
    constexpr int NV = Op::NV, NC = Op::NC, PD = Op::pd2(PAT);
    constexpr int NE = Op::ne(PAT) > 0 ? Op::ne(PAT) : 1;
    constexpr int SV = Op::sv(PAT), SC = Op::sc(PAT) > 0 ? Op::sc(PAT) : 0;
    constexpr int STAGE = (SV + SC) * kPitch2;
    const int lane = threadIdx.x & 31;
    // Windows that touch the mesh boundary run the general row step, about twice the instructions of
    // the fast one, and in a one-wave launch the slowest warp is the launch time.  Each of their
    // strips is therefore split between two warps: warps past the regular nwj2 x nstrips2 take the
    // second halves (g.nslow2 such windows: window 0 and the last nslow2 - 1).
    const int nreg = g.nwj2 * g.nstrips2;
    int wj, wi, half;
    if (gw < nreg) {
        wj = gw % g.nwj2;
        wi = gw / g.nwj2;
        half = (wj == 0 || wj >= g.nwj2 - (g.nslow2 - 1)) ? 1 : 0;
    } else {
        const int e = gw - nreg;
        if (g.nslow2 <= 0 || e >= g.nslow2 * g.nstrips2) return;
        const int si = e % g.nslow2;
        wi = e / g.nslow2;
        wj = si == 0 ? 0 : g.nwj2 - g.nslow2 + si;
        half = 2;
    }
    if (g.nslow2 <= 0) half = 0;
    constexpr int WSM = PD * STAGE + SV * kPitch2;  // the ring + the strip's first vertex row
    unsigned char* const wbase = smem + wib * WSM;
    const unsigned bar0 = smem_addr(smem + nwb * WSM) + wib * ((PD + 1) * 8);
    const int j0 = wj * kOut2 - 1;
    const int jA = j0 + 2 * lane, jB = jA + 1;
    const bool vA = jA >= 0 && jA <= g.ny, vB = jB <= g.ny;
    const bool cA = jA >= 0 && jA < g.ny, cB = jB < g.ny && lane < 31;
    const bool oA = vA && lane >= 1, oB = vB && lane < 31;
    const bool fastwin = j0 >= 1 && j0 + kCols2 <= g.ny;  // every column a valid interior vertex
    const int h2 = (g.S2 + 1) / 2;  // rows of a first half
    const int i0 = wi * g.S2 + (half == 2 ? h2 : 0);
    const int i1 = min(wi * g.S2 + (half == 1 ? h2 : g.S2), g.nx + 1);
    if (i0 >= i1) return;
    const int vlast = min(i1, g.nx);          // last vertex row this strip reads
    const int clast = min(i1 - 1, g.nx - 1);  // last cell row this strip computes
    if (lane == 0) {
#pragma unroll
        for (int u = 0; u <= PD; ++u) mbar_init(bar0 + 8 * u, 1);
        mbar_fence_init();
    }
    __syncwarp();
    double vcA[NV], vcB[NV], rc[NV], carryA[NC], carryB[NC];
#pragma unroll
    for (int k = 0; k < NC; ++k) carryA[k] = carryB[k] = 0.0;
#pragma unroll
    for (int k = 0; k < NV; ++k) vcA[k] = vcB[k] = 0.0;
    int ci = i0 - 1;
    // refill the stage at (sbase, bar) for row step `step` (vertex row step + 1, cell row step)
    auto issue = [&](unsigned char* sbase, unsigned bar, int step) {
        if (lane == 0) {
            unsigned bytes = 0;
            const TmaIssue t{smem_addr(sbase), bar, maps, &bytes};
            if (step + 1 <= vlast) op.tissue_v(g, step + 1, j0, t);
            if constexpr (SC > 0) {
                if (step >= 0 && step <= clast) op.template tissue_c<PAT>(g, step, j0, t.at(SV));
            }
            mbar_expect_tx(bar, bytes);
        }
    };
    // the first vertex row of the strip has its own slots (after the ring) and barrier (index PD), so
    // its copy and the ring's first PD refills are all in flight before the first wait
    unsigned char* const frow = wbase + PD * STAGE;
    if (ci >= 0 && lane == 0) {
        unsigned bytes = 0;
        const TmaIssue t{smem_addr(frow), bar0 + 8 * PD, maps, &bytes};
        op.tissue_v(g, ci, j0, t);
        mbar_expect_tx(t.bar, bytes);
    }
#pragma unroll
    for (int u = 0; u < PD; ++u)
        if (ci + u < i1) issue(wbase + u * STAGE, bar0 + 8 * u, ci + u);
    if (ci >= 0) {
        mbar_wait(bar0 + 8 * PD, 0);
        const int v0 = (int)vid(g, ci, j0);
        if (vA) op.fix_v(g, ci, jA, Slots{frow, 2 * lane, kPitch2, 1, v0}, vcA);
        if (vB) op.fix_v(g, ci, jB, Slots{frow, 2 * lane + 1, kPitch2, 1, v0}, vcB);
    }
#pragma unroll
    for (int k = 0; k < NV; ++k) rc[k] = __shfl_down_sync(PF_FULL, vcA[k], 1);
    // ring position of step ci: stage u at sb with barrier bar, every stage on its phase-th use
    int u = 0;
    unsigned char* sb = wbase;
    unsigned bar = bar0, phase = 0;
    auto step = [&](auto fast_c, auto par_c) {
        constexpr bool FAST = decltype(fast_c)::v != 0;
        constexpr int PE = decltype(par_c)::v;            // parity of cell A (fast form, union-jack), else -1
        constexpr int PO = PE < 0 ? -1 : 1 - PE;          // parity of cell B
        mbar_wait(bar, phase);
        const int v0 = (int)vid(g, ci + 1, j0), c0 = (int)cid(g, ci, j0);  // first items of the staged rows
        const Slots sA{sb, 2 * lane, kPitch2, 1, v0}, sB{sb, 2 * lane + 1, kPitch2, 1, v0};
        const Slots tA{sb + SV * kPitch2, 2 * lane, kPitch2, 1, c0}, tB{sb + SV * kPitch2, 2 * lane + 1, kPitch2, 1, c0};
        double vnA[NV], vnB[NV], rn[NV], eA[NE], eB[NE];
        double a00[NC], a10[NC], a01[NC], a11[NC], b00[NC], b10[NC], b01[NC], b11[NC];
        if constexpr (FAST) {
            op.template fix_v<false>(g, ci + 1, jA, sA, vnA);
            op.template fix_v<false>(g, ci + 1, jB, sB, vnB);
            if constexpr (SC > 0 || Op::ne(PAT) > 0) {
                op.template fix_c<PAT>(g, ci, jA, tA, eA);
                op.template fix_c<PAT>(g, ci, jB, tB, eB);
            }
#pragma unroll
            for (int k = 0; k < NV; ++k) rn[k] = __shfl_down_sync(PF_FULL, vnA[k], 1);
            op.template cell<PAT, NE, PE>(g, ci, jA, vcA, vnA, vcB, vnB, eA, a00, a10, a01, a11, lane >= 1);
            op.template cell<PAT, NE, PO>(g, ci, jB, vcB, vnB, rc, rn, eB, b00, b10, b01, b11, lane < 31);
        } else {
#pragma unroll
            for (int k = 0; k < NV; ++k) vnA[k] = vnB[k] = 0.0;
#pragma unroll
            for (int k = 0; k < NE; ++k) eA[k] = eB[k] = 0.0;
            const bool rowv = ci + 1 <= vlast, crow = ci >= 0 && ci < g.nx, own = ci >= i0;
            if (rowv && vA) op.fix_v(g, ci + 1, jA, sA, vnA);
            if (rowv && vB) op.fix_v(g, ci + 1, jB, sB, vnB);
            if (crow && cA) op.template fix_c<PAT>(g, ci, jA, tA, eA);
            if (crow && cB) op.template fix_c<PAT>(g, ci, jB, tB, eB);
#pragma unroll
            for (int k = 0; k < NV; ++k) rn[k] = __shfl_down_sync(PF_FULL, vnA[k], 1);
#pragma unroll
            for (int k = 0; k < NC; ++k) {
                a00[k] = a10[k] = a01[k] = a11[k] = 0.0;
                b00[k] = b10[k] = b01[k] = b11[k] = 0.0;
            }
            if (crow && cA) op.template cell<PAT, NE, -1>(g, ci, jA, vcA, vnA, vcB, vnB, eA, a00, a10, a01, a11, own && oA);
            if (crow && cB) op.template cell<PAT, NE, -1>(g, ci, jB, vcB, vnB, rc, rn, eB, b00, b10, b01, b11, own && oB);
        }
#pragma unroll
        for (int k = 0; k < NC; ++k) {
            const double l01 = __shfl_up_sync(PF_FULL, b01[k], 1);
            const double l11 = __shfl_up_sync(PF_FULL, b11[k], 1);
            a00[k] += carryA[k] + l01;
            carryA[k] = a10[k] + l11;
            b00[k] += carryB[k] + a01[k];
            carryB[k] = b10[k] + a11[k];
        }
        if constexpr (FAST) {
            if (lane >= 1) op.template out<false>(g, ci, jA, a00, vcA);
            if (lane < 31) op.template out<false>(g, ci, jB, b00, vcB);
        } else {
            if (ci >= i0 && oA) op.out(g, ci, jA, a00, vcA);
            if (ci >= i0 && oB) op.out(g, ci, jB, b00, vcB);
        }
#pragma unroll
        for (int k = 0; k < NV; ++k) { vcA[k] = vnA[k]; vcB[k] = vnB[k]; rc[k] = rn[k]; }
        __syncwarp();  // every lane is done with this stage before the TMA overwrites it
        if (ci + PD < i1) issue(sb, bar, ci + PD);
        ++ci;
        ++u;
        sb += STAGE;
        bar += 8;
        if (u == PD) { u = 0; sb = wbase; bar = bar0; phase ^= 1u; }
    };
    // fast pairs need rows ci .. ci+2 interior and owned: ci >= max(i0, 1), ci + 2 <= nx - 1, ci + 1 < i1
    const int flo = max(i0, 1), fhi = min(i1 - 2, g.nx - 3);
    while (ci < i1) {
        if (fastwin && ci >= flo && ci <= fhi) {
            if constexpr (PAT == PF_UNION_JACK) {
                if (((ci + j0) & 1) == 0) { step(IC<1>{}, IC<0>{}); step(IC<1>{}, IC<1>{}); }
                else { step(IC<1>{}, IC<1>{}); step(IC<1>{}, IC<0>{}); }
            } else {
                step(IC<1>{}, IC<-1>{});
                step(IC<1>{}, IC<-1>{});
            }
        } else {
            step(IC<0>{}, IC<-1>{});
        }
    }
}

struct NoRed {
    static constexpr int MINB = 2;
    __device__ bool enter() const { return true; }
    __device__ void finish() {}
};

// cell scalars E / Gc (per-cell field or the scalar)
__device__ __forceinline__ void putE(const Geo2& g, const Slots& s, int q, long long cell) {
    if (g.E_cell) put1(s, q, g.E_cell, cell);
}
__device__ __forceinline__ double getE(const Geo2& g, const Slots& s, int q) {
    return g.E_cell ? get1(s, q) : g.E;
}
__device__ __forceinline__ void putGc(const Geo2& g, const Slots& s, int q, long long cell) {
    if (g.Gc_cell) put1(s, q, g.Gc_cell, cell);
}
__device__ __forceinline__ double getGc(const Geo2& g, const Slots& s, int q) {
    return g.Gc_cell ? get1(s, q) : g.Gc;
}

// ================================================================================================
// Kuu: y = K(alpha) x, optionally Dirichlet-eliminated (fem.py:233-243, 282-294).
// FUSED: CG step A -- p_out = z + beta p_in (beta = 0 at iteration 0), y = K p_out, pAp reduced
// and gamma = rz / pAp formed by the last block (linalg.py:130-138).
// vertex slots: x|z (0-1), [p_in (2-3)], alpha; cell slots: E, [centre x|z, p_in, alpha]
// ================================================================================================
// EPI != 0: GMG fine-level smoother epilogue (pf_gmg.cu), applied where each output vertex is
// final instead of storing y = K x (see GmgEpi in pf_internal.cuh for the modes).
template <bool FUSED, int EPI = EPI_NONE>
struct OpKuu {
    static constexpr int NV = 3, NC = 2, MINB = 2;
    static constexpr int pd(int pat) { return 4; }
    static constexpr int ne(int pat) { return 1 + 3 * crossed(pat); }
    static constexpr int sv(int) { return FUSED ? 5 : 3; }
    static constexpr int sc(int pat) { return 1 + crossed(pat) * (FUSED ? 5 : 3); }
    const double* alpha;
    const double* x;      // plain: x ; fused: z
    const double* pin;    // fused only
    double* pout;         // fused only
    double* y;
    int bcmode;
    double* scal;
    RedBuf rb;
    double acc;
    GmgEpi e{};
    double ca = 0.0, cb = 0.0, th = 1.0;
    double breg = 0.0;  // persistent PCG (k_pcg_gmg2d): beta held in a register instead of scal[S_BETA]
    int use_breg = 0;

    __device__ bool enter() {
        if constexpr (EPI != EPI_NONE) {
            if (e.live && !(e.live[S_DONE] == 0.0 && e.live[S_FAIL] == 0.0)) return false;
            const Cheb c = cheb_of(e.lam, e.ratio);
            th = c.theta;
            if (EPI == EPI_CHEB || EPI == EPI_CHEB_ADDD) cheb_ab(c, e.k, ca, cb);
            return true;
        }
        if (!FUSED) return true;
        return scal[S_DONE] == 0.0 && scal[S_FAIL] == 0.0;
    }
    // smoother epilogue at a final output vertex: y = (K d)_id, (d0, d1) = d_id (the raw input)
    __device__ __forceinline__ void epi(long long id, double y0, double y1, double d0, double d1) {
        if constexpr (EPI == EPI_CHEB || EPI == EPI_CHEB_ADDD) {
            // res -= D^-1 y ; dnext = a d + b res ; x (+= d) += dnext   (k_cheb_step)
            const double2 dw = bmul(e.Dinv, e.nvD, id, y0, y1);
            double2 r = reinterpret_cast<const double2*>(e.res)[id];
            r.x -= dw.x;
            r.y -= dw.y;
            const double2 dn = make_double2(ca * d0 + cb * r.x, ca * d1 + cb * r.y);
            st2(e.res, id, r.x, r.y);
            st2(e.dnext, id, dn.x, dn.y);
            double2 xv = reinterpret_cast<const double2*>(e.xs)[id];
            if (EPI == EPI_CHEB_ADDD) {
                xv.x += d0;
                xv.y += d1;
            }
            xv.x += dn.x;
            xv.y += dn.y;
            st2(e.xs, id, xv.x, xv.y);
            if (e.rz_first >= 0) {  // PCG r . z with z = this final smoother iterate
                const double2 rv = ld2(e.rcg, id);
                acc += rv.x * xv.x + rv.y * xv.y;
            }
        } else if constexpr (EPI == EPI_RESID) {
            const double2 bv = ld2(e.bvec, id);
            st2(e.rout, id, bv.x - y0, bv.y - y1);
        } else if constexpr (EPI == EPI_RESID_CHEB0) {
            // res = D^-1 (b - y) ; d0 = res / theta   (k_resid + k_cheb0; x += d0 is deferred)
            const double2 bv = ld2(e.bvec, id);
            const double2 rr = bmul(e.Dinv, e.nvD, id, bv.x - y0, bv.y - y1);
            st2(e.res, id, rr.x, rr.y);
            st2(e.dnext, id, rr.x / th, rr.y / th);
        }
    }
    __device__ __forceinline__ double beta() const { return use_breg ? breg : (scal[S_ITER] > 0.0 ? scal[S_BETA] : 0.0); }
    __device__ __forceinline__ double2 xval(long long v) const {  // direct (boundary rows only)
        double2 z = ld2(x, v);
        if (FUSED) {
            const double b = beta();
            const double2 p = ld2(pin, v);
            z.x = z.x + b * p.x;
            z.y = z.y + b * p.y;
        }
        return z;
    }
    __device__ __forceinline__ void stage_vertex(const Slots& s, long long v) const {
        put2(s, 0, x, v);
        if (FUSED) { put2(s, 2, pin, v); put1(s, 4, alpha, v); }
        else put1(s, 2, alpha, v);
    }
    __device__ __forceinline__ double2 staged_x(const Slots& s) const {
        double2 z = get2(s, 0);
        if (FUSED) {
            const double b = beta();
            const double2 p = get2(s, 2);
            z.x = z.x + b * p.x;
            z.y = z.y + b * p.y;
        }
        return z;
    }
    __device__ void issue_v(const Geo2& g, int i, int j, const Slots& s) const { stage_vertex(s, vid(g, i, j)); }
    // v2 engine: tensor maps MX = x|z (16-byte items), MP = p_in, MA = alpha, ME = E per cell
    enum { MX = 0, MP = 1, MA = 2, ME = 3 };
    static constexpr bool V2 = true;
    static constexpr int pd2(int pat) { return pat == PF_CROSSED ? 3 : 4; }
    void maps(const Geo2& g, MapBuilder& mb) const {
        mb.f2(MX, x, g.nv);
        if (FUSED) mb.f2(MP, pin, g.nv);
        mb.f1(MA, alpha, g.nv);
        if (g.E_cell) mb.f1(ME, g.E_cell, g.ncell);
    }
    __device__ __forceinline__ void tstage_vertex(const TmaIssue& t, long long v) const {
        t.put2(0, MX, v);
        if (FUSED) { t.put2(2, MP, v); t.put1(4, MA, v); }
        else t.put1(2, MA, v);
    }
    __device__ void tissue_v(const Geo2& g, int i, int j0, const TmaIssue& t) const { tstage_vertex(t, vid(g, i, j0)); }
    template <int PAT>
    __device__ void tissue_c(const Geo2& g, int ci, int j0, const TmaIssue& t) const {
        if (g.E_cell) t.put1(0, ME, cid(g, ci, j0));
        if constexpr (PAT == PF_CROSSED) tstage_vertex(t.at(1), ctr(g, ci, j0));
    }
    template <bool BND = true>
    __device__ void fix_v(const Geo2& g, int i, int j, const Slots& s, double (&v)[NV]) const {
        const double2 xv = staged_x(s);
        const unsigned m = (BND && bcmode) ? bcbits(g, i, j, vid(g, i, j)) : 0u;
        v[0] = (m & 1u) ? 0.0 : xv.x;
        v[1] = (m & 2u) ? 0.0 : xv.y;
        v[2] = get1(s, FUSED ? 4 : 2);
    }
    template <int PAT>
    __device__ void issue_c(const Geo2& g, int ci, int j, const Slots& s) const {
        putE(g, s, 0, cid(g, ci, j));
        if constexpr (PAT == PF_CROSSED) stage_vertex(s.at(1), ctr(g, ci, j));
    }
    template <int PAT, int NE>
    __device__ void fix_c(const Geo2& g, int ci, int j, const Slots& s, double (&e)[NE]) const {
        e[0] = getE(g, s, 0);
        if constexpr (PAT == PF_CROSSED) {
            const Slots c = s.at(1).sh(g.nc);
            const double2 xv = staged_x(c);
            e[1] = xv.x; e[2] = xv.y; e[3] = get1(c, FUSED ? 4 : 2);
        }
    }
    template <int PAT, int NE, int PARH = -1>
    __device__ void cell(const Geo2& g, int ci, int j, const double (&vc)[NV], const double (&vn)[NV],
                         const double (&rc)[NV], const double (&rn)[NV], const double (&ec)[NE],
                         double (&c00)[NC], double (&c10)[NC], double (&c01)[NC], double (&c11)[NC],
                         bool own) {
        if constexpr (PAT == PF_UNION_JACK || PAT == PF_RIGHT) {
            // Edge form: every union-jack triangle is a right triangle with one cell edge along x
            // and one along y, so both diagonal orientations use the same four edge differences;
            // the parity only decides which vertical edge pairs with which triangle (4 selects on
            // the inputs, 4 on the outputs, instead of mirroring 15 inputs and 10 outputs).
            // right: always the even split; PARH >= 0: the parity is a compile-time constant
            const bool odd = PAT == PF_UNION_JACK && (PARH >= 0 ? PARH != 0 : ((ci + j) & 1) != 0);
            const double ihx = g.ihx, ihy = ihy_at(g, j);
            const double sc = area_at(g, j) * ec[0];
            // corners: 00 = vc (ci, j), 10 = vn (ci+1, j), 01 = rc (ci, j+1), 11 = rn (ci+1, j+1)
            const double bx1 = vn[0] - vc[0], bx2 = vn[1] - vc[1];  // bottom edge (x)
            const double tx1 = rn[0] - rc[0], tx2 = rn[1] - rc[1];  // top edge (x)
            const double ly1 = rc[0] - vc[0], ly2 = rc[1] - vc[1];  // left edge (y)
            const double ry1 = rn[0] - vn[0], ry2 = rn[1] - vn[1];  // right edge (y)
            // triangle on the bottom edge: even (00,10,11) -> right edge ; odd (00,10,01) -> left
            // triangle on the top edge:    even (00,11,01) -> left edge  ; odd (10,11,01) -> right
            const double by1 = odd ? ly1 : ry1, by2 = odd ? ly2 : ry2;
            const double ty1 = odd ? ry1 : ly1, ty2 = odd ? ry2 : ly2;
            const double ab = (vc[2] + vn[2] + (odd ? rc[2] : rn[2])) * (1.0 / 3.0);
            const double at = ((odd ? vn[2] : vc[2]) + rn[2] + rc[2]) * (1.0 / 3.0);
            double fbx1, fbx2, fby1, fby2, ftx1, ftx2, fty1, fty2;  // edge fluxes (x / y), 2 comps
            {
                const double om = 1.0 - ab;
                const double k = (om * om + g.kell) * sc;
                double s0, s1, s2;
                unit_stress(g, bx1 * ihx, by2 * ihy, by1 * ihy + bx2 * ihx, s0, s1, s2);
                fbx1 = k * ihx * s0; fbx2 = k * ihx * s2;
                fby1 = k * ihy * s2; fby2 = k * ihy * s1;
            }
            {
                const double om = 1.0 - at;
                const double k = (om * om + g.kell) * sc;
                double s0, s1, s2;
                unit_stress(g, tx1 * ihx, ty2 * ihy, ty1 * ihy + tx2 * ihx, s0, s1, s2);
                ftx1 = k * ihx * s0; ftx2 = k * ihx * s2;
                fty1 = k * ihy * s2; fty2 = k * ihy * s1;
            }
            const double fr1 = odd ? fty1 : fby1, fr2 = odd ? fty2 : fby2;  // right edge
            const double fl1 = odd ? fby1 : fty1, fl2 = odd ? fby2 : fty2;  // left edge
            c00[0] = -fbx1 - fl1; c00[1] = -fbx2 - fl2;
            c10[0] = fbx1 - fr1;  c10[1] = fbx2 - fr2;
            c01[0] = -ftx1 + fl1; c01[1] = -ftx2 + fl2;
            c11[0] = ftx1 + fr1;  c11[1] = ftx2 + fr2;
            return;
        }
        double U1[5] = {vc[0], vn[0], rc[0], rn[0], 0.0};
        double U2[5] = {vc[1], vn[1], rc[1], rn[1], 0.0};
        double Al[5] = {vc[2], vn[2], rc[2], rn[2], 0.0};
        if constexpr (PAT == PF_CROSSED) { U1[4] = ec[1]; U2[4] = ec[2]; Al[4] = ec[3]; }
        double Y1[5] = {0, 0, 0, 0, 0}, Y2[5] = {0, 0, 0, 0, 0};
        const int par = (PAT == PF_UNION_JACK) ? (PARH >= 0 ? PARH : ((ci + j) & 1)) : 0;
        const double hxs = par ? -g.ihx : g.ihx;
        mirror<PAT>(par, U1);
        mirror<PAT>(par, U2);
        mirror<PAT>(par, Al);
        const double Ec = ec[0];
        for_each_elem<PAT>(par, [&](auto T, auto, auto A, auto B, auto C) {
            const double ab = (Al[A.v] + Al[B.v] + Al[C.v]) * (1.0 / 3.0);
            const double om = 1.0 - ab;
            const double s = (om * om + g.kell) * area_at(g, j) * Ec;
            double e0, e1, e2, s0, s1, s2;
            strain<PAT, T.v, A.v, B.v, C.v>(hxs, ihy_at(g, j), U1, U2, e0, e1, e2);
            unit_stress(g, e0, e1, e2, s0, s1, s2);
            scatter_BT<PAT, T.v, A.v, B.v, C.v>(hxs, ihy_at(g, j), s * s0, s * s1, s * s2, Y1, Y2);
        });
        mirror<PAT>(par, Y1);
        mirror<PAT>(par, Y2);
        c00[0] = Y1[0]; c00[1] = Y2[0];
        c10[0] = Y1[1]; c10[1] = Y2[1];
        c01[0] = Y1[2]; c01[1] = Y2[2];
        c11[0] = Y1[3]; c11[1] = Y2[3];
        if constexpr (PAT == PF_CROSSED) {
            if (own) {
                const long long cv = ctr(g, ci, j);
                if constexpr (EPI != EPI_NONE) {
                    epi(cv, Y1[4], Y2[4], U1[4], U2[4]);
                } else {
                    st2(y, cv, Y1[4], Y2[4]);
                    if (FUSED) {
                        st2(pout, cv, U1[4], U2[4]);
                        acc += U1[4] * Y1[4] + U2[4] * Y2[4];
                    }
                }
            }
        }
    }
    template <bool BND = true>
    __device__ void out(const Geo2& g, int i, int j, const double (&t)[NC], const double (&v)[NV]) {
        const long long id = vid(g, i, j);
        double y0 = t[0], y1 = t[1];
        double p0 = v[0], p1 = v[1];
        const unsigned m = (BND && bcmode) ? bcbits(g, i, j, id) : 0u;
        if (m) {
            const double2 xv = xval(id);
            if (m & 1u) { y0 = xv.x; p0 = xv.x; }
            if (m & 2u) { y1 = xv.y; p1 = xv.y; }
        }
        if constexpr (EPI != EPI_NONE) {
            epi(id, y0, y1, p0, p1);
            return;
        }
        st2(y, id, y0, y1);
        if (FUSED) {
            st2(pout, id, p0, p1);
            acc += p0 * y0 + p1 * y1;
        }
    }
    __device__ void finish() {
        if constexpr (EPI == EPI_CHEB || EPI == EPI_CHEB_ADDD) {
            if (e.rz_first < 0) return;
            double v[1] = {acc};
            double* s = scal;
            const int first = e.rz_first;
            grid_reduce<1>(v, rb, 6, [s, first](double* t) {  // k_cg_rz
                if (!(t[0] > 0.0)) { s[S_FAIL] = 2.0; return; }
                if (!first) s[S_BETA] = t[0] / s[S_RZ];
                s[S_RZ] = t[0];
            });
            return;
        }
        if (EPI != EPI_NONE || !FUSED) return;
        double v[1] = {acc};
        double* s = scal;
        grid_reduce<1>(v, rb, 0, [s](double* tot) {
            s[S_PAP] = tot[0];
            if (!(tot[0] > 0.0)) s[S_FAIL] = 1.0;  // breakdown: p'Ap <= 0 (linalg.py:133-136)
            else s[S_GAMMA] = s[S_RZ] / tot[0];
        });
    }
};

// diag(Kuu) -> dinv = 1/diag; eliminated rows get 1.   vertex: alpha; cell: E, [alpha_c]
struct OpKuuDiag : NoRed {
    static constexpr int NV = 1, NC = 2;
    static constexpr int pd(int) { return 4; }
    static constexpr int ne(int pat) { return 1 + crossed(pat); }
    static constexpr int sv(int) { return 1; }
    static constexpr int sc(int pat) { return 1 + crossed(pat); }
    const double* alpha;
    double* dinv;
    __device__ void issue_v(const Geo2& g, int i, int j, const Slots& s) const { put1(s, 0, alpha, vid(g, i, j)); }
    template <bool BND = true>
    __device__ void fix_v(const Geo2&, int, int, const Slots& s, double (&v)[NV]) const { v[0] = get1(s, 0); }
    template <int PAT>
    __device__ void issue_c(const Geo2& g, int ci, int j, const Slots& s) const {
        putE(g, s, 0, cid(g, ci, j));
        if constexpr (PAT == PF_CROSSED) put1(s, 1, alpha, ctr(g, ci, j));
    }
    template <int PAT, int NE>
    __device__ void fix_c(const Geo2& g, int, int, const Slots& s, double (&e)[NE]) const {
        e[0] = getE(g, s, 0);
        if constexpr (PAT == PF_CROSSED) e[1] = get1(s, 1);
    }
    template <int PAT, int NE, int PARH = -1>
    __device__ void cell(const Geo2& g, int ci, int j, const double (&vc)[NV], const double (&vn)[NV],
                         const double (&rc)[NV], const double (&rn)[NV], const double (&ec)[NE],
                         double (&c00)[NC], double (&c10)[NC], double (&c01)[NC], double (&c11)[NC],
                         bool own) {
        double Al[5] = {vc[0], vn[0], rc[0], rn[0], 0.0};
        if constexpr (PAT == PF_CROSSED) Al[4] = ec[1];
        double Y1[5] = {0, 0, 0, 0, 0}, Y2[5] = {0, 0, 0, 0, 0};
        const int par = (PAT == PF_UNION_JACK) ? (PARH >= 0 ? PARH : ((ci + j) & 1)) : 0;
        mirror<PAT>(par, Al);
        const double Ec = ec[0];
        for_each_elem<PAT>(par, [&](auto T, auto, auto A, auto B, auto C) {
            const double ab = (Al[A.v] + Al[B.v] + Al[C.v]) * (1.0 / 3.0);
            const double om = 1.0 - ab;
            const double s = (om * om + g.kell) * area_at(g, j) * Ec;
            using Sh = Shp<PAT, T.v>;
            const double X2 = g.ihx * g.ihx, Y2h = ihy_at(g, j) * ihy_at(g, j);
            const double bb[3] = {double(Sh::b0 * Sh::b0) * X2, double(Sh::b1 * Sh::b1) * X2,
                                  double(Sh::b2 * Sh::b2) * X2};
            const double cc[3] = {double(Sh::c0 * Sh::c0) * Y2h, double(Sh::c1 * Sh::c1) * Y2h,
                                  double(Sh::c2 * Sh::c2) * Y2h};
            Y1[A.v] += s * (bb[0] * g.D00 + cc[0] * g.D22);
            Y2[A.v] += s * (cc[0] * g.D11 + bb[0] * g.D22);
            Y1[B.v] += s * (bb[1] * g.D00 + cc[1] * g.D22);
            Y2[B.v] += s * (cc[1] * g.D11 + bb[1] * g.D22);
            Y1[C.v] += s * (bb[2] * g.D00 + cc[2] * g.D22);
            Y2[C.v] += s * (cc[2] * g.D11 + bb[2] * g.D22);
        });
        mirror<PAT>(par, Y1);
        mirror<PAT>(par, Y2);
        c00[0] = Y1[0]; c00[1] = Y2[0]; c10[0] = Y1[1]; c10[1] = Y2[1];
        c01[0] = Y1[2]; c01[1] = Y2[2]; c11[0] = Y1[3]; c11[1] = Y2[3];
        if constexpr (PAT == PF_CROSSED) {
            if (own) st2(dinv, ctr(g, ci, j), 1.0 / Y1[4], 1.0 / Y2[4]);
        }
    }
    template <bool BND = true>
    __device__ void out(const Geo2& g, int i, int j, const double (&t)[NC], const double (&)[NV]) {
        const long long id = vid(g, i, j);
        const unsigned m = bcbits(g, i, j, id);
        st2(dinv, id, (m & 1u) ? 1.0 : 1.0 / t[0], (m & 2u) ? 1.0 : 1.0 / t[1]);
    }
};

// ================================================================================================
// Damage block.  kappa_e = (1/2 a'' q + (Gc/c_w) w''/ell) |T|/9 is the element reaction
// coefficient (fem.py:266-276; independent of alpha for AT1/AT2); c = r_alpha - Kaa alpha is its
// affine remainder (solver.py:152-153), c_v = sum_e |T|/3 (-q_e + [AT1] Gc_e/(c_w ell)).
// vertex: u; cell: E, Gc, [u_c]
// ================================================================================================
struct OpKappa : NoRed {
    static constexpr int NV = 2, NC = 1;
    static constexpr int pd(int) { return 4; }
    static constexpr int ne(int pat) { return 2 + 2 * crossed(pat); }
    static constexpr int sv(int) { return 2; }
    static constexpr int sc(int pat) { return 2 + 2 * crossed(pat); }
    const double* u;
    double* kappa;
    double* cvec;
    __device__ void issue_v(const Geo2& g, int i, int j, const Slots& s) const { put2(s, 0, u, vid(g, i, j)); }
    // v2 engine: tensor maps MU = u, ME = E per cell, MGC = Gc per cell
    enum { MU = 0, ME = 1, MGC = 2 };
    static constexpr bool V2 = true;
    static constexpr int pd2(int pat) { return pat == PF_CROSSED ? 3 : 4; }
    void maps(const Geo2& g, MapBuilder& mb) const {
        mb.f2(MU, u, g.nv);
        if (g.E_cell) mb.f1(ME, g.E_cell, g.ncell);
        if (g.Gc_cell) mb.f1(MGC, g.Gc_cell, g.ncell);
    }
    __device__ void tissue_v(const Geo2& g, int i, int j0, const TmaIssue& t) const { t.put2(0, MU, vid(g, i, j0)); }
    template <int PAT>
    __device__ void tissue_c(const Geo2& g, int ci, int j0, const TmaIssue& t) const {
        const long long cell = cid(g, ci, j0);
        if (g.E_cell) t.put1(0, ME, cell);
        if (g.Gc_cell) t.put1(1, MGC, cell);
        if constexpr (PAT == PF_CROSSED) t.put2(2, MU, ctr(g, ci, j0));
    }
    template <bool BND = true>
    __device__ void fix_v(const Geo2&, int, int, const Slots& s, double (&v)[NV]) const {
        const double2 uv = get2(s, 0);
        v[0] = uv.x; v[1] = uv.y;
    }
    template <int PAT>
    __device__ void issue_c(const Geo2& g, int ci, int j, const Slots& s) const {
        const long long cell = cid(g, ci, j);
        putE(g, s, 0, cell);
        putGc(g, s, 1, cell);
        if constexpr (PAT == PF_CROSSED) put2(s, 2, u, ctr(g, ci, j));
    }
    template <int PAT, int NE>
    __device__ void fix_c(const Geo2& g, int, int, const Slots& s, double (&e)[NE]) const {
        e[0] = getE(g, s, 0);
        e[1] = getGc(g, s, 1);
        if constexpr (PAT == PF_CROSSED) {
            const double2 uv = get2(s, 2);
            e[2] = uv.x; e[3] = uv.y;
        }
    }
    template <int PAT, int NE, int PARH = -1>
    __device__ void cell(const Geo2& g, int ci, int j, const double (&vc)[NV], const double (&vn)[NV],
                         const double (&rc)[NV], const double (&rn)[NV], const double (&ec)[NE],
                         double (&c00)[NC], double (&c10)[NC], double (&c01)[NC], double (&c11)[NC],
                         bool own) {
        double U1[5] = {vc[0], vn[0], rc[0], rn[0], 0.0};
        double U2[5] = {vc[1], vn[1], rc[1], rn[1], 0.0};
        if constexpr (PAT == PF_CROSSED) { U1[4] = ec[2]; U2[4] = ec[3]; }
        double Y[5] = {0, 0, 0, 0, 0};
        const int par = (PAT == PF_UNION_JACK) ? (PARH >= 0 ? PARH : ((ci + j) & 1)) : 0;
        const double hxs = par ? -g.ihx : g.ihx;
        mirror<PAT>(par, U1);
        mirror<PAT>(par, U2);
        const long long cell = cid(g, ci, j);
        const double Ec = ec[0];
        const double kc = ec[1] / g.cw;
        for_each_elem<PAT>(par, [&](auto T, auto S, auto A, auto B, auto C) {
            double e0, e1, e2, s0, s1, s2;
            strain<PAT, T.v, A.v, B.v, C.v>(hxs, ihy_at(g, j), U1, U2, e0, e1, e2);
            if (g.eps0) {
                const double e = __ldg(g.eps0 + (long long)(T.v + 2 * par) * g.ny + j);
                e0 -= e; e1 -= e;
            }
            unit_stress(g, e0, e1, e2, s0, s1, s2);
            const double q = Ec * (e0 * s0 + e1 * s1 + e2 * s2);
            const double ar = area_at(g, j);
            const double kap = (q + (g.at2 ? 2.0 * kc / g.ell : 0.0)) * ar * (1.0 / 9.0);
            const double cc = ar * (1.0 / 3.0) * (-q + (g.at2 ? 0.0 : kc / g.ell));
            Y[A.v] += cc; Y[B.v] += cc; Y[C.v] += cc;
            if (own) kappa[(long long)S.v * g.ncell + cell] = kap;
        });
        mirror<PAT>(par, Y);
        c00[0] = Y[0]; c10[0] = Y[1]; c01[0] = Y[2]; c11[0] = Y[3];
        if constexpr (PAT == PF_CROSSED) {
            if (own) cvec[ctr(g, ci, j)] = Y[4];
        }
    }
    template <bool BND = true>
    __device__ void out(const Geo2& g, int i, int j, const double (&t)[NC], const double (&)[NV]) {
        cvec[vid(g, i, j)] = t[0];
    }
};

// Damage Hessian element action: y_m += kappa (x_A + x_B + x_C) + delta (b_m gx + c_m gy),
// delta = 2 (Gc/c_w) ell |T| (diffusion part, fem.py:272-273).
template <int PAT, int T, int A, int B, int C>
__device__ __forceinline__ void elem_kaa(const Geo2& g, int j, double hx, double kap, double kc,
                                         const double (&X)[5], double (&Y)[5]) {
    const double del = 2.0 * kc * g.ell * area_at(g, j);
    double gx, gy;
    grad<PAT, T, A, B, C>(hx, ihy_at(g, j), X, gx, gy);
    grad_scatter<PAT, T, A, B, C>(hx, ihy_at(g, j), kap * ((X[A] + X[B]) + X[C]), del * gx, del * gy, Y);
}

template <int PAT>
__device__ __forceinline__ void put_kappa(const Geo2& g, const double* kappa, long long cell,
                                          const Slots& s, int q) {
#pragma unroll
    for (int k = 0; k < npc_of(PAT); ++k) put1(s, q + k, kappa, (long long)k * g.ncell + cell);
}
template <int PAT, int NE>
__device__ __forceinline__ void get_kappa(const Geo2& g, const Slots& s, int q, int off, double (&e)[NE]) {
#pragma unroll
    for (int k = 0; k < npc_of(PAT); ++k) e[off + k] = get1(s.sh((long long)k * g.ncell), q + k);
}
// v2: element slot k of the warp window's cell row through tensor map m
template <int PAT>
__device__ __forceinline__ void tput_kappa(const Geo2& g, const TmaIssue& t, int q, int m, long long cell) {
#pragma unroll
    for (int k = 0; k < npc_of(PAT); ++k) t.put1(q + k, m, (long long)k * g.ncell + cell);
}

// Kaa apply; MASKED: rows/cols of active vertices (act != 0) are replaced by identity (the
// reduced inactive-block operator J_NN of vi.py:235 embedded in full space).
// vertex slots: x|z, [p_in], [act word]; cell: Gc, kappa x npc, [centre x|z, p_in, act word]
// ec: [Gc, kappa x npc, (centre: x unmasked, active flag)]
// CHEB: the apply feeds one Chebyshev step instead of storing y (the C block of Newton's field
// split, pf_newton.cu cheb_C_dev): at each own vertex r -= (K d)_v ; d' = a d_v + b D^-1 r ;
// x += d' with d' written to a second buffer (the neighbours still read d); a, b = tab[2k-1], tab[2k].
struct KaaCheb {
    double *r, *dnext, *xacc;
    const double* dinv;
    const double* tab;
    int k;
};
template <bool FUSED, bool MASKED, bool CHEB = false>
struct OpKaa {
    static constexpr int NV = 1, NC = 1, MINB = 2;
    static constexpr int VS = 1 + (FUSED ? 1 : 0) + (MASKED ? 1 : 0);  // vertex slots
    static constexpr int pd(int pat) { return pat == PF_CROSSED ? 4 : 6; }
    static constexpr int ne(int pat) { return 1 + npc_of(pat) + 2 * crossed(pat); }
    static constexpr int sv(int) { return VS; }
    static constexpr int sc(int pat) { return 1 + npc_of(pat) + crossed(pat) * VS; }
    const double* kappa;
    const double* x;     // fused: z
    const double* pin;
    double* pout;
    double* y;
    const unsigned char* act;
    double* scal;
    RedBuf rb;
    double acc;
    double breg = 0.0;  // persistent PCG (k_pcg_kaa): beta held in a register instead of scal[S_BETA]
    int use_breg = 0;
    KaaCheb ch{};
    double ca = 0.0, cb = 0.0;
    __device__ bool enter() {
        if constexpr (CHEB) {
            ca = ch.tab[2 * ch.k - 1];
            cb = ch.tab[2 * ch.k];
        }
        if (!FUSED) return true;
        return scal[S_DONE] == 0.0 && scal[S_FAIL] == 0.0;
    }
    __device__ __forceinline__ void store_y(long long id, double dv, double yy) const {
        if constexpr (CHEB) {
            const double ri = ch.r[id] - yy;
            const double dn = ca * dv + cb * ch.dinv[id] * ri;
            ch.r[id] = ri;
            ch.dnext[id] = dn;
            ch.xacc[id] += dn;
        } else {
            y[id] = yy;
        }
    }
    __device__ __forceinline__ double xval(long long v) const {
        double z = __ldg(x + v);
        if (FUSED) {
            const double b = use_breg ? breg : (scal[S_ITER] > 0.0 ? scal[S_BETA] : 0.0);
            z = z + b * __ldg(pin + v);
        }
        return z;
    }
    __device__ __forceinline__ bool is_act(long long v) const { return MASKED && act[v] != 0; }
    __device__ __forceinline__ void stage_vertex(const Slots& s, long long v) const {
        put1(s, 0, x, v);
        if (FUSED) put1(s, 1, pin, v);
        if (MASKED) putb(s, FUSED ? 2 : 1, act, v);
    }
    // (value, active) from a staged vertex
    __device__ __forceinline__ double staged(const Slots& s, long long v, bool& a) const {
        double z = get1(s, 0);
        if (FUSED) {
            const double b = use_breg ? breg : (scal[S_ITER] > 0.0 ? scal[S_BETA] : 0.0);
            z = z + b * get1(s, 1);
        }
        a = MASKED ? (getb(s, FUSED ? 2 : 1, v) != 0u) : false;
        return z;
    }
    __device__ void issue_v(const Geo2& g, int i, int j, const Slots& s) const { stage_vertex(s, vid(g, i, j)); }
    // v2 engine: tensor maps MX = x|z, MP = p_in, MACT = active bytes, MGC = Gc per cell, MK = kappa
    enum { MX = 0, MP = 1, MACT = 2, MGC = 3, MK = 4 };
    static constexpr bool V2 = true;
    static constexpr int pd2(int pat) { return pat == PF_CROSSED ? 3 : 4; }
    void maps(const Geo2& g, MapBuilder& mb) const {
        mb.f1(MX, x, g.nv);
        if (FUSED) mb.f1(MP, pin, g.nv);
        if (MASKED) mb.u8(MACT, act, g.nv);
        if (g.Gc_cell) mb.f1(MGC, g.Gc_cell, g.ncell);
        mb.f1(MK, kappa, (long long)g.npc * g.ncell);
    }
    __device__ __forceinline__ void tstage_vertex(const TmaIssue& t, long long v) const {
        t.put1(0, MX, v);
        if (FUSED) t.put1(1, MP, v);
        if (MASKED) t.putb(FUSED ? 2 : 1, MACT, v);
    }
    __device__ void tissue_v(const Geo2& g, int i, int j0, const TmaIssue& t) const { tstage_vertex(t, vid(g, i, j0)); }
    template <int PAT>
    __device__ void tissue_c(const Geo2& g, int ci, int j0, const TmaIssue& t) const {
        const long long cell = cid(g, ci, j0);
        if (g.Gc_cell) t.put1(0, MGC, cell);
        tput_kappa<PAT>(g, t, 1, MK, cell);
        if constexpr (PAT == PF_CROSSED) tstage_vertex(t.at(1 + npc_of(PAT)), ctr(g, ci, j0));
    }
    template <bool BND = true>
    __device__ void fix_v(const Geo2& g, int i, int j, const Slots& s, double (&v)[NV]) const {
        bool a;
        const double z = staged(s, vid(g, i, j), a);
        v[0] = a ? 0.0 : z;
    }
    template <int PAT>
    __device__ void issue_c(const Geo2& g, int ci, int j, const Slots& s) const {
        const long long cell = cid(g, ci, j);
        putGc(g, s, 0, cell);
        put_kappa<PAT>(g, kappa, cell, s, 1);
        if constexpr (PAT == PF_CROSSED) stage_vertex(s.at(1 + npc_of(PAT)), ctr(g, ci, j));
    }
    template <int PAT, int NE>
    __device__ void fix_c(const Geo2& g, int ci, int j, const Slots& s, double (&e)[NE]) const {
        e[0] = getGc(g, s, 0);
        get_kappa<PAT>(g, s, 1, 1, e);
        if constexpr (PAT == PF_CROSSED) {
            bool a;
            e[5] = staged(s.at(1 + npc_of(PAT)).sh(g.nc), ctr(g, ci, j), a);
            e[6] = a ? 1.0 : 0.0;
        }
    }
    template <int PAT, int NE, int PARH = -1>
    __device__ void cell(const Geo2& g, int ci, int j, const double (&vc)[NV], const double (&vn)[NV],
                         const double (&rc)[NV], const double (&rn)[NV], const double (&ec)[NE],
                         double (&c00)[NC], double (&c10)[NC], double (&c01)[NC], double (&c11)[NC],
                         bool own) {
        if constexpr (PAT == PF_UNION_JACK || PAT == PF_RIGHT) {
            // edge form (see OpKuu::cell): slot 0 is the triangle on the bottom cell edge, slot 1
            // the one on the top edge, in both diagonal orientations
            // right: always the even split; PARH >= 0: the parity is a compile-time constant
            const bool odd = PAT == PF_UNION_JACK && (PARH >= 0 ? PARH != 0 : ((ci + j) & 1) != 0);
            const double ihx = g.ihx, ihy = ihy_at(g, j);
            const double del = 2.0 * (ec[0] / g.cw) * g.ell * area_at(g, j);
            const double x00 = vc[0], x10 = vn[0], x01 = rc[0], x11 = rn[0];
            const double bx = x10 - x00, tx = x11 - x01, ly = x01 - x00, ry = x11 - x10;
            const double bb = ec[1] * ((x00 + x10) + (odd ? x01 : x11));  // reaction, bottom triangle
            const double bt = ec[2] * (((odd ? x10 : x00) + x11) + x01);   // reaction, top triangle
            const double fbx = del * bx * ihx * ihx, ftx = del * tx * ihx * ihx;
            const double fby = del * (odd ? ly : ry) * ihy * ihy, fty = del * (odd ? ry : ly) * ihy * ihy;
            const double fr = odd ? fty : fby, fl = odd ? fby : fty;
            c00[0] = bb + (odd ? 0.0 : bt) - fbx - fl;
            c10[0] = bb + (odd ? bt : 0.0) + fbx - fr;
            c01[0] = bt + (odd ? bb : 0.0) - ftx + fl;
            c11[0] = bt + (odd ? 0.0 : bb) + ftx + fr;
            return;
        }
        double X[5] = {vc[0], vn[0], rc[0], rn[0], 0.0};
        if constexpr (PAT == PF_CROSSED) X[4] = ec[6] != 0.0 ? 0.0 : ec[5];
        double Y[5] = {0, 0, 0, 0, 0};
        const int par = (PAT == PF_UNION_JACK) ? (PARH >= 0 ? PARH : ((ci + j) & 1)) : 0;
        const double hxs = par ? -g.ihx : g.ihx;
        mirror<PAT>(par, X);
        const double kc = ec[0] / g.cw;
        for_each_elem<PAT>(par, [&](auto T, auto S, auto A, auto B, auto C) {
            elem_kaa<PAT, T.v, A.v, B.v, C.v>(g, j, hxs, ec[1 + S.v], kc, X, Y);
        });
        mirror<PAT>(par, Y);
        c00[0] = Y[0]; c10[0] = Y[1]; c01[0] = Y[2]; c11[0] = Y[3];
        if constexpr (PAT == PF_CROSSED) {
            if (own) {
                const long long cv = ctr(g, ci, j);
                const double xc = ec[5];
                const double yy = ec[6] != 0.0 ? xc : Y[4];
                store_y(cv, xc, yy);
                if (FUSED) { pout[cv] = xc; acc += xc * yy; }
            }
        }
    }
    template <bool BND = true>
    __device__ void out(const Geo2& g, int i, int j, const double (&t)[NC], const double (&v)[NV]) {
        const long long id = vid(g, i, j);
        double yy = t[0], p = v[0];
        if (is_act(id)) { p = xval(id); yy = p; }
        store_y(id, p, yy);
        if (FUSED) { pout[id] = p; acc += p * yy; }
    }
    __device__ void finish() {
        if (!FUSED) return;
        double v[1] = {acc};
        double* s = scal;
        grid_reduce<1>(v, rb, 0, [s](double* tot) {
            s[S_PAP] = tot[0];
            if (!(tot[0] > 0.0)) s[S_FAIL] = 1.0;
            else s[S_GAMMA] = s[S_RZ] / tot[0];
        });
    }
};

// diag(Kaa) (masked: active rows 1).  cell: Gc, kappa x npc
template <bool MASKED>
struct OpKaaDiag : NoRed {
    static constexpr int NV = 1, NC = 1;
    static constexpr int pd(int) { return 4; }
    static constexpr int ne(int pat) { return 1 + npc_of(pat); }
    static constexpr int sv(int) { return 0; }
    static constexpr int sc(int pat) { return 1 + npc_of(pat); }
    const double* kappa;
    double* dinv;
    const unsigned char* act;
    __device__ void issue_v(const Geo2&, int, int, const Slots&) const {}
    template <bool BND = true>
    __device__ void fix_v(const Geo2&, int, int, const Slots&, double (&v)[NV]) const { v[0] = 0.0; }
    template <int PAT>
    __device__ void issue_c(const Geo2& g, int ci, int j, const Slots& s) const {
        const long long cell = cid(g, ci, j);
        putGc(g, s, 0, cell);
        put_kappa<PAT>(g, kappa, cell, s, 1);
    }
    template <int PAT, int NE>
    __device__ void fix_c(const Geo2& g, int, int, const Slots& s, double (&e)[NE]) const {
        e[0] = getGc(g, s, 0);
        get_kappa<PAT>(g, s, 1, 1, e);
    }
    template <int PAT, int NE, int PARH = -1>
    __device__ void cell(const Geo2& g, int ci, int j, const double (&)[NV], const double (&)[NV],
                         const double (&)[NV], const double (&)[NV], const double (&ec)[NE],
                         double (&c00)[NC], double (&c10)[NC], double (&c01)[NC], double (&c11)[NC],
                         bool own) {
        double Y[5] = {0, 0, 0, 0, 0};
        const int par = (PAT == PF_UNION_JACK) ? (PARH >= 0 ? PARH : ((ci + j) & 1)) : 0;
        const double kc = ec[0] / g.cw;
        for_each_elem<PAT>(par, [&](auto T, auto S, auto A, auto B, auto C) {
            const double kap = ec[1 + S.v];
            const double del = 2.0 * kc * g.ell * area_at(g, j);
            using Sh = Shp<PAT, T.v>;
            const double X2 = g.ihx * g.ihx, Y2h = ihy_at(g, j) * ihy_at(g, j);
            Y[A.v] += kap + del * (double(Sh::b0 * Sh::b0) * X2 + double(Sh::c0 * Sh::c0) * Y2h);
            Y[B.v] += kap + del * (double(Sh::b1 * Sh::b1) * X2 + double(Sh::c1 * Sh::c1) * Y2h);
            Y[C.v] += kap + del * (double(Sh::b2 * Sh::b2) * X2 + double(Sh::c2 * Sh::c2) * Y2h);
        });
        mirror<PAT>(par, Y);
        c00[0] = Y[0]; c10[0] = Y[1]; c01[0] = Y[2]; c11[0] = Y[3];
        if constexpr (PAT == PF_CROSSED) {
            if (own) {
                const long long cv = ctr(g, ci, j);
                dinv[cv] = (MASKED && act[cv]) ? 1.0 : 1.0 / Y[4];
            }
        }
    }
    template <bool BND = true>
    __device__ void out(const Geo2& g, int i, int j, const double (&t)[NC], const double (&)[NV]) {
        const long long id = vid(g, i, j);
        dinv[id] = (MASKED && act[id]) ? 1.0 : 1.0 / t[0];
    }
};

// ================================================================================================
// Line-search trial of the damage VI (vi.py:209-220): trial = clip(x + mu d, lb, 1)
// (d == null -> trial = x), F = Kaa trial + c, Phi = fb(trial - lb, fb(1 - trial, -F)),
// merit = |Phi|^2 reduced into scal[merit_slot].
// vertex slots: x, d, lb; cell: Gc, kappa x npc, [centre x, d, lb]
// ================================================================================================
struct OpKaaTrial {
    static constexpr int NV = 1, NC = 1, MINB = 2;
    static constexpr int pd(int) { return 4; }
    static constexpr int ne(int pat) { return 1 + npc_of(pat) + crossed(pat); }
    static constexpr int sv(int) { return 3; }
    static constexpr int sc(int pat) { return 1 + npc_of(pat) + 3 * crossed(pat); }
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
    __device__ __forceinline__ void stage_vertex(const Slots& s, long long v) const {
        put1(s, 0, x, v);
        if (d) { put1(s, 1, d, v); put1(s, 2, lb, v); }
    }
    __device__ __forceinline__ double staged(const Slots& s) const {
        const double xv = get1(s, 0);
        if (!d) return xv;
        return fmin(fmax(xv + scal[S_MU] * get1(s, 1), get1(s, 2)), 1.0);
    }
    __device__ void issue_v(const Geo2& g, int i, int j, const Slots& s) const { stage_vertex(s, vid(g, i, j)); }
    // v2 engine: tensor maps MX = x, MD = d, ML = lb, MGC = Gc per cell, MK = kappa
    enum { MX = 0, MD = 1, ML = 2, MGC = 3, MK = 4 };
    static constexpr bool V2 = true;
    static constexpr int pd2(int pat) { return pat == PF_CROSSED ? 3 : 4; }
    void maps(const Geo2& g, MapBuilder& mb) const {
        mb.f1(MX, x, g.nv);
        if (d) { mb.f1(MD, d, g.nv); mb.f1(ML, lb, g.nv); }
        if (g.Gc_cell) mb.f1(MGC, g.Gc_cell, g.ncell);
        mb.f1(MK, kappa, (long long)g.npc * g.ncell);
    }
    __device__ __forceinline__ void tstage_vertex(const TmaIssue& t, long long v) const {
        t.put1(0, MX, v);
        if (d) { t.put1(1, MD, v); t.put1(2, ML, v); }
    }
    __device__ void tissue_v(const Geo2& g, int i, int j0, const TmaIssue& t) const { tstage_vertex(t, vid(g, i, j0)); }
    template <int PAT>
    __device__ void tissue_c(const Geo2& g, int ci, int j0, const TmaIssue& t) const {
        const long long cell = cid(g, ci, j0);
        if (g.Gc_cell) t.put1(0, MGC, cell);
        tput_kappa<PAT>(g, t, 1, MK, cell);
        if constexpr (PAT == PF_CROSSED) tstage_vertex(t.at(1 + npc_of(PAT)), ctr(g, ci, j0));
    }
    template <bool BND = true>
    __device__ void fix_v(const Geo2&, int, int, const Slots& s, double (&v)[NV]) const { v[0] = staged(s); }
    template <int PAT>
    __device__ void issue_c(const Geo2& g, int ci, int j, const Slots& s) const {
        const long long cell = cid(g, ci, j);
        putGc(g, s, 0, cell);
        put_kappa<PAT>(g, kappa, cell, s, 1);
        if constexpr (PAT == PF_CROSSED) stage_vertex(s.at(1 + npc_of(PAT)), ctr(g, ci, j));
    }
    template <int PAT, int NE>
    __device__ void fix_c(const Geo2& g, int, int, const Slots& s, double (&e)[NE]) const {
        e[0] = getGc(g, s, 0);
        get_kappa<PAT>(g, s, 1, 1, e);
        if constexpr (PAT == PF_CROSSED) e[5] = staged(s.at(1 + npc_of(PAT)).sh(g.nc));
    }
    __device__ __forceinline__ void finish_vertex(long long id, double tv, double Fv) {
        const double l = __ldg(lb + id);
        trial[id] = tv;
        F[id] = Fv;
        const double ph = fbphi(tv - l, fbphi(1.0 - tv, -Fv));
        acc_m += ph * ph;
    }
    template <int PAT, int NE, int PARH = -1>
    __device__ void cell(const Geo2& g, int ci, int j, const double (&vc)[NV], const double (&vn)[NV],
                         const double (&rc)[NV], const double (&rn)[NV], const double (&ec)[NE],
                         double (&c00)[NC], double (&c10)[NC], double (&c01)[NC], double (&c11)[NC],
                         bool own) {
        double X[5] = {vc[0], vn[0], rc[0], rn[0], 0.0};
        if constexpr (PAT == PF_CROSSED) X[4] = ec[5];
        double Y[5] = {0, 0, 0, 0, 0};
        const int par = (PAT == PF_UNION_JACK) ? (PARH >= 0 ? PARH : ((ci + j) & 1)) : 0;
        const double hxs = par ? -g.ihx : g.ihx;
        mirror<PAT>(par, X);
        const double kc = ec[0] / g.cw;
        for_each_elem<PAT>(par, [&](auto T, auto S, auto A, auto B, auto C) {
            elem_kaa<PAT, T.v, A.v, B.v, C.v>(g, j, hxs, ec[1 + S.v], kc, X, Y);
        });
        mirror<PAT>(par, Y);
        c00[0] = Y[0]; c10[0] = Y[1]; c01[0] = Y[2]; c11[0] = Y[3];
        if constexpr (PAT == PF_CROSSED) {
            if (own) {
                const long long cv = ctr(g, ci, j);
                finish_vertex(cv, X[4], Y[4] + __ldg(cvec + cv));
            }
        }
    }
    template <bool BND = true>
    __device__ void out(const Geo2& g, int i, int j, const double (&t)[NC], const double (&v)[NV]) {
        const long long id = vid(g, i, j);
        finish_vertex(id, v[0], t[0] + __ldg(cvec + id));
    }
    __device__ void finish() {
        double v[1] = {acc_m};
        double* s = scal;
        const int ms = merit_slot;
        grid_reduce<1>(v, rb, 1, [s, ms](double* tot) { s[ms] = tot[0]; });
    }
};

// ================================================================================================
// Physics pass: energies (fem.py:162-174), r_u (fem.py:177-189), r_alpha (fem.py:202-218) and
// the FB optimality residual (solver.py:104-118).  rows: PF_ROWS_RAW / ZERO / VALUE.
// Reductions -> scal[S_PHYS0 ..]: E_el, E_d, |r_u|^2, |Phi|^2.
// vertex slots: u, alpha; cell: E, Gc, [u_c, alpha_c]
// ================================================================================================
template <int ROWS, bool RELAX = false>
struct OpPhys {
    static constexpr int NV = 3, NC = 3, MINB = RELAX ? 1 : 2;
    static constexpr int pd(int) { return 3; }
    static constexpr int ne(int pat) { return 2 + 3 * crossed(pat); }
    static constexpr int sv(int) { return RELAX ? 5 : 3; }
    static constexpr int sc(int pat) { return 2 + crossed(pat) * (RELAX ? 5 : 3); }
    const double* u;
    const double* alpha;   // RELAX: alpha_prev
    const double* lb;
    double* ru;
    double* ra;
    double* phi;
    double* scal;
    RedBuf rb;
    double eel, ed, nru, nphi;
    // RELAX (north_star part 4): alpha = P[alpha_prev + w_bar (alpha* - alpha_prev)] formed while
    // staging, written at owned vertices; |alpha - alpha_prev|_inf max-reduced into bits[1]
    const double* astar = nullptr;
    double* aout = nullptr;
    double omega = 1.0;
    unsigned long long* bits = nullptr;
    double wb = 1.0, dmax = 0.0;
    int kk = 0;
    bool star = true;
    __device__ bool enter() {
        if constexpr (RELAX) choose_omega(omega, bits[0], wb, kk, star);
        return true;
    }
    __device__ __forceinline__ double relaxed(double a0, double as, double l) const {  // k_relax_apply
        const double cand = star ? as : a0 + wb * (as - a0);
        return fmin(fmax(cand, l), 1.0);
    }
    __device__ void issue_v(const Geo2& g, int i, int j, const Slots& s) const {
        const long long id = vid(g, i, j);
        put2(s, 0, u, id);
        put1(s, 2, alpha, id);
        if (RELAX) { put1(s, 3, astar, id); put1(s, 4, lb, id); }
    }
    // (not on the v2 engine: measured no gain -- the pass is bound by its fp64 work (hypot, energies)
    // and two columns per lane cost 166 registers: 8192^2 union-jack 2.15 vs 2.23 ms, 2048^2 0.249 vs
    // 0.203 ms)
    template <bool BND = true>
    __device__ void fix_v(const Geo2&, int, int, const Slots& s, double (&v)[NV]) const {
        const double2 uv = get2(s, 0);
        v[0] = uv.x; v[1] = uv.y;
        v[2] = RELAX ? relaxed(get1(s, 2), get1(s, 3), get1(s, 4)) : get1(s, 2);
    }
    template <int PAT>
    __device__ void issue_c(const Geo2& g, int ci, int j, const Slots& s) const {
        const long long cell = cid(g, ci, j);
        putE(g, s, 0, cell);
        putGc(g, s, 1, cell);
        if constexpr (PAT == PF_CROSSED) {
            const long long cv = ctr(g, ci, j);
            put2(s, 2, u, cv);
            put1(s, 4, alpha, cv);
            if (RELAX) { put1(s, 5, astar, cv); put1(s, 6, lb, cv); }
        }
    }
    template <int PAT, int NE>
    __device__ void fix_c(const Geo2& g, int, int, const Slots& s, double (&e)[NE]) const {
        e[0] = getE(g, s, 0);
        e[1] = getGc(g, s, 1);
        if constexpr (PAT == PF_CROSSED) {
            const Slots c = s.sh(g.nc);
            const double2 uv = get2(c, 2);
            e[2] = uv.x; e[3] = uv.y;
            e[4] = RELAX ? relaxed(get1(c, 4), get1(c, 5), get1(c, 6)) : get1(c, 4);
        }
    }
    __device__ __forceinline__ void vertex_out(const Geo2& g, long long id, unsigned m, double r0,
                                               double r1, double rav, double av) {
        if (m) {
            if (ROWS == PF_ROWS_ZERO) {
                if (m & 1u) r0 = 0.0;
                if (m & 2u) r1 = 0.0;
            } else if (ROWS == PF_ROWS_VALUE) {
                const double2 uv = ld2(u, id);
                const double2 ub = ld2(g.ubar, id);
                if (m & 1u) r0 = uv.x - ub.x;
                if (m & 2u) r1 = uv.y - ub.y;
            }
        }
        if (ru) st2(ru, id, r0, r1);
        if (ra) ra[id] = rav;
        if (RELAX) {
            aout[id] = av;
            dmax = fmax(dmax, fabs(av - __ldg(alpha + id)));
        }
        nru += r0 * r0 + r1 * r1;
        if (lb) {
            const double ph = fbphi(av - __ldg(lb + id), fbphi(1.0 - av, -rav));
            if (phi) phi[id] = ph;
            nphi += ph * ph;
        }
    }
    template <int PAT, int NE, int PARH = -1>
    __device__ void cell(const Geo2& g, int ci, int j, const double (&vc)[NV], const double (&vn)[NV],
                         const double (&rc)[NV], const double (&rn)[NV], const double (&ec)[NE],
                         double (&c00)[NC], double (&c10)[NC], double (&c01)[NC], double (&c11)[NC],
                         bool own) {
        double U1[5] = {vc[0], vn[0], rc[0], rn[0], 0.0};
        double U2[5] = {vc[1], vn[1], rc[1], rn[1], 0.0};
        double Al[5] = {vc[2], vn[2], rc[2], rn[2], 0.0};
        if constexpr (PAT == PF_CROSSED) { U1[4] = ec[2]; U2[4] = ec[3]; Al[4] = ec[4]; }
        double Y1[5] = {0, 0, 0, 0, 0}, Y2[5] = {0, 0, 0, 0, 0}, Ya[5] = {0, 0, 0, 0, 0};
        const int par = (PAT == PF_UNION_JACK) ? (PARH >= 0 ? PARH : ((ci + j) & 1)) : 0;
        const double hxs = par ? -g.ihx : g.ihx;
        mirror<PAT>(par, U1);
        mirror<PAT>(par, U2);
        mirror<PAT>(par, Al);
        const double Ec = ec[0];
        const double kc = ec[1] / g.cw;
        for_each_elem<PAT>(par, [&](auto T, auto, auto A, auto B, auto C) {
            const double ab = (Al[A.v] + Al[B.v] + Al[C.v]) * (1.0 / 3.0);
            const double om = 1.0 - ab;
            const double a = om * om + g.kell, ap = -2.0 * om;
            const double w = g.at2 ? ab * ab : ab, wp = g.at2 ? 2.0 * ab : 1.0;
            const double ar = area_at(g, j);
            double e0, e1, e2, s0, s1, s2;
            strain<PAT, T.v, A.v, B.v, C.v>(hxs, ihy_at(g, j), U1, U2, e0, e1, e2);
            if (g.eps0) {
                const double e = __ldg(g.eps0 + (long long)(T.v + 2 * par) * g.ny + j);
                e0 -= e; e1 -= e;
            }
            unit_stress(g, e0, e1, e2, s0, s1, s2);
            const double q = Ec * (e0 * s0 + e1 * s1 + e2 * s2);
            const double s = a * ar * Ec;
            scatter_BT<PAT, T.v, A.v, B.v, C.v>(hxs, ihy_at(g, j), s * s0, s * s1, s * s2, Y1, Y2);
            double gx, gy;
            grad<PAT, T.v, A.v, B.v, C.v>(hxs, ihy_at(g, j), Al, gx, gy);
            const double nod = (0.5 * ap * q + kc * wp / g.ell) * ar * (1.0 / 3.0);
            const double del = 2.0 * kc * g.ell * ar;
            grad_scatter<PAT, T.v, A.v, B.v, C.v>(hxs, ihy_at(g, j), nod, del * gx, del * gy, Ya);
            if (own) {
                eel += 0.5 * ar * a * q;
                ed += ar * kc * (w / g.ell + g.ell * (gx * gx + gy * gy));
            }
        });
        mirror<PAT>(par, Y1);
        mirror<PAT>(par, Y2);
        mirror<PAT>(par, Ya);
        c00[0] = Y1[0]; c00[1] = Y2[0]; c00[2] = Ya[0];
        c10[0] = Y1[1]; c10[1] = Y2[1]; c10[2] = Ya[1];
        c01[0] = Y1[2]; c01[1] = Y2[2]; c01[2] = Ya[2];
        c11[0] = Y1[3]; c11[1] = Y2[3]; c11[2] = Ya[3];
        if constexpr (PAT == PF_CROSSED) {
            if (own) vertex_out(g, ctr(g, ci, j), 0u, Y1[4], Y2[4], Ya[4], Al[4]);
        }
    }
    template <bool BND = true>
    __device__ void out(const Geo2& g, int i, int j, const double (&t)[NC], const double (&v)[NV]) {
        const long long id = vid(g, i, j);
        vertex_out(g, id, bcbits(g, i, j, id), t[0], t[1], t[2], v[2]);
    }
    __device__ void finish() {
        if constexpr (RELAX) {
            double dm = dmax;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) dm = fmax(dm, __shfl_xor_sync(PF_FULL, dm, o));
            if ((threadIdx.x & 31) == 0 && dm > 0.0)
                atomicMax(bits + 1, (unsigned long long)__double_as_longlong(dm));
            if (blockIdx.x == 0 && threadIdx.x == 0) {
                scal[S_OMEGABAR] = wb;
                scal[S_AUX1] = (double)kk;
            }
        }
        double v[4] = {eel, ed, nru, nphi};
        double* s = scal;
        grid_reduce<4>(v, rb, 2, [s](double* tot) {
            s[S_PHYS0 + 0] = tot[0];
            s[S_PHYS0 + 1] = tot[1];
            s[S_PHYS0 + 2] = tot[2];
            s[S_PHYS0 + 3] = tot[3];
        });
    }
};

// ================================================================================================
// Elastic right-hand side with symmetric Dirichlet elimination (fem.py:192-199, 297-310):
// b = M (f - K g) + (I - M) ubar = -M r_raw(g) + (I - M) ubar, g = ubar on constrained dofs.
// With LOADONLY the output is f itself (assemble_load_u).  Reduces |b|^2 into scal[S_AUX0].
// vertex slots: alpha; cell: E, [alpha_c]
// ================================================================================================
template <bool LOADONLY>
struct OpRhs {
    static constexpr int NV = 3, NC = 2, MINB = 2;
    static constexpr int pd(int) { return 4; }
    static constexpr int ne(int pat) { return 1 + crossed(pat); }
    static constexpr int sv(int) { return 1; }
    static constexpr int sc(int pat) { return 1 + crossed(pat); }
    const double* alpha;
    double* b;
    double* scal;
    RedBuf rb;
    double acc;
    __device__ bool enter() const { return true; }
    __device__ void issue_v(const Geo2& g, int i, int j, const Slots& s) const { put1(s, 0, alpha, vid(g, i, j)); }
    template <bool BND = true>
    __device__ void fix_v(const Geo2& g, int i, int j, const Slots& s, double (&v)[NV]) const {
        const long long id = vid(g, i, j);
        v[0] = 0.0; v[1] = 0.0;
        if (!LOADONLY) {
            const unsigned m = bcbits(g, i, j, id);
            if (m) {
                const double2 ub = ld2(g.ubar, id);
                if (m & 1u) v[0] = ub.x;
                if (m & 2u) v[1] = ub.y;
            }
        }
        v[2] = get1(s, 0);
    }
    template <int PAT>
    __device__ void issue_c(const Geo2& g, int ci, int j, const Slots& s) const {
        putE(g, s, 0, cid(g, ci, j));
        if constexpr (PAT == PF_CROSSED) put1(s, 1, alpha, ctr(g, ci, j));
    }
    template <int PAT, int NE>
    __device__ void fix_c(const Geo2& g, int, int, const Slots& s, double (&e)[NE]) const {
        e[0] = getE(g, s, 0);
        if constexpr (PAT == PF_CROSSED) e[1] = get1(s, 1);
    }
    template <int PAT, int NE, int PARH = -1>
    __device__ void cell(const Geo2& g, int ci, int j, const double (&vc)[NV], const double (&vn)[NV],
                         const double (&rc)[NV], const double (&rn)[NV], const double (&ec)[NE],
                         double (&c00)[NC], double (&c10)[NC], double (&c01)[NC], double (&c11)[NC],
                         bool own) {
        double U1[5] = {vc[0], vn[0], rc[0], rn[0], 0.0};
        double U2[5] = {vc[1], vn[1], rc[1], rn[1], 0.0};
        double Al[5] = {vc[2], vn[2], rc[2], rn[2], 0.0};
        if constexpr (PAT == PF_CROSSED) Al[4] = ec[1];
        double Y1[5] = {0, 0, 0, 0, 0}, Y2[5] = {0, 0, 0, 0, 0};
        const int par = (PAT == PF_UNION_JACK) ? (PARH >= 0 ? PARH : ((ci + j) & 1)) : 0;
        const double hxs = par ? -g.ihx : g.ihx;
        mirror<PAT>(par, U1);
        mirror<PAT>(par, U2);
        mirror<PAT>(par, Al);
        const double Ec = ec[0];
        for_each_elem<PAT>(par, [&](auto T, auto, auto A, auto B, auto C) {
            const double ab = (Al[A.v] + Al[B.v] + Al[C.v]) * (1.0 / 3.0);
            const double om = 1.0 - ab;
            const double s = (om * om + g.kell) * area_at(g, j) * Ec;
            double e0 = 0.0, e1 = 0.0, e2 = 0.0, s0, s1, s2;
            if (!LOADONLY) strain<PAT, T.v, A.v, B.v, C.v>(hxs, ihy_at(g, j), U1, U2, e0, e1, e2);
            if (g.eps0) {
                const double e = __ldg(g.eps0 + (long long)(T.v + 2 * par) * g.ny + j);
                e0 -= e; e1 -= e;
            }
            unit_stress(g, e0, e1, e2, s0, s1, s2);
            // r_raw = K g - f  ->  B^T s D (Bg - eps0)
            scatter_BT<PAT, T.v, A.v, B.v, C.v>(hxs, ihy_at(g, j), s * s0, s * s1, s * s2, Y1, Y2);
        });
        mirror<PAT>(par, Y1);
        mirror<PAT>(par, Y2);
        c00[0] = Y1[0]; c00[1] = Y2[0]; c10[0] = Y1[1]; c10[1] = Y2[1];
        c01[0] = Y1[2]; c01[1] = Y2[2]; c11[0] = Y1[3]; c11[1] = Y2[3];
        if constexpr (PAT == PF_CROSSED) {
            if (own) {
                const double b0 = -Y1[4], b1 = -Y2[4];
                st2(b, ctr(g, ci, j), b0, b1);
                acc += b0 * b0 + b1 * b1;
            }
        }
    }
    template <bool BND = true>
    __device__ void out(const Geo2& g, int i, int j, const double (&t)[NC], const double (&v)[NV]) {
        const long long id = vid(g, i, j);
        double b0 = -t[0], b1 = -t[1];
        if (!LOADONLY) {
            const unsigned m = bcbits(g, i, j, id);
            if (m & 1u) b0 = v[0];
            if (m & 2u) b1 = v[1];
        }
        st2(b, id, b0, b1);
        acc += b0 * b0 + b1 * b1;
    }
    __device__ void finish() {
        double v[1] = {acc};
        double* s = scal;
        grid_reduce<1>(v, rb, 3, [s](double* tot) { s[S_AUX0] = tot[0]; });  // |b|^2
    }
};

// ================================================================================================
// Coupling blocks (fem.py:246-263): Kua column of element e = (a' |T| E / 3) B^T sigma for each of
// its 3 nodes, sigma = D (B u - eps0).  Kau = Kua^T.  bcmode eliminates Dirichlet rows of Kua
// (columns of Kau).
// ================================================================================================
template <int PAT, int T, int A, int B, int C>
__device__ __forceinline__ void coupling_vec(const Geo2& g, double hx, int et, const double (&U1)[5],
                                             const double (&U2)[5], const double (&Al)[5], double Ec,
                                             int j, double& sc, double& s0, double& s1, double& s2) {
    const double ab = (Al[A] + Al[B] + Al[C]) * (1.0 / 3.0);
    const double ap = -2.0 * (1.0 - ab);
    double e0, e1, e2;
    strain<PAT, T, A, B, C>(hx, ihy_at(g, j), U1, U2, e0, e1, e2);
    if (g.eps0) {
        const double e = __ldg(g.eps0 + (long long)et * g.ny + j);
        e0 -= e; e1 -= e;
    }
    unit_stress(g, e0, e1, e2, s0, s1, s2);
    sc = ap * area_at(g, j) * Ec * (1.0 / 3.0);
}

// vertex slots: u, alpha, xa; cell: E, [u, alpha, xa centre]
struct OpKua : NoRed {
    static constexpr int NV = 4, NC = 2;
    static constexpr int pd(int) { return 3; }
    static constexpr int ne(int pat) { return 1 + 4 * crossed(pat); }
    static constexpr int sv(int) { return 4; }
    static constexpr int sc(int pat) { return 1 + 4 * crossed(pat); }
    const double* u;
    const double* alpha;
    const double* xa;
    double* yu;
    int bcmode;
    __device__ __forceinline__ void stage_vertex(const Slots& s, long long v) const {
        put2(s, 0, u, v); put1(s, 2, alpha, v); put1(s, 3, xa, v);
    }
    __device__ __forceinline__ void staged(const Slots& s, double* v) const {
        const double2 uv = get2(s, 0);
        v[0] = uv.x; v[1] = uv.y; v[2] = get1(s, 2); v[3] = get1(s, 3);
    }
    __device__ void issue_v(const Geo2& g, int i, int j, const Slots& s) const { stage_vertex(s, vid(g, i, j)); }
    template <bool BND = true>
    __device__ void fix_v(const Geo2&, int, int, const Slots& s, double (&v)[NV]) const { staged(s, v); }
    template <int PAT>
    __device__ void issue_c(const Geo2& g, int ci, int j, const Slots& s) const {
        putE(g, s, 0, cid(g, ci, j));
        if constexpr (PAT == PF_CROSSED) stage_vertex(s.at(1), ctr(g, ci, j));
    }
    template <int PAT, int NE>
    __device__ void fix_c(const Geo2& g, int, int, const Slots& s, double (&e)[NE]) const {
        e[0] = getE(g, s, 0);
        if constexpr (PAT == PF_CROSSED) staged(s.at(1), e + 1);
    }
    template <int PAT, int NE, int PARH = -1>
    __device__ void cell(const Geo2& g, int ci, int j, const double (&vc)[NV], const double (&vn)[NV],
                         const double (&rc)[NV], const double (&rn)[NV], const double (&ec)[NE],
                         double (&c00)[NC], double (&c10)[NC], double (&c01)[NC], double (&c11)[NC],
                         bool own) {
        double U1[5] = {vc[0], vn[0], rc[0], rn[0], 0.0};
        double U2[5] = {vc[1], vn[1], rc[1], rn[1], 0.0};
        double Al[5] = {vc[2], vn[2], rc[2], rn[2], 0.0};
        double X[5] = {vc[3], vn[3], rc[3], rn[3], 0.0};
        if constexpr (PAT == PF_CROSSED) { U1[4] = ec[1]; U2[4] = ec[2]; Al[4] = ec[3]; X[4] = ec[4]; }
        double Y1[5] = {0, 0, 0, 0, 0}, Y2[5] = {0, 0, 0, 0, 0};
        const int par = (PAT == PF_UNION_JACK) ? (PARH >= 0 ? PARH : ((ci + j) & 1)) : 0;
        const double hxs = par ? -g.ihx : g.ihx;
        mirror<PAT>(par, U1);
        mirror<PAT>(par, U2);
        mirror<PAT>(par, Al);
        mirror<PAT>(par, X);
        const double Ec = ec[0];
        for_each_elem<PAT>(par, [&](auto T, auto, auto A, auto B, auto C) {
            double sc, s0, s1, s2;
            coupling_vec<PAT, T.v, A.v, B.v, C.v>(g, hxs, T.v + 2 * par, U1, U2, Al, Ec, j, sc, s0, s1, s2);
            const double f = sc * ((X[A.v] + X[B.v]) + X[C.v]);
            scatter_BT<PAT, T.v, A.v, B.v, C.v>(hxs, ihy_at(g, j), f * s0, f * s1, f * s2, Y1, Y2);
        });
        mirror<PAT>(par, Y1);
        mirror<PAT>(par, Y2);
        c00[0] = Y1[0]; c00[1] = Y2[0]; c10[0] = Y1[1]; c10[1] = Y2[1];
        c01[0] = Y1[2]; c01[1] = Y2[2]; c11[0] = Y1[3]; c11[1] = Y2[3];
        if constexpr (PAT == PF_CROSSED) {
            if (own) st2(yu, ctr(g, ci, j), Y1[4], Y2[4]);
        }
    }
    template <bool BND = true>
    __device__ void out(const Geo2& g, int i, int j, const double (&t)[NC], const double (&)[NV]) {
        const long long id = vid(g, i, j);
        const unsigned m = bcmode ? bcbits(g, i, j, id) : 0u;
        st2(yu, id, (m & 1u) ? 0.0 : t[0], (m & 2u) ? 0.0 : t[1]);
    }
};

// vertex slots: u, alpha, xu; cell: E, [u, alpha, xu centre]
struct OpKau : NoRed {
    static constexpr int NV = 5, NC = 1;
    static constexpr int pd(int) { return 3; }
    static constexpr int ne(int pat) { return 1 + 5 * crossed(pat); }
    static constexpr int sv(int) { return 5; }
    static constexpr int sc(int pat) { return 1 + 5 * crossed(pat); }
    const double* u;
    const double* alpha;
    const double* xu;
    double* ya;
    int bcmode;
    __device__ __forceinline__ void stage_vertex(const Slots& s, long long v) const {
        put2(s, 0, u, v); put1(s, 2, alpha, v); put2(s, 3, xu, v);
    }
    __device__ void issue_v(const Geo2& g, int i, int j, const Slots& s) const { stage_vertex(s, vid(g, i, j)); }
    template <bool BND = true>
    __device__ void fix_v(const Geo2& g, int i, int j, const Slots& s, double (&v)[NV]) const {
        const double2 uv = get2(s, 0);
        const double2 xv = get2(s, 3);
        const unsigned m = bcmode ? bcbits(g, i, j, vid(g, i, j)) : 0u;
        v[0] = uv.x; v[1] = uv.y; v[2] = get1(s, 2);
        v[3] = (m & 1u) ? 0.0 : xv.x;
        v[4] = (m & 2u) ? 0.0 : xv.y;
    }
    template <int PAT>
    __device__ void issue_c(const Geo2& g, int ci, int j, const Slots& s) const {
        putE(g, s, 0, cid(g, ci, j));
        if constexpr (PAT == PF_CROSSED) stage_vertex(s.at(1), ctr(g, ci, j));
    }
    template <int PAT, int NE>
    __device__ void fix_c(const Geo2& g, int, int, const Slots& s, double (&e)[NE]) const {
        e[0] = getE(g, s, 0);
        if constexpr (PAT == PF_CROSSED) {
            const Slots c = s.at(1);
            const double2 uv = get2(c, 0);
            const double2 xv = get2(c, 3);
            e[1] = uv.x; e[2] = uv.y; e[3] = get1(c, 2); e[4] = xv.x; e[5] = xv.y;
        }
    }
    template <int PAT, int NE, int PARH = -1>
    __device__ void cell(const Geo2& g, int ci, int j, const double (&vc)[NV], const double (&vn)[NV],
                         const double (&rc)[NV], const double (&rn)[NV], const double (&ec)[NE],
                         double (&c00)[NC], double (&c10)[NC], double (&c01)[NC], double (&c11)[NC],
                         bool own) {
        double U1[5] = {vc[0], vn[0], rc[0], rn[0], 0.0};
        double U2[5] = {vc[1], vn[1], rc[1], rn[1], 0.0};
        double Al[5] = {vc[2], vn[2], rc[2], rn[2], 0.0};
        double X1[5] = {vc[3], vn[3], rc[3], rn[3], 0.0};
        double X2[5] = {vc[4], vn[4], rc[4], rn[4], 0.0};
        if constexpr (PAT == PF_CROSSED) {
            U1[4] = ec[1]; U2[4] = ec[2]; Al[4] = ec[3]; X1[4] = ec[4]; X2[4] = ec[5];
        }
        double Y[5] = {0, 0, 0, 0, 0};
        const int par = (PAT == PF_UNION_JACK) ? (PARH >= 0 ? PARH : ((ci + j) & 1)) : 0;
        const double hxs = par ? -g.ihx : g.ihx;
        mirror<PAT>(par, U1);
        mirror<PAT>(par, U2);
        mirror<PAT>(par, Al);
        mirror<PAT>(par, X1);
        mirror<PAT>(par, X2);
        const double Ec = ec[0];
        for_each_elem<PAT>(par, [&](auto T, auto, auto A, auto B, auto C) {
            double sc, s0, s1, s2, d0, d1, d2;
            coupling_vec<PAT, T.v, A.v, B.v, C.v>(g, hxs, T.v + 2 * par, U1, U2, Al, Ec, j, sc, s0, s1, s2);
            strain<PAT, T.v, A.v, B.v, C.v>(hxs, ihy_at(g, j), X1, X2, d0, d1, d2);  // (B x)^T sigma
            const double f = sc * (d0 * s0 + d1 * s1 + d2 * s2);
            Y[A.v] += f; Y[B.v] += f; Y[C.v] += f;
        });
        mirror<PAT>(par, Y);
        c00[0] = Y[0]; c10[0] = Y[1]; c01[0] = Y[2]; c11[0] = Y[3];
        if constexpr (PAT == PF_CROSSED) {
            if (own) ya[ctr(g, ci, j)] = Y[4];
        }
    }
    template <bool BND = true>
    __device__ void out(const Geo2& g, int i, int j, const double (&t)[NC], const double (&)[NV]) {
        ya[vid(g, i, j)] = t[0];
    }
};

// ================================================================================================
// Newton: reduced coupled Jacobian [[Kuu_bc, Kua_bc], [Kau_bc, Kaa]] on the inactive set
// (solver.py:292-296 + vi.py:235 with index extraction replaced by masks): active damage rows /
// columns (act != 0) become identity.  One pass reads (u, alpha, x_u, x_a).
// vertex slots: u, alpha, xu, xa, [act word]; cell: E, Gc, [centre: same as vertex]
// ec: [E, Gc, (centre u1, u2, alpha, xu1, xu2, xa_masked, xa_raw, act)]
// ================================================================================================
struct OpJac : NoRed {
    static constexpr int NV = 6, NC = 3, MINB = 1;
    static constexpr int pd(int pat) { return pat == PF_CROSSED ? 2 : 3; }
    static constexpr int ne(int pat) { return 2 + 8 * crossed(pat); }
    static constexpr int sv(int) { return 7; }
    static constexpr int sc(int pat) { return 2 + 7 * crossed(pat); }
    const double* u;
    const double* alpha;
    const double* xu;
    const double* xa;
    double* yu;
    double* ya;
    const unsigned char* act;
    __device__ __forceinline__ void stage_vertex(const Slots& s, long long v) const {
        put2(s, 0, u, v); put1(s, 2, alpha, v); put2(s, 3, xu, v); put1(s, 5, xa, v);
        if (act) putb(s, 6, act, v);
    }
    __device__ void issue_v(const Geo2& g, int i, int j, const Slots& s) const { stage_vertex(s, vid(g, i, j)); }
    template <bool BND = true>
    __device__ void fix_v(const Geo2& g, int i, int j, const Slots& s, double (&v)[NV]) const {
        const long long id = vid(g, i, j);
        const double2 uv = get2(s, 0);
        const double2 xv = get2(s, 3);
        const unsigned m = bcbits(g, i, j, id);
        const bool a = act && getb(s, 6, id) != 0u;
        v[0] = uv.x; v[1] = uv.y; v[2] = get1(s, 2);
        v[3] = (m & 1u) ? 0.0 : xv.x;
        v[4] = (m & 2u) ? 0.0 : xv.y;
        v[5] = a ? 0.0 : get1(s, 5);
    }
    template <int PAT>
    __device__ void issue_c(const Geo2& g, int ci, int j, const Slots& s) const {
        const long long cell = cid(g, ci, j);
        putE(g, s, 0, cell);
        putGc(g, s, 1, cell);
        if constexpr (PAT == PF_CROSSED) stage_vertex(s.at(2), ctr(g, ci, j));
    }
    template <int PAT, int NE>
    __device__ void fix_c(const Geo2& g, int ci, int j, const Slots& s, double (&e)[NE]) const {
        e[0] = getE(g, s, 0);
        e[1] = getGc(g, s, 1);
        if constexpr (PAT == PF_CROSSED) {
            const Slots c = s.at(2);
            const long long cv = ctr(g, ci, j);
            const double2 uv = get2(c, 0);
            const double2 xv = get2(c, 3);
            const double xr = get1(c, 5);
            const bool a = act && getb(c, 6, cv) != 0u;
            e[2] = uv.x; e[3] = uv.y; e[4] = get1(c, 2); e[5] = xv.x; e[6] = xv.y;
            e[7] = a ? 0.0 : xr; e[8] = xr; e[9] = a ? 1.0 : 0.0;
        }
    }
    template <int PAT, int NE, int PARH = -1>
    __device__ void cell(const Geo2& g, int ci, int j, const double (&vc)[NV], const double (&vn)[NV],
                         const double (&rc)[NV], const double (&rn)[NV], const double (&ec)[NE],
                         double (&c00)[NC], double (&c10)[NC], double (&c01)[NC], double (&c11)[NC],
                         bool own) {
        double U1[5] = {vc[0], vn[0], rc[0], rn[0], 0.0};
        double U2[5] = {vc[1], vn[1], rc[1], rn[1], 0.0};
        double Al[5] = {vc[2], vn[2], rc[2], rn[2], 0.0};
        double X1[5] = {vc[3], vn[3], rc[3], rn[3], 0.0};
        double X2[5] = {vc[4], vn[4], rc[4], rn[4], 0.0};
        double Xa[5] = {vc[5], vn[5], rc[5], rn[5], 0.0};
        if constexpr (PAT == PF_CROSSED) {
            U1[4] = ec[2]; U2[4] = ec[3]; Al[4] = ec[4]; X1[4] = ec[5]; X2[4] = ec[6]; Xa[4] = ec[7];
        }
        double Y1[5] = {0, 0, 0, 0, 0}, Y2[5] = {0, 0, 0, 0, 0}, Ya[5] = {0, 0, 0, 0, 0};
        const int par = (PAT == PF_UNION_JACK) ? (PARH >= 0 ? PARH : ((ci + j) & 1)) : 0;
        const double hxs = par ? -g.ihx : g.ihx;
        mirror<PAT>(par, U1);
        mirror<PAT>(par, U2);
        mirror<PAT>(par, Al);
        mirror<PAT>(par, X1);
        mirror<PAT>(par, X2);
        mirror<PAT>(par, Xa);
        const double Ec = ec[0];
        const double kc = ec[1] / g.cw;
        for_each_elem<PAT>(par, [&](auto T, auto, auto A, auto B, auto C) {
            const double ab = (Al[A.v] + Al[B.v] + Al[C.v]) * (1.0 / 3.0);
            const double om = 1.0 - ab;
            const double a = om * om + g.kell, ap = -2.0 * om;
            const double ar = area_at(g, j);
            double e0, e1, e2, s0, s1, s2, d0, d1, d2, t0, t1, t2;
            strain<PAT, T.v, A.v, B.v, C.v>(hxs, ihy_at(g, j), U1, U2, e0, e1, e2);
            if (g.eps0) {
                const double e = __ldg(g.eps0 + (long long)(T.v + 2 * par) * g.ny + j);
                e0 -= e; e1 -= e;
            }
            unit_stress(g, e0, e1, e2, s0, s1, s2);          // sigma (unit E)
            strain<PAT, T.v, A.v, B.v, C.v>(hxs, ihy_at(g, j), X1, X2, d0, d1, d2);
            unit_stress(g, d0, d1, d2, t0, t1, t2);          // D B x_u
            const double q = Ec * (e0 * s0 + e1 * s1 + e2 * s2);
            const double sxa = (Xa[A.v] + Xa[B.v]) + Xa[C.v];
            const double cpl = ap * ar * Ec * (1.0 / 3.0);
            // u rows: a|T|E B^T D B x_u + cpl * sxa * B^T sigma
            const double ka = a * ar * Ec, kb = cpl * sxa;
            scatter_BT<PAT, T.v, A.v, B.v, C.v>(hxs, ihy_at(g, j), ka * t0 + kb * s0, ka * t1 + kb * s1,
                                                ka * t2 + kb * s2, Y1, Y2);
            // alpha rows: cpl * (B x_u)^T sigma + Kaa x_a
            const double kap = (q + (g.at2 ? 2.0 * kc / g.ell : 0.0)) * ar * (1.0 / 9.0);
            const double fa = cpl * (d0 * s0 + d1 * s1 + d2 * s2);
            double Yt[5] = {0, 0, 0, 0, 0};
            elem_kaa<PAT, T.v, A.v, B.v, C.v>(g, j, hxs, kap, kc, Xa, Yt);
            Ya[A.v] += fa + Yt[A.v];
            Ya[B.v] += fa + Yt[B.v];
            Ya[C.v] += fa + Yt[C.v];
        });
        mirror<PAT>(par, Y1);
        mirror<PAT>(par, Y2);
        mirror<PAT>(par, Ya);
        c00[0] = Y1[0]; c00[1] = Y2[0]; c00[2] = Ya[0];
        c10[0] = Y1[1]; c10[1] = Y2[1]; c10[2] = Ya[1];
        c01[0] = Y1[2]; c01[1] = Y2[2]; c01[2] = Ya[2];
        c11[0] = Y1[3]; c11[1] = Y2[3]; c11[2] = Ya[3];
        if constexpr (PAT == PF_CROSSED) {
            if (own) {
                const long long cv = ctr(g, ci, j);
                st2(yu, cv, Y1[4], Y2[4]);
                ya[cv] = ec[9] != 0.0 ? ec[8] : Ya[4];
            }
        }
    }
    template <bool BND = true>
    __device__ void out(const Geo2& g, int i, int j, const double (&t)[NC], const double (&v)[NV]) {
        const long long id = vid(g, i, j);
        const unsigned m = bcbits(g, i, j, id);
        double y0 = t[0], y1 = t[1];
        if (m) {
            const double2 xv = ld2(xu, id);
            if (m & 1u) y0 = xv.x;
            if (m & 2u) y1 = xv.y;
        }
        st2(yu, id, y0, y1);
        ya[id] = (act && act[id]) ? __ldg(xa + id) : t[2];
    }
};

}  // namespace pf
