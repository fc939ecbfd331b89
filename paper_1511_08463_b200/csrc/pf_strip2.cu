// pf_strip2.cu -- strip engine v2 (two columns per lane, TMA row tiles): kernel, tensor-map
// plumbing and the launchers of the operators that run on it (engine: pf_strip2d.cuh, strip_pass2).
//
// Tensor maps.  Every staged array is described to the TMA unit as a rank-1 tensor of its
// elements (fp64 or bytes) with a box of one warp window: 64 items (512 B) for 8-byte items, 128
// doubles (1024 B) for the 16-byte vertex pairs of u-like vectors, 64 bytes for masks (8-byte and
// byte boxes carry 2 / 16 extra items: the TMA needs 16-byte aligned starts, measured with
// tools/probe/tma_probe.cu -- an unaligned rank-1 coordinate is an illegal instruction).  The maps
// are encoded on the host per launch (cuTensorMapEncodeTiled through the runtime's driver entry
// point: no link dependency on libcuda), cached by (pointer, length, kind), and travel in the
// kernel's parameter block (__grid_constant__), so CUDA-graph replays carry them too.
#include <cuda.h>

#include <mutex>
#include <unordered_map>

#include "pf_strip2d.cuh"

namespace pf {

static_assert(sizeof(TmaMap) == sizeof(CUtensorMap), "TmaMap must mirror CUtensorMap");

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            p = nullptr;
        return (EncodeTiledFn)p;
    }();
    return fn;
}

enum { TM_F64x1 = 0, TM_F64x2 = 1, TM_U8 = 2 };

struct MapKey {
    const void* p;
    unsigned long long n;
    int kind;
    bool operator==(const MapKey& o) const { return p == o.p && n == o.n && kind == o.kind; }
};
struct MapKeyHash {
    size_t operator()(const MapKey& k) const {
        return std::hash<const void*>()(k.p) ^ (std::hash<unsigned long long>()(k.n) * 1315423911u) ^ (size_t)k.kind;
    }
};

// one rank-1 map: n items of `kind` at p.  false: the TMA path cannot take this array (not 16-byte
// aligned, too long, or no driver entry point) and the caller falls back to the v1 engine.
static bool encode_map(TmaMap* out, const void* p, unsigned long long n, int kind) {
    static std::mutex mu;
    static std::unordered_map<MapKey, TmaMap, MapKeyHash> cache;
    if (!p || n == 0) return false;
    if (reinterpret_cast<uintptr_t>(p) & 15u) return false;
    const MapKey key{p, n, kind};
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(key);
    if (it != cache.end()) { *out = it->second; return true; }
    EncodeTiledFn fn = encode_fn();
    if (!fn) return false;
    const cuuint64_t dim[1] = {kind == TM_F64x2 ? 2 * n : n};
    if (dim[0] >= (1ull << 31)) return false;  // coordinates are int32
    const cuuint64_t stride[1] = {0};
    // 16-byte aligned starts: 8-byte rows may begin one item early, byte rows up to 15 (TmaIssue::put*)
    const cuuint32_t box[1] = {(cuuint32_t)(kind == TM_F64x2 ? 2 * kCols2 : kind == TM_F64x1 ? kCols2 + 2 : kCols2 + 16)};
    const cuuint32_t estr[1] = {1};
    CUtensorMap m;
    const CUresult r = fn(&m, kind == TM_U8 ? CU_TENSOR_MAP_DATA_TYPE_UINT8 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 1,
                          const_cast<void*>(p), dim, stride, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                          CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return false;
    TmaMap t;
    memcpy(&t, &m, sizeof(t));
    if (cache.size() > 4096) cache.clear();
    cache.emplace(key, t);
    *out = t;
    return true;
}

void MapBuilder::f1(int m, const double* p, long long n) { ok = ok && encode_map(&set.m[m], p, (unsigned long long)n, TM_F64x1); }
void MapBuilder::f2(int m, const double* p, long long n) { ok = ok && encode_map(&set.m[m], p, (unsigned long long)n, TM_F64x2); }
void MapBuilder::u8(int m, const unsigned char* p, long long n) { ok = ok && encode_map(&set.m[m], p, (unsigned long long)n, TM_U8); }

constexpr int kBlock2 = 128;  // threads per block of the v2 strip kernels (4 warps)

template <class Op, int PAT>
__global__ void __launch_bounds__(kBlock2, Op::MINB) k_strip2v(const Geo2 g, Op op, const __grid_constant__ TmaSet tm) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    if (!op.enter()) return;  // device-side early exit (solver converged): uniform
    // TMA destinations must be 128-byte aligned; the launch reserves the slack
    unsigned char* smem = smem_raw + ((128u - (smem_addr(smem_raw) & 127u)) & 127u);
    const int wib = __shfl_sync(PF_FULL, (int)(threadIdx.x >> 5), 0);  // warp-uniform for the compiler
    strip_pass2<Op, PAT>(g, op, tm.m, smem, blockIdx.x * (kBlock2 / 32) + wib, wib, kBlock2 / 32);
    op.finish();
}

template <class Op, int PAT>
static constexpr int strip2_smem() {
    return 128 + (kBlock2 / 32) * ((Op::pd2(PAT) * (Op::sv(PAT) + Op::sc(PAT)) + Op::sv(PAT)) * kPitch2 + (Op::pd2(PAT) + 1) * 8);
}

inline int strip2_blocks(const Geo2& g) {
    const long long warps = (long long)(g.nwj2 + g.nslow2) * g.nstrips2;
    return (int)((warps * 32 + kBlock2 - 1) / kBlock2);
}

// Rows per strip.  With R warps resident on the GPU (SMs x this kernel's blocks per SM x 4 warps),
// ns strips of S = ceil(rows / ns) rows run nwj2 ns warps of S + 1 row steps each (one halo row per
// strip).  Blocks start and retire one by one, so the launch behaves like a continuous flow of
// nwj2 (rows + ns) / R steps through the resident slots, plus the tail while the last blocks drain
// (about half a strip and its pipeline fill).  Short strips cost halo rows, long strips cost tail:
//     t(ns) = nwj2 (rows + ns) / R + (S + kRamp) / 2,   minimised over ns (S >= 4, grid <= the
// reduction buffer).  Measured against a whole-wave model (waves x (S + 4), which prefers few long
// waves): 4096^2 union-jack Kuu 0.1485 -> 0.128 ms, 2048^2 0.0481 -> 0.0461 ms (tools/opbench.py with
// PF_STRIP2_WARPS sweeps, profiles/r02t_strip2_sizing.log).
static void size_strips2(Geo2& g, int resident_warps, int nslow) {
    constexpr double kRamp = 3.0;
    const long long rows = g.nx + 1;
    // a mesh that fits one wave of strips of at most 32 rows runs as that one wave (1024^2 .. 2048^2:
    // Kaa 2048^2 union-jack 0.039 vs 0.042 ms, the config-3 slab 0.958 vs 0.976 s/step)
    {
        const long long ns1 = std::max(1LL, (long long)resident_warps / (g.nwj2 + nslow));  // incl. the split halves
        const long long S1 = std::max(4LL, (rows + ns1 - 1) / ns1);
        if (S1 <= 32) {
            g.S2 = (int)S1;
            g.nstrips2 = (int)((rows + S1 - 1) / S1);
            return;
        }
    }
    long long best_ns = 1;
    double best_t = -1.0;
    for (long long ns = 1; ns <= rows; ++ns) {
        const long long S = (rows + ns - 1) / ns;
        if (S < 4 && ns > 1) break;
        const long long warps = (long long)(g.nwj2 + nslow) * ns;
        if ((warps * 32 + kBlock2 - 1) / kBlock2 > kMaxBlocksRed) break;
        const double t = (double)g.nwj2 * (double)(rows + ns) / (double)resident_warps + 0.5 * ((double)S + kRamp);
        if (best_t < 0.0 || t < best_t) { best_t = t; best_ns = ns; }
    }
    const long long S = (rows + best_ns - 1) / best_ns;
    g.S2 = (int)S;
    g.nstrips2 = (int)((rows + S - 1) / S);
}

template <class Op, int PAT>
static cudaError_t launch2_pat(Geo2 g, const Op& op, const TmaSet& tm, cudaStream_t st) {
    constexpr int smem = strip2_smem<Op, PAT>();
    static_assert(smem <= 227 * 1024, "strip stage ring exceeds shared memory");
    static std::atomic<int> occ[kMaxDev];  // blocks per SM of this instantiation (0: not set up yet)
    const int dv = cur_dev();
    if (!occ[dv].load()) {
        cudaError_t e = cudaFuncSetAttribute(k_strip2v<Op, PAT>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
        int nb = 0;
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_strip2v<Op, PAT>, kBlock2, smem);
        if (e != cudaSuccess) return e;
        occ[dv] = nb > 0 ? nb : 1;
    }
    static const long long forced = getenv("PF_STRIP2_WARPS") ? atoll(getenv("PF_STRIP2_WARPS")) : 0;
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dv);
    // boundary windows (general row step): window 0 and every window reaching past column ny - 1;
    // their strips are split between two warps (strip_pass2)
    static const bool split = !(getenv("PF_STRIP2_SPLIT") && atoi(getenv("PF_STRIP2_SPLIT")) == 0);
    int nslow = 0;
    if (split && g.nwj2 >= 4) {
        nslow = 1;
        for (int wj = g.nwj2 - 1; wj > 0 && wj * kOut2 - 1 + kCols2 > g.ny; --wj) ++nslow;
    }
    if (!forced) size_strips2(g, sms * occ[dv].load() * (kBlock2 / 32), nslow);
    g.nslow2 = 0;
    if (nslow > 0 && ((long long)(g.nwj2 + nslow) * g.nstrips2 * 32 + kBlock2 - 1) / kBlock2 <= kMaxBlocksRed) g.nslow2 = nslow;
    k_strip2v<Op, PAT><<<strip2_blocks(g), kBlock2, smem, st>>>(g, op, tm);
    return cudaSuccess;
}

// PF_OK: launched on the v2 engine.  -1: not applicable (the caller runs the v1 engine).
template <class Op>
int run_strip2(Ctx* c, const Op& op, cudaStream_t st, int kind, double bytes) {
    MapBuilder mb;
    op.maps(c->g, mb);
    if (!mb.ok) return -1;
    const Geo2& g = c->g;
    const int slot = prof_begin(c, st);
    cudaError_t e;
    switch (g.pattern) {
        case PF_UNION_JACK: e = launch2_pat<Op, PF_UNION_JACK>(g, op, mb.set, st); break;
        case PF_RIGHT: e = launch2_pat<Op, PF_RIGHT>(g, op, mb.set, st); break;
        default: e = launch2_pat<Op, PF_CROSSED>(g, op, mb.set, st); break;
    }
    if (e != cudaSuccess) return check_cuda(c, e, "strip v2 kernel attribute");
    prof_end(c, st, slot, kind, bytes);
    c->launches++;
    return check_cuda(c, cudaGetLastError(), "strip v2 kernel launch");
}

// the operators that run on the v2 engine
#define PF_V2(...) template int run_strip2<__VA_ARGS__>(Ctx*, const __VA_ARGS__&, cudaStream_t, int, double)
PF_V2(OpKuu<false, EPI_NONE>);
PF_V2(OpKuu<true, EPI_NONE>);
PF_V2(OpKuu<false, EPI_CHEB>);
PF_V2(OpKuu<false, EPI_CHEB_ADDD>);
PF_V2(OpKuu<false, EPI_RESID>);
PF_V2(OpKuu<false, EPI_RESID_CHEB0>);
PF_V2(OpKaa<false, false, false>);
PF_V2(OpKaa<false, true, false>);
PF_V2(OpKaa<false, true, true>);
PF_V2(OpKaa<true, false, false>);
PF_V2(OpKaa<true, true, false>);
PF_V2(OpKaaTrial);
PF_V2(OpKappa);

}  // namespace pf
