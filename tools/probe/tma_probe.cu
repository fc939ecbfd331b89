// TMA rank-1 tensor-map probe: which (dtype, box, coordinate) combinations work on this GPU.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
struct alignas(64) TmaMap { unsigned long long o[16]; };
typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                        const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
__device__ unsigned sa(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__global__ void k(const __grid_constant__ TmaMap m, int c0, int nbytes, unsigned char* out) {
    extern __shared__ __align__(128) unsigned char sm[];
    unsigned bar = sa(sm + 4096);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncwarp();
    for (int i = threadIdx.x; i < 4096; i += 32) sm[i] = 0xEE;
    __syncwarp();
    if (threadIdx.x == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("cp.async.bulk.tensor.1d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2}], [%3];" ::"r"(sa(sm)),
                     "l"((unsigned long long)&m), "r"(c0), "r"(bar) : "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(nbytes) : "memory");
    }
    asm volatile("{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@p bra D;\nbra W;\nD:\n}" ::"r"(bar) : "memory");
    for (int i = threadIdx.x; i < nbytes; i += 32) out[i] = sm[i];
}
int main(int argc, char** argv) {
    const int only = argc > 1 ? atoi(argv[1]) : -1;
    void* fp = nullptr; cudaDriverEntryPointQueryResult q;
    cudaFree(0);
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
    Enc enc = (Enc)fp;
    printf("entry %p q=%d\n", fp, (int)q);
    const int N = 100000;
    std::vector<double> h(N);
    for (int i = 0; i < N; ++i) h[i] = i;
    double* d; cudaMalloc(&d, N * 8); cudaMemcpy(d, h.data(), N * 8, cudaMemcpyHostToDevice);
    unsigned char* out; cudaMalloc(&out, 4096);
    struct Case { int dtype; unsigned box; int c0; const char* name; };
    Case cases[] = {{0, 64, 128, "f64 box64 c0=128 (aligned)"}, {0, 64, 5, "f64 box64 c0=5 (8B aligned)"},
                    {0, 64, -1, "f64 box64 c0=-1"}, {0, 128, 10, "f64 box128 c0=10"}, {0, 128, -2, "f64 box128 c0=-2"},
                    {0, 64, N - 10, "f64 box64 tail OOB"}, {1, 64, 3, "u8 box64 c0=3"}, {1, 64, -1, "u8 box64 c0=-1"},
                    {0, 256, 7, "f64 box256 c0=7"}, {0, 66, 4, "f64 box66 c0=4"}, {0, 66, -2, "f64 box66 c0=-2"},
                    {0, 128, -2, "f64 box128 c0=-2"}, {0, 66, N - 10, "f64 box66 tail OOB"}, {1, 80, 16, "u8 box80 c0=16"},
                    {1, 80, -16, "u8 box80 c0=-16"}, {0, 64, 6, "f64 box64 c0=6"}};
    int idx = -1;
    for (auto& cs : cases) {
        ++idx;
        if (only >= 0 && idx != only) continue;
        CUtensorMap m;
        cuuint64_t dim[1] = {(cuuint64_t)(cs.dtype ? N * 8 : N)};
        cuuint64_t str[1] = {0};
        cuuint32_t box[1] = {cs.box};
        cuuint32_t es[1] = {1};
        CUresult r = enc(&m, cs.dtype ? CU_TENSOR_MAP_DATA_TYPE_UINT8 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 1, d, dim, str, box,
                         es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        TmaMap t; memcpy(&t, &m, 128);
        int nbytes = cs.box * (cs.dtype ? 1 : 8);
        cudaMemset(out, 0xCD, 4096);
        k<<<1, 32, 8192>>>(t, cs.c0, nbytes, out);
        cudaError_t e = cudaDeviceSynchronize();
        printf("%-32s encode=%d run=%s", cs.name, (int)r, cudaGetErrorString(e));
        if (e == cudaSuccess) {
            std::vector<unsigned char> ho(nbytes);
            cudaMemcpy(ho.data(), out, nbytes, cudaMemcpyDeviceToHost);
            if (cs.dtype == 0) { double* p = (double*)ho.data(); printf("  first %.0f %.0f %.0f last %.0f", p[0], p[1], p[2], p[cs.box - 1]); }
            else printf("  first %d %d %d %d", ho[0], ho[1], ho[2], ho[3]);
        } else { printf("\n"); return 1; }
        printf("\n");
    }
    return 0;
}
