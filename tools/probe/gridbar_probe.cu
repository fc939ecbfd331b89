// Grid-barrier latency probe: 148 co-resident CTAs x 512 threads, NB barriers per launch with a
// small dependent store/load between them (so there are writes to publish), several arrival forms.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gridbar_probe gridbar_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

// A: the library's barrier (fence + returning atomic, sense taken from the returned value)
__device__ __forceinline__ void bar_a(unsigned int* bar) {
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
// B: sense kept in a register (read once at kernel start), non-returning red.release
__device__ __forceinline__ void bar_b(unsigned int* bar, unsigned int& sense) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned int inc = blockIdx.x == 0 ? 0x80000000u - (gridDim.x - 1) : 1u;
        asm volatile("red.release.gpu.global.add.u32 [%0], %1;\n" ::"l"(bar), "r"(inc) : "memory");
        unsigned int cur;
        do {
            asm volatile("ld.acquire.gpu.u32 %0, [%1];\n" : "=r"(cur) : "l"(bar) : "memory");
        } while (((sense ^ cur) & 0x80000000u) == 0);
    }
    sense ^= 0x80000000u;
    __syncthreads();
}
// C: as B, fence + relaxed red
__device__ __forceinline__ void bar_c(unsigned int* bar, unsigned int& sense) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned int inc = blockIdx.x == 0 ? 0x80000000u - (gridDim.x - 1) : 1u;
        __threadfence();
        asm volatile("red.relaxed.gpu.global.add.u32 [%0], %1;\n" ::"l"(bar), "r"(inc) : "memory");
        unsigned int cur;
        do {
            asm volatile("ld.acquire.gpu.u32 %0, [%1];\n" : "=r"(cur) : "l"(bar) : "memory");
        } while (((sense ^ cur) & 0x80000000u) == 0);
    }
    sense ^= 0x80000000u;
    __syncthreads();
}
// D: as A with a relaxed poll and one fence after (instead of an acquire load per poll)
__device__ __forceinline__ void bar_d(unsigned int* bar, unsigned int& sense) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned int inc = blockIdx.x == 0 ? 0x80000000u - (gridDim.x - 1) : 1u;
        asm volatile("red.release.gpu.global.add.u32 [%0], %1;\n" ::"l"(bar), "r"(inc) : "memory");
        unsigned int cur;
        do {
            asm volatile("ld.relaxed.gpu.u32 %0, [%1];\n" : "=r"(cur) : "l"(bar) : "memory");
        } while (((sense ^ cur) & 0x80000000u) == 0);
        asm volatile("fence.acq_rel.gpu;\n" ::: "memory");
    }
    sense ^= 0x80000000u;
    __syncthreads();
}

template <int V>
__global__ void __launch_bounds__(512, 1) k(unsigned int* bar, double* x, double* y, int nb, int n) {
    unsigned int sense = 0;
    if (V != 0) sense = *(volatile unsigned int*)bar & 0x80000000u;
    const int tid = blockIdx.x * blockDim.x + threadIdx.x, nth = gridDim.x * blockDim.x;
    double* a = x;
    double* b = y;
    for (int it = 0; it < nb; ++it) {
        for (int i = tid; i < n; i += nth) b[i] = 0.5 * (__ldcg(a + (i + 1) % n) + __ldcg(a + (i + n - 1) % n));
        if (V == 0) bar_a(bar);
        if (V == 1) bar_b(bar, sense);
        if (V == 2) bar_c(bar, sense);
        if (V == 3) bar_d(bar, sense);
        double* t = a; a = b; b = t;
    }
}
template <int V>
__global__ void __launch_bounds__(512, 1) knb(double* x, double* y, int nb, int n) {  // the work alone
    const int tid = blockIdx.x * blockDim.x + threadIdx.x, nth = gridDim.x * blockDim.x;
    double* a = x;
    double* b = y;
    for (int it = 0; it < nb; ++it) {
        for (int i = tid; i < n; i += nth) b[i] = 0.5 * (__ldcg(a + (i + 1) % n) + __ldcg(a + (i + n - 1) % n));
        __syncthreads();
        double* t = a; a = b; b = t;
    }
}

template <int V>
static float run(unsigned int* bar, double* x, double* y, int nb, int n, int grid) {
    void* args[] = {&bar, &x, &y, &nb, &n};
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int w = 0; w < 3; ++w) cudaLaunchCooperativeKernel((void*)k<V>, dim3(grid), dim3(512), args, 0, 0);
    cudaEventRecord(e0);
    for (int w = 0; w < 10; ++w) cudaLaunchCooperativeKernel((void*)k<V>, dim3(grid), dim3(512), args, 0, 0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (cudaGetLastError() != cudaSuccess) printf("error variant %d\n", V);
    return ms / 10.f * 1000.f / nb;  // us per barrier+work
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    unsigned int* bar;
    cudaMalloc(&bar, 256);
    cudaMemset(bar, 0, 256);
    const int nb = 2000;
    for (int n : {1024, 66049, 4 * 66049}) {
        double *x, *y;
        cudaMalloc(&x, n * 8);
        cudaMalloc(&y, n * 8);
        cudaMemset(x, 0, n * 8);
        cudaMemset(y, 0, n * 8);
        void* a2[] = {&x, &y, (void*)&nb, &n};
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaLaunchKernel((void*)knb<0>, dim3(sms), dim3(512), a2, 0, 0);
        cudaEventRecord(e0);
        cudaLaunchKernel((void*)knb<0>, dim3(sms), dim3(512), a2, 0, 0);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("n=%d  work alone %.3f us/phase | ", n, ms * 1000.f / nb);
        printf("A %.3f  ", run<0>(bar, x, y, nb, n, sms));
        printf("B %.3f  ", run<1>(bar, x, y, nb, n, sms));
        printf("C %.3f  ", run<2>(bar, x, y, nb, n, sms));
        printf("D %.3f  us/phase\n", run<3>(bar, x, y, nb, n, sms));
        cudaFree(x);
        cudaFree(y);
    }
    unsigned int h;
    cudaMemcpy(&h, bar, 4, cudaMemcpyDeviceToHost);
    printf("bar word %08x  last error: %s\n", h, cudaGetErrorString(cudaGetLastError()));
    return 0;
}
