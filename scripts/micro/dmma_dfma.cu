// Do FP64 MMA (mma.sync m8n8k4 f64, SASS DMMA) and FP64 FMA (DFMA) share issue capacity?
// Kernels: DFMA-only, DMMA-only, and both interleaved in the same warps.  Prints
// per-second rates; if "both" reaches ~the sum of the separate rates, DMMA is extra FP64
// capacity.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 dmma_dfma.cu -o dmma_dfma
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 4096;

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

template <bool FMA, bool MMA>
__global__ void k(double* out, double s) {
    double f[8], m[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        f[i] = threadIdx.x * 1e-3 + i;
        m[i] = threadIdx.x * 1e-4 + i;
    }
    const double a = s * 0.999, b = s * 1.001;
    for (int it = 0; it < ITERS; ++it) {
        if (FMA) {
#pragma unroll
            for (int r = 0; r < 4; ++r)
#pragma unroll
                for (int i = 0; i < 8; ++i) f[i] = fma(f[i], a, b);
        }
        if (MMA) {
#pragma unroll
            for (int i = 0; i < 8; i += 2) dmma(m[i], m[i + 1], a, b);
        }
    }
    double t = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) t += f[i] + m[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}

template <bool F, bool M>
float run(double* d, int blocks, int threads) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k<F, M><<<blocks, threads>>>(d, 1.0);
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) k<F, M><<<blocks, threads>>>(d, 1.0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    return ms / 5;
}

int main() {
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    const int threads = 256, blocks = nsm * 4;
    double* d;
    cudaMalloc(&d, sizeof(double) * blocks * threads);
    const double warps = blocks * threads / 32.0;
    const float tf = run<true, false>(d, blocks, threads);
    const float tm = run<false, true>(d, blocks, threads);
    const float tb = run<true, true>(d, blocks, threads);
    const double fma_thr = (double)blocks * threads * ITERS * 32;      // thread DFMA per launch
    const double mma_ops = warps * ITERS * 4 * (8.0 * 8 * 4 * 2);     // flops per launch (4 MMAs/iter)
    printf("DFMA only : %.3f ms  %.2f T thread-DFMA/s (%.1f TFLOP/s)\n", tf, fma_thr / tf * 1e-9, 2 * fma_thr / tf * 1e-9);
    printf("DMMA only : %.3f ms  %.1f TFLOP/s\n", tm, mma_ops / tm * 1e-9);
    printf("both      : %.3f ms  (sum of separate %.3f ms, max %.3f ms)\n", tb, tf + tm, tf > tm ? tf : tm);
    printf("=> %s\n", tb < 0.8 * (tf + tm) ? "DMMA and DFMA overlap (separate capacity)" : "DMMA and DFMA share capacity");
    cudaError_t e = cudaGetLastError();
    printf("status %s\n", cudaGetErrorString(e));
    return 0;
}
