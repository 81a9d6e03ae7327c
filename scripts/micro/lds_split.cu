// Shared-memory LDS.128 cost when the lanes of a warp read 1, 2 or 4 distinct 16-byte
// addresses (split by half / quarter warp), with the far field's DFMA mix beside it.
// Question: can two half-warps read two different clusters' weights for the price of one
// broadcast?  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o lds_split lds_split.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int GROUPS, int DFMA_PER_LOAD>
__global__ void __launch_bounds__(256) k_lds(double* out, int iters) {
    __shared__ __align__(16) double w[8 * 4 * 128];  // 8 warps x 4 groups x 128 doubles
    for (int i = threadIdx.x; i < 8 * 4 * 128; i += blockDim.x) w[i] = 1.0 + 1e-3 * i;
    __syncthreads();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int grp = lane / (32 / GROUPS);
    const double* base = w + (wid * 4 + grp) * 128;
    double a0 = lane, a1 = 0.5, a2 = 0.25, a3 = 0.125;
    const double x = 1.0000001;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < 64; j += 2) {
            const double2 v = *reinterpret_cast<const double2*>(base + j);
            a0 = fma(v.x, x, a0);
            a1 = fma(v.y, x, a1);
            if (DFMA_PER_LOAD > 2) {
                a2 = fma(v.x, a0, a2);
                a3 = fma(v.y, a1, a3);
            }
        }
        asm volatile("" ::: "memory");
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3;
}

// LDS.64 variant: one double per load
template <int GROUPS>
__global__ void __launch_bounds__(256) k_lds64(double* out, int iters) {
    __shared__ __align__(16) double w[8 * 4 * 128];
    for (int i = threadIdx.x; i < 8 * 4 * 128; i += blockDim.x) w[i] = 1.0 + 1e-3 * i;
    __syncthreads();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int grp = lane / (32 / GROUPS);
    const double* base = w + (wid * 4 + grp) * 128;
    double a0 = lane, a1 = 0.5;
    const double x = 1.0000001;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < 64; j += 2) {
            double v0, v1;  // exactly two LDS.64 (volatile: not merged, not hoisted)
            asm volatile("ld.volatile.shared.f64 %0, [%1];" : "=d"(v0) : "r"((unsigned)__cvta_generic_to_shared(base + j)));
            asm volatile("ld.volatile.shared.f64 %0, [%1];" : "=d"(v1) : "r"((unsigned)__cvta_generic_to_shared(base + j + 1)));
            a0 = fma(v0, x, a0);
            a1 = fma(v1, x, a1);
        }
        asm volatile("" ::: "memory");
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1;
}

template <int G>
void run64(const char* name, double* out) {
    const int iters = 2000, blocks = 148 * 4;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k_lds64<G><<<blocks, 256>>>(out, 10);
    cudaEventRecord(e0);
    k_lds64<G><<<blocks, 256>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    const double lds = (double)blocks * 8 * iters * 64;  // warp-level LDS.64 instructions
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const double per_sm_clk = ms * 1e-3 * clk * 1e3;
    printf("%-34s %8.3f ms  %.3f clk per warp LDS.64 per SM\n", name, ms, per_sm_clk * 148 / lds);
}

template <int G, int D>
void run(const char* name, double* out) {
    const int iters = 2000, blocks = 148 * 4;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k_lds<G, D><<<blocks, 256>>>(out, 10);
    cudaEventRecord(e0);
    k_lds<G, D><<<blocks, 256>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    const double lds = (double)blocks * 8 * iters * 32;  // warp-level LDS.128 instructions
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const double per_sm_clk = ms * 1e-3 * clk * 1e3;  // SM clocks elapsed
    printf("%-34s %8.3f ms  %.3f clk per warp LDS.128 per SM (%d DFMA per load)\n", name, ms,
           per_sm_clk * 148 / lds, D);
}

int main() {
    double* out;
    cudaMalloc(&out, 148 * 4 * 256 * sizeof(double));
    run<1, 2>("broadcast (1 address)", out);
    run<2, 2>("half warps (2 addresses)", out);
    run<4, 2>("quarter warps (4 addresses)", out);
    run<1, 4>("broadcast + 4 DFMA", out);
    run<2, 4>("half warps + 4 DFMA", out);
    run<4, 4>("quarter warps + 4 DFMA", out);
    run64<1>("LDS.64 broadcast (1 address)", out);
    run64<2>("LDS.64 half warps (2 addresses)", out);
    cudaFree(out);
    return 0;
}
