// Microbenchmark: the k_far per-pair evaluation (harmonic recurrence + 4-column contraction)
// in isolation, weights in shared memory, all lanes busy.  Includes traverse.cu's far_eval.
#include <cstdio>
#include <cuda_runtime.h>
#define ST_MICRO 1
#include "../../paper_1811_12498_b200/csrc/far_eval.cuh"
template <int P>
__global__ void kfar(double* out, int iters) {
    constexpr int H4 = 4 * (P + 1) * (P + 1);
    __shared__ __align__(16) double W[H4];
    for (int i = threadIdx.x; i < H4; i += blockDim.x) W[i] = 1e-3 * (1 + (i % 7));
    __syncthreads();
    double u0 = 0, u1 = 0, u2 = 0;
    double dx0 = 0.3 + 1e-4 * threadIdx.x, dx1 = -0.2, dx2 = 0.25;
    for (int it = 0; it < iters; ++it) {
        const double r2 = dx0 * dx0 + dx1 * dx1 + dx2 * dx2;
        st::far_eval<P, false>(dx0, dx1, dx2, r2, W, u0, u1, u2);
        dx0 += 1e-7;
    }
    if (u0 + u1 + u2 == 1.2345) out[0] = u0;
}
template <int P>
void run(int warps_per_sm, int iters) {
    int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    double* o; cudaMalloc(&o, 8);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int threads = 128, grid = nsm * warps_per_sm / 4;
    kfar<P><<<grid, threads>>>(o, 2);
    cudaEventRecord(e0);
    kfar<P><<<grid, threads>>>(o, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double pairs = (double)grid * threads * iters;
    printf("P=%d warps/SM=%d: %.3e pairs/s\n", P, warps_per_sm, pairs / (ms * 1e-3));
}
int main() {
    for (int w : {8, 12, 16}) run<10>(w, 2000);
    run<12>(12, 1500);
    return 0;
}
