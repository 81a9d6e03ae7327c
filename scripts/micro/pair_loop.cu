// Microbenchmark: the near-field pair loop in isolation (smem-broadcast records, no
// traversal), sweeping unroll depth and resident warps.  Same arithmetic as k_near.
#include <cstdio>
#include <cuda_runtime.h>
#include <cstdint>
__device__ __forceinline__ double rsqrt_dp(double x) {
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    const double e = fma(-x, y * y, 1.0);
    return fma(y * e, fma(e, 0.375, 0.5), y);
}
__device__ __forceinline__ double rsqrt_f32seed(double x) {
    const float yf = rsqrtf(__double2float_rn(x));
    const double y = (double)yf;
    const double e = fma(-x, y * y, 1.0);
    return fma(y * e, fma(e, 0.375, 0.5), y);
}
// seed from an FP32 MUFU.RSQ with the double<->float conversions done in integer
// arithmetic (exponent halved, mantissa repacked), so no FP64-pipe instruction but the
// cubic correction; zero / subnormal / inf / nan inputs give NaN
__device__ __forceinline__ double rsqrt_intseed(double x) {
    const uint32_t hi = (uint32_t)__double2hiint(x), lo = (uint32_t)__double2loint(x);
    const int e = (int)(hi >> 20) - 1023;
    const int ep = e & 1, q = (e - ep) >> 1;
    const uint32_t fb = ((127u + ep) << 23) | ((hi & 0xFFFFFu) << 3) | (lo >> 29);
    float yf;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(yf) : "f"(__uint_as_float(fb)));
    const uint32_t yb = __float_as_uint(yf);
    const uint32_t dhi = (((yb >> 23) - 127u - (uint32_t)q + 1023u) << 20) | ((yb & 0x7FFFFFu) >> 3);
    double y = __hiloint2double((int)dhi, (int)((yb & 7u) << 29));
    y = (hi - 0x00100000u) >= 0x7FE00000u ? __longlong_as_double(0x7FF8000000000000ll) : y;
    const double ee = fma(-x, y * y, 1.0);
    return fma(y * ee, fma(ee, 0.375, 0.5), y);
}
template <int F32>
__device__ __forceinline__ void pair(const double* r, double x0, double x1, double x2, double& u0, double& u1,
                                     double& u2, bool& bad) {
    const double2 p01 = *reinterpret_cast<const double2*>(r);
    const double2 p2f0 = *reinterpret_cast<const double2*>(r + 2);
    const double d0 = x0 - p01.x, d1 = x1 - p01.y, d2 = x2 - p2f0.x;
    const double rr = fma(d2, d2, fma(d1, d1, d0 * d0));
    const double rinv = F32 == 2 ? rsqrt_intseed(rr) : F32 ? rsqrt_f32seed(rr) : rsqrt_dp(rr);
    const double rinv2 = rinv * rinv;
    const double2 f12 = *reinterpret_cast<const double2*>(r + 4);
    const double2 h01 = *reinterpret_cast<const double2*>(r + 6);
    const double2 h2n0 = *reinterpret_cast<const double2*>(r + 8);
    const double2 n12 = *reinterpret_cast<const double2*>(r + 10);
    const double f0 = p2f0.y, f1 = f12.x, f2 = f12.y;
    const double df = fma(d2, f2, fma(d1, f1, d0 * f0));
    const double dh = fma(d2, h2n0.x, fma(d1, h01.y, d0 * h01.x));
    const double dn = fma(d2, n12.y, fma(d1, n12.x, d0 * h2n0.y));
    const double sc = fma(dh * dn, rinv2, df) * rinv2;
    u0 = fma(rinv, fma(d0, sc, f0), u0);
    u1 = fma(rinv, fma(d1, sc, f1), u1);
    u2 = fma(rinv, fma(d2, sc, f2), u2);
}
template <int U, int F32>
__global__ void kpair(double* out, int iters) {
    __shared__ __align__(16) double rec[64 * 12];
    for (int i = threadIdx.x; i < 64 * 12; i += blockDim.x) rec[i] = 0.1 + 0.01 * (i % 12) + 0.001 * (i / 12);
    __syncthreads();
    const double x0 = 1.0 + threadIdx.x * 1e-3, x1 = 2.0, x2 = 3.0;
    double u[U][3] = {};
    bool bad = false;
    for (int it = 0; it < iters; ++it)
        for (int q = 0; q < 64; q += U)
#pragma unroll
            for (int v = 0; v < U; ++v) pair<F32>(rec + 12 * (q + v), x0, x1, x2, u[v & 1][0], u[v & 1][1], u[v & 1][2], bad);
    double s = 0;
    for (int v = 0; v < 2 && v < U; ++v) s += u[v][0] + u[v][1] + u[v][2];
    if (s == 1.2345 || bad) out[0] = s;
}
// two targets per lane share each record's shared-memory loads
__device__ __forceinline__ void pair2(const double* r, double x0, double x1, double x2, double z0, double z1,
                                      double z2, double* u, double* w) {
    const double2 p01 = *reinterpret_cast<const double2*>(r);
    const double2 p2f0 = *reinterpret_cast<const double2*>(r + 2);
    const double2 f12 = *reinterpret_cast<const double2*>(r + 4);
    const double2 h01 = *reinterpret_cast<const double2*>(r + 6);
    const double2 h2n0 = *reinterpret_cast<const double2*>(r + 8);
    const double2 n12 = *reinterpret_cast<const double2*>(r + 10);
    const double f0 = p2f0.y, f1 = f12.x, f2 = f12.y;
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        const double a0 = k ? z0 : x0, a1 = k ? z1 : x1, a2 = k ? z2 : x2;
        double* acc = k ? w : u;
        const double d0 = a0 - p01.x, d1 = a1 - p01.y, d2 = a2 - p2f0.x;
        const double rr = fma(d2, d2, fma(d1, d1, d0 * d0));
        const double rinv = rsqrt_dp(rr);
        const double rinv2 = rinv * rinv;
        const double df = fma(d2, f2, fma(d1, f1, d0 * f0));
        const double dh = fma(d2, h2n0.x, fma(d1, h01.y, d0 * h01.x));
        const double dn = fma(d2, n12.y, fma(d1, n12.x, d0 * h2n0.y));
        const double sc = fma(dh * dn, rinv2, df) * rinv2;
        acc[0] = fma(rinv, fma(d0, sc, f0), acc[0]);
        acc[1] = fma(rinv, fma(d1, sc, f1), acc[1]);
        acc[2] = fma(rinv, fma(d2, sc, f2), acc[2]);
    }
}
template <int U>
__global__ void kpair2(double* out, int iters) {
    __shared__ __align__(16) double rec[64 * 12];
    for (int i = threadIdx.x; i < 64 * 12; i += blockDim.x) rec[i] = 0.1 + 0.01 * (i % 12) + 0.001 * (i / 12);
    __syncthreads();
    const double x0 = 1.0 + threadIdx.x * 1e-3, x1 = 2.0, x2 = 3.0, z0 = 1.5 + threadIdx.x * 1e-3, z1 = 2.5, z2 = 3.5;
    double u[2][3] = {}, w[2][3] = {};
    for (int it = 0; it < iters; ++it)
        for (int q = 0; q < 64; q += U)
#pragma unroll
            for (int v = 0; v < U; ++v) pair2(rec + 12 * (q + v), x0, x1, x2, z0, z1, z2, u[v & 1], w[v & 1]);
    double s = u[0][0] + u[1][1] + u[0][2] + w[0][0] + w[1][1] + w[1][2];
    if (s == 1.2345) out[0] = s;
}
template <int U>
void run2(int threads, int blocks_per_sm, int iters) {
    int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    double* o; cudaMalloc(&o, 8);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int grid = nsm * blocks_per_sm;
    kpair2<U><<<grid, threads>>>(o, 2);
    cudaEventRecord(e0);
    kpair2<U><<<grid, threads>>>(o, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double pairs = (double)grid * threads * iters * 64 * 2;
    printf("2tgt    U=%d warps/SM=%2d: %.3e pairs/s\n", U, threads / 32 * blocks_per_sm, pairs / (ms * 1e-3));
}
template <int U, int F32 = 0>
void run(int threads, int blocks_per_sm, int iters) {
    int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    double* o; cudaMalloc(&o, 8);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int grid = nsm * blocks_per_sm;
    kpair<U, F32><<<grid, threads>>>(o, 2);
    cudaEventRecord(e0);
    kpair<U, F32><<<grid, threads>>>(o, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double pairs = (double)grid * threads * iters * 64;
    printf("%s U=%d warps/SM=%2d: %.3e pairs/s = %.2f T DP-inst/s (30/pair)\n", F32 == 2 ? "intseed" : F32 ? "f32seed" : "rsq64h ", U, threads / 32 * blocks_per_sm,
           pairs / (ms * 1e-3), pairs * 30 / (ms * 1e-3) * 1e-12);
}
int main() {
    for (int wps : {16, 24, 32}) {
        run<4>(256, wps / 8, 400);
        run2<2>(256, wps / 8, 200);
        run2<4>(256, wps / 8, 200);
    }
    return 0;
}
