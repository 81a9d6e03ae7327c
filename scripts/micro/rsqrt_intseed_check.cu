#include <cstdio>
#include <cmath>
#include <cstdint>
#include <cuda_runtime.h>
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
__global__ void k(int n, double* out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double u = (i + 0.5) / n;
    const double x = exp2(-300.0 + 600.0 * u) * (1.0 + 0.618 * ((i * 2654435761u) % 1000003) / 1000003.0);
    out[i] = fabs(rsqrt_intseed(x) - 1.0 / sqrt(x)) * sqrt(x);
}
__global__ void kz(double* o) { o[0] = rsqrt_intseed(0.0); o[1] = rsqrt_intseed(1e-320); o[2] = rsqrt_intseed(INFINITY); o[3] = rsqrt_intseed(4.0); }
int main() {
    const int n = 1 << 22; double* d; cudaMalloc(&d, 8 * n);
    k<<<n / 256, 256>>>(n, d); double* h = new double[n]; cudaMemcpy(h, d, 8 * n, cudaMemcpyDeviceToHost);
    double m = 0; for (int i = 0; i < n; ++i) m = fmax(m, h[i]);
    printf("intseed+cubic max rel err %.3e over 2^-300..2^300\n", m);
    kz<<<1, 1>>>(d); double z[4]; cudaMemcpy(z, d, 32, cudaMemcpyDeviceToHost);
    printf("special: 0 -> %g, subnormal -> %g, inf -> %g, 4 -> %.17g\n", z[0], z[1], z[2], z[3]);
}
