// Accuracy of the MUFU.RSQ64H seed (rsqrt.approx.ftz.f64) and of one quadratic / one cubic
// correction, against 1/sqrt(x) in double, over x spanning many binades.
#include <cstdio>
#include <cmath>
#include <cuda_runtime.h>

__global__ void k(int n, double* out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    // x in [1e-12, 1e4): log-uniform, plus mantissa variety
    const double u = (i + 0.5) / n;
    const double x = exp2(-40.0 + 53.0 * u) * (1.0 + 0.618033988749 * ((i * 2654435761u) % 1000003) / 1000003.0);
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    const double ref = 1.0 / sqrt(x);
    const double e = fma(-x, y * y, 1.0);
    const double yq = fma(y * e, 0.5, y);                  // one Newton (quadratic)
    const double yc = fma(y * e, fma(e, 0.375, 0.5), y);   // cubic correction (production)
    out[4 * i] = fabs(y - ref) / ref;
    out[4 * i + 1] = fabs(yq - ref) / ref;
    out[4 * i + 2] = fabs(yc - ref) / ref;
    out[4 * i + 3] = (yq - ref) / ref;
}

int main() {
    const int n = 1 << 22;
    double* d;
    cudaMalloc(&d, sizeof(double) * 4 * n);
    k<<<(n + 255) / 256, 256>>>(n, d);
    double* h = new double[4 * (size_t)n];
    cudaMemcpy(h, d, sizeof(double) * 4 * n, cudaMemcpyDeviceToHost);
    double m[3] = {0, 0, 0}, bias = 0;
    for (int i = 0; i < n; ++i) {
        for (int j = 0; j < 3; ++j) m[j] = fmax(m[j], h[4 * i + j]);
        bias += h[4 * i + 3];
    }
    printf("seed max rel err %.3e (2^%.1f)\n", m[0], log2(m[0]));
    printf("quadratic max rel err %.3e (2^%.1f), mean signed %.3e\n", m[1], log2(m[1]), bias / n);
    printf("cubic max rel err %.3e (2^%.1f)\n", m[2], log2(m[2]));
    return 0;
}
