// Microbenchmark: DFMA throughput vs operand pattern on one B200 (scripts/micro).
//   A: a_i = fma(a_i, m, c)         two operands shared across chains (reuse-cache friendly)
//   B: a_i = fma(b_i, c_i, a_i)     three distinct registers per instruction
//   C: B with a DMUL/DADD mix like the near-field pair (18 FMA : 10 MUL : 3 ADD)
#include <cstdio>
#include <cuda_runtime.h>
__global__ void kA(double* o, int it, double s) {
    double a[8];
    for (int i = 0; i < 8; ++i) a[i] = s + threadIdx.x + i;
    const double m = 0.999999999, c = 1e-9;
    for (int k = 0; k < it; ++k)
#pragma unroll
        for (int r = 0; r < 16; ++r)
#pragma unroll
            for (int i = 0; i < 8; ++i) a[i] = fma(a[i], m, c);
    double t = 0;
    for (int i = 0; i < 8; ++i) t += a[i];
    if (t == 1.2345) o[0] = t;
}
__global__ void kB(double* o, int it, double s) {
    double a[8], b[8], c[8];
    for (int i = 0; i < 8; ++i) { a[i] = s + threadIdx.x + i; b[i] = 0.999999 + 1e-7 * i; c[i] = 1e-9 * (i + 1); }
    for (int k = 0; k < it; ++k)
#pragma unroll
        for (int r = 0; r < 16; ++r)
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                a[i] = fma(b[i], c[(i + 3) & 7], a[i]);
                b[i] = fma(a[(i + 1) & 7], 1e-12, b[i]);
            }
    double t = 0;
    for (int i = 0; i < 8; ++i) t += a[i] + b[i];
    if (t == 1.2345) o[0] = t;
}
__global__ void kC(double* o, int it, double s) {
    double a[8], b[8];
    for (int i = 0; i < 8; ++i) { a[i] = s + threadIdx.x + i; b[i] = 1.0 + 1e-7 * i; }
    for (int k = 0; k < it; ++k)
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                double x = a[i] * b[i];              // DMUL
                double y = x + a[(i + 1) & 7];       // DADD
                a[i] = fma(y, 1e-9, a[i]);           // DFMA
                b[i] = fma(b[i], x, 1.0) * 0.5;      // DFMA + DMUL
                a[i] = fma(a[i], b[(i + 2) & 7], y); // DFMA
            }
    double t = 0;
    for (int i = 0; i < 8; ++i) t += a[i] + b[i];
    if (t == 1.2345) o[0] = t;
}
template <class K>
double run(K k, int ops_per_iter, int it) {
    int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    double* o; cudaMalloc(&o, 8);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    k<<<nsm * 8, 256>>>(o, 10, 1.0);
    cudaEventRecord(e0);
    k<<<nsm * 8, 256>>>(o, it, 1.0);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double inst = (double)nsm * 8 * 256 * it * ops_per_iter;
    return inst / (ms * 1e-3) * 1e-12;  // T thread-inst/s
}
int main2();
int main() {
    main2();
    printf("A (shared operands)  : %.2f T DP thread-inst/s\n", run(kA, 128, 4000));
    printf("B (distinct operands): %.2f T DP thread-inst/s\n", run(kB, 256, 2000));
    printf("C (mul/add mix)      : %.2f T DP thread-inst/s\n", run(kC, 32 * 6, 4000));
    return 0;
}
// D: one rsqrt.approx.f64 (MUFU.RSQ64H) per R DFMAs per chain
template <int R>
__global__ void kD(double* o, int it, double s) {
    double a[8], y[8];
    for (int i = 0; i < 8; ++i) { a[i] = s + threadIdx.x + i; y[i] = 1.0; }
    for (int k = 0; k < it; ++k)
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            double r;
            asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(a[i] + 2.0));
            y[i] += r;
#pragma unroll
            for (int q = 0; q < R; ++q) a[i] = fma(a[i], 0.999999999, 1e-9);
        }
    double t = 0;
    for (int i = 0; i < 8; ++i) t += a[i] + y[i];
    if (t == 1.2345) o[0] = t;
}
int main2() {
    printf("D R=30 (1 MUFU.RSQ64H per 30 DFMA): %.2f T DFMA thread-inst/s\n", run(kD<30>, 8 * 30, 2000));
    printf("D R=8  (1 MUFU.RSQ64H per 8 DFMA) : %.2f T DFMA thread-inst/s\n", run(kD<8>, 8 * 8, 4000));
    printf("D R=2  (1 MUFU.RSQ64H per 2 DFMA) : %.2f T DFMA thread-inst/s\n", run(kD<2>, 8 * 2, 8000));
    return 0;
}
