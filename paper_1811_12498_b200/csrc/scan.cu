#include "scan.cuh"

#include <cub/device/device_scan.cuh>
#include <thrust/iterator/transform_iterator.h>

namespace st {

namespace {
constexpr int kScanThreads = 1024;

// Block-wide inclusive scan of one value per thread (1024 threads).
template <class T>
__device__ T block_inclusive(T v, T* warp_sums) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        T y = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += y;
    }
    if (lane == 31) warp_sums[wid] = v;
    __syncthreads();
    if (wid == 0) {
        T w = warp_sums[lane];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            T y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += y;
        }
        warp_sums[lane] = w;
    }
    __syncthreads();
    if (wid > 0) v += warp_sums[wid - 1];
    __syncthreads();
    return v;
}
}  // namespace

__global__ void __launch_bounds__(kScanThreads) k_scan_cols(const uint32_t* __restrict__ in,
                                                            uint32_t* __restrict__ out, int nrows,
                                                            int ncols) {
    __shared__ uint32_t warp_sums[32];
    __shared__ uint32_t carry;
    for (int c = 0; c < ncols; ++c) {
        if (threadIdx.x == 0) carry = 0;
        __syncthreads();
        for (int base = 0; base < nrows; base += kScanThreads) {
            const int r = base + threadIdx.x;
            const uint32_t v = r < nrows ? in[(size_t)r * ncols + c] : 0u;
            const uint32_t inc = block_inclusive<uint32_t>(v, warp_sums);
            const uint32_t cy = carry;
            if (r < nrows) out[(size_t)r * ncols + c] = cy + inc - v;
            __syncthreads();
            if (threadIdx.x == kScanThreads - 1) carry = cy + inc;
            __syncthreads();
        }
        if (threadIdx.x == 0) out[(size_t)nrows * ncols + c] = carry;
        __syncthreads();
    }
}

__global__ void __launch_bounds__(kScanThreads) k_scan_i32(const int32_t* __restrict__ in,
                                                           int32_t* __restrict__ out, int nrows) {
    __shared__ int32_t warp_sums[32];
    __shared__ int32_t carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int base = 0; base < nrows; base += kScanThreads) {
        const int r = base + threadIdx.x;
        const int32_t v = r < nrows ? in[r] : 0;
        const int32_t inc = block_inclusive<int32_t>(v, warp_sums);
        const int32_t cy = carry;
        if (r < nrows) out[r] = cy + inc - v;
        __syncthreads();
        if (threadIdx.x == kScanThreads - 1) carry = cy + inc;
        __syncthreads();
    }
    if (threadIdx.x == 0) out[nrows] = carry;
}

// Exclusive scan of nrows uint32 values into uint64 offsets; out[nrows] = total.
__global__ void __launch_bounds__(kScanThreads) k_scan_u32_u64(const uint32_t* __restrict__ in,
                                                               uint64_t* __restrict__ out, int nrows) {
    __shared__ uint64_t warp_sums[32];
    __shared__ uint64_t carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int base = 0; base < nrows; base += kScanThreads) {
        const int r = base + threadIdx.x;
        const uint64_t v = r < nrows ? in[r] : 0u;
        const uint64_t inc = block_inclusive<uint64_t>(v, warp_sums);
        const uint64_t cy = carry;
        if (r < nrows) out[r] = cy + inc - v;
        __syncthreads();
        if (threadIdx.x == kScanThreads - 1) carry = cy + inc;
        __syncthreads();
    }
    if (threadIdx.x == 0) out[nrows] = carry;
}

namespace {
struct ToU64 {
    __host__ __device__ uint64_t operator()(uint32_t v) const { return v; }
};
// Rows beyond one CTA's comfortable range go to CUB's decoupled-lookback scan (single-CTA
// scans of 250K rows took 0.26 ms each at cfg4); small ones stay one launch.
constexpr int kScanOneCta = 16384;
}  // namespace

void launch_scan_u32_u64(const uint32_t* in, uint64_t* out, int nrows, cudaStream_t s) {
    if (nrows <= kScanOneCta) {
        k_scan_u32_u64<<<1, kScanThreads, 0, s>>>(in, out, nrows);
        ST_LAUNCH("k_scan_u32_u64");
        count_launch();
        return;
    }
    // out[0] = 0, out[1..n] = inclusive sums (accumulated in 64 bits)
    const auto it = thrust::make_transform_iterator(in, ToU64());
    size_t tmp = 0;
    ST_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tmp, it, out + 1, nrows, s));
    DevArray<unsigned char> scratch(tmp, s);
    ST_CUDA(cudaMemsetAsync(out, 0, sizeof(uint64_t), s));
    ST_CUDA(cub::DeviceScan::InclusiveSum(scratch.get(), tmp, it, out + 1, nrows, s));
    ST_LAUNCH("cub::DeviceScan (u32 -> u64)");
    count_launch(2);
}

// The 8-column case (the tree build's per-tile octant histograms): every thread scans a
// whole row of 8 counts at once (two 16-B loads), so a level costs nrows / 1024 block-scan
// rounds instead of 8 x that (38 -> ~6 us per level at 8M particles).
__global__ void __launch_bounds__(kScanThreads) k_scan_cols8(const uint32_t* __restrict__ in,
                                                             uint32_t* __restrict__ out, int nrows) {
    __shared__ uint32_t warp_sums[32][8];
    __shared__ uint32_t carry[8];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (threadIdx.x < 8) carry[threadIdx.x] = 0;
    __syncthreads();
    for (int base = 0; base < nrows; base += kScanThreads) {
        const int r = base + threadIdx.x;
        uint32_t v[8], x[8];
        if (r < nrows) {
            const uint4 a = reinterpret_cast<const uint4*>(in)[2 * (size_t)r];
            const uint4 b = reinterpret_cast<const uint4*>(in)[2 * (size_t)r + 1];
            v[0] = a.x, v[1] = a.y, v[2] = a.z, v[3] = a.w, v[4] = b.x, v[5] = b.y, v[6] = b.z, v[7] = b.w;
        } else {
#pragma unroll
            for (int c = 0; c < 8; ++c) v[c] = 0u;
        }
#pragma unroll
        for (int c = 0; c < 8; ++c) x[c] = v[c];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1)
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, x[c], o);
                if (lane >= o) x[c] += y;
            }
        if (lane == 31)
#pragma unroll
            for (int c = 0; c < 8; ++c) warp_sums[wid][c] = x[c];
        __syncthreads();
        if (wid < 8) {  // warp c scans column c of the 32 warp totals
            uint32_t w = warp_sums[lane][wid];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
                if (lane >= o) w += y;
            }
            warp_sums[lane][wid] = w;
        }
        __syncthreads();
        uint32_t cy[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) cy[c] = carry[c] + (wid > 0 ? warp_sums[wid - 1][c] : 0u);
        if (r < nrows) {
            uint4 a, b;
            a.x = cy[0] + x[0] - v[0], a.y = cy[1] + x[1] - v[1], a.z = cy[2] + x[2] - v[2], a.w = cy[3] + x[3] - v[3];
            b.x = cy[4] + x[4] - v[4], b.y = cy[5] + x[5] - v[5], b.z = cy[6] + x[6] - v[6], b.w = cy[7] + x[7] - v[7];
            reinterpret_cast<uint4*>(out)[2 * (size_t)r] = a;
            reinterpret_cast<uint4*>(out)[2 * (size_t)r + 1] = b;
        }
        __syncthreads();
        if (threadIdx.x < 8) carry[threadIdx.x] += warp_sums[31][threadIdx.x];
        __syncthreads();
    }
    if (threadIdx.x < 8) out[(size_t)nrows * 8 + threadIdx.x] = carry[threadIdx.x];
}

void launch_scan_cols(const uint32_t* in, uint32_t* out, int nrows, int ncols, cudaStream_t s) {
    if (ncols == 8) {
        k_scan_cols8<<<1, kScanThreads, 0, s>>>(in, out, nrows);
        ST_LAUNCH("k_scan_cols8");
        count_launch();
        return;
    }
    k_scan_cols<<<1, kScanThreads, 0, s>>>(in, out, nrows, ncols);
    ST_LAUNCH("k_scan_cols");
    count_launch();
}

void launch_scan_i32(const int32_t* in, int32_t* out, int nrows, cudaStream_t s) {
    if (nrows <= kScanOneCta) {
        k_scan_i32<<<1, kScanThreads, 0, s>>>(in, out, nrows);
        ST_LAUNCH("k_scan_i32");
        count_launch();
        return;
    }
    size_t tmp = 0;
    ST_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tmp, in, out + 1, nrows, s));
    DevArray<unsigned char> scratch(tmp, s);
    ST_CUDA(cudaMemsetAsync(out, 0, sizeof(int32_t), s));
    ST_CUDA(cub::DeviceScan::InclusiveSum(scratch.get(), tmp, in, out + 1, nrows, s));
    ST_LAUNCH("cub::DeviceScan (i32)");
    count_launch(2);
}

}  // namespace st
