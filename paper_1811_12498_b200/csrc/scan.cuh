// Small single-CTA scans used by the level-synchronous tree build (row counts are
// at most a few hundred thousand, so one resident CTA is enough).
#pragma once

#include "st_common.cuh"

namespace st {

// Exclusive column scan of a row-major [nrows][ncols] uint32 matrix; out has
// nrows+1 rows, the last one holding the column totals.
__global__ void k_scan_cols(const uint32_t* __restrict__ in, uint32_t* __restrict__ out, int nrows,
                            int ncols);

// Exclusive scan of nrows int32 values; out[nrows] = total (also *total if non-null).
__global__ void k_scan_i32(const int32_t* __restrict__ in, int32_t* __restrict__ out, int nrows);

__global__ void k_scan_u32_u64(const uint32_t* __restrict__ in, uint64_t* __restrict__ out, int nrows);
void launch_scan_u32_u64(const uint32_t* in, uint64_t* out, int nrows, cudaStream_t s);
void launch_scan_cols(const uint32_t* in, uint32_t* out, int nrows, int ncols, cudaStream_t s);
void launch_scan_i32(const int32_t* in, int32_t* out, int nrows, cudaStream_t s);

}  // namespace st
