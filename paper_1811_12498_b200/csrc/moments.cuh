// K2: per-cluster Taylor moments (moments.hpp:34-80) and their fold into the
// far-field weights the traversal kernels contract with.
#pragma once

#include <vector>

#include "st_common.cuh"
#include "tree.cuh"

namespace st {

// Host-side work lists of the moment pass (leaf items and chunk partials, internal
// clusters by level), built from the tree's cluster records read back on stream `s`
// (one synchronisation).  Independent of the order p.
struct MomentsPlan {
    std::vector<int32_t> off, cl, slot;  // leaf work items: first item, cluster, partial slot
    int items = 0, parts = 0;
    std::vector<std::vector<int32_t>> lv;  // internal clusters per level, root level first
};
MomentsPlan plan_moments(const DevTree& tree, cudaStream_t s);

// Cartesian moments of every cluster at order p, combined layout
// M[ncl][E(p)][12]: columns 0..2 = M_j^k (f), 3..11 = M~_jl^k (h_j nu_l, j*3+l).
// `src` is the tree-ordered 12-double source record array.  With a plan, nothing in
// here waits for the host: the kernels can be queued on a second stream.
void compute_moments_device(const DevTree& tree, const double* src, int p, bool sto, bool str,
                            cudaStream_t s, DevArray<double>& M, const MomentsPlan* plan = nullptr);

// Far-field weights in the harmonic basis: W[ncl][(P+1)^2][4] with
// u_i = sum_h b_h W[h][i] + dx_i * sum_h b_h W[h][3]  ("K4").
// P = p + 2 with stresslets, p + 1 without.  `nblk` blocks of E(p) moments.
// pstride: order the blocks of M were computed at (>= p; -1 = p).
void fold_weights_device(const double* M, int nblk, int p, bool sto, bool str, cudaStream_t s,
                         DevArray<double>& W, int pstride = -1);

// Reference-layout export of M (stok[3E], str[9E], trace[E], sym[6E] per block;
// moments.hpp:15-27, derive_stresslet_contractions :67-80).
void export_moments_device(const double* M, int nblk, int p, bool sto, bool str, double* stok,
                           double* strm, double* trace, double* sym, cudaStream_t s);

// Inverse of the export (reference-layout blocks -> combined M), for the per-pair API.
void import_moments_device(int nblk, int p, bool sto, bool str, const double* stok,
                           const double* strm, double* M, cudaStream_t s);

}  // namespace st
