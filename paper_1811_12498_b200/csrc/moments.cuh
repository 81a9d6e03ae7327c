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
    std::vector<int4> info;                // host copy of the tree's cluster records
    std::vector<int32_t> depth;            // depth of each cluster (pre-order id)
};
MomentsPlan plan_moments(const DevTree& tree, cudaStream_t s);

// The moment pass split over `nshards` ranks (multi-GPU).  The tree is
// cut at the shallowest depth L that yields at least 4 * nshards "units" (the clusters at
// depth L and the leaves above it): whole subtrees, each a contiguous pre-order range.
// Units are dealt to the ranks in pre-order, balanced by particle count, so rank r owns the
// contiguous cluster rows [w_cuts[r], w_cuts[r+1]) (the top clusters above depth L that
// fall inside are recomputed by every rank after the exchange).  Each rank computes its
// units' leaf moments, M2M and weights; the ranks exchange the weight rows and the units'
// root moments; every rank then shifts the top levels (M2M) and folds them.  Every
// cluster's moments and weights are computed exactly as the one-rank pass computes them,
// so the result is bit-identical for any rank count.
struct MomentsSplit {
    int depth = 0;                          // L
    std::vector<int32_t> units;             // unit root ids, pre-order
    std::vector<size_t> unit_cuts;          // nshards + 1
    std::vector<size_t> w_cuts;             // nshards + 1 cluster-row cut points
    std::vector<std::vector<int32_t>> top;  // internal clusters above L per level (root first)
    std::vector<int32_t> top_ids;           // the same, flat
};
MomentsSplit split_moments(const MomentsPlan& full, int ncl, int nshards);
// The plan of rank `shard`'s units (leaves and internal clusters at depth >= L).
MomentsPlan shard_moments_plan(const MomentsPlan& full, const MomentsSplit& sp, int shard);
// The plan of the top levels only (no leaves): M2M above depth L, on an M already holding
// the units' moments.
MomentsPlan top_moments_plan(const MomentsSplit& sp);

// Cartesian moments of every cluster at order p, combined layout
// M[ncl][E(p)][12]: columns 0..2 = M_j^k (f), 3..11 = M~_jl^k (h_j nu_l, j*3+l).
// `src` is the tree-ordered 12-double source record array.  With a plan, nothing in
// here waits for the host: the kernels can be queued on a second stream.
// keep = true: M is already allocated (ncl blocks) and holds moments this call must not
// clear (the top-level pass of a split moment pass).
void compute_moments_device(const DevTree& tree, const double* src, int p, bool sto, bool str,
                            cudaStream_t s, DevArray<double>& M, const MomentsPlan* plan = nullptr,
                            bool keep = false);

// Far-field weights in the harmonic basis: W[ncl][(P+1)^2][4] with
// u_i = sum_h b_h W[h][i] + dx_i * sum_h b_h W[h][3]  ("K4").
// P = p + 2 with stresslets, p + 1 without.  `nblk` blocks of E(p) moments.
// pstride: order the blocks of M were computed at (>= p; -1 = p).
void fold_weights_device(const double* M, int nblk, int p, bool sto, bool str, cudaStream_t s,
                         DevArray<double>& W, int pstride = -1);

// The same fold for the listed clusters only (rows, device, n of them), into an existing
// W of ncl rows (split moment pass).
void fold_weights_rows_device(const double* M, const int32_t* rows, int n, int p, bool sto, bool str,
                              cudaStream_t s, double* W);
// dst[i][0..len) = src[rows[i]][0..len) (gather) or the reverse (scatter), device.
void gather_rows_device(const double* src, const int32_t* rows, int n, size_t len, double* dst, bool scatter,
                        cudaStream_t s);

// Reference-layout export of M (stok[3E], str[9E], trace[E], sym[6E] per block;
// moments.hpp:15-27, derive_stresslet_contractions :67-80).
void export_moments_device(const double* M, int nblk, int p, bool sto, bool str, double* stok,
                           double* strm, double* trace, double* sym, cudaStream_t s);

// Inverse of the export (reference-layout blocks -> combined M), for the per-pair API.
void import_moments_device(int nblk, int p, bool sto, bool str, const double* stok,
                           const double* strm, double* M, cudaStream_t s);

}  // namespace st
