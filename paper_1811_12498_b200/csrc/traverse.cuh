// K3-K6: MAC traversal, far field, near field, O(N^2) direct sums.
#pragma once

#include "st_common.cuh"

namespace st {

constexpr uint32_t kNoSkip = 0xffffffffu;

struct TravArgs {
    const double* tx = nullptr;      // targets in batch (Morton) order, xyz
    const uint32_t* tskip = nullptr; // source tree index excluded per target (kNoSkip: none)
    const uint32_t* torig = nullptr; // original target index per batch position
    int nt = 0;
    int w0 = 0, w1 = 0;              // warp (32-target batch) range of this launch
    const double4* geom = nullptr;   // pre-order clusters: centre, radius
    const int4* info = nullptr;      // begin, end, next, is_leaf
    int ncl = 0;
    double th2 = 0.0;                // theta * theta
    const double* W = nullptr;       // far weights [ncl][(P+1)^2][4]
    const double* src = nullptr;     // tree-ordered source records [n][12]
    double* ufar = nullptr;          // far-field sums per batch position [nt][3]
    double* out = nullptr;           // final velocities, original target order [nt][3]
    uint64_t* per_target = nullptr;  // optional {visited, far, direct}, original order
    unsigned long long* stats = nullptr;  // {farfield_evals, direct_pairs, clusters_visited}
    int* err = nullptr;              // set to 1 on a coincident source/target pair
    float* warp_cost = nullptr;      // count pass: per-warp work estimate
    int out_batch = 0;               // 1: write out / per_target in batch order (slot t), not torig[t]
    int* work = nullptr;             // persistent kernels: next batch counter (zeroed per launch)
    // k_far with count = 1 also does the near plan's counting pass (the same DFS): near
    // leaves per target, near entries per batch warp (index warp - w0) and per source leaf,
    // and the statistics (stats, per_target)
    int count = 0;
    uint32_t* cnt_kn = nullptr;      // [nt]
    uint32_t* cnt_wcnt = nullptr;    // [w1 - w0]
    int32_t* cnt_leaf = nullptr;     // [ncl], zeroed by the caller
    // Sparse far events: k_far does not evaluate a cluster accepted by <= sparse_max lanes
    // of the warp (it would idle the other lanes); when counting it counts those entries
    // (per target, per batch warp, per cluster) and the near field's plan evaluates them
    // packed 32 per task (needs W and P).  0 disables deferral.
    int sparse_max = 0;
    int P = 0;                       // far order of W
    uint32_t* cnt_kd = nullptr;      // [nt]
    uint32_t* cnt_wd = nullptr;      // [w1 - w0]
    int32_t* cnt_dcl = nullptr;      // [ncl], zeroed by the caller
};

// Storage for the counting pass shared by k_far and the near field (see TravArgs::count).
struct NearCounts {
    DevArray<uint32_t> kn, wcnt, kd, wd;
    DevArray<int32_t> leaf, dcl;
    int sparse_max = 0;              // the deferral threshold the counting k_far used
    // allocate for a's warp range, zero the bucket counts, and point a's cnt_* fields at them
    void attach(TravArgs& a, cudaStream_t s) {
        kn.alloc(a.nt, s);
        wcnt.alloc(a.w1 - a.w0, s);
        leaf.alloc(a.ncl, s);
        leaf.zero();
        kd.alloc(a.nt, s);
        wd.alloc(a.w1 - a.w0, s);
        dcl.alloc(a.ncl, s);
        dcl.zero();
        a.cnt_kn = kn.get();
        a.cnt_wcnt = wcnt.get();
        a.cnt_leaf = leaf.get();
        a.cnt_kd = kd.get();
        a.cnt_wd = wd.get();
        a.cnt_dcl = dcl.get();
        sparse_max = a.sparse_max;
    }
};

// Far field for warps [w0, w1): P = p + 2 (stresslet) or p + 1.
void launch_far(int P, const TravArgs& a, cudaStream_t s);
// One far order to combine with the near field: its weights (for the deferred sparse
// events), the dense far sums k_far wrote, and the output.
struct FarOrder {
    int P = 0;
    const double* W = nullptr;
    const double* ufar = nullptr;
    double* out = nullptr;
};
// Near field + deferred far events + combine + scatter to original order + counters.  With
// counts (filled by a counting k_far over the same warp range) the near field skips its
// own counting walk.  Orders: the near sums are formed once and combined with each order
// (default: the single order described by a.P, a.W, a.ufar, a.out).
struct NearTimes {
    double near_eval_s = 0.0;        // k_neval (all slabs)
    double far_deferred_s = 0.0;     // k_feval over the deferred sparse far events (all orders)
};
void launch_near(bool sto, bool str, const TravArgs& a, cudaStream_t s, const NearCounts* counts = nullptr,
                 const FarOrder* orders = nullptr, int n_orders = 0, NearTimes* times = nullptr);
// Interaction lists (pre-order cluster ids, DFS order) of the targets in a.tx.
void launch_lists(const TravArgs& a, int cap, int32_t* far, int32_t* near, int64_t* nfar, int64_t* nnear,
                  cudaStream_t s);
// Traversal-only work estimate of every 4th warp of [a.w0, a.w1) into a.warp_cost (for
// multi-GPU shard cuts; the caller fills the warps in between from the preceding sample).
constexpr int kCountStride = 4;
void launch_count(const TravArgs& a, float far_cost, float near_cost, cudaStream_t s);

// O(N^2) contracted direct sum (kernels.hpp:45-83, 123-150): sources are the
// original-order records [n][12]; targets are source indices (self skipped).
void launch_direct(bool sto, bool str, const double* rec, size_t n, const int64_t* tgt, size_t nt,
                   double* u, int* err, cudaStream_t s);
// naive_direct_velocity (kernels.hpp:89-118): tensors S, T formed per pair.
void launch_naive(bool sto, bool str, const double* rec, size_t n, double* u, int* err,
                  cudaStream_t s);

// Per-pair far-field API: n pairs, pair i uses dx[3i..] and weight block i.
void launch_far_pairs(int P, size_t n, const double* dx, const double* W, double* u, cudaStream_t s);
// Reference-order Coulomb coefficients b^k, |k| <= pmax (coulomb.hpp:28-50).
void launch_coulomb(size_t n, const double* dx, int pmax, double* b, cudaStream_t s);
void launch_taylor(size_t n, const double* dx, const double* b, int pmax_b, int order, double* asto,
                   double* astr, cudaStream_t s);

}  // namespace st
