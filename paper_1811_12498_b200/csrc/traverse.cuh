// K3-K6: MAC traversal, far field, near field, O(N^2) direct sums.
#pragma once

#include <functional>

#include <utility>
#include <vector>

#include "st_common.cuh"

namespace st {

constexpr uint32_t kNoSkip = 0xffffffffu;

struct TravArgs {
    const double* tx = nullptr;      // targets in batch (octree-key) order, xyz
    const uint32_t* tskip = nullptr; // source tree index excluded per target (kNoSkip: none)
    const uint32_t* torig = nullptr; // original target index per batch position
    int nt = 0;
    int w0 = 0, w1 = 0;              // warp (32-target batch) range of this launch
    const double4* geom = nullptr;   // pre-order clusters: centre, radius
    const int4* info = nullptr;      // begin, end, next, is_leaf
    int ncl = 0;
    double th2 = 0.0;                // theta * theta
    const double* src = nullptr;     // tree-ordered source records [n][12]
    double* out = nullptr;           // final velocities, original target order [nt][3]
    uint64_t* per_target = nullptr;  // optional {visited, far, direct}, original order
    unsigned long long* stats = nullptr;  // {farfield_evals, direct_pairs, clusters_visited}
    int* err = nullptr;              // set to 1 on a coincident source/target pair
    unsigned long long* warp_cost = nullptr;  // count pass: sampled warps' work estimates (integer)
    int out_batch = 0;               // 1: write out / per_target in batch order (slot t), not torig[t]
    int* work = nullptr;             // persistent kernels: next batch counter (zeroed per launch)
    // far events accepted by <= sparse_max lanes of a warp are evaluated by the packed
    // pass (k_feval) instead of the warp's event list (k_far_list); 0 disables
    int sparse_max = 0;
};

// One far order: its folded weights (P = p + 2 with stresslets, else p + 1), a buffer for
// the dense far sums (nt x 3, batch order) and the output.
struct FarOrder {
    int P = 0;
    const double* W = nullptr;
    double* ufar = nullptr;
    double* out = nullptr;
};
struct EvalTimes {
    double near_s = 0.0;            // k_neval (all slabs)
    double far_s = 0.0;             // k_far_list + k_feval (all slabs and orders)
    std::vector<double> far_order;  // the same per order
    cudaEvent_t origin = nullptr;   // if set: start of the first near / far launch after it
    double near_start_s = 0.0, far_start_s = 0.0;
    // ST_DEBUG_TIMELINE: ms from `origin` at the plan's steps (count walk done, plan sized
    // on the host, write walk done)
    std::vector<std::pair<const char*, double>> plan_ms;
    std::vector<double> plan_host_ms;  // host clock at the same marks, from launch_eval's entry
};
// K3-K5 for the batch warps [a.w0, a.w1): the plan walks (counts, then near entries,
// deferred sparse far entries and each warp's dense far events), then per slab the dense
// far field of every order, the near field once, the packed sparse far events and the
// reduce per order (original order unless a.out_batch); counters into a.stats and
// a.per_target.  Synchronises the stream before returning.
// far_ready (if set): the orders' weights W are produced on another stream; the far
// kernels wait for it (they run after the near field's evaluation).
// before_far (if set): called once, after the first slab's near field is queued and
// before any far kernel (also for an empty shard): the split moment pass completes W
// there (exchange with the other ranks, top levels; capi.cu run_treecode).
// src_ready (if set): the source records a.src are written on another stream; the near
// field's evaluation waits for it (the plan walks before it do not read them).
void launch_eval(bool sto, bool str, const TravArgs& a, const FarOrder* orders, int n_orders, cudaStream_t s,
                 EvalTimes* times = nullptr, cudaEvent_t far_ready = nullptr,
                 const std::function<void()>* before_far = nullptr, cudaEvent_t src_ready = nullptr);
// Interaction lists (pre-order cluster ids, DFS order) of the targets in a.tx.
void launch_lists(const TravArgs& a, int cap, int32_t* far, int32_t* near, int64_t* nfar, int64_t* nnear,
                  cudaStream_t s);
// Traversal-only work estimate of every count_stride(w)-th warp of [a.w0, a.w1) into
// a.warp_cost[(warp - w0) / stride] (for multi-GPU shard cuts; each sample stands for the
// stride warps from it).  Integer units: a dense far event costs 24 x 8 (P+1)^2 (~its warp DP
// instructions), a sparse one (na lanes) 8 (P+1)^2 na (its packed share), a near (lane,
// source) pair 24.  Integers make every prefix sum exact, so the cut is the same however it
// is summed.
constexpr int kCountStride = 4;
// every count_stride(w)-th of w batch warps is walked for the shard cuts: at least every
// 4th, at most ~8K samples (the per-warp cost is smooth along the key order)
// ST_COUNT_SAMPLES overrides the ~8K sampled warps (A/B of the multi-GPU cut cost).
inline int count_samples() {
    static const int v = [] {
        const char* e = getenv("ST_COUNT_SAMPLES");
        const int k = e ? atoi(e) : 8192;
        return k > 0 ? k : 8192;
    }();
    return v;
}
inline int count_stride(int warps) {
    return warps / count_samples() > kCountStride ? warps / count_samples() : kCountStride;
}
void launch_count(const TravArgs& a, uint32_t far_cost, cudaStream_t s);
// Work-balanced contiguous cuts of the warps [0, nwarps) into k shards from the samples
// (sample g = warps [g stride, min((g+1) stride, nwarps))), on the device: cut s is the
// first warp i with prefix(i) + w(i) / 2 >= s total / k (shard_cuts_host's rule, in exact
// integers).  cuts[0..k] (int32).
void launch_shard_cuts(const unsigned long long* samples, int nwarps, int stride, int k, int* cuts,
                       cudaStream_t s);

// O(N^2) contracted direct sum (kernels.hpp:45-83, 123-150): sources are the
// original-order records [n][12]; targets are source indices (self skipped).
void launch_direct(bool sto, bool str, const double* rec, size_t n, const int64_t* tgt, size_t nt,
                   double* u, int* err, cudaStream_t s);
// naive_direct_velocity (kernels.hpp:89-118): tensors S, T formed per pair.
void launch_naive(bool sto, bool str, const double* rec, size_t n, double* u, int* err,
                  cudaStream_t s);

// Per-pair far-field API: n pairs, pair i uses dx[3i..] and weight block i.
// Reserves / frees device `dev`'s near-field entry workspace (ensure_device /
// st_release_workspace).
void reserve_near_workspace(int dev, size_t bytes);
void release_near_workspace(int dev);
void launch_far_pairs(int P, size_t n, const double* dx, const double* W, double* u, cudaStream_t s);
// Reference-order Coulomb coefficients b^k, |k| <= pmax (coulomb.hpp:28-50).
void launch_coulomb(size_t n, const double* dx, int pmax, double* b, cudaStream_t s);
void launch_taylor(size_t n, const double* dx, const double* b, int pmax_b, int order, double* asto,
                   double* astr, cudaStream_t s);

}  // namespace st
