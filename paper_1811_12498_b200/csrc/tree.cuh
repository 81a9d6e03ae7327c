// K1: device octree build, bit-exact with build_tree (cluster_tree.hpp:152-192).
#pragma once

#include <vector>

#include "st_common.cuh"

namespace st {

// Cluster tree in pre-order (id 0 = root), device resident.
struct DevTree {
    size_t n = 0;
    int ncl = 0;
    int depth = 0;
    DevArray<double4> geom;      // center xyz, radius
    DevArray<int4> info;         // begin, end, next (pre-order id after the subtree), is_leaf
    DevArray<double> bbox;       // lo xyz, hi xyz per cluster
    DevArray<int32_t> children;  // 8 per cluster, pre-order ids, -1 padded
    DevArray<int32_t> nchild;    // n_children
    DevArray<uint32_t> perm;     // tree index -> original index (to_original)
    DevArray<uint32_t> to_tree;  // original index -> tree index (the inverse of perm)
    DevArray<int32_t> bylevel;   // pre-order ids in breadth-first (level) order
    std::vector<int> level_start;  // host: bylevel[level_start[d] .. level_start[d+1]) = depth d
};

// Builds the tree of n points (xyz interleaved, device) with leaf capacity n0.
// geometry=false skips bbox/center/radius (used for the target ordering tree).
// key_order (optional): the points' octree-key order (below), when the build made it on the
// way (left empty otherwise) -- the batch order of the same points as targets.
void build_tree_device(const double* d_pos, size_t n, int n0, bool shrink, bool geometry,
                       cudaStream_t s, DevTree& out, DevArray<uint32_t>* key_order = nullptr);

// Batch order of n points (device, xyz): stable order of their 30-bit octree keys (ten
// levels of bisection of the root cube of their tight box, cluster_tree.hpp:163-169, the
// tree build's own first levels); perm[i] is the original index of the i-th point.
// Stream-ordered, no host synchronisation.
void order_targets(const double* d_pos, size_t n, cudaStream_t s, DevArray<uint32_t>& perm);

}  // namespace st
