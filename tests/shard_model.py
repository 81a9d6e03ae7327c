"""Host restatement of the multi-GPU planning of the CUDA path (test infrastructure).

* batch order: 63-bit Morton keys of the targets in their tight box, stably sorted
  (csrc/tree.cu order_targets / k_morton: 21 bits per axis, x in the top bit of each
  triple; CUB radix sort on the keys, original index as the tie order);
* per-warp cost of the shard cuts: csrc/traverse.cu k_count in exact integers: an
  accepted cluster costs 24 cf, cf = 8 (P+1)^2, when more than `sparse_max` lanes accept
  it, cf * lanes otherwise; a near leaf costs 24 * lanes * leaf size; every stride-th warp
  is walked and the others take the preceding sample's cost;
* cuts: st_shard_cuts (the library's host function) on those costs -- the same rule that
  k_shard_cuts evaluates on the device (capi.cu run_treecode).

tests/test_multirank.py shards with it on CPU (gloo); tests/test_gpu_parity.py checks it
against the library's own batch order and shard ranges on a GPU."""
import numpy as np

COUNT_STRIDE = 4      # traverse.cuh kCountStride
SPARSE_MAX = 24       # capi.cu far_sparse_max() default


def _spread21(v):
    v = v.astype(np.uint64) & np.uint64(0x1FFFFF)
    for shift, mask in ((32, 0x1F00000000FFFF), (16, 0x1F0000FF0000FF), (8, 0x100F00F00F00F00F),
                        (4, 0x10C30C30C30C30C3), (2, 0x1249249249249249)):
        v = (v | (v << np.uint64(shift))) & np.uint64(mask)
    return v


def morton_batch_order(xyz):
    """batch position -> original target index."""
    xyz = np.asarray(xyz, np.float64)
    lo, hi = xyz.min(axis=0), xyz.max(axis=0)
    side = 0.0
    for a in range(3):
        side = max(side, hi[a] - lo[a])
    inv = 2097151.0 / side if side > 0.0 else 0.0
    key = np.zeros(len(xyz), np.uint64)
    for a in range(3):
        q = np.minimum(np.maximum((xyz[:, a] - lo[a]) * inv, 0.0), 2097151.0).astype(np.uint64)
        key |= _spread21(q) << np.uint64(2 - a)
    return np.argsort(key, kind="stable").astype(np.int64)


def count_stride(warps):
    return warps // 8192 if warps // 8192 > COUNT_STRIDE else COUNT_STRIDE


def warp_costs(order, far_lists, near_lists, leaf_size, P, sparse_max=SPARSE_MAX):
    """k_count's per-warp cost for the batch order `order` (per-target far / near lists in
    original target order; leaf_size[c] = end - begin of cluster c), in its integer units:
    a dense far event 24 x 8 (P+1)^2, a sparse one 8 (P+1)^2 x its lanes, a near (lane,
    source) pair 24.  Every count_stride-th warp is sampled; the warps after a sample
    take its cost."""
    nt = len(order)
    nw = (nt + 31) // 32
    cf = (P + 1) * (P + 1) * 8
    stride = count_stride(nw)
    cost = np.zeros(nw, np.int64)
    for w in range(0, nw, stride):
        nacc, nleaf = {}, {}
        for t in order[32 * w:32 * w + 32]:
            for c in far_lists[t]:
                nacc[int(c)] = nacc.get(int(c), 0) + 1
            for c in near_lists[t]:
                nleaf[int(c)] = nleaf.get(int(c), 0) + 1
        acc = 0
        for c in set(nacc) | set(nleaf):
            na, nl = nacc.get(c, 0), nleaf.get(c, 0)
            if na:
                acc += 24 * cf if na > sparse_max else cf * na
            if nl:
                acc += 24 * nl * int(leaf_size[c])
        cost[w] = acc
    for w in range(nw):
        if w % stride:
            cost[w] = cost[w - w % stride]
    return cost.astype(np.float64)
