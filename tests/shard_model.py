"""Host restatement of the multi-GPU planning of the CUDA path (test infrastructure).

* batch order: 30-bit octree keys of the targets (ten levels of bisection of the root
  cube of their tight box, x in the low bit of each level's digit), stably sorted
  (csrc/tree.cu order_targets / k_geokey and the tree build's own key sort; CUB radix
  sort on the keys, original index as the tie order);
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


KEY_LEVELS = 10      # tree.cu kKeyLevels


def key_batch_order(xyz):
    """batch position -> original target index: the stable order of the 30-bit octree keys
    (tree.cu k_geokey: ten bisections of the root cube of the points' tight box, k_root;
    cluster_tree.hpp:99-105, 163-169, in the same rounded arithmetic)."""
    xyz = np.asarray(xyz, np.float64)
    lo, hi = xyz.min(axis=0), xyz.max(axis=0)
    side = 0.0
    for a in range(3):
        ext = hi[a] - lo[a]
        side = ext if side < ext else side
    side = side * (1.0 + 1e-12)
    half = side * 0.5
    blo = np.empty(3)
    bhi = np.empty(3)
    for a in range(3):
        c = (lo[a] + hi[a]) * 0.5
        blo[a], bhi[a] = c - half, c + half
    n = len(xyz)
    key = np.zeros(n, np.uint64)
    L = np.tile(blo, (n, 1))
    H = np.tile(bhi, (n, 1))
    for _ in range(KEY_LEVELS):
        slot = np.zeros(n, np.uint64)
        for a in range(3):
            mid = (L[:, a] + H[:, a]) * 0.5
            up = xyz[:, a] >= mid
            slot |= up.astype(np.uint64) << np.uint64(a)
            L[:, a] = np.where(up, mid, L[:, a])
            H[:, a] = np.where(up, H[:, a], mid)
        key = (key << np.uint64(3)) | slot
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
