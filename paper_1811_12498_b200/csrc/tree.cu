// K1: level-synchronous device octree build, bit-exact with the reference's
// recursive build_tree (cluster_tree.hpp:81-192).
//
// The reference recursion (pre-order emplace, geometric bisection with ties
// going up, stable counting-sort scatter, empty children pruned, leaf iff
// count <= N0 or depth >= 64) is equivalent to a breadth-first sequence of
// stable 8-way partitions of every still-splitting segment: particles keep
// their parent-range order inside each child, so the final order is the
// reference's tree order.  Each level is
//   seg_of -> slot + tile histogram -> column scan -> segment bases -> stable
//   scatter -> children records -> compaction of the next active level,
// followed by subtree sizes (bottom-up) and pre-order ids (top-down).
// The first kKeyLevels levels skip the per-level passes over all points: one radix
// sort of each point's octant digits (k_geokey) orders every node's range at once and a
// level's children come from binary searches (k_split_sorted); a second sort restores
// input order inside the leaves.  Levels below kKeyLevels use the partition passes.
// Geometry uses the reference's exact non-FMA expressions (__dadd_rn /
// __dmul_rn), and min / max / max-of-norm2 are order-free exact reductions.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <string>
#include <utility>
#include <vector>

#include "scan.cuh"
#include "tree.cuh"

#include <cooperative_groups.h>
#include <cub/device/device_radix_sort.cuh>

namespace cg = cooperative_groups;

namespace st {

namespace {

constexpr int kTile = 2048;      // elements per partition tile
constexpr int kTileThreads = 256;

__device__ __forceinline__ uint64_t ord_enc(double d) {
    const uint64_t b = static_cast<uint64_t>(__double_as_longlong(d));
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double ord_dec(uint64_t u) {
    const uint64_t b = (u >> 63) ? (u & 0x7fffffffffffffffull) : ~u;
    return __longlong_as_double(static_cast<long long>(b));
}

// norm2 as vec3.hpp:48-52 evaluates it: (a0*a0 + a1*a1) + a2*a2, no contraction.
__device__ __forceinline__ double norm2_rn(double a0, double a1, double a2) {
    return __dadd_rn(__dadd_rn(__dmul_rn(a0, a0), __dmul_rn(a1, a1)), __dmul_rn(a2, a2));
}

template <class T>
__device__ __forceinline__ T warp_min(T v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        T y = __shfl_xor_sync(0xffffffffu, v, o);
        v = y < v ? y : v;
    }
    return v;
}
template <class T>
__device__ __forceinline__ T warp_max(T v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        T y = __shfl_xor_sync(0xffffffffu, v, o);
        v = v < y ? y : v;
    }
    return v;
}

// tight box of all points (cluster_tree.hpp:58-69, 163) into ordered-int atomics.
__global__ void k_tight_all(const double* __restrict__ pos, size_t n,
                            unsigned long long* __restrict__ mm /* lo3 (min), hi3 (max) */) {
    uint64_t lo[3] = {~0ull, ~0ull, ~0ull}, hi[3] = {0, 0, 0};
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
         i += (size_t)gridDim.x * blockDim.x) {
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            const uint64_t e = ord_enc(pos[3 * i + a]);
            lo[a] = e < lo[a] ? e : lo[a];
            hi[a] = hi[a] < e ? e : hi[a];
        }
    }
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        lo[a] = warp_min(lo[a]);
        hi[a] = warp_max(hi[a]);
    }
    // one atomic per block and value (per-warp atomics on 6 addresses serialised)
    __shared__ uint64_t s_lo[32][3], s_hi[32][3];
    const int wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
    if ((threadIdx.x & 31) == 0)
        for (int a = 0; a < 3; ++a) {
            s_lo[wid][a] = lo[a];
            s_hi[wid][a] = hi[a];
        }
    __syncthreads();
    if (threadIdx.x < 3) {
        const int a = threadIdx.x;
        uint64_t l = ~0ull, h = 0;
        for (int w = 0; w < nw; ++w) {
            l = s_lo[w][a] < l ? s_lo[w][a] : l;
            h = h < s_hi[w][a] ? s_hi[w][a] : h;
        }
        atomicMin(&mm[a], (unsigned long long)l);
        atomicMax(&mm[3 + a], (unsigned long long)h);
    }
}

// Root cube (cluster_tree.hpp:163-169): side = max extent * (1 + 1e-12), centred
// on the tight box.  Writes BFS node 0.
__global__ void k_root(const unsigned long long* __restrict__ mm, uint32_t n, uint32_t* nb_begin,
                       uint32_t* nb_end, double* nb_box) {
    double lo[3], hi[3];
    for (int a = 0; a < 3; ++a) {
        lo[a] = ord_dec(mm[a]);
        hi[a] = ord_dec(mm[3 + a]);
    }
    double side = 0.0;
    for (int a = 0; a < 3; ++a) {
        const double ext = __dsub_rn(hi[a], lo[a]);
        side = side < ext ? ext : side;  // std::max(side, ext)
    }
    side = __dmul_rn(side, __dadd_rn(1.0, 1e-12));
    const double half = __dmul_rn(side, 0.5);
    for (int a = 0; a < 3; ++a) {
        const double c = __dmul_rn(__dadd_rn(lo[a], hi[a]), 0.5);
        nb_box[a] = __dsub_rn(c, half);
        nb_box[3 + a] = __dadd_rn(c, half);
    }
    nb_begin[0] = 0;
    nb_end[0] = n;
}

// Active segments of this level: range + geometric midpoint (cluster_tree.hpp:99).
__global__ void k_mkseg(const int32_t* __restrict__ act, int m, const uint32_t* __restrict__ nb_begin,
                        const uint32_t* __restrict__ nb_end, const double* __restrict__ nb_box,
                        uint32_t* seg_begin, uint32_t* seg_end, double* seg_mid) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= m) return;
    const int v = act[s];
    seg_begin[s] = nb_begin[v];
    seg_end[s] = nb_end[v];
    for (int a = 0; a < 3; ++a)
        seg_mid[3 * s + a] = __dmul_rn(__dadd_rn(nb_box[6 * v + a], nb_box[6 * v + 3 + a]), 0.5);
}

// Element -> active segment (segments are disjoint and sorted by begin).
__global__ void k_segof(uint32_t n, const uint32_t* __restrict__ seg_begin,
                        const uint32_t* __restrict__ seg_end, int m, int32_t* __restrict__ seg_of) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int lo = 0, hi = m - 1, found = -1;
    while (lo <= hi) {
        const int mid = (lo + hi) >> 1;
        if (seg_begin[mid] <= i) {
            found = mid;
            lo = mid + 1;
        } else {
            hi = mid - 1;
        }
    }
    seg_of[i] = (found >= 0 && i < seg_end[found]) ? found : -1;
}

// Octant slot, ties go to the upper child (cluster_tree.hpp:101-105), and per-tile
// histograms.  slot 8 marks elements outside every active segment.
__global__ void __launch_bounds__(kTileThreads)
    k_slot_hist(uint32_t n, const double* __restrict__ pos, const uint32_t* __restrict__ perm,
                const int32_t* __restrict__ seg_of, const double* __restrict__ seg_mid,
                uint8_t* __restrict__ slot8, uint32_t* __restrict__ blk_cnt) {
    // counts by warp ballots (lane k keeps the warp's count of slot k), one shared atomic
    // per warp and slot: 8 contended shared-memory counters per element were the kernel's
    // bottleneck
    __shared__ uint32_t cnt[8];
    if (threadIdx.x < 8) cnt[threadIdx.x] = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    uint32_t mine = 0;
    const uint32_t base = blockIdx.x * kTile;
    for (int r = 0; r < kTile / kTileThreads; ++r) {
        const uint32_t i = base + r * kTileThreads + threadIdx.x;
        uint8_t slot = 8;
        if (i < n) {
            const int s = seg_of[i];
            if (s >= 0) {
                const double* p = pos + 3 * (size_t)perm[i];
                const double* mid = seg_mid + 3 * s;
                slot = (p[0] >= mid[0] ? 1 : 0) | (p[1] >= mid[1] ? 2 : 0) | (p[2] >= mid[2] ? 4 : 0);
            }
            slot8[i] = slot;
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const unsigned b = __ballot_sync(0xffffffffu, slot == k);
            if (lane == k) mine += __popc(b);
        }
    }
    if (lane < 8 && mine) atomicAdd(&cnt[lane], mine);
    __syncthreads();
    if (threadIdx.x < 8) blk_cnt[blockIdx.x * 8 + threadIdx.x] = cnt[threadIdx.x];
}

// Global exclusive per-slot prefix P[pos][k] at both ends of every active segment
// (one warp per segment): seg_base[s][k] = P[begin][k], seg_cnt[s][k] = P[end][k] - P[begin][k].
__global__ void k_segbase(int m, const uint32_t* __restrict__ seg_begin,
                          const uint32_t* __restrict__ seg_end, const uint8_t* __restrict__ slot8,
                          const uint32_t* __restrict__ blk_off, uint32_t* __restrict__ seg_base,
                          uint32_t* __restrict__ seg_cnt) {
    const int s = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (s >= m) return;  // whole warps only; no block-level barrier below
    uint32_t P[2] = {0, 0};
    for (int which = 0; which < 2; ++which) {
        const uint32_t p = which ? seg_end[s] : seg_begin[s];
        const uint32_t tile = p / kTile;
        uint32_t c[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        for (uint32_t j = tile * kTile + lane; j < p; j += 32) {
            const uint8_t k = slot8[j];
#pragma unroll
            for (int q = 0; q < 8; ++q) c[q] += (k == q);
        }
        uint32_t mine = 0;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
#pragma unroll
            for (int o = 16; o; o >>= 1) c[q] += __shfl_xor_sync(0xffffffffu, c[q], o);
            if (q == lane) mine = c[q];
        }
        if (lane < 8) P[which] = blk_off[tile * 8 + lane] + mine;
    }
    if (lane < 8) {
        seg_base[s * 8 + lane] = P[0];
        seg_cnt[s * 8 + lane] = P[1] - P[0];
    }
}

// Stable scatter: new position = segment begin + child offset + stable rank.
__global__ void __launch_bounds__(kTileThreads)
    k_scatter(uint32_t n, const uint8_t* __restrict__ slot8, const int32_t* __restrict__ seg_of,
              const uint32_t* __restrict__ blk_off, const uint32_t* __restrict__ seg_begin,
              const uint32_t* __restrict__ seg_base, const uint32_t* __restrict__ seg_cnt,
              const uint32_t* __restrict__ perm_in, uint32_t* __restrict__ perm_out) {
    __shared__ uint32_t warp_cnt[kTileThreads / 32][8];
    __shared__ uint32_t run[8];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const unsigned lt = (1u << lane) - 1u;
    if (threadIdx.x < 8) run[threadIdx.x] = 0;
    const uint32_t base = blockIdx.x * kTile;
    for (int r = 0; r < kTile / kTileThreads; ++r) {
        const uint32_t i = base + r * kTileThreads + threadIdx.x;
        const uint8_t slot = i < n ? slot8[i] : 8;
        uint32_t rank_w = 0;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const unsigned msk = __ballot_sync(0xffffffffu, slot == k);
            if (lane == 0) warp_cnt[wid][k] = __popc(msk);
            if (slot == k) rank_w = __popc(msk & lt);
        }
        __syncthreads();
        uint32_t before = 0;
        if (slot < 8) {
            before = run[slot];
            for (int w = 0; w < wid; ++w) before += warp_cnt[w][slot];
        }
        __syncthreads();
        if (threadIdx.x < 8) {
            uint32_t t = 0;
            for (int w = 0; w < kTileThreads / 32; ++w) t += warp_cnt[w][threadIdx.x];
            run[threadIdx.x] += t;
        }
        if (i < n) {
            if (slot < 8) {
                const int s = seg_of[i];
                const uint32_t grank = blk_off[blockIdx.x * 8 + slot] + before + rank_w;
                uint32_t child_off = 0;
                for (int k = 0; k < slot; ++k) child_off += seg_cnt[s * 8 + k];
                const uint32_t np = seg_begin[s] + child_off + (grank - seg_base[s * 8 + slot]);
                perm_out[np] = perm_in[i];
            } else {
                perm_out[i] = perm_in[i];
            }
        }
        __syncthreads();
    }
}

__global__ void k_nch(int m, const uint32_t* __restrict__ seg_cnt, int32_t* __restrict__ nch) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= m) return;
    int c = 0;
    for (int k = 0; k < 8; ++k) c += seg_cnt[s * 8 + k] != 0;
    nch[s] = c;
}

// Child clusters in slot order (cluster_tree.hpp:125-137), empty slots pruned.
__global__ void k_children(int m, const int32_t* __restrict__ act, const uint32_t* __restrict__ seg_begin,
                           const uint32_t* __restrict__ seg_cnt, const int32_t* __restrict__ chbase,
                           int next_start, int n0, int child_depth, const double* box_in,
                           double* nb_box, uint32_t* __restrict__ nb_begin,
                           uint32_t* __restrict__ nb_end, int32_t* __restrict__ nb_first,
                           int32_t* __restrict__ nb_nch, int32_t* __restrict__ act_flag) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= m) return;
    const int v = act[s];
    double glo[3], ghi[3], mid[3];
    for (int a = 0; a < 3; ++a) {
        glo[a] = box_in[6 * v + a];
        ghi[a] = box_in[6 * v + 3 + a];
        mid[a] = __dmul_rn(__dadd_rn(glo[a], ghi[a]), 0.5);
    }
    uint32_t off = seg_begin[s];
    int c = next_start + chbase[s];
    nb_first[v] = c;
    nb_nch[v] = chbase[s + 1] - chbase[s];
    for (int k = 0; k < 8; ++k) {
        const uint32_t cnt = seg_cnt[s * 8 + k];
        if (!cnt) continue;
        for (int a = 0; a < 3; ++a) {
            const bool up = (k >> a) & 1;
            nb_box[6 * c + a] = up ? mid[a] : glo[a];
            nb_box[6 * c + 3 + a] = up ? ghi[a] : mid[a];
        }
        nb_begin[c] = off;
        nb_end[c] = off + cnt;
        nb_first[c] = -1;
        nb_nch[c] = 0;
        // cluster_tree.hpp:96: leaf iff count <= N0 or depth >= 64
        act_flag[c - next_start] = (cnt > (uint32_t)n0 && child_depth < 64) ? 1 : 0;
        off += cnt;
        ++c;
    }
}

__global__ void k_compact(int C, int next_start, const int32_t* __restrict__ flag,
                          const int32_t* __restrict__ pos, int32_t* __restrict__ act) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c < C && flag[c]) act[pos[c]] = next_start + c;
}

// subtree sizes, bottom-up one level per launch; with `mm`, also the tight boxes of the
// level's internal clusters from their children's
__global__ void k_subtree(int v0, int v1, const int32_t* __restrict__ first,
                          const int32_t* __restrict__ nch, int32_t* __restrict__ size,
                          unsigned long long* __restrict__ mm) {
    const int v = v0 + blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= v1) return;
    int s = 1;
    const int k = nch[v];
    for (int j = 0; j < k; ++j) s += size[first[v] + j];
    size[v] = s;
    if (mm && k) {
        uint64_t lo[3] = {~0ull, ~0ull, ~0ull}, hi[3] = {0ull, 0ull, 0ull};
        for (int j = 0; j < k; ++j) {
            const unsigned long long* c = mm + 6 * (size_t)(first[v] + j);
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                lo[a] = c[a] < lo[a] ? c[a] : lo[a];
                hi[a] = hi[a] < c[3 + a] ? c[3 + a] : hi[a];
            }
        }
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            mm[6 * (size_t)v + a] = lo[a];
            mm[6 * (size_t)v + 3 + a] = hi[a];
        }
    }
}

__global__ void k_preorder(int v0, int v1, const int32_t* __restrict__ first,
                           const int32_t* __restrict__ nch, const int32_t* __restrict__ size,
                           int32_t* __restrict__ pre) {
    const int v = v0 + blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= v1) return;
    if (v == 0) pre[0] = 0;
    int run = pre[v] + 1;
    for (int j = 0; j < nch[v]; ++j) {
        pre[first[v] + j] = run;
        run += size[first[v] + j];
    }
}

// bbox and centre = (lo + hi) * 0.5 (cluster_tree.hpp:15, 88-89).
__global__ void k_center(int T, int shrink, const unsigned long long* __restrict__ mm,
                         const double* __restrict__ nb_box, double* __restrict__ fbox,
                         double* __restrict__ center) {
    const int v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= T) return;
    for (int a = 0; a < 3; ++a) {
        const double lo = shrink ? ord_dec(mm[6 * v + a]) : nb_box[6 * v + a];
        const double hi = shrink ? ord_dec(mm[6 * v + 3 + a]) : nb_box[6 * v + 3 + a];
        fbox[6 * v + a] = lo;
        fbox[6 * v + 3 + a] = hi;
        center[3 * v + a] = __dmul_rn(__dadd_rn(lo, hi), 0.5);
    }
}

// to_tree[perm[t]] = t
__global__ void k_invperm(uint32_t n, const uint32_t* __restrict__ perm, uint32_t* __restrict__ to_tree) {
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t < n) to_tree[perm[t]] = t;
}

// positions in tree order, once, so the geometry passes over every level read them
// contiguously (they gathered 24-byte records through perm per level before)
__global__ void k_tree_pos(uint32_t n, const uint32_t* __restrict__ perm, const double* __restrict__ pos,
                           double* __restrict__ tpos) {
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    const double* p = pos + 3 * (size_t)perm[t];
    tpos[3 * (size_t)t] = p[0];
    tpos[3 * (size_t)t + 1] = p[1];
    tpos[3 * (size_t)t + 2] = p[2];
}

__global__ void k_finalize(int T, int geometry, const int32_t* __restrict__ pre,
                           const int32_t* __restrict__ size, const uint32_t* __restrict__ nb_begin,
                           const uint32_t* __restrict__ nb_end, const int32_t* __restrict__ nb_first,
                           const int32_t* __restrict__ nb_nch, const double* __restrict__ center,
                           const unsigned long long* __restrict__ r2max, const double* __restrict__ fbox,
                           double4* __restrict__ geom, int4* __restrict__ info, double* __restrict__ bbox,
                           int32_t* __restrict__ children, int32_t* __restrict__ nchild,
                           int32_t* __restrict__ bylevel) {
    const int v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= T) return;
    const int p = pre[v];
    bylevel[v] = p;
    const int nc = nb_nch[v];
    info[p] = make_int4((int)nb_begin[v], (int)nb_end[v], p + size[v], nc == 0 ? 1 : 0);
    nchild[p] = nc;
    for (int j = 0; j < 8; ++j) children[8 * p + j] = j < nc ? pre[nb_first[v] + j] : -1;
    if (geometry) {
        const double r = __dsqrt_rn(__longlong_as_double((long long)r2max[v]));
        geom[p] = make_double4(center[3 * v], center[3 * v + 1], center[3 * v + 2], r);
        for (int a = 0; a < 6; ++a) bbox[6 * p + a] = fbox[6 * v + a];
    }
}

// ---- keyed levels: one radix sort replaces the first kKeyLevels partition passes ----
//
// The reference's bisection is a pure function of the point and the root cube: at depth d
// the octant is decided against the midpoint of the depth-d box, whose bounds are the
// parent's bound or the parent's midpoint (cluster_tree.hpp:99-105, 125-137).  Each point
// descends kKeyLevels levels with the same rn arithmetic as k_children / k_mkseg and
// records its octant digits, most significant first.  A stable sort of these keys puts
// every depth-d node (d <= kKeyLevels) into one contiguous, slot-ordered range, so a
// level's children are found by binary search in the sorted keys instead of by a
// histogram + scatter pass over all n points.  Inside a node at depth kKeyLevels the
// points keep their input order (stable sort), which is what the partition passes
// continue from if a node there still splits.  Inside a leaf the reference keeps input
// order, which the key sort does not: k_leafkey + a second stable sort restore it.
constexpr int kKeyLevels = 10;  // 30-bit keys

__global__ void k_geokey(uint32_t n, const double* __restrict__ pos, const double* __restrict__ root_box,
                         uint32_t* __restrict__ key, uint32_t* __restrict__ idx) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double lo[3], hi[3], p[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        lo[a] = root_box[a];
        hi[a] = root_box[3 + a];
        p[a] = pos[3 * (size_t)i + a];
    }
    uint32_t k = 0;
#pragma unroll
    for (int d = 0; d < kKeyLevels; ++d) {
        uint32_t slot = 0;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            const double mid = __dmul_rn(__dadd_rn(lo[a], hi[a]), 0.5);
            const bool up = p[a] >= mid;
            slot |= (up ? 1u : 0u) << a;
            lo[a] = up ? mid : lo[a];
            hi[a] = up ? hi[a] : mid;
        }
        k = (k << 3) | slot;
    }
    key[i] = k;
    idx[i] = i;
}

// Children of the active segments at depth d < kKeyLevels from the sorted keys: 8 threads
// per segment, thread k finds the first position whose depth-d digit is >= k.
__global__ void k_split_sorted(int m, int d, const int32_t* __restrict__ act, const uint32_t* __restrict__ nb_begin,
                               const uint32_t* __restrict__ nb_end, const uint32_t* __restrict__ skey,
                               uint32_t* __restrict__ seg_begin, uint32_t* __restrict__ seg_cnt) {
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    const int s = g >> 3, k = g & 7;
    const bool live = s < m;
    const int v = live ? act[s] : 0;
    const uint32_t b = live ? nb_begin[v] : 0, e = live ? nb_end[v] : 0;
    const int sh = 3 * (kKeyLevels - 1 - d);
    uint32_t lo = b, hi = e;  // first t in [b, e) with digit(t) >= k, else e
    while (lo < hi) {
        const uint32_t mid = lo + ((hi - lo) >> 1);
        if ((int)((skey[mid] >> sh) & 7u) < k) lo = mid + 1;
        else hi = mid;
    }
    // the next slot's start (lane k + 1 of the same 8-group; e after slot 7)
    const uint32_t nxt = __shfl_down_sync(0xffffffffu, lo, 1, 8);
    if (!live) return;
    const uint32_t end_k = k == 7 ? e : nxt;
    seg_cnt[8 * s + k] = end_k - lo;
    if (k == 0) seg_begin[s] = b;
}

// All keyed levels in one cooperative launch (no host round trip per level).  Every block
// walks the levels in lockstep, grid-wide barriers between the phases of a level:
//   A  8 threads per active segment binary-search its children's ranges (k_split_sorted)
//   B  block 0: child counts -> exclusive scan over the segments (chbase), C
//   C  children records and next-level flags (k_children)
//   D  block 0: scan of the flags -> next active list, level bookkeeping
// Sizes are bounded up front: an active segment holds more than n0 points, so a level has
// at most mcap = n / (n0 + 1) of them and at most 8 mcap children.
struct KeyedLevels {
    int n0 = 0;
    int mcap = 0, tcap = 0;
    const uint32_t* skey = nullptr;
    uint32_t* nb_begin = nullptr;
    uint32_t* nb_end = nullptr;
    double* nb_box = nullptr;
    int32_t* nb_first = nullptr;
    int32_t* nb_nch = nullptr;
    int32_t* act[2] = {nullptr, nullptr};  // ping-pong active lists [mcap]
    uint32_t* seg_cnt = nullptr;           // [8 mcap]
    int32_t* chbase = nullptr;             // [mcap + 1]
    int32_t* flag = nullptr;               // [8 mcap + 1] (exclusive scan in place)
    int32_t* state = nullptr;              // m, total, depth, which act, overflow, level_start[kKeyLevels + 2]
};
constexpr int kKeyThreads = 512;
enum { KS_M = 0, KS_TOTAL, KS_DEPTH, KS_ACT, KS_OVER, KS_LS };

// block-wide exclusive scan of int32 values in place over [0, cnt); returns the total
__device__ int block_scan_inplace(int32_t* a, int cnt, int32_t* sh) {
    const int per = (cnt + kKeyThreads - 1) / kKeyThreads;
    const int i0 = min(cnt, (int)threadIdx.x * per), i1 = min(cnt, i0 + per);
    int sum = 0;
    for (int i = i0; i < i1; ++i) sum += a[i];
    sh[threadIdx.x] = sum;
    __syncthreads();
    for (int o = 1; o < kKeyThreads; o <<= 1) {
        const int y = threadIdx.x >= (unsigned)o ? sh[threadIdx.x - o] : 0;
        __syncthreads();
        sh[threadIdx.x] += y;
        __syncthreads();
    }
    int run = sh[threadIdx.x] - sum;
    for (int i = i0; i < i1; ++i) {
        const int x = a[i];
        a[i] = run;
        run += x;
    }
    const int total = sh[kKeyThreads - 1];
    __syncthreads();
    return total;
}

__global__ void __launch_bounds__(kKeyThreads) k_keyed_levels(const KeyedLevels K) {
    cg::grid_group grid = cg::this_grid();
    __shared__ int32_t sh[kKeyThreads];
    const int gtid = blockIdx.x * blockDim.x + threadIdx.x, gsz = gridDim.x * blockDim.x;
    for (;;) {
        const int m = *(volatile int32_t*)&K.state[KS_M];
        const int depth = *(volatile int32_t*)&K.state[KS_DEPTH];
        const int total = *(volatile int32_t*)&K.state[KS_TOTAL];
        const int32_t* act = K.act[*(volatile int32_t*)&K.state[KS_ACT]];
        int32_t* act2 = K.act[1 - *(volatile int32_t*)&K.state[KS_ACT]];
        if (m == 0 || depth >= kKeyLevels || K.state[KS_OVER]) break;
        // A: child ranges
        const int sh3 = 3 * (kKeyLevels - 1 - depth);
        for (int g = gtid; g < 8 * m; g += gsz) {
            const int sg = g >> 3, k = g & 7;
            const int v = act[sg];
            uint32_t lo = K.nb_begin[v], hi = K.nb_end[v];
            while (lo < hi) {
                const uint32_t mid = lo + ((hi - lo) >> 1);
                if ((int)((K.skey[mid] >> sh3) & 7u) < k) lo = mid + 1;
                else hi = mid;
            }
            K.seg_cnt[g] = lo;  // start of slot k; counts in B
        }
        grid.sync();
        // B: counts, children per segment, exclusive scan
        if (blockIdx.x == 0) {
            for (int sg = threadIdx.x; sg < m; sg += blockDim.x) {
                const uint32_t e = K.nb_end[act[sg]];
                int c = 0;
                for (int k = 0; k < 8; ++k) {
                    const uint32_t st = K.seg_cnt[8 * sg + k], en = k == 7 ? e : K.seg_cnt[8 * sg + k + 1];
                    c += en > st;
#ifdef ST_DEBUG_CHECKS
                    // slot ranges tile the parent's range in slot order (debug builds)
                    if (en < st || (k == 0 && st != K.nb_begin[act[sg]])) K.state[KS_OVER] = 2;
#endif
                }
                K.chbase[sg] = c;
            }
            __syncthreads();
            const int C = block_scan_inplace(K.chbase, m, sh);
            if (threadIdx.x == 0) {
                K.chbase[m] = C;
                if (total + C > K.tcap || C > 8 * K.mcap) K.state[KS_OVER] = 1;
            }
        }
        grid.sync();
        if (K.state[KS_OVER]) break;
        const int C = K.chbase[m];
        // C: children records (cluster_tree.hpp:125-137), flags of the next level's splits
        for (int sg = gtid; sg < m; sg += gsz) {
            const int v = act[sg];
            double glo[3], ghi[3], mid[3];
            for (int a = 0; a < 3; ++a) {
                glo[a] = K.nb_box[6 * v + a];
                ghi[a] = K.nb_box[6 * v + 3 + a];
                mid[a] = __dmul_rn(__dadd_rn(glo[a], ghi[a]), 0.5);
            }
            const uint32_t e = K.nb_end[v];
            int c = total + K.chbase[sg];
            K.nb_first[v] = c;
            K.nb_nch[v] = K.chbase[sg + 1] - K.chbase[sg];
            for (int k = 0; k < 8; ++k) {
                const uint32_t st = K.seg_cnt[8 * sg + k], en = k == 7 ? e : K.seg_cnt[8 * sg + k + 1];
                if (en <= st) continue;
                for (int a = 0; a < 3; ++a) {
                    const bool up = (k >> a) & 1;
                    K.nb_box[6 * c + a] = up ? mid[a] : glo[a];
                    K.nb_box[6 * c + 3 + a] = up ? ghi[a] : mid[a];
                }
                K.nb_begin[c] = st;
                K.nb_end[c] = en;
                K.nb_first[c] = -1;
                K.nb_nch[c] = 0;
                // cluster_tree.hpp:96: leaf iff count <= N0 or depth >= 64
                K.flag[c - total] = (en - st > (uint32_t)K.n0 && depth + 1 < 64) ? 1 : 0;
                ++c;
            }
        }
        grid.sync();
        // D: next active list
        if (blockIdx.x == 0) {
            const int m2 = block_scan_inplace(K.flag, C, sh);
            for (int c = threadIdx.x; c < C; c += blockDim.x) {
                const int next = c + 1 < C ? K.flag[c + 1] : m2;
                if (next > K.flag[c]) act2[K.flag[c]] = total + c;
            }
            if (threadIdx.x == 0) {
                K.state[KS_LS + depth + 1] = total;
                K.state[KS_TOTAL] = total + C;
                K.state[KS_DEPTH] = depth + 1;
                K.state[KS_M] = m2;
                K.state[KS_ACT] = 1 - K.state[KS_ACT];
            }
        }
        grid.sync();
    }
}

// Leaf key of every point: the leaf's pre-order id (leaves in pre-order = tree order),
// stored at the point's input index.  One warp per cluster; internal clusters skip.
__global__ void k_leafkey(int T, const int32_t* __restrict__ nb_nch, const uint32_t* __restrict__ nb_begin,
                          const uint32_t* __restrict__ nb_end, const int32_t* __restrict__ pre,
                          const uint32_t* __restrict__ perm, uint32_t* __restrict__ lkey) {
    const int v = (int)((blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5);
    if (v >= T || nb_nch[v] != 0) return;
    const uint32_t key = (uint32_t)pre[v];
    for (uint32_t t = nb_begin[v] + (threadIdx.x & 31); t < nb_end[v]; t += 32) lkey[perm[t]] = key;
}

// ---- geometry ----
// Tight boxes: one pass over the points for the leaves, then each level from its children
// (min / max are exact and order-free, so a parent's box is its children's).  Points are
// in tree order, so the lanes of a warp that share a leaf are consecutive: a segmented
// reduction towards the run's first lane (shuffle down, kept while the neighbour is in the
// same leaf) leaves one atomic per run.  Radii (which need every point again, against the
// cluster's own centre) go by fixed-size chunks of each cluster's range.
// leaf_of[t] = the leaf (BFS id) holding tree position t; one warp per cluster
__global__ void k_leaf_of(int T, const int32_t* __restrict__ nb_nch, const uint32_t* __restrict__ nb_begin,
                          const uint32_t* __restrict__ nb_end, int32_t* __restrict__ leaf_of) {
    const int v = (int)((blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5);
    if (v >= T || nb_nch[v] != 0) return;
    for (uint32_t t = nb_begin[v] + (threadIdx.x & 31); t < nb_end[v]; t += 32) leaf_of[t] = v;
}

// segmented reduction over runs of equal `key` (consecutive lanes); returns true on a
// run's first lane, which then holds the run's reduction
template <class T, class Op>
__device__ __forceinline__ bool seg_reduce(int key, T& v, Op op) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const T y = __shfl_down_sync(0xffffffffu, v, o);
        const int k = __shfl_down_sync(0xffffffffu, key, o);
        if (lane + o < 32 && k == key) v = op(v, y);
    }
    const int prev = __shfl_up_sync(0xffffffffu, key, 1);
    return lane == 0 || prev != key;
}

// tight boxes of the leaves (cluster_tree.hpp:88)
__global__ void __launch_bounds__(256) k_leaf_minmax(uint32_t n, const double* __restrict__ tpos,
                                                     const int32_t* __restrict__ leaf_of,
                                                     unsigned long long* __restrict__ mm) {
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    uint64_t lo[3] = {~0ull, ~0ull, ~0ull}, hi[3] = {0ull, 0ull, 0ull};
    int v = -1;
    if (t < n) {
        v = leaf_of[t];
#pragma unroll
        for (int a = 0; a < 3; ++a) lo[a] = hi[a] = ord_enc(tpos[3 * (size_t)t + a]);
    }
    auto mn = [](uint64_t x, uint64_t y) { return y < x ? y : x; };
    auto mx = [](uint64_t x, uint64_t y) { return x < y ? y : x; };
    bool head = false;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        head = seg_reduce(v, lo[a], mn);
        seg_reduce(v, hi[a], mx);
    }
    if (head && v >= 0) {
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            atomicMin(&mm[6 * v + a], (unsigned long long)lo[a]);
            atomicMax(&mm[6 * v + 3 + a], (unsigned long long)hi[a]);
        }
    }
}

constexpr int kGeomChunk = 4096;  // points per radius work item

__global__ void k_nchunk(int T, const uint32_t* __restrict__ b, const uint32_t* __restrict__ e,
                         int32_t* __restrict__ nck) {
    const int v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v < T) nck[v] = (int32_t)((e[v] - b[v] + kGeomChunk - 1) / kGeomChunk);
}

// radius^2 = max over the cluster of norm2(p - c) (cluster_tree.hpp:90-93); non-negative
// doubles order like their bit patterns, so u64 atomicMax is exact.  One block per chunk of
// a cluster's range; the grid is an upper bound of the chunk count (no host round trip),
// blocks past item_off[T] exit.
__global__ void __launch_bounds__(256) k_radius(int T, const int32_t* __restrict__ item_off,
                                                const uint32_t* __restrict__ nb_begin,
                                                const uint32_t* __restrict__ nb_end,
                                                const double* __restrict__ tpos,
                                                const double* __restrict__ center,
                                                unsigned long long* __restrict__ r2max) {
    const int item = blockIdx.x;
    if (item >= item_off[T]) return;
    int lo = 0, hi = T - 1;  // the cluster whose chunks hold `item`
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (item_off[mid] <= item) lo = mid;
        else hi = mid - 1;
    }
    const int v = lo;
    const uint32_t b = nb_begin[v] + (uint32_t)(item - item_off[v]) * kGeomChunk;
    const uint32_t e = min(nb_end[v], b + kGeomChunk);
    const double c0 = center[3 * v], c1 = center[3 * v + 1], c2 = center[3 * v + 2];
    uint64_t m = 0;
    for (uint32_t t = b + threadIdx.x; t < e; t += blockDim.x) {
        const double* p = tpos + 3 * (size_t)t;
        const double r2 = norm2_rn(__dsub_rn(p[0], c0), __dsub_rn(p[1], c1), __dsub_rn(p[2], c2));
        const uint64_t q = static_cast<uint64_t>(__double_as_longlong(r2));
        m = m < q ? q : m;
    }
    m = warp_max(m);
    if ((threadIdx.x & 31) == 0) atomicMax(&r2max[v], (unsigned long long)m);
}

__global__ void k_iota(uint32_t* p, uint32_t n) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) p[i] = i;
}

__global__ void k_zero_hi(unsigned long long* mm, int T) {
    const int v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v < T) mm[6 * v + 3] = mm[6 * v + 4] = mm[6 * v + 5] = 0ull;
}

template <class T>
void grow(DevArray<T>& a, size_t need, size_t used, cudaStream_t s) {
    if (a.size() >= need) return;
    size_t cap = std::max<size_t>(need, a.size() * 2);
    DevArray<T> b(cap, s);
    if (used) ST_CUDA(cudaMemcpyAsync(b.get(), a.get(), used * sizeof(T), cudaMemcpyDeviceToDevice, s));
    a = std::move(b);
}

inline unsigned blocks(size_t n, int t) { return (unsigned)((n + t - 1) / t); }

}  // namespace

void build_tree_device(const double* d_pos, size_t n_sz, int n0, bool shrink, bool geometry,
                       cudaStream_t s, DevTree& out, DevArray<uint32_t>* key_order) {
    if (n_sz == 0) fail(ST_INVALID_ARGUMENT, "build_tree: empty particle set");
    if (n0 < 1) fail(ST_INVALID_ARGUMENT, "build_tree: leaf capacity must be >= 1");
    if (n_sz >= 0x7fffffffull) fail(ST_INVALID_ARGUMENT, "build_tree: more than 2^31-1 particles");
    const uint32_t n = (uint32_t)n_sz;
    const int ntiles = (int)blocks(n, kTile);
    // ST_DEBUG_BUILD=1: device-time marks of the build's phases (stderr)
    static const bool dbg = getenv("ST_DEBUG_BUILD") != nullptr;
    std::vector<std::pair<const char*, Event>> marks;
    std::vector<double> host_ms;  // host clock at each mark (is the GPU waiting for the host?)
    const auto h0 = std::chrono::steady_clock::now();
    auto mark = [&](const char* what) {
        if (!dbg) return;
        marks.emplace_back(what, Event());
        marks.back().second.record(s);
        host_ms.push_back(std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - h0).count());
    };
    mark("start");

    // BFS node storage (grown per level)
    size_t cap = 64;
    DevArray<uint32_t> nb_begin(cap, s), nb_end(cap, s);
    DevArray<double> nb_box(6 * cap, s);
    DevArray<int32_t> nb_first(cap, s), nb_nch(cap, s);

    DevArray<unsigned long long> mm(6, s);
    {
        ST_CUDA(cudaMemsetAsync(mm.get(), 0xff, 3 * sizeof(unsigned long long), s));
        ST_CUDA(cudaMemsetAsync(mm.get() + 3, 0x00, 3 * sizeof(unsigned long long), s));
        const unsigned g = std::min<unsigned>(blocks(n, 256), 148 * 8);
        k_tight_all<<<g, 256, 0, s>>>(d_pos, n, mm.get());
        ST_LAUNCH("k_tight_all");
        k_root<<<1, 1, 0, s>>>(mm.get(), n, nb_begin.get(), nb_end.get(), nb_box.get());
        ST_LAUNCH("k_root");
        count_launch(2);
    }
    // root: first/nch = leaf until split
    ST_CUDA(cudaMemsetAsync(nb_first.get(), 0xff, sizeof(int32_t), s));
    ST_CUDA(cudaMemsetAsync(nb_nch.get(), 0, sizeof(int32_t), s));

    // keyed levels (k_geokey): ST_TREE_PARTITION=1 forces the partition passes from the root
    static const bool partition_only = getenv("ST_TREE_PARTITION") != nullptr;
    const bool keyed = !partition_only && n > (uint32_t)n0;
    DevArray<uint32_t> perm(n, s), perm2, skey;
    if (keyed) {
        DevArray<uint32_t> key(n, s), idx(n, s);
        skey.alloc(n, s);
        k_geokey<<<blocks(n, 256), 256, 0, s>>>(n, d_pos, nb_box.get(), key.get(), idx.get());
        ST_LAUNCH("k_geokey");
        size_t tmp = 0;
        ST_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, key.get(), skey.get(), idx.get(), perm.get(), (int)n, 0,
                                                3 * kKeyLevels, s));
        DevArray<char> scratch(tmp, s);
        ST_CUDA(cub::DeviceRadixSort::SortPairs(scratch.get(), tmp, key.get(), skey.get(), idx.get(), perm.get(),
                                                (int)n, 0, 3 * kKeyLevels, s));
        count_launch(1 + 5);  // + the sort's passes
    } else {
        k_iota<<<blocks(n, 256), 256, 0, s>>>(perm.get(), n);  // cluster_tree.hpp:160-161
        ST_LAUNCH("k_iota");
        count_launch();
    }
    mark("root");

    // partition-pass state, allocated only if a level below the keyed ones splits
    DevArray<int32_t> seg_of;
    DevArray<uint8_t> slot8;
    DevArray<uint32_t> blk_cnt, blk_off;

    std::vector<int> level_start{0};
    int total = 1;
    int m = n > (uint32_t)n0 ? 1 : 0;
    DevArray<int32_t> act(std::max(m, 1), s);
    if (m) ST_CUDA(cudaMemsetAsync(act.get(), 0, sizeof(int32_t), s));
    int depth = 0;
    bool deep = false;

    // the keyed levels in one cooperative launch when their sizes are bounded (mcap: at most
    // n / (n0 + 1) splitting segments per level); ST_TREE_LEVEL_LOOP=1 keeps the per-level
    // host loop below
    static const bool level_loop = getenv("ST_TREE_LEVEL_LOOP") != nullptr;
    const long long mcap_ll = (long long)n / ((long long)n0 + 1) + 1;
    if (keyed && m && !level_loop && mcap_ll <= 65536) {
        const int mcap = (int)mcap_ll;
        const int tcap = 1 + 8 * kKeyLevels * mcap;
        grow(nb_begin, tcap, total, s);
        grow(nb_end, tcap, total, s);
        grow(nb_first, tcap, total, s);
        grow(nb_nch, tcap, total, s);
        grow(nb_box, 6 * (size_t)tcap, 6 * (size_t)total, s);
        DevArray<int32_t> actb[2] = {DevArray<int32_t>(mcap, s), DevArray<int32_t>(mcap, s)};
        DevArray<uint32_t> kseg((size_t)8 * mcap, s);
        DevArray<int32_t> kch(mcap + 1, s), kflag((size_t)8 * mcap + 1, s), kst(KS_LS + kKeyLevels + 2, s);
        constexpr int NS = KS_LS + kKeyLevels + 2;
        int32_t* st0 = static_cast<int32_t*>(pinned_stage(NS * sizeof(int32_t)));
        memset(st0, 0, NS * sizeof(int32_t));
        st0[KS_M] = 1;
        st0[KS_TOTAL] = 1;
        ST_CUDA(cudaMemcpyAsync(kst.get(), st0, NS * sizeof(int32_t), cudaMemcpyHostToDevice, s));
        ST_CUDA(cudaMemsetAsync(actb[0].get(), 0, sizeof(int32_t), s));
        KeyedLevels K;
        K.n0 = n0;
        K.mcap = mcap;
        K.tcap = tcap;
        K.skey = skey.get();
        K.nb_begin = nb_begin.get();
        K.nb_end = nb_end.get();
        K.nb_box = nb_box.get();
        K.nb_first = nb_first.get();
        K.nb_nch = nb_nch.get();
        K.act[0] = actb[0].get();
        K.act[1] = actb[1].get();
        K.seg_cnt = kseg.get();
        K.chbase = kch.get();
        K.flag = kflag.get();
        K.state = kst.get();
        static int grid = [] {
            int dev = 0, sms = 0, per = 0;
            ST_CUDA(cudaGetDevice(&dev));
            ST_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
            ST_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_keyed_levels, kKeyThreads, 0));
            return std::max(1, std::min(sms, sms * per));
        }();
        void* args[] = {&K};
        ST_CUDA(cudaLaunchCooperativeKernel((const void*)k_keyed_levels, grid, kKeyThreads, args, 0, s));
        ST_LAUNCH("k_keyed_levels");
        count_launch();
        int32_t* st1 = static_cast<int32_t*>(pinned_stage(NS * sizeof(int32_t)));
        ST_CUDA(cudaMemcpyAsync(st1, kst.get(), NS * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
        st0 = st1;
        ST_CUDA(cudaStreamSynchronize(s));
        if (st0[KS_OVER] == 2) fail(ST_RUNTIME_ERROR, "build_tree: keyed levels' slot ranges do not tile a segment");
        if (st0[KS_OVER]) fail(ST_RUNTIME_ERROR, "build_tree: keyed levels exceeded their bound");
        depth = st0[KS_DEPTH];
        for (int d = 1; d <= depth; ++d) level_start.push_back(st0[KS_LS + d]);
        total = st0[KS_TOTAL];
        m = st0[KS_M];
        act = DevArray<int32_t>(std::max(m, 1), s);
        if (m)
            ST_CUDA(cudaMemcpyAsync(act.get(), actb[st0[KS_ACT]].get(), sizeof(int32_t) * m, cudaMemcpyDeviceToDevice,
                                    s));
        mark("keyed levels");
    }

    while (m > 0) {
        DevArray<uint32_t> seg_begin(m, s), seg_end, seg_base, seg_cnt((size_t)8 * m, s);
        DevArray<double> seg_mid;
        DevArray<int32_t> nch(m, s), chbase(m + 1, s);

        if (keyed && depth < kKeyLevels) {
            k_split_sorted<<<blocks((size_t)8 * m, 128), 128, 0, s>>>(m, depth, act.get(), nb_begin.get(),
                                                                      nb_end.get(), skey.get(), seg_begin.get(),
                                                                      seg_cnt.get());
            ST_LAUNCH("k_split_sorted");
            count_launch();
        } else {
            deep = true;  // perm is no longer the plain key order
            if (!seg_of.size()) {
                skey.reset();
                seg_of.alloc(n, s);
                slot8.alloc(n, s);
                blk_cnt.alloc((size_t)ntiles * 8, s);
                blk_off.alloc((size_t)(ntiles + 1) * 8, s);
                perm2.alloc(n, s);
            }
            seg_end.alloc(m, s);
            seg_base.alloc((size_t)8 * m, s);
            seg_mid.alloc((size_t)3 * m, s);
            k_mkseg<<<blocks(m, 128), 128, 0, s>>>(act.get(), m, nb_begin.get(), nb_end.get(), nb_box.get(),
                                                   seg_begin.get(), seg_end.get(), seg_mid.get());
            ST_LAUNCH("k_mkseg");
            k_segof<<<blocks(n, 256), 256, 0, s>>>(n, seg_begin.get(), seg_end.get(), m, seg_of.get());
            ST_LAUNCH("k_segof");
            k_slot_hist<<<ntiles, kTileThreads, 0, s>>>(n, d_pos, perm.get(), seg_of.get(), seg_mid.get(),
                                                        slot8.get(), blk_cnt.get());
            ST_LAUNCH("k_slot_hist");
            launch_scan_cols(blk_cnt.get(), blk_off.get(), ntiles, 8, s);
            k_segbase<<<blocks((size_t)2 * m * 32, 256), 256, 0, s>>>(m, seg_begin.get(), seg_end.get(),
                                                                      slot8.get(), blk_off.get(),
                                                                      seg_base.get(), seg_cnt.get());
            ST_LAUNCH("k_segbase");
            k_scatter<<<ntiles, kTileThreads, 0, s>>>(n, slot8.get(), seg_of.get(), blk_off.get(),
                                                      seg_begin.get(), seg_base.get(), seg_cnt.get(),
                                                      perm.get(), perm2.get());
            ST_LAUNCH("k_scatter");
            perm.swap(perm2);
            count_launch(5);
        }
        k_nch<<<blocks(m, 128), 128, 0, s>>>(m, seg_cnt.get(), nch.get());
        ST_LAUNCH("k_nch");
        launch_scan_i32(nch.get(), chbase.get(), m, s);
        count_launch(2);
        // sized by the bound C <= 8m so the children are made without waiting for C; one
        // host round trip per level reads C and the next level's split count together
        const int Cmax = 8 * m;
        const size_t need = (size_t)total + Cmax;
        grow(nb_begin, need, total, s);
        grow(nb_end, need, total, s);
        grow(nb_first, need, total, s);
        grow(nb_nch, need, total, s);
        grow(nb_box, 6 * need, 6 * (size_t)total, s);

        DevArray<int32_t> flag(Cmax, s), fpos(Cmax + 1, s);
        ST_CUDA(cudaMemsetAsync(flag.get(), 0, sizeof(int32_t) * Cmax, s));
        k_children<<<blocks(m, 128), 128, 0, s>>>(m, act.get(), seg_begin.get(), seg_cnt.get(),
                                                  chbase.get(), total, n0, depth + 1, nb_box.get(),
                                                  nb_box.get(), nb_begin.get(), nb_end.get(),
                                                  nb_first.get(), nb_nch.get(), flag.get());
        ST_LAUNCH("k_children");
        launch_scan_i32(flag.get(), fpos.get(), Cmax, s);
        count_launch();
        int32_t* cm = static_cast<int32_t*>(pinned_stage(2 * sizeof(int32_t)));  // C, next level's split count
        ST_CUDA(cudaMemcpyAsync(&cm[0], chbase.get() + m, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
        ST_CUDA(cudaMemcpyAsync(&cm[1], fpos.get() + Cmax, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
        ST_CUDA(cudaStreamSynchronize(s));
        const int C = cm[0], m2 = cm[1];
        DevArray<int32_t> act2(std::max(m2, 1), s);
        if (m2) {
            k_compact<<<blocks(C, 256), 256, 0, s>>>(C, total, flag.get(), fpos.get(), act2.get());
            ST_LAUNCH("k_compact");
            count_launch();
        }
        act = std::move(act2);
        level_start.push_back(total);
        total += C;
        m = m2;
        ++depth;
        mark("level");
    }
    level_start.push_back(total);
    const int T = total;
    const int L = (int)level_start.size() - 1;

    // geometry, first half: positions in tree order (any order inside a leaf serves the
    // order-free reductions, so this need not wait for the leaf sort below) and the
    // leaves' tight boxes; the subtree pass folds them upwards
    DevArray<double> tpos, center, fbox;
    DevArray<unsigned long long> r2max, nmm;
    if (geometry) {
        tpos.alloc(3 * (size_t)n, s);
        k_tree_pos<<<blocks(n, 256), 256, 0, s>>>(n, perm.get(), d_pos, tpos.get());
        ST_LAUNCH("k_tree_pos");
        count_launch();
        if (shrink) {
            DevArray<int32_t> leaf_of(n, s);
            k_leaf_of<<<blocks((size_t)32 * T, 256), 256, 0, s>>>(T, nb_nch.get(), nb_begin.get(), nb_end.get(),
                                                                  leaf_of.get());
            ST_LAUNCH("k_leaf_of");
            nmm.alloc(6 * (size_t)T, s);
            // lo slots = +inf ordering (all ones), hi slots = 0
            nmm.fill_bytes(0xff);
            k_zero_hi<<<blocks(T, 256), 256, 0, s>>>(nmm.get(), T);
            ST_LAUNCH("k_zero_hi");
            k_leaf_minmax<<<blocks(n, 256), 256, 0, s>>>(n, tpos.get(), leaf_of.get(), nmm.get());
            ST_LAUNCH("k_leaf_minmax");
            count_launch(3);
        }
    }

    DevArray<int32_t> size(T, s), pre(T, s);
    for (int d = L - 1; d >= 0; --d) {
        const int v0 = level_start[d], v1 = level_start[d + 1];
        k_subtree<<<blocks(v1 - v0, 128), 128, 0, s>>>(v0, v1, nb_first.get(), nb_nch.get(), size.get(), nmm.get());
        ST_LAUNCH("k_subtree");
        count_launch();
    }
    for (int d = 0; d < L; ++d) {
        const int v0 = level_start[d], v1 = level_start[d + 1];
        k_preorder<<<blocks(v1 - v0, 128), 128, 0, s>>>(v0, v1, nb_first.get(), nb_nch.get(), size.get(),
                                                         pre.get());
        ST_LAUNCH("k_preorder");
        count_launch();
    }
    mark("subtree+preorder");

    // geometry, second half: centres, then radii against them
    if (geometry) {
        center.alloc(3 * (size_t)T, s);
        fbox.alloc(6 * (size_t)T, s);
        r2max.alloc(T, s);
        r2max.zero();
        k_center<<<blocks(T, 128), 128, 0, s>>>(T, shrink ? 1 : 0, nmm.get(), nb_box.get(), fbox.get(),
                                                center.get());
        ST_LAUNCH("k_center");
        DevArray<int32_t> nck(T, s), ioff(T + 1, s);
        k_nchunk<<<blocks(T, 256), 256, 0, s>>>(T, nb_begin.get(), nb_end.get(), nck.get());
        ST_LAUNCH("k_nchunk");
        launch_scan_i32(nck.get(), ioff.get(), T, s);
        // chunks <= sum over levels of (points / chunk + clusters of the level)
        const size_t items_ub = (size_t)L * (n / kGeomChunk) + (size_t)T;
        k_radius<<<(unsigned)items_ub, 256, 0, s>>>(T, ioff.get(), nb_begin.get(), nb_end.get(), tpos.get(),
                                                    center.get(), r2max.get());
        ST_LAUNCH("k_radius");
        count_launch(3);
        tpos.reset();
    }
    mark("geometry");

    if (keyed) {
        // inside each leaf, input order (the reference's stable partitions): sort the points
        // by (leaf pre-order id, input index) -- a stable sort of the leaf ids over the
        // input indices
        seg_of.reset();
        slot8.reset();
        perm2.reset();
        DevArray<uint32_t> lkey(n, s), lkey2(n, s), idx(n, s), perm_out(n, s);
        k_leafkey<<<blocks((size_t)32 * T, 256), 256, 0, s>>>(T, nb_nch.get(), nb_begin.get(), nb_end.get(),
                                                              pre.get(), perm.get(), lkey.get());
        ST_LAUNCH("k_leafkey");
        k_iota<<<blocks(n, 256), 256, 0, s>>>(idx.get(), n);
        ST_LAUNCH("k_iota");
        int bits = 1;
        while (bits < 32 && (1ull << bits) < (unsigned long long)T) ++bits;
        size_t tmp = 0;
        ST_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, lkey.get(), lkey2.get(), idx.get(), perm_out.get(),
                                                (int)n, 0, bits, s));
        DevArray<char> scratch(tmp, s);
        ST_CUDA(cub::DeviceRadixSort::SortPairs(scratch.get(), tmp, lkey.get(), lkey2.get(), idx.get(),
                                                perm_out.get(), (int)n, 0, bits, s));
        if (key_order && !deep) *key_order = std::move(perm);
        perm = std::move(perm_out);
        count_launch(2 + 3);
    }
    mark("leaf order");
    out.n = n;
    out.ncl = T;
    out.depth = L - 1;
    out.geom.alloc(geometry ? T : 0, s);
    out.bbox.alloc(geometry ? 6 * (size_t)T : 0, s);
    out.info.alloc(T, s);
    out.children.alloc(8 * (size_t)T, s);
    out.nchild.alloc(T, s);
    out.bylevel.alloc(T, s);
    out.level_start = level_start;

    k_finalize<<<blocks(T, 128), 128, 0, s>>>(T, geometry ? 1 : 0, pre.get(), size.get(), nb_begin.get(),
                                              nb_end.get(), nb_first.get(), nb_nch.get(), center.get(),
                                              r2max.get(), fbox.get(), out.geom.get(), out.info.get(),
                                              out.bbox.get(), out.children.get(), out.nchild.get(),
                                              out.bylevel.get());
    ST_LAUNCH("k_finalize");
    count_launch();
    out.to_tree.alloc(n, s);
    k_invperm<<<blocks(n, 256), 256, 0, s>>>(n, perm.get(), out.to_tree.get());
    ST_LAUNCH("k_invperm");
    count_launch();
    out.perm = std::move(perm);
    mark("finalize");
    if (dbg) {
        ST_CUDA(cudaStreamSynchronize(s));
        std::string line = "[build] n " + std::to_string(n) + " levels " + std::to_string(depth) + ":";
        for (size_t i = 1; i < marks.size(); ++i) {
            float ms = 0.f;
            ST_CUDA(cudaEventElapsedTime(&ms, marks[i - 1].second.e, marks[i].second.e));
            char buf[96];
            snprintf(buf, sizeof buf, " %s %.3f (host %.3f)", marks[i].first, ms, host_ms[i] - host_ms[i - 1]);
            line += buf;
        }
        fprintf(stderr, "%s ms\n", line.c_str());
    }
}

void order_targets(const double* d_pos, size_t n, cudaStream_t s, DevArray<uint32_t>& perm) {
    perm.alloc(n, s);
    if (!n) return;
    DevArray<unsigned long long> mm(6, s);
    ST_CUDA(cudaMemsetAsync(mm.get(), 0xff, 3 * sizeof(unsigned long long), s));
    ST_CUDA(cudaMemsetAsync(mm.get() + 3, 0x00, 3 * sizeof(unsigned long long), s));
    const unsigned g = (unsigned)std::min<size_t>((n + 255) / 256, 148 * 8);
    k_tight_all<<<g, 256, 0, s>>>(d_pos, n, mm.get());
    ST_LAUNCH("k_tight_all");
    DevArray<uint32_t> rng(2, s);
    DevArray<double> box(6, s);
    k_root<<<1, 1, 0, s>>>(mm.get(), (uint32_t)n, rng.get(), rng.get() + 1, box.get());
    ST_LAUNCH("k_root");
    DevArray<uint32_t> key(n, s), key2(n, s), idx(n, s);
    k_geokey<<<(unsigned)((n + 255) / 256), 256, 0, s>>>((uint32_t)n, d_pos, box.get(), key.get(), idx.get());
    ST_LAUNCH("k_geokey");
    size_t tmp = 0;
    ST_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, key.get(), key2.get(), idx.get(), perm.get(), (int)n, 0,
                                            3 * kKeyLevels, s));
    DevArray<char> scratch(tmp, s);
    ST_CUDA(cub::DeviceRadixSort::SortPairs(scratch.get(), tmp, key.get(), key2.get(), idx.get(), perm.get(), (int)n,
                                            0, 3 * kKeyLevels, s));
    count_launch(3 + 5);
}

}  // namespace st
