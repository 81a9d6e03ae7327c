// C ABI of libstokestree_b200.so (include/stokestree_c.h): validation with the
// reference's error taxonomy and messages, device buffer management, and the
// orchestration of K1 (tree) -> K2 (moments + fold) -> K3/K4 (far) -> K5 (near).
#include <cuda.h>

#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <map>
#include <cmath>
#include <cstring>
#include <functional>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "moments.cuh"
#include "staging.cuh"
#include "nccl_comm.cuh"
#include "traverse.cuh"
#include "tree.cuh"

namespace st {
thread_local uint64_t g_launches = 0;

// pinned staging blocks of this host thread: `cur` is bumped; blocks outgrown during a
// call are kept until the next reset (copies may still read them)
struct PinnedArena {
    struct Block {
        char* p = nullptr;
        size_t size = 0;
    };
    Block cur;
    size_t used = 0;
    std::vector<Block> old;
    ~PinnedArena() {
        for (auto& b : old) cudaFreeHost(b.p);
        if (cur.p) cudaFreeHost(cur.p);
    }
};
static thread_local PinnedArena g_pinned;

void* pinned_stage(size_t bytes) {
    PinnedArena& a = g_pinned;
    bytes = (bytes + 15) & ~size_t(15);
    if (a.used + bytes > a.cur.size) {
        if (a.cur.p) a.old.push_back(a.cur);
        const size_t sz = std::max<size_t>({bytes, 2 * a.cur.size, size_t(1) << 20});
        void* p = nullptr;
        ST_CUDA(cudaMallocHost(&p, sz));
        a.cur = {static_cast<char*>(p), sz};
        a.used = 0;
    }
    void* r = a.cur.p + a.used;
    a.used += bytes;
    return r;
}

void pinned_reset() {
    PinnedArena& a = g_pinned;
    for (auto& b : a.old) cudaFreeHost(b.p);
    a.old.clear();
    a.used = 0;
}
}  // namespace st

using namespace st;

namespace {

thread_local std::string g_last_error;

st_status set_error(st_status s, const std::string& m) {
    g_last_error = m;
    return s;
}

template <class F>
st_status guarded(F&& f) {
    try {
        pinned_reset();
        f();
        g_last_error.clear();
        return ST_OK;
    } catch (const Error& e) {
        return set_error(e.status, e.what());
    } catch (const std::bad_alloc&) {
        return set_error(ST_RUNTIME_ERROR, "out of host memory");
    } catch (const std::exception& e) {
        return set_error(ST_RUNTIME_ERROR, e.what());
    }
}

// ------------------------------------------------------------ device context

// Private per-device pools (st_common.cuh).
std::mutex g_pool_mu;
cudaMemPool_t g_pool[64] = {};

}  // namespace

cudaMemPool_t st::device_pool() {
    int dev = 0;
    ST_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(g_pool_mu);
    cudaMemPool_t& p = g_pool[dev & 63];
    if (!p) {
        cudaMemPoolProps props = {};
        props.allocType = cudaMemAllocationTypePinned;
        props.handleTypes = cudaMemHandleTypeNone;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = dev;
        ST_CUDA(cudaMemPoolCreate(&p, &props));
        uint64_t thr = UINT64_MAX;
        ST_CUDA(cudaMemPoolSetAttribute(p, cudaMemPoolAttrReleaseThreshold, &thr));
    }
    return p;
}

void st::pool_grant_peer(int owner, int peer) {
    int cur = 0;
    ST_CUDA(cudaGetDevice(&cur));
    ST_CUDA(cudaSetDevice(owner));
    cudaMemPool_t p = device_pool();
    ST_CUDA(cudaSetDevice(cur));
    cudaMemAccessDesc d = {};
    d.location.type = cudaMemLocationTypeDevice;
    d.location.id = peer;
    d.flags = cudaMemAccessFlagsProtReadWrite;
    ST_CUDA(cudaMemPoolSetAccess(p, &d, 1));
}

namespace {

// Per-device check done once (cudaGetDeviceProperties is slow and takes driver locks;
// it must not sit inside every call's timed path).
std::mutex g_dev_mu;
int g_dev_state[64] = {0};  // 0 unknown, 1 ok, 2 wrong architecture

void ensure_device() {
    int dev = 0;
    const cudaError_t e = cudaGetDevice(&dev);
    int ndev = 0;
    if (e != cudaSuccess || cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        fail(ST_CUDA_ERROR, std::string("no CUDA device available (") + cudaGetErrorString(e) +
                                "); the treecode has no CPU fallback");
    }
    if (dev >= 64) return;
    std::lock_guard<std::mutex> lk(g_dev_mu);
    if (g_dev_state[dev] == 0) {
        int major = 0, minor = 0;
        ST_CUDA(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev));
        ST_CUDA(cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev));
        g_dev_state[dev] = major == 10 ? 1 : 2;
        if (major == 10) {
            cudaMemPool_t pool = device_pool();
            // Map a block of pool memory once and keep it: a stream-ordered allocation that
            // has to grow the pool was measured to block the host for 10-550 ms (GB-size
            // requests at cfg4), mid-call.  8% of the device, at most half of what is free
            // (ST_POOL_RESERVE_GB overrides); larger problems still grow the pool as needed.
            size_t fr = 0, tot = 0;
            if (cudaMemGetInfo(&fr, &tot) == cudaSuccess) {
                size_t reserve = tot / 100 * 8;
                if (const char* env = getenv("ST_POOL_RESERVE_GB")) reserve = (size_t)(atof(env) * 1e9);
                reserve = std::min(reserve, fr / 2);
                void* p = nullptr;
                if (reserve && cudaMallocFromPoolAsync(&p, reserve, pool, 0) == cudaSuccess) {
                    cudaFreeAsync(p, 0);
                    cudaStreamSynchronize(0);
                }
                cudaGetLastError();
                // the near field's entry workspace: 2 GB (65M entries; cfg1 needs 0.6 GB), at
                // most a tenth of what is free (ST_NEAR_RESERVE_GB overrides)
                size_t near = std::min<size_t>(2000000000ull, fr / 10);
                if (const char* env = getenv("ST_NEAR_RESERVE_GB")) near = (size_t)(atof(env) * 1e9);
                if (near) reserve_near_workspace(dev, near);
            }
        } else {
            fail(ST_CUDA_ERROR, "device " + std::to_string(dev) + " is sm_" + std::to_string(major) +
                                    std::to_string(minor) + "; this library is built for sm_100a");
        }
    }
    if (g_dev_state[dev] == 2) fail(ST_CUDA_ERROR, "device is not sm_100; this library is built for sm_100a");
}

struct OwnedStream {
    cudaStream_t s = nullptr;
    OwnedStream() { ST_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking)); }
    ~OwnedStream() {
        if (s) cudaStreamDestroy(s);
    }
};


inline unsigned nblocks(size_t n, int t) { return (unsigned)((n + t - 1) / t); }

// ------------------------------------------------------------ small kernels
// 12-double source record [y, f, h, nu] gathered by `perm` (identity if null).
__global__ void k_pack(size_t n, const uint32_t* __restrict__ perm, const double* __restrict__ pos,
                       const double* __restrict__ f, const double* __restrict__ h,
                       const double* __restrict__ nu, double* __restrict__ rec,
                       uint32_t* __restrict__ to_tree) {
    const size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    if (t >= n) return;
    const size_t o = perm ? perm[t] : t;
    double* r = rec + 12 * t;
    for (int a = 0; a < 3; ++a) {
        r[a] = pos[3 * o + a];
        r[3 + a] = f ? f[3 * o + a] : 0.0;
        r[6 + a] = h ? h[3 * o + a] : 0.0;
        r[9 + a] = nu ? nu[3 * o + a] : 0.0;
    }
    if (to_tree) to_tree[o] = (uint32_t)t;
}

// The same records written from the original order: coalesced reads of the caller's
// arrays, each record stored whole (six 16-byte stores) at its tree position.
__global__ void k_pack_tree(size_t n, const uint32_t* __restrict__ to_tree, const double* __restrict__ pos,
                            const double* __restrict__ f, const double* __restrict__ h,
                            const double* __restrict__ nu, double* __restrict__ rec) {
    const size_t o = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    if (o >= n) return;
    double v[12];
    for (int a = 0; a < 3; ++a) {
        v[a] = pos[3 * o + a];
        v[3 + a] = f ? f[3 * o + a] : 0.0;
        v[6 + a] = h ? h[3 * o + a] : 0.0;
        v[9 + a] = nu ? nu[3 * o + a] : 0.0;
    }
    double2* r = reinterpret_cast<double2*>(rec + 12 * (size_t)to_tree[o]);
#pragma unroll
    for (int q = 0; q < 6; ++q) r[q] = make_double2(v[2 * q], v[2 * q + 1]);
}

// Targets in batch order: positions, original index, excluded source tree index.
__global__ void k_targets(size_t nt, const uint32_t* __restrict__ tperm, const double* __restrict__ tpos,
                          const uint32_t* __restrict__ to_tree, double* __restrict__ tx,
                          uint32_t* __restrict__ torig, uint32_t* __restrict__ tskip) {
    const size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    if (t >= nt) return;
    const uint32_t o = tperm[t];
    for (int a = 0; a < 3; ++a) tx[3 * t + a] = tpos[3 * (size_t)o + a];
    torig[t] = o;
    tskip[t] = to_tree ? to_tree[o] : kNoSkip;
}

// batch order -> original order (multi-device gather on device 0)
__global__ void k_unbatch(size_t nt, const uint32_t* __restrict__ torig, const double* __restrict__ ub,
                          const uint64_t* __restrict__ pb, double* __restrict__ u, uint64_t* __restrict__ pt) {
    const size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    if (t >= nt) return;
    const size_t o = torig[t];
    for (int a = 0; a < 3; ++a) u[3 * o + a] = ub[3 * t + a];
    if (pt)
        for (int a = 0; a < 3; ++a) pt[3 * o + a] = pb[3 * t + a];
}

// validate(ps, sel) (particles.hpp:41-70) on device: first failing index per check
// {position finite, f finite, h finite, nu finite, nu unit (+-1e-12)}.
__global__ void k_validate(size_t n, const double* __restrict__ pos, const double* __restrict__ f,
                           const double* __restrict__ h, const double* __restrict__ nu, int str,
                           unsigned long long* __restrict__ first_bad) {
    const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    auto fin3 = [](const double* a) { return isfinite(a[0]) && isfinite(a[1]) && isfinite(a[2]); };
    if (!fin3(pos + 3 * i)) atomicMin(&first_bad[0], (unsigned long long)i);
    if (f && !fin3(f + 3 * i)) atomicMin(&first_bad[1], (unsigned long long)i);
    if (h && !fin3(h + 3 * i)) atomicMin(&first_bad[2], (unsigned long long)i);
    if (nu) {
        const double* v = nu + 3 * i;
        if (!fin3(v)) atomicMin(&first_bad[3], (unsigned long long)i);
        if (str) {
            const double n2 = __dadd_rn(__dadd_rn(__dmul_rn(v[0], v[0]), __dmul_rn(v[1], v[1])),
                                        __dmul_rn(v[2], v[2]));
            const double len = __dsqrt_rn(n2);
            if (fabs(__dsub_rn(len, 1.0)) > 1e-12) atomicMin(&first_bad[4], (unsigned long long)i);
        }
    }
}

__global__ void k_fp64_peak(double* out, int iters, double seed) {
    double a0 = seed + threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5,
           a6 = a0 + 6, a7 = a0 + 7;
    const double m = 0.999999999, c = 1e-9;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            a0 = fma(a0, m, c); a1 = fma(a1, m, c); a2 = fma(a2, m, c); a3 = fma(a3, m, c);
            a4 = fma(a4, m, c); a5 = fma(a5, m, c); a6 = fma(a6, m, c); a7 = fma(a7, m, c);
        }
    }
    const double r = ((a0 + a1) + (a2 + a3)) + ((a4 + a5) + (a6 + a7));
    if (r == 12345.678) out[0] = r;  // practically never; keeps the chains live
}

// ------------------------------------------------------------ validation (host side)
void validate_params(const st_params* p) {
    if (!p) fail(ST_INVALID_ARGUMENT, "params: null");
    if (p->order < 0 || p->order > 16) fail(ST_INVALID_ARGUMENT, "params: order must be in [0, 16]");
    if (!(p->theta > 0.0) || !(p->theta < 1.0))
        fail(ST_INVALID_ARGUMENT, "params: theta must lie strictly in (0,1)");
    if (p->leaf_capacity < 1) fail(ST_INVALID_ARGUMENT, "params: leaf capacity must be >= 1");
    if (p->workers < 1) fail(ST_INVALID_ARGUMENT, "params: workers must be >= 1");
    if (!p->stokeslet && !p->stresslet)
        fail(ST_INVALID_ARGUMENT, "params: at least one kernel must be enabled");
    if (p->devices < 1) fail(ST_INVALID_ARGUMENT, "params: devices must be >= 1");
}

// Host-visible part of validate(ps, sel): selection, emptiness, presence ("length").
void validate_shape(const st_particles* ps, bool sto, bool str) {
    if (!sto && !str) fail(ST_INVALID_ARGUMENT, "kernel selection: at least one kernel must be enabled");
    if (!ps || ps->n == 0) fail(ST_INVALID_ARGUMENT, "particle set is empty");
    auto need = [](const double* a, const char* name) {
        if (!a)
            fail(ST_INVALID_ARGUMENT, std::string("particle array '") + name + "' has mismatched length");
    };
    need(ps->position, "position");
    if (sto) need(ps->force_weight, "force_weight");
    if (str) {
        need(ps->dipole_weight, "dipole_weight");
        need(ps->normal, "normal");
    }
}

// validate(ps, sel)'s value checks (particles.hpp:47-69) on the host, in the reference's
// order: every array in turn (position, force_weight, dipole_weight, normal), then the
// unit normals.  Used by the O(N^2) direct entry points, whose range checks follow it.
void validate_values_host(const st_particles* ps, bool sto, bool str) {
    const size_t n = ps->n;
    auto finite = [n](const double* a, const char* name) {
        for (size_t i = 0; i < 3 * n; ++i)
            if (!std::isfinite(a[i]))
                fail(ST_INVALID_ARGUMENT, std::string("particle array '") + name + "' contains a non-finite value");
    };
    finite(ps->position, "position");
    if (sto) finite(ps->force_weight, "force_weight");
    if (str) {
        finite(ps->dipole_weight, "dipole_weight");
        finite(ps->normal, "normal");
        for (size_t i = 0; i < n; ++i) {
            const double* v = ps->normal + 3 * i;
            const double len = std::sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]);
            if (std::fabs(len - 1.0) > 1e-12)
                fail(ST_INVALID_ARGUMENT, "normal " + std::to_string(i) + " is not unit length");
        }
    }
}

// Device part of validate(ps, sel) on device-resident arrays.
// ------------------------------------------------------------ device-resident inputs
struct DevParticles {
    size_t n = 0;
    const double *pos = nullptr, *f = nullptr, *h = nullptr, *nu = nullptr;
    DevArray<double> own_pos, own_f, own_h, own_nu;
};

void upload(const st_particles* ps, bool need_f, bool need_hn, DevParticles& d, cudaStream_t s) {
    d.n = ps->n;
    auto up = [&](const double* src, DevArray<double>& dst) -> const double* {
        if (!src) return nullptr;
        dst.alloc(3 * ps->n, s);
        h2d(dst.get(), src, 3 * ps->n * sizeof(double), s);
        return dst.get();
    };
    d.pos = up(ps->position, d.own_pos);
    d.f = need_f ? up(ps->force_weight, d.own_f) : nullptr;
    d.h = need_hn ? up(ps->dipole_weight, d.own_h) : nullptr;
    d.nu = need_hn ? up(ps->normal, d.own_nu) : nullptr;
}

// ------------------------------------------------------------ the treecode
struct RunOut {
    unsigned long long vflags[6] = {~0ull, ~0ull, ~0ull, ~0ull, ~0ull, ~0ull};  // first bad index per check
    int domain_err = 0;
    uint64_t stats[3] = {0, 0, 0};
    double t_build = 0, t_moments = 0, t_traverse = 0, t_total = 0, t_far = 0, t_near = 0;
};

// validate(ps, sel) messages in the reference's order (particles.hpp:41-70), then the
// coincident-pair domain error of the direct sums (kernels.hpp:52): validation first.
void raise_flags(const RunOut& ro) {
    const char* names[4] = {"position", "force_weight", "dipole_weight", "normal"};
    for (int k = 0; k < 4; ++k)
        if (ro.vflags[k] != ~0ull)
            fail(ST_INVALID_ARGUMENT, std::string("particle array '") + names[k] + "' contains a non-finite value");
    if (ro.vflags[4] != ~0ull) fail(ST_INVALID_ARGUMENT, "normal " + std::to_string(ro.vflags[4]) + " is not unit length");
    if (ro.vflags[5] != ~0ull) fail(ST_INVALID_ARGUMENT, "targets: non-finite position");
    if (ro.domain_err & 2) fail(ST_RUNTIME_ERROR, "MAC accepted a cluster containing the target");
    if (ro.domain_err & 1) fail(ST_DOMAIN_ERROR, "direct sum: coincident particles");
}


// Far events (clusters) accepted by at most this many of a warp's 32 lanes are not
// evaluated by k_far, which would idle the other lanes, but packed 32 per task by the near
// field's plan: 24 measured best (cfg1 -2%, cfg4 -6%); ST_FAR_SPARSE overrides, 0 disables.
int far_sparse_max() {
    static const int v = [] {
        const char* e = getenv("ST_FAR_SPARSE");
        return e ? std::max(0, std::min(31, atoi(e))) : 24;
    }();
    return v;
}

struct ShardOut {
    int w0 = 0, w1 = 0;         // warp (32-target batch) range evaluated
    DevArray<uint32_t> torig;   // batch position -> original target index (if requested)
};

bool moments_inline() {
    const char* v = getenv("ST_MOMENTS_INLINE");
    return v && v[0] == '1';
}

// The particle arrays other than positions may still be in flight on another stream:
// `weights_ready` (if set) is waited for after the tree build, which needs positions only.
// Validation runs on the device after that wait and is read back with the results;
// callers raise in the reference's order with raise_flags().
// exchange (if set and nshards > 1): the moment pass is split over the ranks
// (moments.cuh MomentsSplit); the callback moves the rows between them before the far field.
struct SplitExchange {
    st_exchange_fn fn = nullptr;
    void* ctx = nullptr;
};

void run_treecode(const DevParticles& src, const double* d_targets, size_t nt_in, const st_params& prm,
                  double* d_out, uint64_t* d_per_target, int shard, int nshards, cudaStream_t s,
                  RunOut& ro, bool out_batch = false, ShardOut* so = nullptr,
                  cudaEvent_t weights_ready = nullptr, const SplitExchange* xchg = nullptr,
                  cudaEvent_t targets_ready = nullptr) {
    const bool sto = prm.stokeslet != 0, str = prm.stresslet != 0;
    const size_t n = src.n;
    const bool same = d_targets == nullptr;
    const size_t nt = same ? n : nt_in;
    if (nt >= 0x7fffffffull - 64) fail(ST_INVALID_ARGUMENT, "too many targets");
    Event e0, e1, e2, e3;
    e0.record(s);
    // Second stream: the batch order of disjoint targets (positions only) overlaps the tree
    // build; then K2 (below).  Declared before every array whose stream-ordered free goes
    // to it.  Targets that are the sources take the build's own key order.
    AuxStream aux;
    ST_CUDA(cudaStreamWaitEvent(aux.s, e0.e, 0));
    const double* tpos = same ? src.pos : d_targets;
    DevArray<uint32_t> tperm;
    if (!same) {
        if (targets_ready) ST_CUDA(cudaStreamWaitEvent(aux.s, targets_ready, 0));
        order_targets(tpos, nt, aux.s, tperm);
    }
    Event esort;
    esort.record(aux.s);

    // K1: tree over the sources, tree-ordered source records
    DevTree tree;
    build_tree_device(src.pos, n, prm.leaf_capacity, prm.shrink != 0, true, s, tree, same ? &tperm : nullptr);
    if (same && tperm.size() != nt) order_targets(tpos, nt, s, tperm);  // the build made no key order
    const MomentsPlan mplan = plan_moments(tree, s);  // host lists now: K2 below never waits on the host
    // Validation and the tree-ordered source records on the second stream: only the near
    // field (and the moments after them there) read the records, so they overlap the
    // target ordering, the shard cut and the plan walks on s (launch_eval waits for `erec`
    // before the near field's evaluation).
    e1.record(s);  // the tree (positions only)
    ST_CUDA(cudaStreamWaitEvent(aux.s, e1.e, 0));
    if (weights_ready) ST_CUDA(cudaStreamWaitEvent(aux.s, weights_ready, 0));
    DevArray<unsigned long long> vflags(6, aux.s);
    vflags.fill_bytes(0xff);
    k_validate<<<nblocks(n, 256), 256, 0, aux.s>>>(n, src.pos, sto ? src.f : nullptr, str ? src.h : nullptr,
                                                    str ? src.nu : nullptr, str ? 1 : 0, vflags.get());
    ST_LAUNCH("k_validate");
    if (d_targets) {
        k_validate<<<nblocks(nt_in, 256), 256, 0, aux.s>>>(nt_in, d_targets, nullptr, nullptr, nullptr, 0,
                                                            vflags.get() + 5);
        ST_LAUNCH("k_validate");
    }
    count_launch(d_targets ? 2 : 1);
    DevArray<double> rec(12 * n, aux.s);
    const DevArray<uint32_t>& to_tree = tree.to_tree;
    k_pack_tree<<<nblocks(n, 256), 256, 0, aux.s>>>(n, to_tree.get(), src.pos, sto ? src.f : nullptr,
                                                    str ? src.h : nullptr, str ? src.nu : nullptr, rec.get());
    ST_LAUNCH("k_pack_tree");
    count_launch();
    Event erec;
    erec.record(aux.s);

    // batch order of the targets: their 30-bit octree-key order (one radix sort, from the
    // build or on the second stream above)
    ST_CUDA(cudaStreamWaitEvent(s, esort.e, 0));
    DevArray<double> tx(3 * nt, s), ufar(3 * nt, s);
    DevArray<uint32_t> torig(nt, s), tskip(nt, s);
    k_targets<<<nblocks(nt, 256), 256, 0, s>>>(nt, tperm.get(), tpos, same ? to_tree.get() : nullptr,
                                               tx.get(), torig.get(), tskip.get());
    ST_LAUNCH("k_targets");
    count_launch();
    Event et, ec;  // timeline: targets ordered, shard cuts known
    et.record(s);

    DevArray<unsigned long long> d_stats(3, s);
    DevArray<int> d_err(1, s), d_work(2, s);
    d_stats.zero();
    d_err.zero();

    TravArgs a;
    a.tx = tx.get();
    a.tskip = tskip.get();
    a.torig = torig.get();
    a.nt = (int)nt;
    const int nwarps = (int)((nt + 31) / 32);
    a.w0 = 0;
    a.w1 = nwarps;
    a.geom = tree.geom.get();
    a.info = tree.info.get();
    a.ncl = tree.ncl;
    a.th2 = prm.theta * prm.theta;
    a.src = rec.get();
    a.out = d_out;
    a.per_target = d_per_target;
    a.stats = d_stats.get();
    a.err = d_err.get();
    a.out_batch = out_batch ? 1 : 0;
    a.work = d_work.get();
    const int P = prm.order + (str ? 2 : 1);

    if (nshards > 1) {
        // work-balanced contiguous warp ranges, identical on every rank (deterministic):
        // sampled counting walk and the cut on the device, two integers back to the host
        const int stride = count_stride(nwarps);
        DevArray<unsigned long long> cost((nwarps + stride - 1) / stride, s);
        DevArray<int> dcuts(nshards + 1, s);
        a.warp_cost = cost.get();
        a.sparse_max = far_sparse_max();
        launch_count(a, (uint32_t)((P + 1) * (P + 1) * 8), s);
        launch_shard_cuts(cost.get(), nwarps, stride, nshards, dcuts.get(), s);
        int* wr = static_cast<int*>(pinned_stage(2 * sizeof(int)));
        ST_CUDA(cudaMemcpyAsync(wr, dcuts.get() + shard, 2 * sizeof(int), cudaMemcpyDeviceToHost, s));
        ST_CUDA(cudaStreamSynchronize(s));
        a.w0 = wr[0];
        a.w1 = wr[1];
        a.warp_cost = nullptr;
    }
    ec.record(s);

    // K2: moments at order p, folded into the far-field weights, on the second stream: only
    // the far field needs them, so they overlap the plan walks and the near field
    // (launch_eval waits for `e2` before the far kernels).  Queued after the target order
    // and the shard cut: its host-side plan lists are pageable uploads, which wait for the
    // second stream to drain (the record pack) -- s must have its work queued by then.
    Event em;
    em.record(aux.s);
    DevArray<double> M, W;
    const bool split = xchg && xchg->fn && nshards > 1;
    const int Pw = prm.order + (str ? 2 : 1);
    const size_t w_row = (size_t)4 * (Pw + 1) * (Pw + 1), m_row = (size_t)12 * mi_count(prm.order);
    MomentsSplit sp;
    DevArray<double> Mu;                   // moments of the split's subtree roots, packed
    DevArray<int32_t> d_units, d_top;      // unit roots, top clusters (device lists)
    if (!split) {
        compute_moments_device(tree, rec.get(), prm.order, sto, str, aux.s, M, &mplan);
        fold_weights_device(M.get(), tree.ncl, prm.order, sto, str, aux.s, W);
        M.reset();
    } else {
        // this rank's subtrees only: leaves, M2M up to depth L, their weights and roots
        sp = split_moments(mplan, tree.ncl, nshards);
        const MomentsPlan own = shard_moments_plan(mplan, sp, shard);
        compute_moments_device(tree, rec.get(), prm.order, sto, str, aux.s, M, &own);
        W.alloc((size_t)tree.ncl * w_row, aux.s);
        const size_t u0 = sp.unit_cuts[shard], u1 = sp.unit_cuts[shard + 1];
        std::vector<int32_t> rows;
        if (u0 < u1) {
            const int lo = sp.units[u0], hi = mplan.info[sp.units[u1 - 1]].z;
            for (int v = lo; v < hi; ++v)
                if (!(mplan.depth[v] < sp.depth && !mplan.info[v].w)) rows.push_back(v);
        }
        DevArray<int32_t> d_rows(rows.size(), aux.s);
        if (!rows.empty())
            ST_CUDA(cudaMemcpyAsync(d_rows.get(), pinned_copy(rows.data(), rows.size()), rows.size() * 4,
                                    cudaMemcpyHostToDevice, aux.s));
        fold_weights_rows_device(M.get(), d_rows.get(), (int)rows.size(), prm.order, sto, str, aux.s, W.get());
        d_units.alloc(sp.units.size(), aux.s);
        ST_CUDA(cudaMemcpyAsync(d_units.get(), pinned_copy(sp.units.data(), sp.units.size()), sp.units.size() * 4,
                                cudaMemcpyHostToDevice, aux.s));
        Mu.alloc(sp.units.size() * m_row, aux.s);
        gather_rows_device(M.get(), d_units.get() + u0, (int)(u1 - u0), m_row, Mu.get() + u0 * m_row, false, aux.s);
        d_top.alloc(sp.top_ids.size(), aux.s);
        if (!sp.top_ids.empty())
            ST_CUDA(cudaMemcpyAsync(d_top.get(), pinned_copy(sp.top_ids.data(), sp.top_ids.size()),
                                    sp.top_ids.size() * 4, cudaMemcpyHostToDevice,
                                    aux.s));
    }
    e2.record(aux.s);
    // ST_MOMENTS_INLINE=1 (measurement only): nothing overlaps the moment pass, so
    // time_moments_s is its own duration (bench.py's moments roofline)
    if (moments_inline()) ST_CUDA(cudaStreamWaitEvent(s, e2.e, 0));
    // split: after this rank's rows exist, the exchange, then every rank shifts and folds
    // the top levels itself; queued on s before the first far kernel (launch_eval)
    std::function<void()> complete_weights = [&] {
        ST_CUDA(cudaStreamWaitEvent(s, e2.e, 0));
        st_shard_exchange ex;
        ex.shard = shard;
        ex.n_shards = nshards;
        ex.w = W.get();
        ex.w_row = w_row;
        ex.ncl = (size_t)tree.ncl;
        ex.w_cuts = sp.w_cuts.data();
        ex.m = Mu.get();
        ex.m_row = m_row;
        ex.n_units = sp.units.size();
        ex.m_cuts = sp.unit_cuts.data();
        ex.stream = s;
        if (xchg->fn(xchg->ctx, &ex) != 0) fail(ST_RUNTIME_ERROR, "shard exchange callback failed");
        gather_rows_device(Mu.get(), d_units.get(), (int)sp.units.size(), m_row, M.get(), true, s);
        const MomentsPlan top = top_moments_plan(sp);
        compute_moments_device(tree, rec.get(), prm.order, sto, str, s, M, &top, true);
        fold_weights_rows_device(M.get(), d_top.get(), (int)sp.top_ids.size(), prm.order, sto, str, s, W.get());
    };

    a.sparse_max = far_sparse_max();
    FarOrder fo;
    fo.P = P;
    fo.W = W.get();
    fo.ufar = ufar.get();
    fo.out = d_out;
    EvalTimes tm;
    tm.origin = e0.e;
    launch_eval(sto, str, a, &fo, 1, s, &tm, e2.e, split ? &complete_weights : nullptr, erec.e);
    ST_CUDA(cudaStreamWaitEvent(s, erec.e, 0));  // vflags (read below) were written on aux
    e3.record(s);

    ST_CUDA(cudaMemcpyAsync(&ro.domain_err, d_err.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
    ST_CUDA(cudaMemcpyAsync(ro.stats, d_stats.get(), sizeof ro.stats, cudaMemcpyDeviceToHost, s));
    ST_CUDA(cudaMemcpyAsync(ro.vflags, vflags.get(), sizeof ro.vflags, cudaMemcpyDeviceToHost, s));
    ST_CUDA(cudaStreamSynchronize(s));
    ro.t_build = secs(e0, e1);
    ro.t_moments = secs(em, e2);    // on the second stream, overlapped with the traversal
    ro.t_traverse = secs(e1, e3);   // targets, plan walks, far and near fields, reduce
    ro.t_total = secs(e0, e3);
    // kernel times: far = dense events (k_far_list) + deferred sparse events (k_feval);
    // near = the leaf sums (k_neval).  Walks, scans and the reduce count in t_traverse only.
    ro.t_far = tm.far_s;
    ro.t_near = tm.near_s;
    static const bool timeline = getenv("ST_DEBUG_TIMELINE") != nullptr;
    if (timeline) {  // ms from the call's first event: when each phase started / ended
        std::string plan;
        for (size_t k = 0; k < tm.plan_ms.size(); ++k)
            plan += std::string(" | ") + tm.plan_ms[k].first + " " + std::to_string(tm.plan_ms[k].second).substr(0, 6) +
                    " (host +" + std::to_string(tm.plan_host_ms[k]).substr(0, 5) + ")";
        fprintf(stderr, "[timeline] build end %.3f | moments %.3f - %.3f (aux stream) | targets ordered %.3f | "
                "cuts %.3f%s | near %.3f - %.3f | far start %.3f | end %.3f\n", 1e3 * ro.t_build, 1e3 * secs(e0, em),
                1e3 * secs(e0, e2), 1e3 * secs(e0, et), 1e3 * secs(e0, ec), plan.c_str(), 1e3 * tm.near_start_s,
                1e3 * (tm.near_start_s + tm.near_s), 1e3 * tm.far_start_s, 1e3 * ro.t_total);
    }
    if (so) {
        so->w0 = a.w0;
        so->w1 = a.w1;
        so->torig = std::move(torig);
    }
}

void fill_stats(st_stats* st, const RunOut& ro) {
    if (!st) return;
    st->farfield_evals = ro.stats[0];
    st->direct_pairs = ro.stats[1];
    st->clusters_visited = ro.stats[2];
    st->time_build_s = ro.t_build;
    st->time_moments_s = ro.t_moments;
    st->time_traverse_s = ro.t_traverse;
    st->time_total_s = ro.t_total;
    st->time_far_s = ro.t_far;
    st->time_near_s = ro.t_near;
}

void shard_cuts_impl(size_t n, const double* w, int k, size_t* cuts) {
    double total = 0.0;
    for (size_t i = 0; i < n; ++i) total += w[i] > 0 ? w[i] : 0.0;
    cuts[0] = 0;
    double run = 0.0;
    size_t i = 0;
    for (int sIdx = 1; sIdx < k; ++sIdx) {
        // run + w/2 < total s / k, multiplied out (exact for integer weights below 2^48,
        // the form k_shard_cuts evaluates in integers)
        const double target = 2.0 * total * sIdx;
        while (i < n && 2.0 * k * run + k * (w[i] > 0 ? w[i] : 0.0) < target) {
            run += w[i] > 0 ? w[i] : 0.0;
            ++i;
        }
        cuts[sIdx] = std::max(cuts[sIdx - 1], i);
    }
    cuts[k] = n;
}

// Order sweep (SURVEY 8f "order-sweep reuse"): one tree, one moment pass at the largest
// order (lower orders are graded prefixes), ONE near-field pass (it does not depend on
// p), then per order only the fold + far field.  Each order's velocities are
// bit-identical to a standalone call at that order.
void run_sweep(const DevParticles& src, const double* d_targets, size_t nt_in, const st_params& prm,
               const int* orders, int n_orders, double* d_out /* n_orders x 3 nt, original order */,
               double* far_s /* n_orders */, cudaStream_t s, RunOut& ro) {
    const bool sto = prm.stokeslet != 0, str = prm.stresslet != 0;
    const size_t n = src.n;
    const bool same = d_targets == nullptr;
    const size_t nt = same ? n : nt_in;
    int pmax = 0;
    for (int i = 0; i < n_orders; ++i) pmax = std::max(pmax, orders[i]);
    Event e0, e1, e2, e3;
    e0.record(s);
    DevTree tree;
    DevArray<uint32_t> tperm;
    build_tree_device(src.pos, n, prm.leaf_capacity, prm.shrink != 0, true, s, tree, same ? &tperm : nullptr);
    const MomentsPlan mplan = plan_moments(tree, s);
    DevArray<unsigned long long> vflags(6, s);
    vflags.fill_bytes(0xff);
    k_validate<<<nblocks(n, 256), 256, 0, s>>>(n, src.pos, sto ? src.f : nullptr, str ? src.h : nullptr,
                                                str ? src.nu : nullptr, str ? 1 : 0, vflags.get());
    ST_LAUNCH("k_validate");
    if (d_targets) {
        k_validate<<<nblocks(nt, 256), 256, 0, s>>>(nt, d_targets, nullptr, nullptr, nullptr, 0, vflags.get() + 5);
        ST_LAUNCH("k_validate");
    }
    DevArray<double> rec(12 * n, s);
    const DevArray<uint32_t>& to_tree = tree.to_tree;
    k_pack_tree<<<nblocks(n, 256), 256, 0, s>>>(n, to_tree.get(), src.pos, sto ? src.f : nullptr,
                                                str ? src.h : nullptr, str ? src.nu : nullptr, rec.get());
    ST_LAUNCH("k_pack_tree");
    count_launch(3);
    e1.record(s);
    // moments at the largest order and every order's fold on a second stream (see
    // run_treecode); the far kernels wait for e2
    AuxStream aux;
    ST_CUDA(cudaStreamWaitEvent(aux.s, e1.e, 0));
    Event em;
    em.record(aux.s);
    DevArray<double> M;
    compute_moments_device(tree, rec.get(), pmax, sto, str, aux.s, M, &mplan);
    const double* tpos = same ? src.pos : d_targets;
    if (tperm.size() != nt) order_targets(tpos, nt, s, tperm);
    DevArray<double> tx(3 * nt, s);
    DevArray<uint32_t> torig(nt, s), tskip(nt, s);
    k_targets<<<nblocks(nt, 256), 256, 0, s>>>(nt, tperm.get(), tpos, same ? to_tree.get() : nullptr, tx.get(),
                                               torig.get(), tskip.get());
    ST_LAUNCH("k_targets");
    count_launch();
    DevArray<unsigned long long> d_stats(3, s);
    DevArray<int> d_err(1, s), d_work(2, s);
    d_stats.zero();
    d_err.zero();
    TravArgs a;
    a.tx = tx.get();
    a.tskip = tskip.get();
    a.torig = torig.get();
    a.nt = (int)nt;
    a.w0 = 0;
    a.w1 = (int)((nt + 31) / 32);
    a.geom = tree.geom.get();
    a.info = tree.info.get();
    a.ncl = tree.ncl;
    a.th2 = prm.theta * prm.theta;
    a.src = rec.get();
    a.stats = d_stats.get();
    a.err = d_err.get();
    a.work = d_work.get();
    // one plan, one near-field pass; per order the fold, the dense far events, the packed
    // sparse ones and the reduce: each order is bit-identical to a standalone call
    a.sparse_max = far_sparse_max();
    std::vector<DevArray<double>> Ws(n_orders), ufars(n_orders);
    std::vector<FarOrder> fo(n_orders);
    for (int i = 0; i < n_orders; ++i) {
        fold_weights_device(M.get(), tree.ncl, orders[i], sto, str, aux.s, Ws[i], pmax);
        ufars[i].alloc(3 * nt, s);
        fo[i].P = orders[i] + (str ? 2 : 1);
        fo[i].W = Ws[i].get();
        fo[i].ufar = ufars[i].get();
        fo[i].out = d_out + 3 * nt * i;
    }
    M.reset();
    e2.record(aux.s);
    EvalTimes tm;
    launch_eval(sto, str, a, fo.data(), n_orders, s, &tm, e2.e);
    for (int i = 0; i < n_orders; ++i)
        if (far_s) far_s[i] = tm.far_order[i];
    e3.record(s);
    ST_CUDA(cudaMemcpyAsync(&ro.domain_err, d_err.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
    ST_CUDA(cudaMemcpyAsync(ro.stats, d_stats.get(), sizeof ro.stats, cudaMemcpyDeviceToHost, s));
    ST_CUDA(cudaMemcpyAsync(ro.vflags, vflags.get(), sizeof ro.vflags, cudaMemcpyDeviceToHost, s));
    ST_CUDA(cudaStreamSynchronize(s));
    ro.t_build = secs(e0, e1);
    ro.t_moments = secs(em, e2);    // on the second stream, overlapped with the traversal
    ro.t_traverse = secs(e1, e3);   // targets, plan walks, far and near fields, reduce
    ro.t_total = secs(e0, e3);
}

// In-process exchange of the split moment pass (multi_device): every device thread
// publishes its rows, waits for the others (a host barrier), pulls the other devices'
// rows over NVLink (cudaMemcpyPeerAsync after the owner's event), and waits again before
// any owner may free its buffers.  A thread that fails breaks the barrier for the others.
struct PeerGroup {
    int D = 0;
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0, gen = 0;
    bool broken = false;
    std::vector<st_shard_exchange> ex;
    std::vector<int> dev;
    std::vector<cudaEvent_t> ready;
    void wait() {
        std::unique_lock<std::mutex> lk(mu);
        if (broken) fail(ST_RUNTIME_ERROR, "devices: another device failed");
        const int g = gen;
        if (++arrived == D) {
            arrived = 0;
            ++gen;
            cv.notify_all();
        } else {
            cv.wait(lk, [&] { return gen != g || broken; });
            if (broken) fail(ST_RUNTIME_ERROR, "devices: another device failed");
        }
    }
    void fail_all() {
        std::lock_guard<std::mutex> lk(mu);
        broken = true;
        cv.notify_all();
    }
};
struct PeerCtx {
    PeerGroup* g;
    int d;
};

int peer_exchange(void* vctx, const st_shard_exchange* ex) {
    PeerCtx* c = static_cast<PeerCtx*>(vctx);
    PeerGroup& g = *c->g;
    cudaStream_t s = static_cast<cudaStream_t>(ex->stream);
    ST_CUDA(cudaEventRecord(g.ready[c->d], s));
    g.ex[c->d] = *ex;
    g.wait();  // every device's rows are queued and its event recorded
    for (int q = 0; q < g.D; ++q) {
        if (q == c->d) continue;
        const st_shard_exchange& o = g.ex[q];
        ST_CUDA(cudaStreamWaitEvent(s, g.ready[q], 0));
        const size_t r0 = o.w_cuts[q], r1 = o.w_cuts[q + 1], u0 = o.m_cuts[q], u1 = o.m_cuts[q + 1];
        if (r1 > r0)
            ST_CUDA(cudaMemcpyPeerAsync(ex->w + r0 * ex->w_row, g.dev[c->d], o.w + r0 * o.w_row, g.dev[q],
                                        (r1 - r0) * o.w_row * sizeof(double), s));
        if (u1 > u0)
            ST_CUDA(cudaMemcpyPeerAsync(ex->m + u0 * ex->m_row, g.dev[c->d], o.m + u0 * o.m_row, g.dev[q],
                                        (u1 - u0) * o.m_row * sizeof(double), s));
    }
    ST_CUDA(cudaStreamSynchronize(s));
    g.wait();  // nobody reads another device's buffers any more
    return 0;
}

// Replicated-data multi-GPU in one process (PAPER.md:986-1030 with GPUs for MPI ranks):
// one host thread per logical device uploads the inputs, rebuilds the (bit-identical)
// tree and moments and evaluates its work-balanced shard of the key-ordered batches.
// The shard's epilogue (k_nreduce, and the count walk for per-target statistics) stores
// straight into device 0's output in original order -- NVLink peer stores from the
// kernel, no gather or scatter pass.  Logical devices beyond the physical count share
// GPUs round-robin (same results, no speedup).
void multi_device(const st_particles* src, const double* targets, size_t n_targets, const st_params& prm,
                  double* u_out, uint64_t* per_target, RunOut& ro_all, double& t_h2d, double& t_d2h) {
    const bool sto = prm.stokeslet != 0, str = prm.stresslet != 0;
    const int D = prm.devices;
    int ndev = 0;
    ST_CUDA(cudaGetDeviceCount(&ndev));
    const size_t nt = targets ? n_targets : src->n;
    int dev0 = 0;
    ST_CUDA(cudaGetDevice(&dev0));
    for (int d = 1; d < std::min(D, ndev); ++d) {  // peer stores into device 0
        const int dev = (dev0 + d) % ndev;
        int can = 0;
        ST_CUDA(cudaDeviceCanAccessPeer(&can, dev, dev0));
        if (!can) fail(ST_CUDA_ERROR, "devices > 1: GPU " + std::to_string(dev) + " cannot access GPU " +
                                          std::to_string(dev0) + " (NVLink peer access required)");
        ST_CUDA(cudaSetDevice(dev));
        const cudaError_t e = cudaDeviceEnablePeerAccess(dev0, 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) cuda_check(e, "cudaDeviceEnablePeerAccess");
        cudaGetLastError();
        pool_grant_peer(dev0, dev);  // the output buffers below come from device 0's pool
    }
    // the split moment pass copies weight rows between every pair of devices
    for (int a = 0; a < std::min(D, ndev); ++a)
        for (int b = 0; b < std::min(D, ndev); ++b) {
            const int da = (dev0 + a) % ndev, db = (dev0 + b) % ndev;
            int can = 0;
            if (da == db || cudaDeviceCanAccessPeer(&can, db, da) != cudaSuccess || !can) continue;
            ST_CUDA(cudaSetDevice(db));
            const cudaError_t e = cudaDeviceEnablePeerAccess(da, 0);
            if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) cuda_check(e, "cudaDeviceEnablePeerAccess");
            cudaGetLastError();
            pool_grant_peer(da, db);
        }
    ST_CUDA(cudaSetDevice(dev0));
    OwnedStream os0, os0w;
    cudaStream_t s0 = os0.s;
    // the host arrays cross PCIe once, to device 0 (positions and targets first, the weight
    // arrays after them on a second stream); every other device copies them from device 0
    // over NVLink (peer copies) as each part lands
    Event h0, pos_ready, w_ready0;
    h0.record(s0);
    DevParticles src0;
    src0.n = src->n;
    auto up0 = [&](const double* h, DevArray<double>& dst, cudaStream_t st) -> const double* {
        if (!h) return nullptr;
        dst.alloc(3 * src->n, st);
        h2d(dst.get(), h, 3 * src->n * sizeof(double), st);
        return dst.get();
    };
    src0.pos = up0(src->position, src0.own_pos, s0);
    DevArray<double> tg0;
    if (targets) {
        tg0.alloc(3 * nt, s0);
        h2d(tg0.get(), targets, 3 * nt * sizeof(double), s0);
    }
    pos_ready.record(s0);
    ST_CUDA(cudaStreamWaitEvent(os0w.s, pos_ready.e, 0));
    src0.f = sto ? up0(src->force_weight, src0.own_f, os0w.s) : nullptr;
    src0.h = str ? up0(src->dipole_weight, src0.own_h, os0w.s) : nullptr;
    src0.nu = str ? up0(src->normal, src0.own_nu, os0w.s) : nullptr;
    w_ready0.record(os0w.s);
    DevArray<double> du(3 * nt, s0);
    DevArray<uint64_t> dpt(per_target ? 3 * nt : 0, s0);
    ST_CUDA(cudaStreamSynchronize(s0));  // allocations complete before other devices store into them
    std::vector<RunOut> ros(D);
    std::vector<std::exception_ptr> errs(D);
    // the moment pass split over the devices, rows exchanged device to device (peer_exchange)
    PeerGroup grp;
    grp.D = D;
    grp.ex.resize(D);
    grp.dev.resize(D);
    grp.ready.assign(D, nullptr);
    for (int d = 0; d < D; ++d) {
        grp.dev[d] = (dev0 + d) % ndev;
        ST_CUDA(cudaSetDevice(grp.dev[d]));
        ST_CUDA(cudaEventCreateWithFlags(&grp.ready[d], cudaEventDisableTiming));
    }
    ST_CUDA(cudaSetDevice(dev0));
    std::vector<PeerCtx> pctx(D);
    auto work = [&](int d) {
        try {
            const int dev = (dev0 + d) % ndev;
            ST_CUDA(cudaSetDevice(dev));
            ensure_device();
            OwnedStream os, os2;
            cudaStream_t s = d == 0 ? s0 : os.s;
            pctx[d] = PeerCtx{&grp, d};
            SplitExchange x;
            x.fn = peer_exchange;
            x.ctx = &pctx[d];
            if (d == 0) {
                run_treecode(src0, targets ? tg0.get() : nullptr, nt, prm, du.get(), per_target ? dpt.get() : nullptr,
                             d, D, s, ros[d], false, nullptr, w_ready0.e, &x);
            } else {
                // device 0's copies, peer to peer: positions (and targets) on the compute stream,
                // the weight arrays on a second stream that run_treecode waits for after the build
                DevParticles dp;
                dp.n = src->n;
                auto peer = [&](const double* from, DevArray<double>& dst, cudaStream_t st) -> const double* {
                    if (!from) return nullptr;
                    dst.alloc(3 * src->n, st);
                    ST_CUDA(cudaMemcpyPeerAsync(dst.get(), dev, from, dev0, 3 * src->n * sizeof(double), st));
                    return dst.get();
                };
                ST_CUDA(cudaStreamWaitEvent(s, pos_ready.e, 0));
                dp.pos = peer(src0.pos, dp.own_pos, s);
                DevArray<double> dt;
                if (targets) {
                    dt.alloc(3 * nt, s);
                    ST_CUDA(cudaMemcpyPeerAsync(dt.get(), dev, tg0.get(), dev0, 3 * nt * sizeof(double), s));
                }
                ST_CUDA(cudaStreamWaitEvent(os2.s, w_ready0.e, 0));
                dp.f = peer(src0.f, dp.own_f, os2.s);
                dp.h = peer(src0.h, dp.own_h, os2.s);
                dp.nu = peer(src0.nu, dp.own_nu, os2.s);
                Event wd;
                wd.record(os2.s);
                run_treecode(dp, targets ? dt.get() : nullptr, nt, prm, du.get(), per_target ? dpt.get() : nullptr, d,
                             D, s, ros[d], false, nullptr, wd.e, &x);
                // the weight copies' stream-ordered frees are on os2: wait before it goes
                ST_CUDA(cudaStreamSynchronize(os2.s));
            }
            raise_flags(ros[d]);
        } catch (...) {
            errs[d] = std::current_exception();
            grp.fail_all();
        }
    };
    std::vector<std::thread> th;
    for (int d = 1; d < D; ++d) th.emplace_back(work, d);
    work(0);
    for (auto& t : th) t.join();  // every shard's stream has completed (run_treecode synchronises)
    for (int d = 0; d < D; ++d) {
        cudaSetDevice(grp.dev[d]);
        cudaEventDestroy(grp.ready[d]);
    }
    ST_CUDA(cudaSetDevice(dev0));
    for (auto& e : errs)
        if (e) std::rethrow_exception(e);
    Event d0, d1;
    d0.record(s0);
    d2h(u_out, du.get(), 3 * nt * sizeof(double), s0);
    if (per_target) d2h(per_target, dpt.get(), 3 * nt * sizeof(uint64_t), s0);
    d1.record(s0);
    ST_CUDA(cudaStreamSynchronize(s0));
    t_d2h = secs(d0, d1);
    t_h2d = secs(h0, w_ready0);  // the one PCIe upload (device 0); the rest moved over NVLink
    for (const RunOut& r : ros) {
        for (int k = 0; k < 3; ++k) ro_all.stats[k] += r.stats[k];
        ro_all.t_build = std::max(ro_all.t_build, r.t_build);
        ro_all.t_moments = std::max(ro_all.t_moments, r.t_moments);
        ro_all.t_traverse = std::max(ro_all.t_traverse, r.t_traverse);
        ro_all.t_total = std::max(ro_all.t_total, r.t_total);
        ro_all.t_far = std::max(ro_all.t_far, r.t_far);
        ro_all.t_near = std::max(ro_all.t_near, r.t_near);
    }
}

}  // namespace

void st::shard_cuts_host(size_t n, const double* w, int k, size_t* cuts) { shard_cuts_impl(n, w, k, cuts); }

namespace st {
st_status io_set_error(st_status s, const std::string& m) {
    g_last_error = m;
    return s;
}
}  // namespace st

// ====================================================================== C ABI
struct st_tree {
    OwnedStream own;  // declared first: destroyed after the arrays that free on it
    DevTree tree;
    DevArray<double> rec;  // tree-ordered source records (ClusterTree::particles)
    size_t n = 0;
    bool sto = false, str = false;
    cudaStream_t s = nullptr;
};

extern "C" {

int st_abi_version(void) { return ST_ABI_VERSION; }

st_status st_release_workspace(void) {
    return guarded([&] {
        int dev = 0;
        ST_CUDA(cudaGetDevice(&dev));
        ST_CUDA(cudaDeviceSynchronize());
        release_near_workspace(dev);
        ST_CUDA(cudaMemPoolTrimTo(device_pool(), 0));
    });
}

const char* st_last_error(void) { return g_last_error.c_str(); }

st_status st_device_count(int* out) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) n = 0;
    cudaGetLastError();
    if (out) *out = n;
    return ST_OK;
}

st_status st_params_validate(const st_params* p) {
    return guarded([&] { validate_params(p); });
}

st_status st_treecode_velocity_ex(const st_particles* src, const double* targets, size_t n_targets,
                                  const st_params* params, double* u_out, uint64_t* per_target,
                                  st_stats* stats) {
    return guarded([&] {
        g_launches = 0;
        validate_params(params);
        const bool sto = params->stokeslet != 0, str = params->stresslet != 0;
        validate_shape(src, sto, str);
        if (targets && n_targets == 0) fail(ST_INVALID_ARGUMENT, "targets: empty target set");
        if (!u_out) fail(ST_INVALID_ARGUMENT, "u_out: null");
        ensure_device();
        if (params->devices > 1) {
            RunOut ro;
            double th = 0, td = 0;
            multi_device(src, targets, n_targets, *params, u_out, per_target, ro, th, td);
            fill_stats(stats, ro);
            if (stats) {
                stats->time_h2d_s = th;
                stats->time_d2h_s = td;
                stats->gpu_launches = g_launches;
            }
            return;
        }
        OwnedStream os, os2;
        cudaStream_t s = os.s, s2 = os2.s;
        Event h0, h1, wready, d0, d1;
        h0.record(s);
        ST_CUDA(cudaStreamWaitEvent(s2, h0.e, 0));
        // positions (and targets) first on the compute stream: the tree build needs only
        // them; f, h, nu follow on a second stream and overlap the build
        DevParticles d;
        d.n = src->n;
        auto up = [&](const double* hsrc, DevArray<double>& dst, cudaStream_t st) -> const double* {
            if (!hsrc) return nullptr;
            dst.alloc(3 * src->n, st);
            h2d(dst.get(), hsrc, 3 * src->n * sizeof(double), st);
            return dst.get();
        };
        d.pos = up(src->position, d.own_pos, s);
        const size_t nt = targets ? n_targets : src->n;
        // ... after the positions: sharing the PCIe link with them would only delay the build.
        // Disjoint targets next (their ordering runs beside the build), then the weights.
        Event hpos, tready;
        hpos.record(s);
        ST_CUDA(cudaStreamWaitEvent(s2, hpos.e, 0));
        DevArray<double> dt;
        if (targets) {
            dt.alloc(3 * nt, s2);
            h2d(dt.get(), targets, 3 * nt * sizeof(double), s2);
            tready.record(s2);
        }
        d.f = sto ? up(src->force_weight, d.own_f, s2) : nullptr;
        d.h = str ? up(src->dipole_weight, d.own_h, s2) : nullptr;
        d.nu = str ? up(src->normal, d.own_nu, s2) : nullptr;
        wready.record(s2);
        DevArray<double> du(3 * nt, s);
        DevArray<uint64_t> dpt(per_target ? 3 * nt : 0, s);
        RunOut ro;
        run_treecode(d, targets ? dt.get() : nullptr, nt, *params, du.get(), per_target ? dpt.get() : nullptr, 0,
                     1, s, ro, false, nullptr, wready.e, nullptr, targets ? tready.e : nullptr);
        raise_flags(ro);
        d0.record(s);
        d2h(u_out, du.get(), 3 * nt * sizeof(double), s);
        if (per_target) d2h(per_target, dpt.get(), 3 * nt * sizeof(uint64_t), s);
        d1.record(s);
        ST_CUDA(cudaStreamSynchronize(s));
        // stream-ordered frees of the s2 uploads must not race the compute stream
        ST_CUDA(cudaStreamSynchronize(s2));
        fill_stats(stats, ro);
        if (stats) {
            stats->time_h2d_s = secs(h0, wready);
            stats->time_d2h_s = secs(d0, d1);
            stats->gpu_launches = g_launches;
        }
    });
}

st_status st_treecode_velocity_sweep(const st_particles* src, const double* targets, size_t n_targets,
                                     const st_params* params, const int* orders, int n_orders, double* u_out,
                                     double* far_seconds, st_stats* stats) {
    return guarded([&] {
        g_launches = 0;
        validate_params(params);
        if (!orders || n_orders < 1) fail(ST_INVALID_ARGUMENT, "sweep: no orders");
        for (int i = 0; i < n_orders; ++i)
            if (orders[i] < 0 || orders[i] > 16) fail(ST_INVALID_ARGUMENT, "params: order must be in [0, 16]");
        const bool sto = params->stokeslet != 0, str = params->stresslet != 0;
        validate_shape(src, sto, str);
        if (targets && n_targets == 0) fail(ST_INVALID_ARGUMENT, "targets: empty target set");
        if (!u_out) fail(ST_INVALID_ARGUMENT, "u_out: null");
        ensure_device();
        OwnedStream os;
        cudaStream_t s = os.s;
        DevParticles d;
        upload(src, sto, str, d, s);
        const size_t nt = targets ? n_targets : src->n;
        DevArray<double> dt;
        if (targets) {
            dt.alloc(3 * nt, s);
            h2d(dt.get(), targets, 3 * nt * sizeof(double), s);
        }
        DevArray<double> du(3 * nt * (size_t)n_orders, s);
        RunOut ro;
        run_sweep(d, targets ? dt.get() : nullptr, nt, *params, orders, n_orders, du.get(), far_seconds, s, ro);
        raise_flags(ro);
        d2h(u_out, du.get(), du.bytes(), s);
        ST_CUDA(cudaStreamSynchronize(s));
        fill_stats(stats, ro);
        if (stats) stats->gpu_launches = g_launches;
    });
}

st_status st_treecode_velocity(const st_particles* src, const st_params* params, double* u_out,
                               st_stats* stats) {
    return st_treecode_velocity_ex(src, nullptr, 0, params, u_out, nullptr, stats);
}

st_status st_treecode_shard_device(const st_particles* src, const double* targets, size_t n_targets,
                                   const st_params* params, int shard, int n_shards, double* u_batch,
                                   uint32_t* batch_to_original, size_t* t0, size_t* t1, void* stream,
                                   st_stats* stats) {
    return guarded([&] {
        g_launches = 0;
        validate_params(params);
        const bool sto = params->stokeslet != 0, str = params->stresslet != 0;
        validate_shape(src, sto, str);
        if (n_shards < 1 || shard < 0 || shard >= n_shards) fail(ST_INVALID_ARGUMENT, "shard out of range");
        if (targets && n_targets == 0) fail(ST_INVALID_ARGUMENT, "targets: empty target set");
        if (!u_batch) fail(ST_INVALID_ARGUMENT, "u_batch: null");
        ensure_device();
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        DevParticles d;
        d.n = src->n;
        d.pos = src->position;
        d.f = sto ? src->force_weight : nullptr;
        d.h = str ? src->dipole_weight : nullptr;
        d.nu = str ? src->normal : nullptr;
        const size_t nt = targets ? n_targets : src->n;
        RunOut ro;
        ShardOut so;
        run_treecode(d, targets, nt, *params, u_batch, nullptr, shard, n_shards, s, ro, true, &so);
        raise_flags(ro);
        if (t0) *t0 = std::min(nt, (size_t)so.w0 * 32);
        if (t1) *t1 = std::min(nt, (size_t)so.w1 * 32);
        if (batch_to_original)
            ST_CUDA(cudaMemcpyAsync(batch_to_original, so.torig.get(), nt * sizeof(uint32_t), cudaMemcpyDeviceToDevice,
                                    s));
        fill_stats(stats, ro);
        if (stats) stats->gpu_launches = g_launches;
    });
}

st_status st_unbatch_device(size_t n, const uint32_t* batch_to_original, const double* u_batch, double* u_out,
                            void* stream) {
    return guarded([&] {
        if (!n) return;
        if (!batch_to_original || !u_batch || !u_out) fail(ST_INVALID_ARGUMENT, "unbatch: null pointer");
        ensure_device();
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        k_unbatch<<<nblocks(n, 256), 256, 0, s>>>(n, batch_to_original, u_batch, nullptr, u_out, nullptr);
        ST_LAUNCH("k_unbatch");
        count_launch();
    });
}

namespace {
std::mutex g_ipc_mu;
std::map<void*, void*> g_ipc_open;  // pointer handed out by st_ipc_open -> mapped allocation base
}  // namespace

st_status st_ipc_export(const void* dptr, unsigned char handle[64], size_t* offset) {
    return guarded([&] {
        if (!dptr || !handle || !offset) fail(ST_INVALID_ARGUMENT, "ipc_export: null pointer");
        ensure_device();
        using GetRange = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
        static GetRange get_range = [] {
            void* fn = nullptr;
            cudaDriverEntryPointQueryResult q{};
            ST_CUDA(cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q));
            if (!fn || q != cudaDriverEntryPointSuccess) fail(ST_CUDA_ERROR, "ipc_export: cuMemGetAddressRange missing");
            return reinterpret_cast<GetRange>(fn);
        }();
        CUdeviceptr base = 0;
        size_t bytes = 0;
        if (get_range(&base, &bytes, reinterpret_cast<CUdeviceptr>(dptr)) != CUDA_SUCCESS)
            fail(ST_INVALID_ARGUMENT, "ipc_export: not a device allocation");
        cudaIpcMemHandle_t h;
        ST_CUDA(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)));
        static_assert(sizeof h == 64, "CUDA IPC handles are 64 bytes");
        std::memcpy(handle, &h, sizeof h);
        *offset = static_cast<size_t>(reinterpret_cast<CUdeviceptr>(dptr) - base);
    });
}

st_status st_ipc_open(const unsigned char handle[64], size_t offset, void** dptr) {
    return guarded([&] {
        if (!handle || !dptr) fail(ST_INVALID_ARGUMENT, "ipc_open: null pointer");
        ensure_device();
        cudaIpcMemHandle_t h;
        std::memcpy(&h, handle, sizeof h);
        void* base = nullptr;
        ST_CUDA(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess));
        *dptr = static_cast<char*>(base) + offset;
        std::lock_guard<std::mutex> lk(g_ipc_mu);
        g_ipc_open[*dptr] = base;
    });
}

st_status st_ipc_close(void* dptr) {
    return guarded([&] {
        void* base = nullptr;
        {
            std::lock_guard<std::mutex> lk(g_ipc_mu);
            auto it = g_ipc_open.find(dptr);
            if (it == g_ipc_open.end()) fail(ST_INVALID_ARGUMENT, "ipc_close: pointer not from st_ipc_open");
            base = it->second;
            g_ipc_open.erase(it);
        }
        ST_CUDA(cudaIpcCloseMemHandle(base));
    });
}

st_status st_treecode_velocity_device(const st_particles* src, const double* targets, size_t n_targets,
                                      const st_params* params, double* u_out, int shard, int n_shards,
                                      void* stream, st_stats* stats) {
    return st_treecode_velocity_device_ev(src, targets, n_targets, params, u_out, shard, n_shards, stream, nullptr,
                                          stats);
}

st_status st_treecode_velocity_device_ev(const st_particles* src, const double* targets, size_t n_targets,
                                         const st_params* params, double* u_out, int shard, int n_shards,
                                         void* stream, void* weights_ready, st_stats* stats) {
    return st_treecode_velocity_device_ev2(src, targets, n_targets, params, u_out, shard, n_shards, stream, nullptr,
                                           weights_ready, stats);
}

st_status st_treecode_velocity_device_ev2(const st_particles* src, const double* targets, size_t n_targets,
                                          const st_params* params, double* u_out, int shard, int n_shards,
                                          void* stream, void* targets_ready, void* weights_ready,
                                          st_stats* stats) {
    return guarded([&] {
        g_launches = 0;
        validate_params(params);
        const bool sto = params->stokeslet != 0, str = params->stresslet != 0;
        validate_shape(src, sto, str);
        if (n_shards < 1 || shard < 0 || shard >= n_shards) fail(ST_INVALID_ARGUMENT, "shard out of range");
        if (targets && n_targets == 0) fail(ST_INVALID_ARGUMENT, "targets: empty target set");
        ensure_device();
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        DevParticles d;
        d.n = src->n;
        d.pos = src->position;
        d.f = sto ? src->force_weight : nullptr;
        d.h = str ? src->dipole_weight : nullptr;
        d.nu = str ? src->normal : nullptr;
        RunOut ro;
        run_treecode(d, targets, targets ? n_targets : src->n, *params, u_out, nullptr, shard, n_shards, s, ro,
                     false, nullptr, static_cast<cudaEvent_t>(weights_ready), nullptr,
                     static_cast<cudaEvent_t>(targets_ready));
        raise_flags(ro);
        fill_stats(stats, ro);
        if (stats) stats->gpu_launches = g_launches;
    });
}

}  // extern "C"

struct st_comm {
    NcclComm* c = nullptr;
};

extern "C" {

st_status st_nccl_unique_id(unsigned char id[128]) {
    return guarded([&] {
        if (!id) fail(ST_INVALID_ARGUMENT, "nccl: null id");
        nccl_unique_id(id);
    });
}

st_status st_nccl_comm_init(const unsigned char id[128], int n_ranks, int rank, st_comm** comm) {
    return guarded([&] {
        if (!id || !comm) fail(ST_INVALID_ARGUMENT, "nccl: null argument");
        ensure_device();
        st_comm* c = new st_comm;
        try {
            c->c = nccl_comm_init(id, n_ranks, rank);
        } catch (...) {
            delete c;
            throw;
        }
        *comm = c;
    });
}

void st_nccl_comm_free(st_comm* comm) {
    if (!comm) return;
    nccl_comm_free(comm->c);
    delete comm;
}

st_status st_treecode_velocity_nccl(const st_particles* src, const double* targets, size_t n_targets,
                                    const st_params* params, double* u_out, const st_comm* comm, void* stream,
                                    st_stats* stats) {
    return guarded([&] {
        g_launches = 0;
        validate_params(params);
        if (!comm || !comm->c) fail(ST_INVALID_ARGUMENT, "nccl: null communicator");
        const bool sto = params->stokeslet != 0, str = params->stresslet != 0;
        validate_shape(src, sto, str);
        if (targets && n_targets == 0) fail(ST_INVALID_ARGUMENT, "targets: empty target set");
        ensure_device();
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        const int rank = nccl_rank(comm->c), world = nccl_ranks(comm->c);
        const size_t nt = targets ? n_targets : src->n;
        DevParticles d;
        d.n = src->n;
        d.pos = src->position;
        d.f = sto ? src->force_weight : nullptr;
        d.h = str ? src->dipole_weight : nullptr;
        d.nu = str ? src->normal : nullptr;
        ST_CUDA(cudaMemsetAsync(u_out, 0, 3 * nt * sizeof(double), s));
        SplitExchange x;
        x.fn = nccl_exchange;
        x.ctx = comm->c;
        RunOut ro;
        run_treecode(d, targets, nt, *params, u_out, nullptr, rank, world, s, ro, false, nullptr, nullptr,
                     world > 1 ? &x : nullptr);
        // the gather before any error is raised: a domain error is found by the rank whose
        // shard holds the coincident pair, and every rank must take part in the collective
        // counters: the three statistics, then how many ranks saw each error bit
        unsigned long long* h = static_cast<unsigned long long*>(pinned_stage(5 * sizeof(unsigned long long)));
        for (int k = 0; k < 3; ++k) h[k] = ro.stats[k];
        h[3] = (unsigned long long)(ro.domain_err & 1);
        h[4] = (unsigned long long)((ro.domain_err >> 1) & 1);
        DevArray<unsigned long long> dst(5, s);
        ST_CUDA(cudaMemcpyAsync(dst.get(), h, 5 * sizeof(unsigned long long), cudaMemcpyHostToDevice, s));
        nccl_gather(comm->c, u_out, 3 * nt, dst.get(), 5, s);
        ST_CUDA(cudaMemcpyAsync(h, dst.get(), 5 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
        ST_CUDA(cudaStreamSynchronize(s));
        for (int k = 0; k < 3; ++k) ro.stats[k] = h[k];
        ro.domain_err = (h[3] ? 1 : 0) | (h[4] ? 2 : 0);
        raise_flags(ro);
        fill_stats(stats, ro);
        if (stats) stats->gpu_launches = g_launches;
    });
}

st_status st_treecode_velocity_device_split(const st_particles* src, const double* targets, size_t n_targets,
                                            const st_params* params, double* u_out, int shard, int n_shards,
                                            void* stream, st_exchange_fn exchange, void* ctx, st_stats* stats) {
    return guarded([&] {
        g_launches = 0;
        validate_params(params);
        const bool sto = params->stokeslet != 0, str = params->stresslet != 0;
        validate_shape(src, sto, str);
        if (n_shards < 1 || shard < 0 || shard >= n_shards) fail(ST_INVALID_ARGUMENT, "shard out of range");
        if (targets && n_targets == 0) fail(ST_INVALID_ARGUMENT, "targets: empty target set");
        ensure_device();
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        DevParticles d;
        d.n = src->n;
        d.pos = src->position;
        d.f = sto ? src->force_weight : nullptr;
        d.h = str ? src->dipole_weight : nullptr;
        d.nu = str ? src->normal : nullptr;
        RunOut ro;
        SplitExchange x;
        x.fn = exchange;
        x.ctx = ctx;
        run_treecode(d, targets, targets ? n_targets : src->n, *params, u_out, nullptr, shard, n_shards, s, ro,
                     false, nullptr, nullptr, &x);
        raise_flags(ro);
        fill_stats(stats, ro);
        if (stats) stats->gpu_launches = g_launches;
    });
}

st_status st_interaction_lists(const st_particles* src, const st_params* params, const size_t* target_index,
                               const double* points, size_t n_sel, size_t cap, int32_t* far, int32_t* near,
                               int64_t* n_far, int64_t* n_near) {
    return guarded([&] {
        validate_params(params);
        validate_shape(src, params->stokeslet != 0, params->stresslet != 0);
        if (!points && !target_index && n_sel) fail(ST_INVALID_ARGUMENT, "interaction_lists: no targets");
        if (!n_sel) return;
        ensure_device();
        OwnedStream os;
        cudaStream_t s = os.s;
        DevParticles d;
        upload(src, false, false, d, s);
        DevTree tree;
        build_tree_device(d.pos, d.n, params->leaf_capacity, params->shrink != 0, true, s, tree);
        DevArray<uint32_t> to_tree(d.n, s);
        DevArray<double> rec(12 * d.n, s);
        k_pack<<<nblocks(d.n, 256), 256, 0, s>>>(d.n, tree.perm.get(), d.pos, nullptr, nullptr, nullptr, rec.get(),
                                                 to_tree.get());
        ST_LAUNCH("k_pack");
        // selected targets (positions; self exclusion only matters for the counts, not the lists)
        std::vector<double> hx(3 * n_sel);
        if (points) {
            std::copy(points, points + 3 * n_sel, hx.begin());
        } else {
            for (size_t i = 0; i < n_sel; ++i) {
                if (target_index[i] >= src->n) fail(ST_INVALID_ARGUMENT, "interaction_lists: target out of range");
                for (int a = 0; a < 3; ++a) hx[3 * i + a] = src->position[3 * target_index[i] + a];
            }
        }
        DevArray<double> tx(3 * n_sel, s);
        ST_CUDA(cudaMemcpyAsync(tx.get(), hx.data(), hx.size() * sizeof(double), cudaMemcpyHostToDevice, s));
        DevArray<int32_t> dfar(n_sel * cap, s), dnear(n_sel * cap, s);
        DevArray<int64_t> dnf(n_sel, s), dnn(n_sel, s);
        dfar.fill_bytes(0xff);
        dnear.fill_bytes(0xff);
        TravArgs a;
        a.tx = tx.get();
        a.nt = (int)n_sel;
        a.geom = tree.geom.get();
        a.info = tree.info.get();
        a.ncl = tree.ncl;
        a.th2 = params->theta * params->theta;
        launch_lists(a, (int)cap, dfar.get(), dnear.get(), dnf.get(), dnn.get(), s);
        if (far) ST_CUDA(cudaMemcpyAsync(far, dfar.get(), dfar.bytes(), cudaMemcpyDeviceToHost, s));
        if (near) ST_CUDA(cudaMemcpyAsync(near, dnear.get(), dnear.bytes(), cudaMemcpyDeviceToHost, s));
        if (n_far) ST_CUDA(cudaMemcpyAsync(n_far, dnf.get(), dnf.bytes(), cudaMemcpyDeviceToHost, s));
        if (n_near) ST_CUDA(cudaMemcpyAsync(n_near, dnn.get(), dnn.bytes(), cudaMemcpyDeviceToHost, s));
        ST_CUDA(cudaStreamSynchronize(s));
    });
}

// The callers have validated shapes and values on the host (then the target range, as
// in the reference, kernels.hpp:125-127, 143-146).
static void direct_common(const st_particles* src, int sto, int str, const std::vector<int64_t>& tg,
                          double* u_out, bool naive) {
    ensure_device();
    OwnedStream os;
    cudaStream_t s = os.s;
    DevParticles d;
    upload(src, sto != 0, str != 0, d, s);
    DevArray<double> rec(12 * d.n, s);
    k_pack<<<nblocks(d.n, 256), 256, 0, s>>>(d.n, nullptr, d.pos, d.f, d.h, d.nu, rec.get(), nullptr);
    ST_LAUNCH("k_pack");
    DevArray<int> err(1, s);
    err.zero();
    const size_t nt = naive ? d.n : tg.size();
    DevArray<double> du(3 * std::max<size_t>(nt, 1), s);
    if (naive) {
        launch_naive(sto != 0, str != 0, rec.get(), d.n, du.get(), err.get(), s);
    } else if (nt) {
        DevArray<int64_t> dtg(nt, s);
        ST_CUDA(cudaMemcpyAsync(dtg.get(), tg.data(), nt * sizeof(int64_t), cudaMemcpyHostToDevice, s));
        launch_direct(sto != 0, str != 0, rec.get(), d.n, dtg.get(), nt, du.get(), err.get(), s);
    }
    int herr = 0;
    ST_CUDA(cudaMemcpyAsync(&herr, err.get(), sizeof herr, cudaMemcpyDeviceToHost, s));
    if (nt) d2h(u_out, du.get(), 3 * nt * sizeof(double), s);
    ST_CUDA(cudaStreamSynchronize(s));
    if (herr)
        // naive_direct_velocity forms the Stokeslet before the stresslet (kernels.hpp:98-112)
        fail(ST_DOMAIN_ERROR, naive ? (sto ? "stokeslet: coincident points" : "stresslet: coincident points")
                                    : "direct sum: coincident particles");
}

st_status st_direct_velocity(const st_particles* src, int sto, int str, size_t first, size_t last,
                             double* u_out) {
    return guarded([&] {
        validate_shape(src, sto != 0, str != 0);
        validate_values_host(src, sto != 0, str != 0);
        if (first > last || last > src->n)
            fail(ST_INVALID_ARGUMENT, "contracted_direct_velocity: bad target range");
        std::vector<int64_t> tg(last - first);
        for (size_t i = first; i < last; ++i) tg[i - first] = (int64_t)i;
        direct_common(src, sto, str, tg, u_out, false);
    });
}

st_status st_direct_velocity_at(const st_particles* src, int sto, int str, const size_t* targets,
                                size_t n_targets, double* u_out) {
    return guarded([&] {
        validate_shape(src, sto != 0, str != 0);
        validate_values_host(src, sto != 0, str != 0);
        std::vector<int64_t> tg(n_targets);
        for (size_t i = 0; i < n_targets; ++i) {
            if (targets[i] >= src->n)
                fail(ST_INVALID_ARGUMENT, "contracted_direct_velocity_at: target out of range");
            tg[i] = (int64_t)targets[i];
        }
        direct_common(src, sto, str, tg, u_out, false);
    });
}

st_status st_naive_direct_velocity(const st_particles* src, int sto, int str, double* u_out) {
    return guarded([&] {
        validate_shape(src, sto != 0, str != 0);
        validate_values_host(src, sto != 0, str != 0);
        direct_common(src, sto, str, {}, u_out, true);
    });
}

st_status st_build_tree(const st_particles* src, int leaf_capacity, int shrink, st_tree** out) {
    return guarded([&] {
        if (!out) fail(ST_INVALID_ARGUMENT, "build_tree: null output");
        *out = nullptr;
        if (!src || src->n == 0) fail(ST_INVALID_ARGUMENT, "build_tree: empty particle set");
        if (!src->position) fail(ST_INVALID_ARGUMENT, "build_tree: null positions");
        if (leaf_capacity < 1) fail(ST_INVALID_ARGUMENT, "build_tree: leaf capacity must be >= 1");
        ensure_device();
        auto* t = new st_tree();
        try {
            t->s = t->own.s;
            t->n = src->n;
            t->sto = src->force_weight != nullptr;
            t->str = src->dipole_weight != nullptr && src->normal != nullptr;
            DevParticles d;
            upload(src, t->sto, t->str, d, t->s);
            build_tree_device(d.pos, d.n, leaf_capacity, shrink != 0, true, t->s, t->tree);
            t->rec.alloc(12 * d.n, t->s);
            k_pack<<<nblocks(d.n, 256), 256, 0, t->s>>>(d.n, t->tree.perm.get(), d.pos, d.f, d.h, d.nu,
                                                        t->rec.get(), nullptr);
            ST_LAUNCH("k_pack");
            ST_CUDA(cudaStreamSynchronize(t->s));
        } catch (...) {
            delete t;
            throw;
        }
        *out = t;
    });
}

size_t st_tree_num_clusters(const st_tree* t) { return t ? (size_t)t->tree.ncl : 0; }
size_t st_tree_num_particles(const st_tree* t) { return t ? t->n : 0; }

st_status st_tree_export(const st_tree* t, int64_t* begin_end, double* geom, int32_t* children,
                         int32_t* meta, uint32_t* to_original) {
    return guarded([&] {
        if (!t) fail(ST_INVALID_ARGUMENT, "tree: null");
        const int ncl = t->tree.ncl;
        cudaStream_t s = t->s;
        std::vector<int4> info(ncl);
        std::vector<double4> g(ncl);
        std::vector<double> bb(6 * (size_t)ncl);
        std::vector<int32_t> ch(8 * (size_t)ncl), nch(ncl);
        ST_CUDA(cudaMemcpyAsync(info.data(), t->tree.info.get(), sizeof(int4) * ncl, cudaMemcpyDeviceToHost, s));
        ST_CUDA(cudaMemcpyAsync(g.data(), t->tree.geom.get(), sizeof(double4) * ncl, cudaMemcpyDeviceToHost, s));
        ST_CUDA(cudaMemcpyAsync(bb.data(), t->tree.bbox.get(), sizeof(double) * 6 * ncl, cudaMemcpyDeviceToHost, s));
        ST_CUDA(cudaMemcpyAsync(ch.data(), t->tree.children.get(), sizeof(int32_t) * 8 * ncl,
                                cudaMemcpyDeviceToHost, s));
        ST_CUDA(cudaMemcpyAsync(nch.data(), t->tree.nchild.get(), sizeof(int32_t) * ncl, cudaMemcpyDeviceToHost, s));
        if (to_original)
            ST_CUDA(cudaMemcpyAsync(to_original, t->tree.perm.get(), sizeof(uint32_t) * t->n,
                                    cudaMemcpyDeviceToHost, s));
        ST_CUDA(cudaStreamSynchronize(s));
        for (int v = 0; v < ncl; ++v) {
            if (begin_end) {
                begin_end[2 * v] = info[v].x;
                begin_end[2 * v + 1] = info[v].y;
            }
            if (geom) {
                double* q = geom + 10 * (size_t)v;
                q[0] = g[v].x;
                q[1] = g[v].y;
                q[2] = g[v].z;
                q[3] = g[v].w;
                for (int a = 0; a < 6; ++a) q[4 + a] = bb[6 * (size_t)v + a];
            }
            if (children)
                for (int j = 0; j < 8; ++j) children[8 * (size_t)v + j] = ch[8 * (size_t)v + j];
            if (meta) {
                meta[2 * v] = nch[v];
                meta[2 * v + 1] = info[v].w;
            }
        }
    });
}

void st_tree_free(st_tree* t) { delete t; }

st_status st_compute_moments(const st_tree* t, int order, int sto, int str, double* stok, double* strm,
                             double* trace, double* sym) {
    return guarded([&] {
        if (!t) fail(ST_INVALID_ARGUMENT, "tree: null");
        if (order < 0 || order > 16) fail(ST_INVALID_ARGUMENT, "compute_moments: order outside table range");
        if (!sto && !str) fail(ST_INVALID_ARGUMENT, "kernel selection: at least one kernel must be enabled");
        if ((sto && !t->sto) || (str && !t->str))
            fail(ST_INVALID_ARGUMENT, "compute_moments: tree was built without the weights of this kernel");
        cudaStream_t s = t->s;
        DevArray<double> M;
        compute_moments_device(t->tree, t->rec.get(), order, sto != 0, str != 0, s, M);
        const size_t E = mi_count(order), ncl = t->tree.ncl;
        DevArray<double> a(sto ? 3 * E * ncl : 0, s), b(str ? 9 * E * ncl : 0, s), c(str ? E * ncl : 0, s),
            d(str ? 6 * E * ncl : 0, s);
        export_moments_device(M.get(), (int)ncl, order, sto != 0, str != 0, a.get(), b.get(), c.get(), d.get(), s);
        auto down = [&](double* h, const DevArray<double>& x) {
            if (h && x.size()) ST_CUDA(cudaMemcpyAsync(h, x.get(), x.bytes(), cudaMemcpyDeviceToHost, s));
        };
        down(stok, a);
        down(strm, b);
        down(trace, c);
        down(sym, d);
        ST_CUDA(cudaStreamSynchronize(s));
    });
}

st_status st_coulomb_coeffs(size_t n, const double* dx, int pmax, double* b_out) {
    return guarded([&] {
        if (pmax < 0) fail(ST_INVALID_ARGUMENT, "MultiIndexTable: pmax must be >= 0");
        for (size_t i = 0; i < n; ++i) {
            const double r2 = dx[3 * i] * dx[3 * i] + dx[3 * i + 1] * dx[3 * i + 1] + dx[3 * i + 2] * dx[3 * i + 2];
            if (!(r2 > 0.0)) fail(ST_DOMAIN_ERROR, "coulomb_coeffs: zero displacement");
        }
        if (!n) return;
        ensure_device();
        OwnedStream os;
        cudaStream_t s = os.s;
        const size_t E = mi_count(pmax);
        DevArray<double> ddx(3 * n, s), db(E * n, s);
        ST_CUDA(cudaMemcpyAsync(ddx.get(), dx, 3 * n * sizeof(double), cudaMemcpyHostToDevice, s));
        launch_coulomb(n, ddx.get(), pmax, db.get(), s);
        ST_CUDA(cudaMemcpyAsync(b_out, db.get(), db.bytes(), cudaMemcpyDeviceToHost, s));
        ST_CUDA(cudaStreamSynchronize(s));
    });
}

st_status st_taylor_coeffs(size_t n, const double* dx, const double* b, int pmax_b, int order, double* a_sto,
                           double* a_str) {
    return guarded([&] {
        if (pmax_b < 0 || order < 0) fail(ST_INVALID_ARGUMENT, "MultiIndexTable: pmax must be >= 0");
        if (a_sto && order + 1 > pmax_b)
            fail(ST_INVALID_ARGUMENT, "stokeslet_taylor_coeff: coefficients not deep enough");
        if (a_str && order + 2 > pmax_b)
            fail(ST_INVALID_ARGUMENT, "stresslet_taylor_coeff: coefficients not deep enough");
        if (!b)
            for (size_t i = 0; i < n; ++i) {
                const double r2 = dx[3 * i] * dx[3 * i] + dx[3 * i + 1] * dx[3 * i + 1] + dx[3 * i + 2] * dx[3 * i + 2];
                if (!(r2 > 0.0)) fail(ST_DOMAIN_ERROR, "coulomb_coeffs: zero displacement");
            }
        if (!n || (!a_sto && !a_str)) return;
        ensure_device();
        OwnedStream os;
        cudaStream_t s = os.s;
        const size_t EB = mi_count(pmax_b), E = mi_count(order);
        DevArray<double> ddx(3 * n, s), db(EB * n, s), da(a_sto ? 9 * E * n : 0, s), dt(a_str ? 27 * E * n : 0, s);
        ST_CUDA(cudaMemcpyAsync(ddx.get(), dx, ddx.bytes(), cudaMemcpyHostToDevice, s));
        if (b) ST_CUDA(cudaMemcpyAsync(db.get(), b, db.bytes(), cudaMemcpyHostToDevice, s));
        else launch_coulomb(n, ddx.get(), pmax_b, db.get(), s);
        launch_taylor(n, ddx.get(), db.get(), pmax_b, order, a_sto ? da.get() : nullptr, a_str ? dt.get() : nullptr, s);
        if (a_sto) ST_CUDA(cudaMemcpyAsync(a_sto, da.get(), da.bytes(), cudaMemcpyDeviceToHost, s));
        if (a_str) ST_CUDA(cudaMemcpyAsync(a_str, dt.get(), dt.bytes(), cudaMemcpyDeviceToHost, s));
        ST_CUDA(cudaStreamSynchronize(s));
    });
}

st_status st_farfield_pairs(size_t n, const double* dx, int order, int sto, int str, const double* stok,
                            const double* strm, const double* /*trace*/, const double* /*sym*/,
                            double* u_out) {
    return guarded([&] {
        if (order < 0 || order > 16) fail(ST_INVALID_ARGUMENT, "farfield: order out of range");
        if (!sto && !str) fail(ST_INVALID_ARGUMENT, "kernel selection: at least one kernel must be enabled");
        if ((sto && !stok) || (str && !strm)) fail(ST_INVALID_ARGUMENT, "farfield: moment order mismatch");
        for (size_t i = 0; i < n; ++i) {
            const double r2 = dx[3 * i] * dx[3 * i] + dx[3 * i + 1] * dx[3 * i + 1] + dx[3 * i + 2] * dx[3 * i + 2];
            if (!(r2 > 0.0)) fail(ST_DOMAIN_ERROR, "coulomb_coeffs: zero displacement");
        }
        if (!n) return;
        ensure_device();
        OwnedStream os;
        cudaStream_t s = os.s;
        const size_t E = mi_count(order);
        DevArray<double> ddx(3 * n, s), a(sto ? 3 * E * n : 0, s), b(str ? 9 * E * n : 0, s), M(12 * E * n, s), W,
            du(3 * n, s);
        ST_CUDA(cudaMemcpyAsync(ddx.get(), dx, 3 * n * sizeof(double), cudaMemcpyHostToDevice, s));
        if (sto) ST_CUDA(cudaMemcpyAsync(a.get(), stok, a.bytes(), cudaMemcpyHostToDevice, s));
        if (str) ST_CUDA(cudaMemcpyAsync(b.get(), strm, b.bytes(), cudaMemcpyHostToDevice, s));
        import_moments_device((int)n, order, sto != 0, str != 0, a.get(), b.get(), M.get(), s);
        fold_weights_device(M.get(), (int)n, order, sto != 0, str != 0, s, W);
        launch_far_pairs(order + (str ? 2 : 1), n, ddx.get(), W.get(), du.get(), s);
        ST_CUDA(cudaMemcpyAsync(u_out, du.get(), du.bytes(), cudaMemcpyDeviceToHost, s));
        ST_CUDA(cudaStreamSynchronize(s));
    });
}

st_status st_relative_error(size_t n, const double* u_ref, const double* u_test, double* out) {
    return guarded([&] {
        if (n == 0) fail(ST_INVALID_ARGUMENT, "relative_error: empty fields");
        double num = 0.0, den = 0.0;
        for (size_t i = 0; i < n; ++i) {
            const double* a = u_ref + 3 * i;
            const double* b = u_test + 3 * i;
            const double d0 = a[0] - b[0], d1 = a[1] - b[1], d2 = a[2] - b[2];
            num += d0 * d0 + d1 * d1 + d2 * d2;
            den += a[0] * a[0] + a[1] * a[1] + a[2] * a[2];
        }
        if (den == 0.0) fail(ST_DOMAIN_ERROR, "relative_error: reference field is identically zero");
        *out = std::sqrt(num / den);
    });
}

st_status st_shard_cuts(size_t n_units, const double* weights, int n_shards, size_t* cuts) {
    return guarded([&] {
        if (n_shards < 1) fail(ST_INVALID_ARGUMENT, "shard_cuts: n_shards must be >= 1");
        if (!cuts || (n_units && !weights)) fail(ST_INVALID_ARGUMENT, "shard_cuts: null buffer");
        shard_cuts_host(n_units, weights, n_shards, cuts);
    });
}

st_status st_fp64_peak(double seconds, double* tflops) {
    return guarded([&] {
        ensure_device();
        OwnedStream os;
        cudaStream_t s = os.s;
        int dev = 0, nsm = 0;
        ST_CUDA(cudaGetDevice(&dev));
        ST_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
        DevArray<double> sink(1, s);
        const int blocks = nsm * 8, threads = 256;
        Event a, b;
        int iters = 256;
        double t = 0.0;
        for (;;) {
            a.record(s);
            k_fp64_peak<<<blocks, threads, 0, s>>>(sink.get(), iters, 1.0);
            ST_LAUNCH("k_fp64_peak");
            b.record(s);
            ST_CUDA(cudaStreamSynchronize(s));
            t = secs(a, b);
            if (t >= seconds || iters > (1 << 24)) break;
            iters *= std::max(2, (int)std::min(16.0, seconds / std::max(t, 1e-6)));
        }
        const double fmas = (double)blocks * threads * iters * 16.0 * 8.0;
        *tflops = 2.0 * fmas / t * 1e-12;
    });
}

}  // extern "C"
