// Shared host/device plumbing for the sm_100a treecode kernels.
#pragma once

#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <cstring>
#include <cstdlib>

#include <cstddef>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>

#include "stokestree_c.h"

namespace st {

// Error carrying the C-ABI status it maps to (ST_* in stokestree_c.h).
struct Error : std::runtime_error {
    st_status status;
    Error(st_status s, const std::string& m) : std::runtime_error(m), status(s) {}
};

[[noreturn]] inline void fail(st_status s, const std::string& m) { throw Error(s, m); }

inline void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess)
        fail(ST_CUDA_ERROR, std::string(what) + ": " + cudaGetErrorName(e) + " (" +
                                cudaGetErrorString(e) + ")");
}
#define ST_CUDA(call) ::st::cuda_check((call), #call)
#define ST_LAUNCH(what) ::st::cuda_check(cudaGetLastError(), what)

// Contiguous work-balanced cut points cuts[0..k] of n units with weights w (st_shard_cuts).
void shard_cuts_host(size_t n, const double* w, int k, size_t* cuts);

// Kernel-launch counter (reported as st_stats.gpu_launches).
extern thread_local uint64_t g_launches;
inline void count_launch(uint64_t k = 1) { g_launches += k; }

// Pinned host staging for the small host<->device transfers inside a call (plan lists up,
// counts and cuts down).  A pageable transfer is not asynchronous: an upload first waits for
// its stream to drain and a download goes through the driver's staging copy, so the host
// stalls behind the other stream's kernels (measured: 2-2.4 ms at cfg2 / cfg4 before the
// plan could be sized).  Per host thread, grow-only; pinned_reset() at each C-ABI entry
// (every call synchronises its streams before returning, so the previous call's copies
// are done with it).
void* pinned_stage(size_t bytes);  // 16-byte aligned, valid until the next pinned_reset()
void pinned_reset();
template <class T>
T* pinned_copy(const T* src, size_t n) {
    T* p = static_cast<T*>(pinned_stage(n * sizeof(T)));
    if (n) memcpy(p, src, n * sizeof(T));
    return p;
}

// Timing event (move-only; destroyed with its owner).
struct Event {
    cudaEvent_t e = nullptr;
    Event() { ST_CUDA(cudaEventCreate(&e)); }
    Event(const Event&) = delete;
    Event& operator=(const Event&) = delete;
    Event(Event&& o) noexcept : e(o.e) { o.e = nullptr; }
    ~Event() {
        if (e) cudaEventDestroy(e);
    }
    void record(cudaStream_t s) { ST_CUDA(cudaEventRecord(e, s)); }
};
// A non-blocking stream owned by one call (destroyed after its queued work completes).
// ST_AUX_PRIORITY=1: the second stream gets the device's highest priority (the moment pass
// then finishes before the near field's persistent CTAs take every SM, but starves the
// target order and the plan walks instead: measured zero-sum, r02o); default priority.
inline int aux_priority() {
    static const int v = [] {
        const char* e = getenv("ST_AUX_PRIORITY");
        if (!e || e[0] != '1') return 0;
        int least = 0, greatest = 0;
        if (cudaDeviceGetStreamPriorityRange(&least, &greatest) != cudaSuccess) {
            cudaGetLastError();
            return 0;
        }
        return greatest;
    }();
    return v;
}
struct AuxStream {
    cudaStream_t s = nullptr;
    AuxStream() { ST_CUDA(cudaStreamCreateWithPriority(&s, cudaStreamNonBlocking, aux_priority())); }
    AuxStream(const AuxStream&) = delete;
    AuxStream& operator=(const AuxStream&) = delete;
    ~AuxStream() {
        if (s) cudaStreamDestroy(s);
    }
};
inline double secs(const Event& a, const Event& b) {
    float ms = 0.f;
    ST_CUDA(cudaEventElapsedTime(&ms, a.e, b.e));
    return ms * 1e-3;
}

// The library's private stream-ordered memory pool on the current device (created on
// first use; the process's default pool is left as the host application configured it).
// Its release threshold is raised so memory is recycled across calls; st_release_workspace
// trims it.
cudaMemPool_t device_pool();
// Let device `peer` read/write allocations from `owner`'s pool (NVLink stores into
// another GPU's output: peer access alone does not cover pool memory).
void pool_grant_peer(int owner, int peer);

// Stream-ordered device array (cudaMallocFromPoolAsync on device_pool()).
template <class T>
class DevArray {
public:
    DevArray() = default;
    DevArray(size_t n, cudaStream_t s) { alloc(n, s); }
    DevArray(const DevArray&) = delete;
    DevArray& operator=(const DevArray&) = delete;
    DevArray(DevArray&& o) noexcept { swap(o); }
    DevArray& operator=(DevArray&& o) noexcept {
        if (this != &o) {
            reset();
            swap(o);
        }
        return *this;
    }
    ~DevArray() { reset(); }

    void alloc(size_t n, cudaStream_t s) {
        reset();
        stream_ = s;
        n_ = n;
        if (n) {
            static const bool dbg = getenv("ST_DEBUG_ALLOC") != nullptr;
            const auto t0 = std::chrono::steady_clock::now();
            ST_CUDA(cudaMallocFromPoolAsync(reinterpret_cast<void**>(&p_), n * sizeof(T), device_pool(), s));
            if (dbg) {
                const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
                if (ms > 1.0) fprintf(stderr, "[alloc] %.1f MB took %.1f ms\n", n * sizeof(T) / 1e6, ms);
            }
        }
    }
    void reset() {
        if (p_) cudaFreeAsync(p_, stream_);
        p_ = nullptr;
        n_ = 0;
    }
    void zero() {
        if (n_) ST_CUDA(cudaMemsetAsync(p_, 0, n_ * sizeof(T), stream_));
    }
    void fill_bytes(int v) {
        if (n_) ST_CUDA(cudaMemsetAsync(p_, v, n_ * sizeof(T), stream_));
    }
    T* get() const { return p_; }
    size_t size() const { return n_; }
    size_t bytes() const { return n_ * sizeof(T); }
    T* release() {
        T* p = p_;
        p_ = nullptr;
        n_ = 0;
        return p;
    }
    void swap(DevArray& o) noexcept {
        std::swap(p_, o.p_);
        std::swap(n_, o.n_);
        std::swap(stream_, o.stream_);
    }

private:
    T* p_ = nullptr;
    size_t n_ = 0;
    cudaStream_t stream_ = nullptr;
};

// Multi-index helpers shared by host and device.
__host__ __device__ constexpr int mi_count(int p) { return (p + 1) * (p + 2) * (p + 3) / 6; }
// Graded-lex flat index (multi_index.hpp:36-44) of k with |k| = s:
// offset(s) + position of (k1,k2) in the k1-major, k2-minor enumeration.
__host__ __device__ inline int mi_flat(int k1, int k2, int k3) {
    const int s = k1 + k2 + k3;
    // entries before grade s: mi_count(s-1); within grade: k1 blocks of sizes (s+1), s, ...
    const int before = s == 0 ? 0 : mi_count(s - 1);
    // sum_{a<k1} (s - a + 1) = k1*(s+1) - k1*(k1-1)/2
    return before + k1 * (s + 1) - k1 * (k1 - 1) / 2 + k2;
}
// Harmonic (k3 <= 1) basis index: grade s occupies [s^2, (s+1)^2): k3 = 0 entries
// (s-j, j, 0) at j = 0..s, then k3 = 1 entries (s-1-j, j, 1) at s+1+j.
__host__ __device__ inline int harm_index(int k1, int k2, int k3) {
    const int s = k1 + k2 + k3;
    return s * s + (k3 == 0 ? k2 : s + 1 + k2);
}
__host__ __device__ constexpr int harm_count(int P) { return (P + 1) * (P + 1); }

}  // namespace st
