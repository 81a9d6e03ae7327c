// Host <-> device copies of the caller's host arrays.  The reference's callers hold
// their particles in pageable std::vector<Vec3> storage (particles.hpp:29-36); a plain
// cudaMemcpyAsync from pageable memory goes through the driver's staging at ~11 GB/s and
// blocks the calling thread.  Here pageable ranges are cut into chunks that a small pool
// of host threads memcpy into a cached ring of pinned slots, each slot's DMA overlapping
// the copy of the next chunk.  Pinned, registered, managed and device memory skip the
// ring (one cudaMemcpyAsync).
#pragma once

#include <atomic>
#include <condition_variable>
#include <cstring>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <thread>
#include <vector>

#include "st_common.cuh"

namespace st {

// Fixed pool of host threads for parallel memcpy.  Each job has its own state, so a
// worker that wakes late only ever sees an exhausted job; the caller takes part.
class CopyPool {
public:
    static CopyPool& get() {
        static CopyPool pool;
        return pool;
    }
    // run fn(i) for i in [0, n) across the pool and the caller; returns when all are done
    void parallel_for(int n, const std::function<void(int)>& fn) {
        if (n <= 1 || workers_.empty()) {
            for (int i = 0; i < n; ++i) fn(i);
            return;
        }
        auto job = std::make_shared<Job>();
        job->fn = &fn;
        job->n = n;
        {
            std::lock_guard<std::mutex> lk(mu_);
            job_ = job;
            ++gen_;
        }
        cv_.notify_all();
        work(*job);
        std::unique_lock<std::mutex> lk(job->mu);
        job->cv.wait(lk, [&] { return job->done == job->n; });
    }
    int threads() const { return (int)workers_.size() + 1; }
    ~CopyPool() {
        {
            std::lock_guard<std::mutex> lk(mu_);
            stop_ = true;
            ++gen_;
        }
        cv_.notify_all();
        for (auto& t : workers_) t.join();
    }

private:
    struct Job {
        const std::function<void(int)>* fn = nullptr;
        int n = 0;
        std::atomic<int> next{0};
        int done = 0;  // guarded by mu
        std::mutex mu;
        std::condition_variable cv;
    };
    CopyPool() {
        const unsigned hc = std::thread::hardware_concurrency();
        const int nw = (int)std::min(7u, hc > 2 ? hc / 2 - 1 : 0u);
        for (int i = 0; i < nw; ++i) workers_.emplace_back([this] { loop(); });
    }
    static void work(Job& j) {
        int done = 0;
        for (int i = j.next.fetch_add(1); i < j.n; i = j.next.fetch_add(1)) {
            (*j.fn)(i);
            ++done;
        }
        if (done) {
            std::lock_guard<std::mutex> lk(j.mu);
            j.done += done;
            if (j.done == j.n) j.cv.notify_all();
        }
    }
    void loop() {
        uint64_t seen = 0;
        for (;;) {
            std::shared_ptr<Job> job;
            {
                std::unique_lock<std::mutex> lk(mu_);
                cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
                if (stop_) return;
                seen = gen_;
                job = job_;
            }
            if (job) work(*job);
        }
    }
    std::vector<std::thread> workers_;
    std::mutex mu_;
    std::condition_variable cv_;
    std::shared_ptr<Job> job_;
    uint64_t gen_ = 0;
    bool stop_ = false;
};

// Cached pinned ring.  Rings are kept in a process-wide free list and lent to one caller
// at a time (concurrent callers -- e.g. the per-device threads of devices > 1 -- never
// share a slot, and per-call threads do not pin new memory every call).
class Stager {
public:
    static constexpr size_t kChunk = size_t(4) << 20;  // bytes per slot
    static constexpr int kSlots = 4;

    struct Lease {
        Stager* s;
        Lease() : s(acquire()) {}
        ~Lease() { release(s); }
        Stager* operator->() const { return s; }
    };
    static bool pageable(const void* p) {
        cudaPointerAttributes a{};
        const cudaError_t e = cudaPointerGetAttributes(&a, p);
        cudaGetLastError();
        return e == cudaSuccess && a.type == cudaMemoryTypeUnregistered;
    }
    // Enqueue host -> device on s.  Returns once the source may be reused (pageable data
    // copied into the ring; the DMAs may still be running).
    void h2d(void* dst, const void* src, size_t bytes, cudaStream_t s) {
        if (!bytes) return;
        if (!pageable(src) || bytes < (size_t(256) << 10)) {
            ST_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, s));
            return;
        }
        ensure();
        for (size_t off = 0; off < bytes; off += kChunk) {
            const size_t len = std::min(kChunk, bytes - off);
            const int k = slot_++ % kSlots;
            ST_CUDA(cudaEventSynchronize(ev_[k]));  // the slot's previous DMA has finished
            par_copy(buf_[k], static_cast<const char*>(src) + off, len);
            ST_CUDA(cudaMemcpyAsync(static_cast<char*>(dst) + off, buf_[k], len, cudaMemcpyHostToDevice, s));
            ST_CUDA(cudaEventRecord(ev_[k], s));
        }
    }
    // Device -> host after everything already enqueued on s; returns when dst is complete.
    void d2h(void* dst, const void* src, size_t bytes, cudaStream_t s) {
        if (!bytes) return;
        if (!pageable(dst) || bytes < (size_t(256) << 10)) {
            ST_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, s));
            ST_CUDA(cudaStreamSynchronize(s));
            return;
        }
        ensure();
        const size_t nchunk = (bytes + kChunk - 1) / kChunk;
        auto issue = [&](size_t c) {
            const size_t off = c * kChunk, len = std::min(kChunk, bytes - off);
            const int k = (int)(c % kSlots);
            ST_CUDA(cudaMemcpyAsync(buf_[k], static_cast<const char*>(src) + off, len, cudaMemcpyDeviceToHost, s));
            ST_CUDA(cudaEventRecord(ev_[k], s));
        };
        for (size_t c = 0; c < std::min<size_t>(nchunk, kSlots - 1); ++c) issue(c);
        for (size_t c = 0; c < nchunk; ++c) {
            if (c + kSlots - 1 < nchunk) issue(c + kSlots - 1);  // keep the DMA engine busy
            const int k = (int)(c % kSlots);
            ST_CUDA(cudaEventSynchronize(ev_[k]));
            const size_t off = c * kChunk, len = std::min(kChunk, bytes - off);
            par_copy(static_cast<char*>(dst) + off, buf_[k], len);
        }
    }
private:
    static std::mutex& pool_mu() {
        static std::mutex m;
        return m;
    }
    // per device: a ring's events belong to the device current when it was made
    static std::vector<Stager*>& free_list(int dev) {
        static std::map<int, std::vector<Stager*>> m;  // rings live until exit
        return m[dev];
    }
    static Stager* acquire() {
        int dev = 0;
        ST_CUDA(cudaGetDevice(&dev));
        std::lock_guard<std::mutex> lk(pool_mu());
        auto& v = free_list(dev);
        if (v.empty()) {
            Stager* s = new Stager();
            s->dev_ = dev;
            return s;
        }
        Stager* s = v.back();
        v.pop_back();
        return s;
    }
    static void release(Stager* s) {
        std::lock_guard<std::mutex> lk(pool_mu());
        free_list(s->dev_).push_back(s);
    }
    void ensure() {
        if (buf_[0]) return;
        for (int k = 0; k < kSlots; ++k) {
            ST_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&buf_[k]), kChunk, cudaHostAllocPortable));
            ST_CUDA(cudaEventCreateWithFlags(&ev_[k], cudaEventDisableTiming));
        }
    }
    static void par_copy(void* dst, const void* src, size_t len) {
        CopyPool& pool = CopyPool::get();
        const int parts = std::max(1, std::min(pool.threads(), (int)(len >> 18)));  // >= 256 KB each
        const size_t step = ((len + parts - 1) / parts + 63) & ~size_t(63);
        pool.parallel_for(parts, [&](int i) {
            const size_t a = std::min(len, i * step), b = std::min(len, a + step);
            if (b > a) std::memcpy(static_cast<char*>(dst) + a, static_cast<const char*>(src) + a, b - a);
        });
    }
    int dev_ = 0;
    char* buf_[kSlots] = {};
    cudaEvent_t ev_[kSlots] = {};
    size_t slot_ = 0;
};

inline void h2d(void* dst, const void* src, size_t bytes, cudaStream_t s) { Stager::Lease()->h2d(dst, src, bytes, s); }
inline void d2h(void* dst, const void* src, size_t bytes, cudaStream_t s) { Stager::Lease()->d2h(dst, src, bytes, s); }

}  // namespace st
