// One process per GPU with NCCL inside the library: the communicator, the split moment
// pass's exchange as NCCL broadcasts, and the gather of every rank's shard as one NCCL
// sum.  NCCL is loaded at first use (dlopen of libnccl.so.2 -- the one already in the
// process when PyTorch is, else the system's), so the library itself does not depend on
// it.  The reference runs its workers as threads of one process over one output vector
// (engine.hpp:157-169); here each rank evaluates its work-balanced shard of the
// key-ordered target batches (capi.cu run_treecode) and NCCL assembles the result.
#include <dlfcn.h>

#include <mutex>
#include <string>

#include <nccl.h>

#include "nccl_comm.cuh"

namespace st {

namespace {

struct NcclApi {
    void* lib = nullptr;
    ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
    ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    ncclResult_t (*broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                               cudaStream_t) = nullptr;
    ncclResult_t (*group_start)() = nullptr;
    ncclResult_t (*group_end)() = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;
};

const NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    static std::string why;
    std::call_once(once, [] {
        for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
            api.lib = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
            if (api.lib) break;
        }
        if (!api.lib) {
            why = std::string("NCCL: cannot load libnccl.so.2 (") + dlerror() + ")";
            return;
        }
        auto sym = [](const char* n) {
            void* p = dlsym(api.lib, n);
            if (!p) why = std::string("NCCL: missing symbol ") + n;
            return p;
        };
        api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(sym("ncclGetUniqueId"));
        api.comm_init_rank = reinterpret_cast<decltype(api.comm_init_rank)>(sym("ncclCommInitRank"));
        api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(sym("ncclCommDestroy"));
        api.broadcast = reinterpret_cast<decltype(api.broadcast)>(sym("ncclBroadcast"));
        api.all_reduce = reinterpret_cast<decltype(api.all_reduce)>(sym("ncclAllReduce"));
        api.group_start = reinterpret_cast<decltype(api.group_start)>(sym("ncclGroupStart"));
        api.group_end = reinterpret_cast<decltype(api.group_end)>(sym("ncclGroupEnd"));
        api.error_string = reinterpret_cast<decltype(api.error_string)>(sym("ncclGetErrorString"));
    });
    if (!why.empty()) fail(ST_NCCL_ERROR, why);
    return api;
}

void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) fail(ST_NCCL_ERROR, std::string(what) + ": " + nccl().error_string(r));
}

}  // namespace

struct NcclComm {
    ncclComm_t comm = nullptr;
    int n_ranks = 0, rank = 0, device = 0;
};

void nccl_unique_id(unsigned char out[128]) {
    static_assert(sizeof(ncclUniqueId) == 128, "NCCL unique id size");
    ncclUniqueId id;
    nccl_check(nccl().get_unique_id(&id), "ncclGetUniqueId");
    memcpy(out, &id, sizeof id);
}

NcclComm* nccl_comm_init(const unsigned char id[128], int n_ranks, int rank) {
    if (n_ranks < 1 || rank < 0 || rank >= n_ranks) fail(ST_INVALID_ARGUMENT, "nccl: rank out of range");
    ncclUniqueId uid;
    memcpy(&uid, id, sizeof uid);
    NcclComm* c = new NcclComm;
    c->n_ranks = n_ranks;
    c->rank = rank;
    ST_CUDA(cudaGetDevice(&c->device));
    const ncclResult_t r = nccl().comm_init_rank(&c->comm, n_ranks, uid, rank);
    if (r != ncclSuccess) {
        delete c;
        nccl_check(r, "ncclCommInitRank");
    }
    return c;
}

void nccl_comm_free(NcclComm* c) {
    if (!c) return;
    if (c->comm) nccl().comm_destroy(c->comm);
    delete c;
}

int nccl_rank(const NcclComm* c) { return c->rank; }
int nccl_ranks(const NcclComm* c) { return c->n_ranks; }

// the split moment pass's exchange: every rank's weight rows and subtree-root moments
// broadcast from their producer, in place, on the call's stream (one NCCL group)
int nccl_exchange(void* ctx, const st_shard_exchange* ex) {
    const NcclComm* c = static_cast<const NcclComm*>(ctx);
    const NcclApi& api = nccl();
    cudaStream_t s = static_cast<cudaStream_t>(ex->stream);
    if (api.group_start() != ncclSuccess) return 1;
    for (int r = 0; r < ex->n_shards; ++r) {
        const size_t w0 = ex->w_cuts[r], w1 = ex->w_cuts[r + 1];
        const size_t m0 = ex->m_cuts[r], m1 = ex->m_cuts[r + 1];
        if (w1 > w0 && api.broadcast(ex->w + w0 * ex->w_row, ex->w + w0 * ex->w_row, (w1 - w0) * ex->w_row,
                                     ncclDouble, r, c->comm, s) != ncclSuccess)
            return 1;
        if (m1 > m0 && api.broadcast(ex->m + m0 * ex->m_row, ex->m + m0 * ex->m_row, (m1 - m0) * ex->m_row,
                                     ncclDouble, r, c->comm, s) != ncclSuccess)
            return 1;
    }
    return api.group_end() == ncclSuccess ? 0 : 1;
}

// every rank's u (zeros outside its shard) summed into every rank's u: each target has
// exactly one writer, so the sums reproduce one GPU's values; counters (u64) summed likewise
void nccl_gather(const NcclComm* c, double* u, size_t n_doubles, unsigned long long* counters, size_t n_counters,
                 cudaStream_t s) {
    const NcclApi& api = nccl();
    nccl_check(api.group_start(), "ncclGroupStart");
    nccl_check(api.all_reduce(u, u, n_doubles, ncclDouble, ncclSum, c->comm, s), "ncclAllReduce (velocities)");
    nccl_check(api.all_reduce(counters, counters, n_counters, ncclUint64, ncclSum, c->comm, s),
               "ncclAllReduce (counters)");
    nccl_check(api.group_end(), "ncclGroupEnd");
}

}  // namespace st
