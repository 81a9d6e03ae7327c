// NCCL inside the library (nccl_comm.cu): communicator, split-moment exchange, gather.
#pragma once

#include "st_common.cuh"

namespace st {

struct NcclComm;
void nccl_unique_id(unsigned char out[128]);
NcclComm* nccl_comm_init(const unsigned char id[128], int n_ranks, int rank);  // on the current device
void nccl_comm_free(NcclComm* c);
int nccl_rank(const NcclComm* c);
int nccl_ranks(const NcclComm* c);
// st_exchange_fn for run_treecode's split moment pass (ctx = the NcclComm)
int nccl_exchange(void* ctx, const st_shard_exchange* ex);
// u[n_doubles] and counters[n_counters] (device) summed over the ranks, in place, on stream s
void nccl_gather(const NcclComm* c, double* u, size_t n_doubles, unsigned long long* counters, size_t n_counters,
                 cudaStream_t s);

}  // namespace st
