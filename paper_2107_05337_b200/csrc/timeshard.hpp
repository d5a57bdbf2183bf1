// Transports of the time-sharded MGRIT driver (timeshard.cpp).
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <memory>
#include <utility>

namespace phi {

/// One rank of the level-0 time partition: a halo shift (rank r -> r + 1) and
/// an allgather in rank order, both on device buffers, ordered on `s`.
struct Comm {
    int rank = 0, size = 1;
    virtual ~Comm() = default;
    /// send: n values to rank + 1 (null on the last rank); recv: n values from
    /// rank - 1 (null on rank 0)
    virtual void shift(const double* send, double* recv, size_t count, cudaStream_t s) = 0;
    /// recv[r * count ..] = rank r's send, r = 0 .. size - 1
    virtual void allgather(const double* send, double* recv, size_t count, cudaStream_t s) = 0;
};

/// ncclUniqueId (nccl.h: NCCL_UNIQUE_ID_BYTES = 128)
struct NcclUniqueId {
    char internal[128];
};
NcclUniqueId nccl_unique_id();
std::unique_ptr<Comm> make_nccl_comm(const NcclUniqueId& id, int nranks, int rank);

/// Host-callback transport (phi_comm_ops in include/phi_engine.h): host buffers,
/// callbacks return 0 on success.
struct CommOps {
    void* ctx;
    int (*shift)(void* ctx, const double* send, double* recv, long long count);
    int (*allgather)(void* ctx, const double* send, double* recv, long long count);
};
std::unique_ptr<Comm> make_ops_comm(const CommOps& ops, int nranks, int rank);

/// Contiguous near-equal split of the coarse intervals: [j0, j1).
std::pair<int, int> shard_of(int n_intervals, int n_ranks, int rank);

}  // namespace phi
