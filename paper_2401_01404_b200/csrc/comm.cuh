// comm.cuh — collectives used by the node-sharded NNDescent.
//
// Two implementations behind one interface:
//   * NcclComm: one process per GPU, NCCL over NVLink/NVSwitch (libnccl.so.2 loaded at
//     nrg_comm_init time, so a single-GPU user never needs NCCL);
//   * LoopbackComm: W contexts in one process (one host thread per virtual rank),
//     exchanging device buffers through host-side barriers + device copies; lets the
//     sharded path be verified on one GPU without kernels that wait on each other.
// All calls are collective (every rank calls them in the same order) and synchronous
// with respect to the calling rank's stream.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "common.cuh"
#include "../../include/netrec_b200.h"

namespace nrg {

struct Comm {
    int rank = 0, world = 1;
    virtual ~Comm() = default;
    // every rank contributes `bytes` from send; recv holds world * bytes, rank-ordered
    virtual void allgather(const void* send, void* recv, size_t bytes, cudaStream_t s) = 0;
    // variable-size all-gather: rank r contributes counts[r] bytes; recv holds them back to back
    virtual void allgatherv(const void* send, void* recv, const std::vector<size_t>& bytes, cudaStream_t s) = 0;
    // send_bytes[r] bytes from send + send_off[r] to rank r; recv_bytes[r] into recv + recv_off[r]
    virtual void alltoallv(const void* send, const std::vector<size_t>& send_bytes, const std::vector<size_t>& send_off,
                           void* recv, const std::vector<size_t>& recv_bytes, const std::vector<size_t>& recv_off,
                           cudaStream_t s) = 0;
    // host scalars (small): element-wise sum / max across ranks, broadcast from rank 0
    virtual void allreduce_u64(uint64_t* v, int n, bool max, cudaStream_t s) = 0;
    virtual void bcast_f64(double* v, int n, cudaStream_t s) = 0;
};

Comm* make_nccl_comm(const uint8_t id[128], int rank, int world, int device);
Comm* make_host_comm(const nrg_host_transport& t, int rank, int world);

// alltoallv plan of one key exchange from the world x world request-count matrix
// (row = requester, column = owner): byte counts / offsets of `rank` as sender and as
// owner; returns the number of keys `rank` receives
uint64_t route_plan(int world, int rank, const uint64_t* mat, std::vector<size_t>& sb, std::vector<size_t>& so,
                    std::vector<size_t>& rb, std::vector<size_t>& ro);
int nccl_unique_id(uint8_t id[128]);
// every collective of `cm` on seeded patterns, verified on every rank (collective call)
void comm_selftest(Comm& cm, cudaStream_t s);

struct LoopbackGroup;
LoopbackGroup* loopback_group_create(int world);
void loopback_group_destroy(LoopbackGroup* g);
Comm* make_loopback_comm(LoopbackGroup* g, int rank);

// owner rank of a pair key in the key-sharded distance cache (independent of the
// cache's slot hash so every rank's table stays uniformly loaded)
__host__ __device__ __forceinline__ int key_owner(uint64_t key, int world) {
    return (int)((mix64(key ^ 0x5bd1e9955bd1e995ULL) >> 33) % (uint64_t)world);
}

// contiguous node-range shard of a level's n nodes (local indices)
inline void shard_range(uint64_t n, int rank, int world, uint64_t& lo, uint64_t& hi) {
    lo = n * (uint64_t)rank / (uint64_t)world;
    hi = n * (uint64_t)(rank + 1) / (uint64_t)world;
}

}  // namespace nrg
