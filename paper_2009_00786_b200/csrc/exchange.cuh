// Cross-shard exchange of the sharded search.
//
// The dataset is split into contiguous series ranges, one shard per device
// (or per process). Two exchanges combine the shards:
//   * seed BSF: after every shard refined its query's own leaf, the minimum of
//     the shards' best-so-far distances becomes every shard's BSF, so each
//     shard prunes against the global seed, not its local one (the SharedBsf
//     of the reference, src/query.cpp:35-42, across shards). Any shard's BSF is
//     the distance of a real series, so pruning against it keeps the exact
//     answer; ties survive (strict pruning).
//   * results: every shard's (distance, position) per query; the answer is the
//     lexicographic minimum - scan_nn's lowest-position tie rule across its
//     range partition (src/scan.cpp:54-59).
// Transports:
//   * NCCL (one communicator rank per shard, shards on distinct devices, in one
//     process via ncclCommInitAll or one process per device via
//     ncclCommInitRank): ncclAllReduce(ncclUint64, ncclMin) of the BSF bit
//     patterns (non-negative doubles order as their bits) inside the captured
//     query graph, and ncclAllGather of the per-shard result records followed
//     by a merge kernel. NCCL is loaded at run time (dlopen), preferring the
//     copy the process already has (torch's), so single-GPU use never needs it.
//   * local (several shards on one device in one process, for tests and
//     over-decomposition): the same exchanges over device memory, with host
//     barriers between the shards' threads.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <memory>
#include <stdexcept>
#include <vector>

namespace tsg {

struct QueryWork;
struct DevResult;

struct NcclError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

enum Transport { kTransportNone = 0, kTransportLocal = 1, kTransportNccl = 2 };

// One shard's endpoint.
class Exchange {
public:
    virtual ~Exchange() = default;
    virtual Transport transport() const = 0;
    // Whether seed_bsf may be recorded into a CUDA graph capture.
    virtual bool capturable() const = 0;
    // Buffers for batches of up to nq queries (called before any capture).
    virtual void reserve(uint32_t nq) = 0;
    // Every query's BSF (work[q].bsf_bits) becomes the minimum over all shards.
    // Collective: every shard calls it for the same batch, in the same order.
    virtual void seed_bsf(QueryWork* work, uint32_t nq, cudaStream_t st) = 0;
    // NCCL only: all-gather this shard's final results (device, nq records) and
    // merge them into merged (device, nq records) on st. Collective.
    virtual void merge_results(const DevResult* local, uint32_t nq, DevResult* merged, cudaStream_t st) = 0;
    // A shard failed: peers blocked in (or later entering) a host barrier throw
    // instead of waiting forever. reset() re-arms the group for the next call.
    virtual void abort() {}
    virtual void reset() {}
    int nranks = 1, rank = 0;
};

// NCCL communicator handle (ncclComm_t) kept opaque outside exchange.cu.
using CommHandle = void*;

// 128-byte NCCL unique id.
void nccl_unique_id(unsigned char out[128]);
// ncclCommInitRank on the current device.
CommHandle nccl_comm_init_rank(int nranks, int rank, const unsigned char id[128]);
// ncclCommInitAll over distinct devices.
std::vector<CommHandle> nccl_comm_init_all(const std::vector<int>& devices);
void nccl_comm_destroy(CommHandle c);
int nccl_version();

std::unique_ptr<Exchange> make_nccl_exchange(CommHandle comm, int nranks, int rank, int device);

// Shared state of the local shards of one index.
struct LocalGroup;
std::shared_ptr<LocalGroup> make_local_group(int shards, int device);
std::unique_ptr<Exchange> make_local_exchange(std::shared_ptr<LocalGroup> g, int shard);

// Lexicographic (distance, position) merge of `shards` device result arrays of
// nq records each (all on the current device) into host_out[nq]; statistics
// add up. Used for the local transport (the NCCL one merges after its gather).
void merge_results_local(const std::vector<const DevResult*>& shards, uint32_t nq, DevResult* host_out,
                         cudaStream_t st);

}  // namespace tsg
