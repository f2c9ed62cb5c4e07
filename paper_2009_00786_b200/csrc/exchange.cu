// Cross-shard exchange (see exchange.cuh): NCCL loaded at run time, the
// local device-memory transport, and the merge / BSF kernels both share.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>

#include "common.cuh"
#include "exchange.cuh"
#include "kernels.cuh"

namespace tsg {

namespace {

// ------------------------------------------------------------------ NCCL
// The handful of entry points used, resolved from the libnccl.so.2 the process
// already has (torch loads its own), else from the system library.
struct NcclApi {
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    ncclResult_t (*GetVersion)(int*) = nullptr;
    std::string error;
};

const NcclApi& nccl() {
    static const NcclApi api = [] {
        NcclApi a;
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h) {
            const char* env = std::getenv("TSG_NCCL_LIB");
            for (const char* name : {env, "libnccl.so.2", "libnccl.so"}) {
                if (!name) continue;
                h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
                if (h) break;
            }
        }
        if (!h) {
            a.error = std::string("NCCL is not loadable: ") + (dlerror() ? dlerror() : "libnccl.so.2 not found");
            return a;
        }
        auto sym = [&](const char* name) {
            void* p = dlsym(h, name);
            if (!p && a.error.empty()) a.error = std::string("NCCL symbol missing: ") + name;
            return p;
        };
        a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(sym("ncclGetUniqueId"));
        a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(sym("ncclCommInitRank"));
        a.CommInitAll = reinterpret_cast<decltype(a.CommInitAll)>(sym("ncclCommInitAll"));
        a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(sym("ncclCommDestroy"));
        a.AllReduce = reinterpret_cast<decltype(a.AllReduce)>(sym("ncclAllReduce"));
        a.AllGather = reinterpret_cast<decltype(a.AllGather)>(sym("ncclAllGather"));
        a.GetErrorString = reinterpret_cast<decltype(a.GetErrorString)>(sym("ncclGetErrorString"));
        a.GetVersion = reinterpret_cast<decltype(a.GetVersion)>(sym("ncclGetVersion"));
        return a;
    }();
    if (!api.error.empty()) throw NcclError(api.error);
    return api;
}

void nccl_check(ncclResult_t r, const char* what) {
    if (r == ncclSuccess) return;
    throw NcclError(std::string(what) + ": " + nccl().GetErrorString(r));
}

// ---------------------------------------------------------------- kernels
constexpr int kMaxShards = 16;
struct PeerBsf {
    const unsigned long long* p[kMaxShards];
    int n;
};

__global__ void k_pack_bsf(const QueryWork* __restrict__ work, uint32_t nq, unsigned long long* __restrict__ out) {
    const uint32_t q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q < nq) out[q] = ld_volatile_u64(&work[q].bsf_bits);
}

// BSF bits of non-negative doubles (and +inf) order as unsigned integers.
__global__ void k_import_bsf(QueryWork* __restrict__ work, uint32_t nq, PeerBsf peers) {
    const uint32_t q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= nq) return;
    unsigned long long m = ~0ull;
    for (int k = 0; k < peers.n; ++k) m = min(m, peers.p[k][q]);
    if (m < ld_volatile_u64(&work[q].bsf_bits)) atomicMin(&work[q].bsf_bits, m);
}

// One thread per query: lexicographic (distance, position) minimum over the
// shards' records (an unanswered shard reports +inf / 0xFFFFFFFF), counters
// summed, overflow flags or-ed.
__global__ void k_merge_results(const DevResult* __restrict__ g, int shards, uint32_t nq, DevResult* __restrict__ out) {
    const uint32_t q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= nq) return;
    DevResult acc = g[q];
    for (int k = 1; k < shards; ++k) {
        const DevResult& r = g[static_cast<uint64_t>(k) * nq + q];
        if (r.distance < acc.distance || (r.distance == acc.distance && r.position < acc.position)) {
            acc.distance = r.distance;
            acc.position = r.position;
        }
        acc.flags |= r.flags;
        for (int s = 0; s < 6; ++s) acc.stats[s] += r.stats[s];
        acc.boxes += r.boxes;
        acc.fine_calcs += r.fine_calcs;
    }
    out[q] = acc;
}

unsigned grid_for(uint32_t nq) { return (nq + 127) / 128; }

// ------------------------------------------------------------ NCCL endpoint
class NcclExchange final : public Exchange {
public:
    NcclExchange(CommHandle comm, int nr, int r, int device) : comm_(static_cast<ncclComm_t>(comm)), device_(device) {
        nranks = nr;
        rank = r;
    }
    ~NcclExchange() override {
        int prev = 0;
        cudaGetDevice(&prev);
        cudaSetDevice(device_);
        cudaFree(bsf_);
        cudaFree(gathered_);
        cudaSetDevice(prev);
    }
    Transport transport() const override { return kTransportNccl; }
    bool capturable() const override { return true; }
    void reserve(uint32_t nq) override {
        if (nq <= cap_) return;
        cudaFree(bsf_);
        cudaFree(gathered_);
        bsf_ = nullptr;
        gathered_ = nullptr;
        TSG_CUDA(cudaMalloc(&bsf_, nq * sizeof(unsigned long long)));
        TSG_CUDA(cudaMalloc(&gathered_, static_cast<size_t>(nranks) * nq * sizeof(DevResult)));
        cap_ = nq;
    }
    void seed_bsf(QueryWork* work, uint32_t nq, cudaStream_t st) override {
        reserve(nq);
        k_pack_bsf<<<grid_for(nq), 128, 0, st>>>(work, nq, bsf_);
        TSG_LAUNCHED();
        nccl_check(nccl().AllReduce(bsf_, bsf_, nq, ncclUint64, ncclMin, comm_, st), "ncclAllReduce(seed BSF)");
        PeerBsf p{};
        p.p[0] = bsf_;
        p.n = 1;
        k_import_bsf<<<grid_for(nq), 128, 0, st>>>(work, nq, p);
        TSG_LAUNCHED();
    }
    void merge_results(const DevResult* local, uint32_t nq, DevResult* merged, cudaStream_t st) override {
        reserve(nq);
        nccl_check(nccl().AllGather(local, gathered_, nq * sizeof(DevResult), ncclUint8, comm_, st),
                   "ncclAllGather(results)");
        k_merge_results<<<grid_for(nq), 128, 0, st>>>(gathered_, nranks, nq, merged);
        TSG_LAUNCHED();
    }

private:
    ncclComm_t comm_;
    int device_;
    uint32_t cap_ = 0;
    unsigned long long* bsf_ = nullptr;
    DevResult* gathered_ = nullptr;
};

}  // namespace

// ------------------------------------------------------------ local endpoint
struct LocalGroup {
    int shards = 0, device = 0;
    // generation barrier over the shards' host threads
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    uint64_t generation = 0;
    bool aborted = false;
    // per shard: its BSF snapshot of the current batch, and the events that
    // order the snapshot's writes and the peers' reads
    std::vector<unsigned long long*> snap;
    std::vector<uint32_t> snap_cap;
    std::vector<cudaEvent_t> packed, imported;
    std::vector<unsigned char> started;  // per shard, written by its own thread (not vector<bool>: no shared words)

    void arrive_and_wait() {
        std::unique_lock<std::mutex> lk(mu);
        if (aborted) throw std::runtime_error("exchange: another shard of the search failed");
        const uint64_t gen = generation;
        if (++arrived == shards) {
            arrived = 0;
            ++generation;
            cv.notify_all();
            return;
        }
        cv.wait(lk, [&] { return generation != gen || aborted; });
        if (generation == gen) throw std::runtime_error("exchange: another shard of the search failed");
    }
    void abort() {
        std::lock_guard<std::mutex> lk(mu);
        aborted = true;
        cv.notify_all();
    }
    void reset() {
        std::lock_guard<std::mutex> lk(mu);
        aborted = false;
        arrived = 0;
    }
    ~LocalGroup() {
        int prev = 0;
        cudaGetDevice(&prev);
        cudaSetDevice(device);
        for (auto p : snap) cudaFree(p);
        for (auto e : packed) if (e) cudaEventDestroy(e);
        for (auto e : imported) if (e) cudaEventDestroy(e);
        cudaSetDevice(prev);
    }
};

namespace {

class LocalExchange final : public Exchange {
public:
    LocalExchange(std::shared_ptr<LocalGroup> g, int shard) : g_(std::move(g)) {
        nranks = g_->shards;
        rank = shard;
    }
    Transport transport() const override { return kTransportLocal; }
    bool capturable() const override { return false; }  // host barriers
    void reserve(uint32_t nq) override {
        LocalGroup& g = *g_;
        if (g.snap_cap[rank] >= nq) return;
        cudaFree(g.snap[rank]);
        g.snap[rank] = nullptr;
        TSG_CUDA(cudaMalloc(&g.snap[rank], nq * sizeof(unsigned long long)));
        g.snap_cap[rank] = nq;
    }
    // Batch protocol (every shard thread, same batch):
    //   1. wait until every peer finished reading this shard's previous snapshot,
    //      then snapshot the BSFs and record `packed`;            barrier A
    //   2. wait for every peer's `packed`, take the minimum, record `imported`; barrier B
    // Peers read snapshots, never the live work arrays, which a shard that ran
    // ahead may already have reset for its next batch.
    void seed_bsf(QueryWork* work, uint32_t nq, cudaStream_t st) override {
        LocalGroup& g = *g_;
        reserve(nq);
        if (g.started[rank])
            for (int k = 0; k < nranks; ++k)
                if (k != rank) TSG_CUDA(cudaStreamWaitEvent(st, g.imported[k], 0));
        k_pack_bsf<<<grid_for(nq), 128, 0, st>>>(work, nq, g.snap[rank]);
        TSG_LAUNCHED();
        TSG_CUDA(cudaEventRecord(g.packed[rank], st));
        g.arrive_and_wait();
        PeerBsf p{};
        for (int k = 0; k < nranks; ++k) {
            if (k == rank) continue;
            TSG_CUDA(cudaStreamWaitEvent(st, g.packed[k], 0));
            p.p[p.n++] = g.snap[k];
        }
        k_import_bsf<<<grid_for(nq), 128, 0, st>>>(work, nq, p);
        TSG_LAUNCHED();
        TSG_CUDA(cudaEventRecord(g.imported[rank], st));
        g.started[rank] = 1;
        g.arrive_and_wait();
    }
    void merge_results(const DevResult*, uint32_t, DevResult*, cudaStream_t) override {
        throw std::logic_error("local exchange: results merge on the host thread (merge_results_local)");
    }
    void abort() override { g_->abort(); }
    void reset() override { g_->reset(); }

private:
    std::shared_ptr<LocalGroup> g_;
};

}  // namespace

void nccl_unique_id(unsigned char out[128]) {
    ncclUniqueId id;
    nccl_check(nccl().GetUniqueId(&id), "ncclGetUniqueId");
    static_assert(sizeof(id) == 128, "ncclUniqueId is 128 bytes");
    std::memcpy(out, &id, sizeof(id));
}

CommHandle nccl_comm_init_rank(int nranks, int rank, const unsigned char id[128]) {
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof(uid));
    ncclComm_t c = nullptr;
    nccl_check(nccl().CommInitRank(&c, nranks, uid, rank), "ncclCommInitRank");
    return c;
}

std::vector<CommHandle> nccl_comm_init_all(const std::vector<int>& devices) {
    std::vector<ncclComm_t> c(devices.size(), nullptr);
    nccl_check(nccl().CommInitAll(c.data(), static_cast<int>(devices.size()), devices.data()), "ncclCommInitAll");
    return std::vector<CommHandle>(c.begin(), c.end());
}

void nccl_comm_destroy(CommHandle c) {
    if (c) nccl().CommDestroy(static_cast<ncclComm_t>(c));
}

int nccl_version() {
    int v = 0;
    nccl_check(nccl().GetVersion(&v), "ncclGetVersion");
    return v;
}

std::unique_ptr<Exchange> make_nccl_exchange(CommHandle comm, int nranks, int rank, int device) {
    if (nranks > kMaxShards) throw std::invalid_argument("exchange: at most 16 shards");
    return std::make_unique<NcclExchange>(comm, nranks, rank, device);
}

std::shared_ptr<LocalGroup> make_local_group(int shards, int device) {
    if (shards > kMaxShards) throw std::invalid_argument("exchange: at most 16 shards");
    auto g = std::make_shared<LocalGroup>();
    g->shards = shards;
    g->device = device;
    g->snap.assign(shards, nullptr);
    g->snap_cap.assign(shards, 0);
    g->packed.assign(shards, nullptr);
    g->imported.assign(shards, nullptr);
    g->started.assign(shards, 0);
    for (int k = 0; k < shards; ++k) {
        TSG_CUDA(cudaEventCreateWithFlags(&g->packed[k], cudaEventDisableTiming));
        TSG_CUDA(cudaEventCreateWithFlags(&g->imported[k], cudaEventDisableTiming));
    }
    return g;
}

std::unique_ptr<Exchange> make_local_exchange(std::shared_ptr<LocalGroup> g, int shard) {
    return std::make_unique<LocalExchange>(std::move(g), shard);
}

void merge_results_local(const std::vector<const DevResult*>& shards, uint32_t nq, DevResult* host_out,
                         cudaStream_t st) {
    const int R = static_cast<int>(shards.size());
    DevResult *g = nullptr, *m = nullptr;
    TSG_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&g), static_cast<size_t>(R) * nq * sizeof(DevResult), st));
    TSG_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&m), nq * sizeof(DevResult), st));
    for (int k = 0; k < R; ++k)
        TSG_CUDA(cudaMemcpyAsync(g + static_cast<uint64_t>(k) * nq, shards[k], nq * sizeof(DevResult),
                                 cudaMemcpyDeviceToDevice, st));
    k_merge_results<<<grid_for(nq), 128, 0, st>>>(g, R, nq, m);
    TSG_LAUNCHED();
    TSG_CUDA(cudaMemcpyAsync(host_out, m, nq * sizeof(DevResult), cudaMemcpyDeviceToHost, st));
    TSG_CUDA(cudaFreeAsync(g, st));
    TSG_CUDA(cudaFreeAsync(m, st));
    TSG_CUDA(cudaStreamSynchronize(st));
}

}  // namespace tsg
