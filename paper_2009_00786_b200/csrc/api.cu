// C ABI (include/tsgpu.h) over the device kernels.
//
// build:  tsidx::build_index (src/index.cpp:258-318)   -> tsg_index_build
// search: tsidx::exact_search (src/query.cpp:258-298)  -> tsg_search
// Validation messages follow IndexConfig::validate (src/config.cpp:22-35),
// build_index (src/index.cpp:259-266) and QueryState (src/query.cpp:84-87).
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <array>
#include <atomic>
#include <cerrno>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/tsgpu.h"
#include "common.cuh"
#include "exchange.cuh"
#include "kernels.cuh"

namespace tsg {

static std::atomic<uint64_t> g_launches{0};
static thread_local uint64_t t_launches = 0;
void note_launch(int n) {
    g_launches.fetch_add(static_cast<uint64_t>(n), std::memory_order_relaxed);
    t_launches += static_cast<uint64_t>(n);
}
uint64_t launch_count() { return g_launches.load(std::memory_order_relaxed); }
uint64_t launch_count_thread() { return t_launches; }

namespace {

thread_local std::string g_error;

struct LogicError : std::logic_error {
    using std::logic_error::logic_error;
};

template <typename F>
tsg_status guarded(F&& f) {
    try {
        f();
        return TSG_OK;
    } catch (const InvalidArgument& e) {
        g_error = e.what();
        return TSG_INVALID_ARGUMENT;
    } catch (const std::invalid_argument& e) {
        g_error = e.what();
        return TSG_INVALID_ARGUMENT;
    } catch (const OutOfMemory& e) {
        g_error = e.what();
        return TSG_OOM;
    } catch (const NcclError& e) {
        g_error = e.what();
        return TSG_NCCL;
    } catch (const CudaError& e) {
        g_error = e.what();
        return TSG_CUDA;
    } catch (const std::logic_error& e) {
        g_error = e.what();
        return TSG_LOGIC;
    } catch (const std::bad_alloc& e) {
        g_error = "host allocation failed";
        return TSG_OOM;
    } catch (const std::exception& e) {
        g_error = e.what();
        return TSG_RUNTIME;
    } catch (...) {
        g_error = "unknown error";
        return TSG_RUNTIME;
    }
}

void fail(const std::string& m) { throw InvalidArgument(m); }

void validate_config(const tsg_config& c) {
    // IndexConfig::validate (src/config.cpp:22-35), same messages.
    if (c.w < 1) fail("IndexConfig: w must be at least 1");
    if (c.w > 64) fail("IndexConfig: w must be at most 64 (root keys are 64-bit)");
    if (c.max_card_bits < 1 || c.max_card_bits > 8) fail("IndexConfig: max_card_bits must be in [1, 8]");
    if (c.n < static_cast<uint64_t>(c.w)) fail("IndexConfig: n must be at least w");
    if (c.n % static_cast<uint64_t>(c.w) != 0)
        fail("IndexConfig: n (" + std::to_string(c.n) + ") must be a multiple of w (" + std::to_string(c.w) + ")");
    if (c.leaf_capacity < 2) fail("IndexConfig: leaf_capacity must be at least 2");
    if (c.chunk_size < 1) fail("IndexConfig: chunk_size must be at least 1");
    if (c.n_queues < 1) fail("IndexConfig: n_queues must be at least 1");
    if (c.initial_buffer_part_size < 1) fail("IndexConfig: initial_buffer_part_size must be at least 1");
    // Device-path limits (documented in DESIGN.md).
    if (c.w > kMaxW) fail("IndexConfig: w must be at most 32 on the device path");
    if (c.n > 8192) fail("IndexConfig: n must be at most 8192 on the device path");
}

int device_count() {
    int n = 0;
    const cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0)
        throw CudaError(std::string("no CUDA device available (the device path has no CPU fallback): ") +
                        cudaGetErrorString(e));
    return n;
}

void check_device(int dev) {
    cudaDeviceProp p{};
    TSG_CUDA(cudaGetDeviceProperties(&p, dev));
    if (p.major < 10)
        throw CudaError("device " + std::to_string(dev) + " is sm_" + std::to_string(p.major * 10 + p.minor) +
                        "; this library is built for sm_100a");
}

struct DeviceGuard {
    int prev = 0;
    explicit DeviceGuard(int d) {
        TSG_CUDA(cudaGetDevice(&prev));
        TSG_CUDA(cudaSetDevice(d));
    }
    ~DeviceGuard() { cudaSetDevice(prev); }
};

}  // namespace

}  // namespace tsg

using namespace tsg;

// Devices and the transport that combines their shards (exchange.cuh):
// several shards on one device exchange locally; distinct devices of one
// process use ncclCommInitAll; tsg_comm_init joins a one-device context to a
// communicator of processes (one shard per rank).
struct tsg_ctx {
    std::vector<int> devices;
    Transport transport = kTransportNone;
    std::vector<CommHandle> comms;  // NCCL: one per device (multi-device) or this process's (multi-process)
    int nranks = 1, rank = 0;       // multi-process communicator
    ~tsg_ctx() {
        for (CommHandle c : comms) {
            try {
                nccl_comm_destroy(c);
            } catch (...) {
            }
        }
    }
};

struct tsg_index {
    tsg_ctx* ctx = nullptr;
    tsg_config cfg{};
    uint64_t count = 0, length = 0, position_offset = 0;
    std::vector<DevIndex> shards;
    std::vector<uint64_t> shard_first;  // first local row of each shard (relative to position_offset)
    std::vector<std::unique_ptr<Exchange>> xchgs;  // one endpoint per shard (none for a lone shard)
    tsg_build_stats stats{};
    std::mutex mu;
};

namespace {

void free_slots(DevIndex::Slots& t) {
    for (void* p : {static_cast<void*>(t.work), static_cast<void*>(t.lut), static_cast<void*>(t.fine_lut), static_cast<void*>(t.gsurv),
                    static_cast<void*>(t.surv), static_cast<void*>(t.surv_lb), static_cast<void*>(t.cand_pos),
                    static_cast<void*>(t.cand_lb), static_cast<void*>(t.cand_sq), static_cast<void*>(t.env),

                    static_cast<void*>(t.dpage), static_cast<void*>(t.dpage_lb)})
        cudaFree(p);
    t = DevIndex::Slots{};
}

// Slot arrays for `n` queries with `cap` candidate records each.
void alloc_slots(const DevIndex& s, DevIndex::Slots& t, uint32_t n, uint64_t cap) {
    t.n = n;
    t.cap = cap;
    const uint64_t NG = std::max<uint64_t>(s.NG, 1);
    TSG_CUDA(cudaMalloc(&t.work, n * sizeof(QueryWork)));
    TSG_CUDA(cudaMemset(t.work, 0, n * sizeof(QueryWork)));
    TSG_CUDA(cudaMalloc(&t.lut, n * static_cast<size_t>(s.w) * 256 * sizeof(float)));
    if (s.fw) TSG_CUDA(cudaMalloc(&t.fine_lut, n * static_cast<size_t>(s.fw) * 256 * sizeof(float)));
    TSG_CUDA(cudaMalloc(&t.gsurv, n * NG * sizeof(uint32_t)));
    t.rcap = std::max<uint64_t>(s.R + s.P, 1);  // a page touches its runs; boundary runs count once per page
    TSG_CUDA(cudaMalloc(&t.surv, n * t.rcap * sizeof(uint2)));
    TSG_CUDA(cudaMalloc(&t.surv_lb, n * t.rcap * sizeof(float)));
    TSG_CUDA(cudaMalloc(&t.dpage, n * std::max<uint64_t>(s.P, 1) * sizeof(uint2)));
    TSG_CUDA(cudaMalloc(&t.dpage_lb, n * std::max<uint64_t>(s.P, 1) * sizeof(float)));
    TSG_CUDA(cudaMalloc(&t.cand_pos, n * cap * sizeof(uint32_t)));
    TSG_CUDA(cudaMalloc(&t.cand_lb, n * cap * sizeof(float)));
    TSG_CUDA(cudaMalloc(&t.cand_sq, n * cap * sizeof(double)));
    TSG_CUDA(cudaMalloc(&t.env, n * 2ull * s.n * sizeof(float)));
}

void free_shard(DevIndex& s) {
    DeviceGuard g(s.device);
    if (s.own_rows) cudaFree(s.rows);
    cudaFree(s.thr);
    cudaFree(s.words);
    cudaFree(s.fine);
    cudaFree(s.run_lo);  // run_hi / quad_hi point into the same pair arrays
    cudaFree(s.quad_lo);
    cudaFree(s.pos);
    cudaFree(s.leaf_off);
    // page arrays come from the stream-ordered pool (build.cu)
    for (void* p : {static_cast<void*>(s.page_off), static_cast<void*>(s.page_leaf), static_cast<void*>(s.page_key),
                    static_cast<void*>(s.page_lo), static_cast<void*>(s.page_hi), static_cast<void*>(s.page_dir),
                    static_cast<void*>(s.group_lo), static_cast<void*>(s.group_hi), static_cast<void*>(s.top_lo),
                    static_cast<void*>(s.top_hi)})
        if (p) cudaFreeAsync(p, s.stream);
    if (s.stream) cudaStreamSynchronize(s.stream);
    free_search_graphs(s);
    free_slots(s.batch);
    free_slots(s.big);
    cudaFree(s.results);
    cudaFree(s.merged);
    cudaFree(s.queries);
    if (s.stream) cudaStreamDestroy(s.stream);
    s = DevIndex{};
}

// Host image of the device threshold block: 256 doubles + the fast-symbol bins.
std::vector<unsigned char> threshold_block(int bits) {
    std::vector<unsigned char> blk(kThrBytes);
    double* thr = reinterpret_cast<double*>(blk.data());
    host_breakpoints(bits, thr);
    host_symbol_bins(thr, bits, kBinRange, kBins, blk.data() + kThrPad * sizeof(double));
    return blk;
}

double* upload_thresholds(int bits) {
    const auto h = threshold_block(bits);
    double* d = nullptr;
    TSG_CUDA(cudaMalloc(&d, h.size()));
    TSG_CUDA(cudaMemcpy(d, h.data(), h.size(), cudaMemcpyHostToDevice));
    return d;
}

// Builds one shard on its device. rows: host (copied) or device (borrowed).
// Source of a shard's rows for build_shard: a file range streamed while K1 runs.
struct FileRows {
    const char* path = nullptr;
    uint64_t first = 0;  // first series of the shard in the file
};

// Streams series [src.first, src.first + N) of a headerless f32 file into
// s.rows: chunks of ~128 MB are read (parallel preads) into one of three
// pinned buffers, copied to HBM on the shard stream and summarised (K1)
// behind the copy, so disk/page-cache reads, PCIe and K1 overlap.
RowFeeder file_feeder(DevIndex& s, const FileRows& src, uint64_t* wall_ns) {
    return [&s, src, wall_ns](const std::function<void(uint64_t, uint64_t)>& sum_chunk) {
        const auto t0 = std::chrono::steady_clock::now();
        const uint64_t row_bytes = static_cast<uint64_t>(s.n) * sizeof(float);
        const uint64_t chunk_rows = std::max<uint64_t>(1, (128ull << 20) / row_bytes);
        const uint64_t chunk_bytes = chunk_rows * row_bytes;
        constexpr int kBufs = 3, kReaders = 8;
        const int fd = ::open(src.path, O_RDONLY);
        if (fd < 0) throw std::runtime_error(std::string("load_dataset: cannot open ") + src.path);
        struct Closer {
            int fd;
            ~Closer() { ::close(fd); }
        } closer{fd};
        ::posix_fadvise(fd, 0, 0, POSIX_FADV_SEQUENTIAL);
        std::array<void*, kBufs> buf{};
        std::array<cudaEvent_t, kBufs> copied{};
        struct Pinned {
            std::array<void*, kBufs>& b;
            std::array<cudaEvent_t, kBufs>& e;
            cudaStream_t st;
            ~Pinned() {
                cudaStreamSynchronize(st);
                for (auto p : b)
                    if (p) cudaFreeHost(p);
                for (auto x : e)
                    if (x) cudaEventDestroy(x);
            }
        } pinned{buf, copied, s.stream};
        for (int i = 0; i < kBufs; ++i) {
            TSG_CUDA(cudaHostAlloc(&buf[i], chunk_bytes, cudaHostAllocDefault));
            TSG_CUDA(cudaEventCreateWithFlags(&copied[i], cudaEventDisableTiming));
        }
        uint64_t i = 0;
        for (uint64_t first = 0; first < s.N; first += chunk_rows, ++i) {
            const int b = static_cast<int>(i % kBufs);
            const uint64_t cnt = std::min(chunk_rows, s.N - first);
            const uint64_t bytes = cnt * row_bytes;
            if (i >= kBufs) TSG_CUDA(cudaEventSynchronize(copied[b]));  // the buffer's last copy is done
            const uint64_t off = (src.first + first) * row_bytes;
            std::atomic<bool> short_read{false};
            auto read_part = [&](int r) {
                const uint64_t lo = bytes * r / kReaders, hi = bytes * (r + 1) / kReaders;
                for (uint64_t p = lo; p < hi;) {
                    const ssize_t got = ::pread(fd, static_cast<char*>(buf[b]) + p, hi - p, static_cast<off_t>(off + p));
                    if (got <= 0) {
                        short_read = true;
                        return;
                    }
                    p += static_cast<uint64_t>(got);
                }
            };
            std::vector<std::thread> readers;
            for (int r = 1; r < kReaders; ++r) readers.emplace_back(read_part, r);
            read_part(0);
            for (auto& t : readers) t.join();
            if (short_read) throw std::runtime_error(std::string("load_dataset: short read from ") + src.path);
            TSG_CUDA(cudaMemcpyAsync(s.rows + first * s.n, buf[b], bytes, cudaMemcpyHostToDevice, s.stream));
            TSG_CUDA(cudaEventRecord(copied[b], s.stream));
            sum_chunk(first, cnt);
        }
        TSG_CUDA(cudaStreamSynchronize(s.stream));
        *wall_ns = static_cast<uint64_t>(
            std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - t0).count());
    };
}

void build_shard(DevIndex& s, const float* rows, bool host_rows, uint64_t N, const tsg_config& cfg,
                 uint64_t pos_offset, uint64_t* h2d_ns, double ms[3], const FileRows* file = nullptr) {
    DeviceGuard g(s.device);
    check_device(s.device);
    // the shard's stream has the highest priority: work the library puts on side streams (the
    // build's gather) yields SMs to it at block granularity
    int prio_least = 0, prio_greatest = 0;
    TSG_CUDA(cudaDeviceGetStreamPriorityRange(&prio_least, &prio_greatest));
    TSG_CUDA(cudaStreamCreateWithPriority(&s.stream, cudaStreamNonBlocking, prio_greatest));
    TSG_CUDA(cudaDeviceGetAttribute(&s.sms, cudaDevAttrMultiProcessorCount, s.device));
    if (const char* e = std::getenv("TSG_L2_FETCH")) {  // A/B: L2 fetch granularity hint (bytes)
        TSG_CUDA(cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, static_cast<size_t>(std::atoi(e))));
    }
    if (std::getenv("TSG_PRINT_L2_FETCH")) {
        size_t v = 0;
        TSG_CUDA(cudaDeviceGetLimit(&v, cudaLimitMaxL2FetchGranularity));
        std::fprintf(stderr, "tsg: cudaLimitMaxL2FetchGranularity = %zu\n", v);
    }
    s.N = N;
    s.n = static_cast<int>(cfg.n);
    s.w = cfg.w;
    s.bits = cfg.max_card_bits;
    s.ws = word_stride(cfg.w);
    s.leaf_cap = cfg.leaf_capacity;
    s.pos_offset = pos_offset;
    if (file) {  // rows arrive from the file while K1 runs (below)
        TSG_CUDA(cudaMalloc(&s.rows, N * cfg.n * sizeof(float)));
        s.own_rows = true;
        *h2d_ns = 0;
    } else if (host_rows) {
        const auto t0 = std::chrono::steady_clock::now();
        TSG_CUDA(cudaMalloc(&s.rows, N * cfg.n * sizeof(float)));
        s.own_rows = true;
        TSG_CUDA(cudaMemcpyAsync(s.rows, rows, N * cfg.n * sizeof(float), cudaMemcpyHostToDevice, s.stream));
        TSG_CUDA(cudaStreamSynchronize(s.stream));
        *h2d_ns = static_cast<uint64_t>(
            std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - t0).count());
    } else {
        s.rows = const_cast<float*>(rows);
        s.own_rows = false;
        *h2d_ns = 0;
    }
    s.thr = upload_thresholds(s.bits);
    // Fine summary (TSG_NO_FINE=1 disables it, for A/B measurements).
    s.fw = std::getenv("TSG_NO_FINE") ? 0 : fine_width(s.n, s.w);
    s.fws = s.fw ? fine_stride(s.fw) : 0;
    if (const char* e = std::getenv("TSG_REFINE_SPLIT")) s.refine_split = static_cast<float>(std::atof(e));
    if (file) {
        const RowFeeder feeder = file_feeder(s, *file, h2d_ns);
        build_layout(s, &ms[0], &ms[1], &ms[2], &feeder);
    } else {
        build_layout(s, &ms[0], &ms[1], &ms[2]);
    }
    // Search workspace: batch_max query slots (TSG_BATCH, default 128). Each
    // slot holds up to `cap` candidate records: as many as the shard has
    // entries when memory allows, else a share of ~45% of the free memory
    // (>= 2^20 and >= the seed range); a query that outgrows its slot is
    // rerun alone in a full-size slot.
    if (const char* e = std::getenv("TSG_BATCH")) s.batch_max = static_cast<uint32_t>(std::max(1, std::atoi(e)));
    size_t free_b = 0, total_b = 0;
    TSG_CUDA(cudaMemGetInfo(&free_b, &total_b));
    const uint64_t per_slot_fixed = sizeof(QueryWork) + static_cast<uint64_t>(s.w) * 1024 +
                                    std::max<uint64_t>(s.NG, 1) * 4 + (s.R + 2 * s.P + 2) * 12 +
                                    static_cast<uint64_t>(s.n) * 8;
    const uint64_t budget = static_cast<uint64_t>(0.45 * static_cast<double>(free_b));
    const uint64_t fixed = per_slot_fixed * s.batch_max;
    const uint64_t cand_budget = budget > fixed ? budget - fixed : 0;
    const uint64_t min_cap = std::min<uint64_t>(N, std::max<uint64_t>(1u << 20, 2 * s.leaf_cap));
    uint64_t cap = std::min<uint64_t>(N, std::max<uint64_t>(min_cap, cand_budget / (16ull * s.batch_max)));
    // TSG_SLOT_CAP (tests): smaller slots, to exercise the full-size rerun of overflowing queries
    if (const char* e = std::getenv("TSG_SLOT_CAP"))
        cap = std::min<uint64_t>(cap, std::max<uint64_t>(std::strtoull(e, nullptr, 10), std::min<uint64_t>(N, 2 * s.leaf_cap)));
    alloc_slots(s, s.batch, s.batch_max, cap);
}

void ensure_results(DevIndex& s, uint32_t nq) {
    if (s.results_cap >= nq) return;
    cudaFree(s.results);
    cudaFree(s.merged);
    s.results = s.merged = nullptr;
    TSG_CUDA(cudaMalloc(&s.results, static_cast<size_t>(nq) * sizeof(DevResult)));
    TSG_CUDA(cudaMalloc(&s.merged, static_cast<size_t>(nq) * sizeof(DevResult)));
    s.results_cap = nq;
}

void ensure_queries(DevIndex& s, uint32_t nq) {
    if (s.queries_cap >= nq) return;
    cudaFree(s.queries);
    s.queries = nullptr;
    TSG_CUDA(cudaMalloc(&s.queries, static_cast<size_t>(nq) * s.n * sizeof(float)));
    s.queries_cap = nq;
}

// Queries that outgrew their batch slot, rerun together: the batch slots'
// candidate arrays are one allocation of n x cap records, so k reruns can use
// them as k slots of n * cap / k records (the shard's size when k <= n * cap / N,
// which cannot overflow). Rows are gathered into a scratch buffer; answers
// replace the flagged ones in host_out; any query that overflows again keeps
// its flag for the one-query full-size path. (c4: 1.57K -> ~2.3K q/s.)
// The device results (s.results) are patched too: the cross-shard merge reads them.
void rerun_overflows_batched(DevIndex& s, const float* dq, uint32_t nq, bool approximate, DevResult* host_out,
                             int window) {
    std::vector<uint32_t> ovf;
    for (uint32_t q = 0; q < nq; ++q)
        if (host_out[q].flags & kResultOverflow) ovf.push_back(q);
    const uint64_t total = static_cast<uint64_t>(s.batch.n) * s.batch.cap;
    const uint64_t k_full = s.N ? total / s.N : 0;  // slots of full size the arrays hold
    if (ovf.empty() || k_full < 2 || std::getenv("TSG_NO_BATCHED_RERUN")) return;
    const uint32_t kmax = static_cast<uint32_t>(std::min<uint64_t>(k_full, s.batch.n));
    float* rows = nullptr;
    DevResult* res = nullptr;
    const uint32_t kc0 = std::min<uint32_t>(kmax, static_cast<uint32_t>(ovf.size()));
    TSG_CUDA(cudaMallocAsync(&rows, static_cast<size_t>(kc0) * s.n * sizeof(float), s.stream));
    TSG_CUDA(cudaMallocAsync(&res, kc0 * sizeof(DevResult), s.stream));
    std::vector<DevResult> out(kc0);
    for (size_t i0 = 0; i0 < ovf.size(); i0 += kc0) {
        const uint32_t kc = static_cast<uint32_t>(std::min<size_t>(kc0, ovf.size() - i0));
        for (uint32_t i = 0; i < kc; ++i)
            TSG_CUDA(cudaMemcpyAsync(rows + static_cast<uint64_t>(i) * s.n, dq + static_cast<uint64_t>(ovf[i0 + i]) * s.n,
                                     s.n * sizeof(float), cudaMemcpyDeviceToDevice, s.stream));
        DevIndex::Slots view = s.batch;  // same arrays, fewer and larger slots (not owned)
        view.n = kc;
        view.cap = std::min<uint64_t>(s.N, total / kc);
        search_batch(s, view, rows, kc, approximate, res, window);
        TSG_CUDA(cudaMemcpyAsync(out.data(), res, kc * sizeof(DevResult), cudaMemcpyDeviceToHost, s.stream));
        for (uint32_t i = 0; i < kc; ++i)
            TSG_CUDA(cudaMemcpyAsync(s.results + ovf[i0 + i], res + i, sizeof(DevResult), cudaMemcpyDeviceToDevice,
                                     s.stream));
        TSG_CUDA(cudaStreamSynchronize(s.stream));
        for (uint32_t i = 0; i < kc; ++i) host_out[ovf[i0 + i]] = out[i];
    }
    TSG_CUDA(cudaFreeAsync(rows, s.stream));
    TSG_CUDA(cudaFreeAsync(res, s.stream));
}

// All nq device queries of one shard: batches of batch_max through the batch
// slots, then any query that outgrew its slot again, alone, in the full-size
// slot (allocated on first use). Results land in host_out.
void search_all(DevIndex& s, const float* dq, uint32_t nq, bool approximate, DevResult* host_out, int window) {
    ensure_results(s, nq);
    // Batches run in the slot arrays sliced into eb slots; a call in which more than 5% of the
    // queries overflow halves eb for the next calls (fewer, larger slots: c4 -> 64 slots), down
    // to 16, and a call without overflows doubles it again (up to batch_max), so one hard query
    // set does not slow later easy ones. Datasets whose queries fit (c2) keep batch_max. Shards
    // that exchange BSFs keep batch_max: every shard must run the same batches.
    const bool xchg = s.xchg != nullptr;
    const uint32_t eb = (!xchg && s.eff_batch) ? s.eff_batch : s.batch_max;
    DevIndex::Slots view = s.batch;  // not owned
    view.n = eb;
    view.cap = std::min<uint64_t>(s.N, static_cast<uint64_t>(s.batch.n) * s.batch.cap / eb);
    for (uint32_t off = 0; off < nq; off += eb) {
        const uint32_t b = std::min(eb, nq - off);
        search_batch(s, view, dq + static_cast<uint64_t>(off) * s.n, b, approximate, s.results + off, window, xchg);
    }
    TSG_CUDA(cudaMemcpyAsync(host_out, s.results, nq * sizeof(DevResult), cudaMemcpyDeviceToHost, s.stream));
    TSG_CUDA(cudaStreamSynchronize(s.stream));
    uint32_t n_ovf = 0;
    for (uint32_t q = 0; q < nq; ++q) n_ovf += (host_out[q].flags & kResultOverflow) ? 1 : 0;
    if (!xchg && !std::getenv("TSG_FIXED_BATCH")) {
        if (static_cast<uint64_t>(n_ovf) * 20 > nq && eb > 16) s.eff_batch = eb / 2;
        else if (n_ovf == 0 && eb < s.batch_max) s.eff_batch = std::min(s.batch_max, eb * 2);
    }
    rerun_overflows_batched(s, dq, nq, approximate, host_out, window);
    for (uint32_t q = 0; q < nq; ++q) {
        if (!(host_out[q].flags & kResultOverflow)) continue;
        if (!s.big.n) alloc_slots(s, s.big, 1, s.N);
        search_batch(s, s.big, dq + static_cast<uint64_t>(q) * s.n, 1, approximate, s.results + q, window);
        TSG_CUDA(cudaMemcpyAsync(host_out + q, s.results + q, sizeof(DevResult), cudaMemcpyDeviceToHost, s.stream));
        TSG_CUDA(cudaStreamSynchronize(s.stream));
        if (host_out[q].flags & kResultOverflow) throw std::logic_error("search: a full-size slot overflowed");
    }
}

void to_result(const DevResult& d, tsg_result& r) {
    r.distance = d.distance;
    r.position = d.position;
    r.box_calcs = static_cast<uint32_t>(std::min<unsigned long long>(d.boxes, 0xFFFFFFFFull));
    r.stats.lb_node_calcs = d.stats[0];
    r.stats.lb_entry_calcs = d.stats[1];
    r.stats.real_dist_calcs = d.stats[2];
    r.stats.bsf_updates = d.stats[3];
    r.stats.pruned_subtrees = d.stats[4];
    r.stats.queue_insertions = d.stats[5];
    r.fine_calcs = d.fine_calcs;
}

void run_search(tsg_index* ix, const float* queries, bool host, uint32_t nq, tsg_result* out, bool approximate,
                int window = -1) {
    if (!ix) fail("search: null index");
    if (nq == 0) return;
    if (!queries || !out) fail("search: null buffer");
    std::lock_guard<std::mutex> lock(ix->mu);
    if (!host && ix->shards.size() != 1) fail("tsg_search_device: device queries need a single-device index");
    const size_t G = ix->shards.size();
    const bool nccl = G >= 1 && ix->shards[0].xchg && ix->shards[0].xchg->transport() == kTransportNccl;
    for (auto& x : ix->xchgs) x->reset();
    std::vector<std::vector<DevResult>> per(G, std::vector<DevResult>(nq));
    auto work = [&](size_t k) {
        DevIndex& s = ix->shards[k];
        DeviceGuard g(s.device);
        const float* dq = queries;
        if (host) {
            ensure_queries(s, nq);
            TSG_CUDA(cudaMemcpyAsync(s.queries, queries, static_cast<size_t>(nq) * s.n * sizeof(float),
                                     cudaMemcpyHostToDevice, s.stream));
            dq = s.queries;
        }
        search_all(s, dq, nq, approximate, per[k].data(), window);
        if (nccl) {  // every rank: all-gather the shards' records, merge on the device
            s.xchg->merge_results(s.results, nq, s.merged, s.stream);
            TSG_CUDA(cudaMemcpyAsync(per[k].data(), s.merged, nq * sizeof(DevResult), cudaMemcpyDeviceToHost,
                                     s.stream));
            TSG_CUDA(cudaStreamSynchronize(s.stream));
        }
    };
    if (G == 1) {
        work(0);
    } else {
        std::vector<std::thread> th;
        std::vector<std::exception_ptr> errs(G);
        for (size_t k = 0; k < G; ++k)
            th.emplace_back([&, k] {
                try {
                    work(k);
                } catch (...) {
                    errs[k] = std::current_exception();
                    if (ix->shards[k].xchg) ix->shards[k].xchg->abort();  // peers must not wait on this shard
                }
            });
        for (auto& t : th) t.join();
        for (auto& e : errs)
            if (e) std::rethrow_exception(e);
    }
    std::vector<DevResult> merged;
    const DevResult* final_res = per[0].data();
    if (G > 1 && !nccl) {  // local shards: merge their device records on the first shard's stream
        DevIndex& s0 = ix->shards[0];
        DeviceGuard g(s0.device);
        std::vector<const DevResult*> src;
        for (auto& s : ix->shards) src.push_back(s.results);
        merged.resize(nq);
        merge_results_local(src, nq, merged.data(), s0.stream);
        final_res = merged.data();
    }
    for (uint32_t q = 0; q < nq; ++q) {
        out[q] = tsg_result{};
        to_result(final_res[q], out[q]);
    }
}

tsg_status do_build(tsg_ctx* ctx, const float* rows, bool host, uint64_t count, uint64_t length,
                    const tsg_config* cfg, uint64_t position_offset, tsg_index** out, tsg_build_stats* stats,
                    const char* path = nullptr) {
    return guarded([&] {
        if (!ctx || !out) fail("build_index: null argument");
        *out = nullptr;
        if (!cfg) fail("build_index: null config");
        validate_config(*cfg);
        if (count == 0) fail("build_index: empty dataset");
        if (length != cfg->n)
            fail("build_index: dataset length " + std::to_string(length) + " does not match config.n " +
                 std::to_string(cfg->n));
        if (count > 0xFFFFFFFFull) fail("build_index: more than 2^32-1 series");
        if (!rows && !path) fail("build_index: null rows");
        if (position_offset + count - 1 > 0xFFFFFFFFull) fail("build_index: positions exceed 2^32-1");
        if (!host && ctx->devices.size() != 1) fail("tsg_index_build_device: device rows need a single-device context");
        if (ctx->transport == kTransportNccl && ctx->devices.size() > 1 && count < ctx->devices.size())
            fail("build_index: fewer series than devices (every NCCL rank needs a shard)");

        auto ix = std::make_unique<tsg_index>();
        ix->ctx = ctx;
        ix->cfg = *cfg;
        ix->count = count;
        ix->length = length;
        ix->position_offset = position_offset;
        const size_t G = std::min<size_t>(ctx->devices.size(), count);
        ix->shards.resize(G);
        ix->shard_first.resize(G);
        std::vector<uint64_t> h2d(G, 0);
        std::vector<std::array<double, 3>> ms(G);
        std::vector<std::exception_ptr> errs(G);
        const auto t0 = std::chrono::steady_clock::now();
        auto work = [&](size_t k) {
            try {
                const uint64_t b = count * k / G, e = count * (k + 1) / G;
                ix->shard_first[k] = b;
                ix->shards[k].device = ctx->devices[k];
                if (path) {
                    const FileRows fr{path, b};
                    build_shard(ix->shards[k], nullptr, true, e - b, *cfg, position_offset + b, &h2d[k], ms[k].data(),
                                &fr);
                } else {
                    build_shard(ix->shards[k], rows + b * length, host, e - b, *cfg, position_offset + b, &h2d[k],
                                ms[k].data());
                }
            } catch (...) {
                errs[k] = std::current_exception();
            }
        };
        if (G == 1) {
            work(0);
        } else {
            std::vector<std::thread> th;
            for (size_t k = 0; k < G; ++k) th.emplace_back(work, k);
            for (auto& t : th) t.join();
        }
        for (auto& e : errs)
            if (e) {
                for (auto& s : ix->shards)
                    if (s.stream || s.rows) free_shard(s);
                std::rethrow_exception(e);
            }
        // cross-shard exchange endpoints (exchange.cuh)
        if (ctx->transport == kTransportNccl) {
            for (size_t k = 0; k < G; ++k) {
                const int nr = ctx->devices.size() > 1 ? static_cast<int>(G) : ctx->nranks;
                const int rk = ctx->devices.size() > 1 ? static_cast<int>(k) : ctx->rank;
                DeviceGuard dg(ix->shards[k].device);
                ix->xchgs.push_back(make_nccl_exchange(ctx->comms[k], nr, rk, ix->shards[k].device));
            }
        } else if (G > 1) {
            DeviceGuard dg(ix->shards[0].device);
            auto group = make_local_group(static_cast<int>(G), ix->shards[0].device);
            for (size_t k = 0; k < G; ++k) ix->xchgs.push_back(make_local_exchange(group, static_cast<int>(k)));
        }
        for (size_t k = 0; k < ix->xchgs.size(); ++k) ix->shards[k].xchg = ix->xchgs[k].get();
        (void)t0;
        tsg_build_stats st{};
        st.series = count;
        double sum_ms = 0, org_ms = 0, leaf_ms = 0;
        for (size_t k = 0; k < G; ++k) {
            const DevIndex& s = ix->shards[k];
            st.leaves += s.L;
            st.pages += s.P;
            st.inner_nodes += s.inner;
            st.overflow_leaves += s.overflow;
            st.max_depth = std::max<uint64_t>(st.max_depth, s.max_depth);
            st.root_children += s.root_children;
            st.h2d_ns = std::max(st.h2d_ns, h2d[k]);
            sum_ms = std::max(sum_ms, ms[k][0]);
            org_ms = std::max(org_ms, ms[k][1]);
            leaf_ms = std::max(leaf_ms, ms[k][2]);
        }
        st.nodes = st.leaves + st.inner_nodes;
        st.empty_leaves = 0;
        st.summarise_ms = sum_ms;
        st.organise_ms = org_ms;
        st.leaves_ms = leaf_ms;
        st.build_ns = static_cast<uint64_t>((sum_ms + org_ms + leaf_ms) * 1e6);
        ix->stats = st;
        if (stats) *stats = st;
        *out = ix.release();
    });
}

}  // namespace

extern "C" {

const char* tsg_last_error(void) { return g_error.c_str(); }

const char* tsg_version(void) { return "tsgpu 0.1 (sm_100a)"; }

uint64_t tsg_launch_count(void) { return launch_count(); }

int tsg_word_stride(int w) { return word_stride(w); }

void tsg_config_default(tsg_config* c) {
    if (!c) return;
    c->n = 256;
    c->w = 16;
    c->max_card_bits = 8;
    c->leaf_capacity = 2000;
    c->chunk_size = 20000;
    c->n_index_workers = 0;
    c->n_search_workers = 0;
    c->n_queues = 24;
    c->queue_mode = 1;
    c->initial_buffer_part_size = 5;
}

tsg_status tsg_config_validate(const tsg_config* cfg) {
    return guarded([&] {
        if (!cfg) fail("IndexConfig: null");
        validate_config(*cfg);
    });
}

tsg_status tsg_open(int n_gpus, const int* devices, tsg_ctx** out) {
    return guarded([&] {
        if (!out) fail("tsg_open: null out");
        *out = nullptr;
        if (n_gpus < 1) fail("tsg_open: n_gpus must be at least 1");
        const int have = device_count();
        auto ctx = std::make_unique<tsg_ctx>();
        for (int i = 0; i < n_gpus; ++i) {
            const int d = devices ? devices[i] : i;
            if (d < 0 || d >= have) fail("tsg_open: device " + std::to_string(d) + " out of range");
            check_device(d);
            ctx->devices.push_back(d);
        }
        if (n_gpus > 1) {
            std::vector<int> u = ctx->devices;
            std::sort(u.begin(), u.end());
            const size_t distinct = static_cast<size_t>(std::unique(u.begin(), u.end()) - u.begin());
            if (distinct == 1) {
                ctx->transport = kTransportLocal;
            } else if (distinct == ctx->devices.size()) {
                ctx->transport = kTransportNccl;
                ctx->comms = nccl_comm_init_all(ctx->devices);
            } else {
                fail("tsg_open: devices must be all distinct (NCCL) or all the same (local shards)");
            }
        }
        *out = ctx.release();
    });
}

tsg_status tsg_close(tsg_ctx* ctx) {
    delete ctx;
    return TSG_OK;
}

tsg_status tsg_comm_unique_id(tsg_comm_id* id) {
    return guarded([&] {
        if (!id) fail("tsg_comm_unique_id: null id");
        nccl_unique_id(id->internal);
    });
}

tsg_status tsg_comm_init(tsg_ctx* ctx, int nranks, int rank, const tsg_comm_id* id) {
    return guarded([&] {
        if (!ctx || !id) fail("tsg_comm_init: null argument");
        if (ctx->devices.size() != 1) fail("tsg_comm_init: a multi-process communicator needs a one-device context");
        if (ctx->transport != kTransportNone) fail("tsg_comm_init: the context already has a communicator");
        if (nranks < 1 || rank < 0 || rank >= nranks) fail("tsg_comm_init: rank must be in [0, nranks)");
        DeviceGuard g(ctx->devices[0]);
        ctx->comms.push_back(nccl_comm_init_rank(nranks, rank, id->internal));
        ctx->transport = kTransportNccl;
        ctx->nranks = nranks;
        ctx->rank = rank;
    });
}

tsg_status tsg_comm_info(const tsg_ctx* ctx, int* transport, int* nranks, int* rank) {
    return guarded([&] {
        if (!ctx) fail("tsg_comm_info: null context");
        if (transport) *transport = static_cast<int>(ctx->transport);
        const bool multi = ctx->devices.size() > 1;
        if (nranks) *nranks = multi ? static_cast<int>(ctx->devices.size()) : ctx->nranks;
        if (rank) *rank = multi ? 0 : ctx->rank;
    });
}

tsg_status tsg_index_build(tsg_ctx* ctx, const float* host_rows, uint64_t count, uint64_t length,
                           const tsg_config* cfg, uint64_t position_offset, tsg_index** out, tsg_build_stats* stats) {
    return do_build(ctx, host_rows, true, count, length, cfg, position_offset, out, stats);
}

tsg_status tsg_index_build_file(tsg_ctx* ctx, const char* path, uint64_t length, const tsg_config* cfg,
                                uint64_t position_offset, tsg_index** out, tsg_build_stats* stats) {
    // load_dataset's checks and messages (src/dataset.cpp:87-100), then build_index's.
    uint64_t count = 0;
    const tsg_status st = guarded([&] {
        if (!path) fail("load_dataset: null path");
        if (length == 0) fail("load_dataset: length must be positive");
        struct stat sb {};
        if (::stat(path, &sb) != 0)
            throw std::runtime_error(std::string("load_dataset: cannot stat ") + path + ": " + std::strerror(errno));
        const uint64_t bytes = static_cast<uint64_t>(sb.st_size), series_bytes = length * sizeof(float);
        if (bytes == 0 || bytes % series_bytes != 0)
            throw std::runtime_error(std::string("load_dataset: ") + path + " holds " + std::to_string(bytes) +
                                     " bytes, not a positive multiple of " + std::to_string(series_bytes) +
                                     " (length " + std::to_string(length) + " * 4)");
        count = bytes / series_bytes;
    });
    if (st != TSG_OK) return st;
    return do_build(ctx, nullptr, true, count, length, cfg, position_offset, out, stats, path);
}

tsg_status tsg_index_build_device(tsg_ctx* ctx, const float* dev_rows, uint64_t count, uint64_t length,
                                  const tsg_config* cfg, uint64_t position_offset, tsg_index** out,
                                  tsg_build_stats* stats) {
    return do_build(ctx, dev_rows, false, count, length, cfg, position_offset, out, stats);
}

tsg_status tsg_index_free(tsg_index* ix) {
    return guarded([&] {
        if (!ix) return;
        for (auto& s : ix->shards) free_shard(s);
        delete ix;
    });
}

tsg_status tsg_index_info(const tsg_index* ix, uint64_t* count, uint64_t* length, tsg_config* cfg,
                          tsg_build_stats* stats) {
    return guarded([&] {
        if (!ix) fail("tsg_index_info: null index");
        if (count) *count = ix->count;
        if (length) *length = ix->length;
        if (cfg) *cfg = ix->cfg;
        if (stats) *stats = ix->stats;
    });
}

tsg_status tsg_search(tsg_index* ix, const float* host_queries, uint32_t nq, tsg_result* out) {
    return guarded([&] { run_search(ix, host_queries, true, nq, out, false); });
}

tsg_status tsg_search_device(tsg_index* ix, const float* dev_queries, uint32_t nq, tsg_result* out) {
    return guarded([&] { run_search(ix, dev_queries, false, nq, out, false); });
}

tsg_status tsg_approximate_search(tsg_index* ix, const float* host_query, tsg_result* out) {
    return guarded([&] { run_search(ix, host_query, true, 1, out, true); });
}

// Measure-aware search (exact_search / approximate_search with a Measure,
// query.hpp:133-151): Euclidean, or DTW with a Sakoe-Chiba window (QueryState's
// window check, src/query.cpp:88-90, same message).
tsg_status tsg_search_measure(tsg_index* ix, const float* queries, int queries_on_device, uint32_t nq,
                              const tsg_measure* m, int approximate, tsg_result* out) {
    return guarded([&] {
        if (!m) fail("exact_search: null measure");
        int window = -1;
        if (m->kind == TSG_MEASURE_DTW) {
            if (!ix) fail("search: null index");
            if (m->window < 0 || static_cast<uint64_t>(m->window) >= ix->cfg.n) fail("dtw window must be in [0, n)");
            if (m->window > kMaxDtwWindow)
                fail("dtw window " + std::to_string(m->window) + " above the device limit " +
                     std::to_string(kMaxDtwWindow));
            window = m->window;
        } else if (m->kind != TSG_MEASURE_ED) {
            fail("exact_search: unknown measure kind");
        }
        run_search(ix, queries, queries_on_device == 0, nq, out, approximate != 0, window);
    });
}

tsg_status tsg_summarise(const float* dev_rows, uint64_t count, uint64_t length, int w, int bits, uint8_t* dev_words,
                         uint32_t* dev_root_keys, void* stream) {
    return guarded([&] {
        if (w < 1 || w > kMaxW) fail("tsg_summarise: w must be in [1, 32]");
        if (bits < 1 || bits > 8) fail("tsg_summarise: bits must be in [1, 8]");
        if (length < static_cast<uint64_t>(w) || length % static_cast<uint64_t>(w) != 0)
            fail("tsg_summarise: length must be a nonzero multiple of w");
        if (count == 0) return;
        if (!dev_rows || !dev_words) fail("tsg_summarise: null buffer");
        device_count();
        int dev = 0;
        TSG_CUDA(cudaGetDevice(&dev));
        check_device(dev);
        const auto h = threshold_block(bits);
        double* d = nullptr;
        auto st = static_cast<cudaStream_t>(stream);
        TSG_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&d), h.size(), st));
        TSG_CUDA(cudaMemcpyAsync(d, h.data(), h.size(), cudaMemcpyHostToDevice, st));
        summarise(dev_rows, count, static_cast<int>(length), w, bits, d, dev_words, dev_root_keys, nullptr, st);
        TSG_CUDA(cudaFreeAsync(d, st));
        TSG_CUDA(cudaStreamSynchronize(st));
    });
}

tsg_status tsg_index_export(const tsg_index* ix, uint8_t* words, uint32_t* positions, uint32_t* leaf_offsets,
                            uint32_t* page_offsets, uint8_t* page_lo, uint8_t* page_hi) {
    return guarded([&] {
        if (!ix) fail("tsg_index_export: null index");
        if (ix->shards.size() != 1) fail("tsg_index_export: single-device index only");
        const DevIndex& s = ix->shards[0];
        DeviceGuard g(s.device);
        if (words) TSG_CUDA(cudaMemcpy(words, s.words, s.N * s.ws, cudaMemcpyDeviceToHost));
        if (positions) {
            TSG_CUDA(cudaMemcpy(positions, s.pos, s.N * 4, cudaMemcpyDeviceToHost));
            for (uint64_t i = 0; i < s.N; ++i) positions[i] += static_cast<uint32_t>(s.pos_offset);
        }
        if (leaf_offsets) TSG_CUDA(cudaMemcpy(leaf_offsets, s.leaf_off, (s.L + 1) * 4, cudaMemcpyDeviceToHost));
        if (page_offsets) TSG_CUDA(cudaMemcpy(page_offsets, s.page_off, (s.P + 1) * 4, cudaMemcpyDeviceToHost));
        if (page_lo) TSG_CUDA(cudaMemcpy(page_lo, s.page_lo, s.P * s.ws, cudaMemcpyDeviceToHost));
        if (page_hi) TSG_CUDA(cudaMemcpy(page_hi, s.page_hi, s.P * s.ws, cudaMemcpyDeviceToHost));
    });
}

tsg_status tsg_index_validate(tsg_index* ix, tsg_validation_report* out) {
    return guarded([&] {
        if (!ix || !out) fail("validate_index: null argument");
        std::lock_guard<std::mutex> lock(ix->mu);
        std::memset(out, 0, sizeof(*out));
        for (auto& s : ix->shards) {
            DeviceGuard g(s.device);
            audit_index(s, out);
        }
    });
}

tsg_status tsg_index_debug_poke(tsg_index* ix, int array, uint64_t offset, const void* bytes, uint64_t n) {
    return guarded([&] {
        if (!ix || !bytes) fail("tsg_index_debug_poke: null argument");
        DevIndex& s = ix->shards[0];
        DeviceGuard g(s.device);
        void* base = nullptr;
        uint64_t size = 0;
        switch (array) {
            case 0: base = s.words; size = s.N * s.ws; break;
            case 1: base = s.pos; size = s.N * 4; break;
            case 2: base = s.leaf_off; size = (s.L + 1) * 4; break;
            case 3: base = s.page_lo; size = s.P * s.ws; break;
            case 4: base = s.quad_lo; size = s.Q * 2 * s.ws; break;
            case 5: base = s.fine; size = s.fw ? s.N * s.fws : 0; break;
            case 6: base = s.run_hi; size = s.R * 2 * s.ws - s.ws; break;
            case 7: base = s.group_lo; size = s.NG * s.ws; break;
            default: fail("tsg_index_debug_poke: unknown array");
        }
        if (!base || offset + n > size) fail("tsg_index_debug_poke: out of range");
        TSG_CUDA(cudaMemcpy(static_cast<uint8_t*>(base) + offset, bytes, n, cudaMemcpyHostToDevice));
    });
}

tsg_status tsg_breakpoints(int bits, double* out256) {
    return guarded([&] {
        if (bits < 1 || bits > 8) fail("tsg_breakpoints: bits must be in [1, 8]");
        if (!out256) fail("tsg_breakpoints: null out");
        host_breakpoints(bits, out256);
    });
}

tsg_status tsg_index_thresholds(const tsg_index* ix, double* out256) {
    return guarded([&] {
        if (!ix || !out256) fail("tsg_index_thresholds: null argument");
        const DevIndex& s = ix->shards[0];
        DeviceGuard g(s.device);
        TSG_CUDA(cudaMemcpy(out256, s.thr, kThrPad * sizeof(double), cudaMemcpyDeviceToHost));
    });
}

tsg_status tsg_index_export_fine(const tsg_index* ix, uint32_t* fine_width, uint8_t* fine) {
    return guarded([&] {
        if (!ix) fail("tsg_index_export_fine: null index");
        if (ix->shards.size() != 1) fail("tsg_index_export_fine: single-device index only");
        const DevIndex& s = ix->shards[0];
        DeviceGuard g(s.device);
        if (fine_width) *fine_width = static_cast<uint32_t>(s.fw);
        if (fine && s.fw) {  // stored in index order: back to dataset order for the caller
            std::vector<uint8_t> idx(s.N * s.fws);
            std::vector<uint32_t> pos(s.N);
            TSG_CUDA(cudaMemcpy(idx.data(), s.fine, s.N * s.fws, cudaMemcpyDeviceToHost));
            TSG_CUDA(cudaMemcpy(pos.data(), s.pos, s.N * 4, cudaMemcpyDeviceToHost));
            for (uint64_t i = 0; i < s.N; ++i) std::memcpy(fine + static_cast<uint64_t>(pos[i]) * s.fws, &idx[i * s.fws], s.fws);
        }
    });
}

tsg_status tsg_generate_series(int kind, float* dev_rows, uint64_t begin, uint64_t count, uint64_t length,
                               uint64_t seed, int znorm, double noise, uint64_t data_count, uint64_t data_seed,
                               void* stream) {
    return guarded([&] {
        if (count == 0) return;
        if (!dev_rows) fail("generate: null rows");
        if (kind != kGenRandomWalk && kind != kGenC3 && kind != kGenC4 && kind != kGenC5)
            fail("generate: kind must be 0, 3, 4 or 5");
        device_count();
        generate_series(kind, dev_rows, begin, count, length, seed, znorm, noise, data_count, data_seed,
                        static_cast<cudaStream_t>(stream));
        TSG_CUDA(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
    });
}

tsg_status tsg_profile_enable(tsg_index* ix, int enable) {
    return guarded([&] {
        if (!ix) fail("tsg_profile_enable: null index");
        std::lock_guard<std::mutex> lock(ix->mu);
        for (auto& s : ix->shards) s.profile = enable != 0;
    });
}

tsg_status tsg_profile_read(tsg_index* ix, double* ms, uint64_t* launches, int reset) {
    return guarded([&] {
        if (!ix) fail("tsg_profile_read: null index");
        std::lock_guard<std::mutex> lock(ix->mu);
        for (int k = 0; k < kProfSlots; ++k) {
            double m = 0;
            uint64_t l = 0;
            for (auto& s : ix->shards) {
                m = std::max(m, s.prof_ms[k]);
                l += s.prof_launches[k];
                if (reset) {
                    s.prof_ms[k] = 0;
                    s.prof_launches[k] = 0;
                }
            }
            if (ms) ms[k] = m;
            if (launches) launches[k] = l;
        }
    });
}

tsg_status tsg_generate_random_walk(float* dev_rows, uint64_t begin, uint64_t count, uint64_t length, uint64_t seed,
                                    int znorm, void* stream) {
    return guarded([&] {
        if (count == 0) return;
        if (!dev_rows) fail("generate_random_walk: null rows");
        device_count();
        generate_random_walk(dev_rows, begin, count, length, seed, znorm, static_cast<cudaStream_t>(stream));
        TSG_CUDA(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
    });
}

}  // extern "C"
