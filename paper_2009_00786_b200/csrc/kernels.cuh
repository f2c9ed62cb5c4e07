// Device-side index layout and the host launchers of every kernel.
#pragma once

#include <cuda_runtime.h>
#include <cstdint>
#include <functional>

#include "common.cuh"

struct tsg_validation_report;  // include/tsgpu.h

namespace tsg {

class Exchange;

// Entries per page: the unit of the leaf-level lower bound and of work
// distribution in the LB scan (a leaf is split into ceil(size/kPage) pages).
constexpr uint32_t kPage = 128;

// Flat structure-of-arrays index of one device shard. Replaces the
// reference's pointer tree (IndexNode / LeafEntries / RootTable,
// include/tsidx/index.hpp:19-75): words and positions are sorted by the
// plane-major iSAX key (root key first), leaves are contiguous ranges,
// pages are contiguous sub-ranges of leaves with their own symbol boxes.
struct DevIndex {
    int device = 0;
    cudaStream_t stream = nullptr;
    uint64_t N = 0;           // series on this shard
    int n = 0, w = 0, bits = 0, ws = 16;
    uint64_t leaf_cap = 0;
    int key_bits = 64;        // sort-key bits the build ordered entries by (build.cu)
    uint64_t pos_offset = 0;  // global position of local row 0
    float* rows = nullptr;    // [N][n] original order
    bool own_rows = false;
    double* thr = nullptr;    // [256] thresholds for `bits`, +inf padded
    uint8_t* words = nullptr; // [N][ws] index order
    // Fine summary (fine_width): [N][fws] quantised 2w half-segment means
    // (fine_quant), index order (row i = the series of entry i). fw = 0: none.
    uint8_t* fine = nullptr;
    int fw = 0, fws = 0;
    uint32_t* pos = nullptr;  // [N] local row of each index entry
    uint32_t* leaf_off = nullptr;  // [L+1]
    uint64_t L = 0;
    uint32_t* page_off = nullptr;   // [P+1] entry offsets (pages tile [0, N))
    uint32_t* page_leaf = nullptr;  // [P]
    uint64_t* page_key = nullptr;   // [P] sort key of each page's first entry
    uint8_t* page_lo = nullptr;     // [P][ws] per-segment min symbol
    uint8_t* page_hi = nullptr;     // [P][ws] per-segment max symbol
    uint8_t* group_lo = nullptr;    // [NG][ws] per-segment min symbol of pages [kGroup g, kGroup g + kGroup)
    uint8_t* group_hi = nullptr;    // [NG][ws] per-segment max symbol
    uint64_t NG = 0;                // ceil(P / kGroup)
    uint8_t* top_lo = nullptr;      // [NT][ws] per-segment min symbol of groups [kGroup t, kGroup t + kGroup)
    uint8_t* top_hi = nullptr;      // [NT][ws] per-segment max symbol
    uint64_t NT = 0;                // ceil(NG / kGroup): the level above groups
    // Run and quad boxes are stored as (min, max) pairs, 2 ws bytes per box
    // (run_hi = run_lo + ws, stride 2 ws): a run's four quad boxes are one
    // 128-byte line, and B200 fetches a whole 128-byte line from HBM for any
    // random read (profiles/micro/dram_granularity.cu), so separate min / max
    // arrays would pull two lines per run, each half used.
    uint8_t* run_lo = nullptr;      // [R] pairs: per-segment min symbol of entries [kRun r, kRun r + kRun)
    uint8_t* run_hi = nullptr;      // run_lo + ws: per-segment max symbol (interior pointer)
    uint64_t R = 0;                 // ceil(N / kRun)
    uint8_t* quad_lo = nullptr;     // [Q] pairs: per-segment min symbol of entries [kQuad q, kQuad q + kQuad)
    uint8_t* quad_hi = nullptr;     // quad_lo + ws: per-segment max symbol (interior pointer)
    uint64_t Q = 0;                 // ceil(N / kQuad)
    uint64_t P = 0;
    uint64_t root_children = 0;
    uint64_t inner = 0, max_depth = 0, overflow = 0;
    uint64_t* page_dir = nullptr;   // [(P + 255) / 256] page_key of every 256th page
    // Search workspace: per-query slots of one batch (every kernel of the
    // pipeline runs once per batch over all its queries), and a single slot
    // with room for every entry, for queries that outgrow a batch slot.
    struct Slots {
        uint32_t n = 0;                 // slots allocated
        uint64_t cap = 0;               // candidate records per slot
        struct QueryWork* work = nullptr;  // [n]
        float* lut = nullptr;           // [n][w][256] squared-gap tables
        float* fine_lut = nullptr;      // [n][fw][256] squared-gap tables of the fine summary
        uint32_t* gsurv = nullptr;      // [n][NG] surviving page groups
        uint64_t rcap = 0;              // run-list capacity per slot (every run of the shard)
        uint2* surv = nullptr;          // [n][rcap] surviving runs' entry ranges: wave 0 front, wave 1 back
        float* surv_lb = nullptr;       // [n][rcap] their box bounds
        uint2* dpage = nullptr;         // [n][P] deferred pages' entry ranges
        float* dpage_lb = nullptr;      // [n][P] their box bounds
        uint32_t* cand_pos = nullptr;   // [n][cap] candidate entries: refinement wave A front, B back
        float* cand_lb = nullptr;       // [n][cap]
        double* cand_sq = nullptr;      // [n][cap]
        float* env = nullptr;           // [n][2][len] DTW: the query's upper / lower Keogh envelope
    };
    Slots batch, big;
    uint32_t batch_max = 128;       // queries per batch (TSG_BATCH)
    uint32_t eff_batch = 0;         // queries per batch after overflow feedback (search_all; 0 = batch_max)
    struct DevResult* results = nullptr;  // [results_cap]
    uint32_t results_cap = 0;
    float* queries = nullptr;      // staging for host queries
    uint32_t queries_cap = 0;
    int sms = 148;
    float refine_split = 0.3f;     // wave-0 page-bound fraction of the seed bound (TSG_REFINE_SPLIT)
    // per-kernel profiling (tsg_profile_enable)
    bool profile = false;
    void* graphs = nullptr;  // search_batch's CUDA graphs of the batch pipeline (search.cu)
    class Exchange* xchg = nullptr;  // cross-shard exchange endpoint (exchange.cuh; owned by the index)
    struct DevResult* merged = nullptr;  // [results_cap] NCCL merge output
    double prof_ms[8] = {0};
    uint64_t prof_launches[8] = {0};
};

constexpr int kProfSlots = 8;
constexpr int kGroup = 8;  // pages per group box (the level above pages)
constexpr int kRun = 16;  // entries per run box (the sub-page filter level)
constexpr int kQuad = 4;  // entries per quad box (the level below runs)

// Per-query device scratch (reset by the prepare kernel).
constexpr unsigned kTieCap = 64;
enum WorkCounter {
    kNextBound = 0, kNextScan0, kNextRefine0, kNextBound1, kNextScan1, kNextRefine1, kNextFine0, kNextFine1, kNextCount
};
struct QueryWork {
    unsigned long long bsf_bits;  // best squared distance so far (double bits)
    // candidate records: wave A (low 32 bits, from the front, after the seed
    // range) and wave B (high 32 bits, from the back), reserved together
    unsigned long long cand;
    unsigned int nseed;
    unsigned int seed_begin, seed_end;  // index range refined as the seed
    unsigned int ngroups;               // surviving page groups
    // surviving runs: wave 0 (low 32 bits, bound <= split x seed bound, front of
    // the run list) and wave 1 (high 32 bits, back of the list)
    unsigned long long runs;
    unsigned int ndefer;                // pages deferred to the second bound pass (bound > split x seed bound)
    unsigned int next[kNextCount];      // work-chunk counters of the persistent kernels
    unsigned int done_blocks;           // finalize's last-block counter
    unsigned int best_pos;
    unsigned int overflow;              // candidates outgrew the slot: rerun in the big slot
    float scan_bound;                   // BSF bound the page/word filters used
    unsigned long long boxes;           // run / quad box bounds evaluated
    unsigned long long stats[6];  // SearchStats order
    unsigned long long fine_calcs;      // fine-summary lower bounds evaluated
    unsigned char qsym[32];
    // every refined row whose sum was within the BSF when it finished (a
    // superset of the answer and its sqrt ties); finalize scans this list,
    // or all candidate records when more than kTieCap were noted
    unsigned int nties;
    unsigned int tie_row[kTieCap];
    double tie_sq[kTieCap];
};

constexpr uint32_t kResultOverflow = 1u;  // DevResult.flags: answer invalid, rerun with a full-size slot

struct DevResult {
    double distance;
    uint32_t position;
    uint32_t flags;
    unsigned long long stats[6];
    unsigned long long boxes;
    unsigned long long fine_calcs;
};

// K1. fine (may be null): the fine summary rows (fine_width(n, w) symbols,
// stride fine_stride) of the same series. record_stride > 0: words and fine
// rows are written with that stride (interleaved records, the build's layout).
void summarise(const float* rows, uint64_t count, int n, int w, int bits, const double* d_thr,
               uint8_t* words, uint32_t* root_keys, uint64_t* sort_keys, cudaStream_t stream,
               uint8_t* fine = nullptr, int key_bits = 64, int record_stride = 0);

// Streams the shard's rows into ix.rows chunk by chunk: for each chunk it
// enqueues the rows' arrival on ix.stream and then calls sum_chunk(first,
// count), which enqueues K1 for those rows on the same stream.
using RowFeeder = std::function<void(const std::function<void(uint64_t, uint64_t)>& sum_chunk)>;

// K1 + K2 + K3: summarise, sort, gather, leaves, pages, boxes. Fills the
// index arrays of `ix` (rows/thr/N/n/w/bits/leaf_cap must be set; with a
// feeder the rows arrive while K1 runs). Device ms per phase.
void build_layout(DevIndex& ix, double* ms_summarise, double* ms_organise, double* ms_leaves,
                  const RowFeeder* feeder = nullptr);

// Query pipeline for nq device queries in slots [0, nq) of `slots`; writes
// results[0..nq). Queries flagged kResultOverflow must be rerun with a slot
// of capacity N (api.cu's search_all does that).
// window < 0: Euclidean; window >= 0: DTW with that Sakoe-Chiba window
// (Measure::dtw, src/query.cpp:88-92,138-145).
// Destroys the shard's cached search graphs (free_shard).
void free_search_graphs(DevIndex& ix);
// exchange: this batch takes part in the cross-shard seed-BSF exchange of
// ix.xchg (every shard runs the same batches; reruns of overflowing queries
// do not exchange).
void search_batch(DevIndex& ix, const DevIndex::Slots& slots, const float* d_queries, uint32_t nq, bool approximate,
                  struct DevResult* results, int window = -1, bool exchange = false);
constexpr int kMaxDtwWindow = 255;  // the device DTW keeps a band diagonal in registers (8 cells per lane)

// validate_index (audit.cu): adds this shard's audit to *out.
void audit_index(DevIndex& ix, ::tsg_validation_report* out);

// Input generators (not on the timed path), see generate.cu.
enum GenKind {
    kGenRandomWalk = 0,  // the reference's random walks (BASELINE configs 1-2)
    kGenC3 = 3,          // AR(1) + sinusoid (config 3)
    kGenC4 = 4,          // Gaussian mixture (config 4)
    kGenC5 = 5,          // noisy dataset rows (config 5 queries)
    kGenC4Comp = 100,    // internal: mixture components
    kGenC5Rows = 101,    // internal: rows chosen by c5 queries
    kGenC5Noise = 102,   // internal: c5 noise on regenerated rows
};
void generate_random_walk(float* rows, uint64_t begin, uint64_t count, uint64_t length,
                          uint64_t seed, int znorm, cudaStream_t stream);
void generate_series(int kind, float* rows, uint64_t begin, uint64_t count, uint64_t length, uint64_t seed,
                     int znorm, double noise, uint64_t data_count, uint64_t data_seed, cudaStream_t stream);

}  // namespace tsg
