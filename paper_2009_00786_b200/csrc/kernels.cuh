// Device-side index layout and the host launchers of every kernel.
#pragma once

#include <cuda_runtime.h>
#include <cstdint>

namespace tsg {

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
    uint64_t pos_offset = 0;  // global position of local row 0
    float* rows = nullptr;    // [N][n] original order
    bool own_rows = false;
    double* thr = nullptr;    // [256] thresholds for `bits`, +inf padded
    uint8_t* words = nullptr; // [N][ws] index order
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
    uint8_t* run_lo = nullptr;      // [R][ws] per-segment min symbol of entries [kRun r, kRun r + kRun)
    uint8_t* run_hi = nullptr;      // [R][ws] per-segment max symbol
    uint64_t R = 0;                 // ceil(N / kRun)
    uint64_t P = 0;
    uint64_t root_children = 0;
    uint64_t inner = 0, max_depth = 0, overflow = 0;
    uint64_t* page_dir = nullptr;   // [(P + 255) / 256] page_key of every 256th page
    // search workspace: kLanes query lanes, each a stream with private
    // scratch, so consecutive queries of a batch run concurrently.
    struct Lane {
        cudaStream_t stream = nullptr;  // lane 0 uses the index stream
        cudaEvent_t done = nullptr;
        struct QueryWork* work = nullptr;
        float* lut = nullptr;          // [w][256] squared-gap table of the lane's query
        uint32_t* gsurv = nullptr;     // [NG] surviving page groups
        uint2* surv = nullptr;         // [P] surviving pages' entry ranges: wave 0 from the front, wave 1 from the back
        float* surv_lb = nullptr;      // [P] their box bounds
        uint32_t* cand_pos = nullptr;  // [cap]
        float* cand_lb = nullptr;      // [cap]
        double* cand_sq = nullptr;     // [cap]
    };
    static constexpr int kLanes = 16;
    Lane lanes[kLanes];
    int nlanes = 1;                // lanes in use (TSG_QUERY_LANES, default 8)
    cudaGraphExec_t graph = nullptr;  // the last query batch, captured (updated in place when the shape repeats)
    struct GraphKey {
        const float* queries = nullptr;
        uint32_t nq = 0;
        bool approximate = false;
        int nlanes = 0;
        int kernels = 0;  // launches the graph holds
    } graph_key;
    uint64_t cand_cap = 0;
    struct DevResult* results = nullptr;  // [results_cap]
    uint32_t results_cap = 0;
    float* queries = nullptr;      // staging for host queries
    uint32_t queries_cap = 0;
    int sms = 148;
    float refine_split = 0.5f;     // wave-0 page-bound fraction of the seed bound (TSG_REFINE_SPLIT)
    // per-kernel profiling (tsg_profile_enable)
    bool profile = false;
    double prof_ms[8] = {0};
    uint64_t prof_launches[8] = {0};
};

constexpr int kProfSlots = 8;
constexpr int kGroup = 8;  // pages per group box (the level above pages)
constexpr int kRun = 16;  // entries per run box (the sub-page filter level)

// Per-query device scratch (reset by the prep kernel).
struct QueryWork {
    unsigned long long bsf_bits;  // best squared distance so far (double bits)
    unsigned long long seed_key;  // (page LB float bits << 32) | page
    unsigned int ncand;
    unsigned int nseed;
    unsigned int work_next;
    unsigned int best_pos;
    unsigned int seed_begin, seed_end;  // index range refined as the seed
    unsigned int nsurv;                 // surviving pages, wave 0 (bound <= split x seed bound)
    unsigned int nsurv_hi;              // surviving pages, wave 1 (stored from the back of surv)
    unsigned int nhigh;                 // wave-1 candidates, stored at the top of the candidate arrays
    unsigned int ngroups;               // surviving page groups
    unsigned int done_blocks;           // finalize's last-block counter
    float scan_bound;                   // BSF bound the page/word filters used
    unsigned long long stats[6];  // SearchStats order
    double qpaa[32];
    unsigned char qsym[32];
};

struct DevResult {
    double distance;
    uint32_t position;
    uint32_t reserved;
    unsigned long long stats[6];
};

// K1
void summarise(const float* rows, uint64_t count, int n, int w, int bits, const double* d_thr,
               uint8_t* words, uint32_t* root_keys, uint64_t* sort_keys, cudaStream_t stream);

// K2 + K3: sort, gather, leaves, pages, boxes. Fills the index arrays of
// `ix` (rows/thr/N/n/w/bits/leaf_cap must be set). Device ms per phase.
void build_layout(DevIndex& ix, double* ms_summarise, double* ms_organise, double* ms_leaves);

// Query pipeline for nq device queries; writes ix.results[0..nq).
void search_batch(DevIndex& ix, const float* d_queries, uint32_t nq, bool approximate);

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
