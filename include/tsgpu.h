/*
 * tsgpu.h — C ABI of the B200-native tsidx hot path (iSAX build + exact
 * Euclidean 1-NN). One shared library: paper_2009_00786_b200/libtsgpu.so.
 *
 * Plain pointers and sizes, no exceptions and no torch types cross this
 * boundary. Each entry point names the reference interface it replaces
 * (paths relative to /root/reference/proj/core):
 *
 *   tsg_index_build          <- tsidx::build_index(Dataset, IndexConfig)
 *                               include/tsidx/index.hpp:158, src/index.cpp:258-318
 *   tsg_search               <- tsidx::exact_search(const Index&, span<const float>,
 *                               Measure, SearchOptions)  include/tsidx/query.hpp:150-151,
 *                               src/query.cpp:258-298 (Measure::ed(); any Measure:
 *                               tsg_search_measure)
 *   tsg_index_validate       <- tsidx::validate_index  include/tsidx/index.hpp:202,
 *                               src/index.cpp:332-484
 *   tsg_approximate_search   <- tsidx::approximate_search  include/tsidx/query.hpp:133-134
 *   tsg_config               <- tsidx::IndexConfig          include/tsidx/config.hpp:12-32
 *   tsg_config_validate      <- IndexConfig::validate       src/config.cpp:22-35
 *   tsg_build_stats          <- tsidx::BuildStats           include/tsidx/index.hpp:121-132
 *   tsg_search_stats         <- tsidx::SearchStats          include/tsidx/query.hpp:17-27
 *   tsg_summarise            <- paa_into + symbols_from_paa + root_key_from_symbols
 *                               (the summarization hot loop, src/index.cpp:162-167)
 *
 * Error contract: every call returns a tsg_status. TSG_INVALID_ARGUMENT is
 * what the reference throws as std::invalid_argument, TSG_LOGIC as
 * std::logic_error, TSG_RUNTIME as std::runtime_error. The message of the
 * last failure on the calling thread is tsg_last_error().
 *
 * There is no CPU fallback: without a usable sm_100 device every compute
 * call fails with TSG_CUDA.
 */
#ifndef TSGPU_H
#define TSGPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum tsg_status {
    TSG_OK = 0,
    TSG_INVALID_ARGUMENT = 1,
    TSG_RUNTIME = 2,
    TSG_LOGIC = 3,
    TSG_CUDA = 4,
    TSG_NCCL = 5,
    TSG_OOM = 6
} tsg_status;

/* Mirrors tsidx::IndexConfig field for field (include/tsidx/config.hpp:12-32).
 * The worker / queue fields are accepted, validated and ignored: the device
 * path has no worker threads or leaf queues (their role is played by the
 * grid and by LB-ordered candidate refinement). */
typedef struct tsg_config {
    uint64_t n;                       /* series length, multiple of w */
    int32_t w;                        /* PAA segments, 1..32 on the device path */
    int32_t max_card_bits;            /* 1..8 */
    uint64_t leaf_capacity;           /* >= 2 */
    uint64_t chunk_size;              /* >= 1 (ignored) */
    uint32_t n_index_workers;         /* ignored */
    uint32_t n_search_workers;        /* ignored */
    uint32_t n_queues;                /* >= 1 (ignored) */
    int32_t queue_mode;               /* 0 single, 1 multi (ignored) */
    uint64_t initial_buffer_part_size;/* >= 1 (ignored) */
} tsg_config;

/* tsidx::BuildStats (include/tsidx/index.hpp:121-132) plus device timings. */
typedef struct tsg_build_stats {
    uint64_t build_ns;        /* device work of the build (CUDA events), excludes H2D */
    uint64_t series;
    uint64_t nodes;
    uint64_t inner_nodes;
    uint64_t leaves;
    uint64_t empty_leaves;
    uint64_t overflow_leaves;
    uint64_t max_depth;       /* root children are depth 1 */
    /* device-path extras */
    uint64_t root_children;   /* distinct root keys */
    uint64_t pages;           /* leaf pages (<= 128 entries each): the device LB / work unit */
    uint64_t h2d_ns;          /* host->device copy of the rows (0 for device input) */
    double summarise_ms;      /* K1 */
    double organise_ms;       /* K2 sort */
    double leaves_ms;         /* K2 gather (side stream) overlapped with K3 leaves / pages / boxes */
} tsg_build_stats;

/* tsidx::SearchStats (include/tsidx/query.hpp:17-27). Device meaning:
 * lb_node_calcs = leaf-box lower bounds, lb_entry_calcs = word lower bounds,
 * real_dist_calcs = full Euclidean refinements, bsf_updates = strict BSF
 * improvements, pruned_subtrees = pruned leaves, queue_insertions =
 * compacted candidates. */
typedef struct tsg_search_stats {
    uint64_t lb_node_calcs;
    uint64_t lb_entry_calcs;
    uint64_t real_dist_calcs;
    uint64_t bsf_updates;
    uint64_t pruned_subtrees;
    uint64_t queue_insertions;
} tsg_search_stats;

/* tsidx::SearchResult: distance, position (global dataset row), stats. */
typedef struct tsg_result {
    double distance;
    uint32_t position;
    uint32_t box_calcs;  /* quad (4-entry) box bounds evaluated (saturates at 2^32-1); group, page and
                            run boxes count in stats.lb_node_calcs */
    tsg_search_stats stats;
    uint64_t fine_calcs;  /* fine-summary (2w half-segment) lower bounds evaluated before refinement */
} tsg_result;

typedef struct tsg_ctx tsg_ctx;
typedef struct tsg_index tsg_index;

const char* tsg_last_error(void);
const char* tsg_version(void);

/* Defaults of IndexConfig (w=16, 8 bits, leaf 2000, chunk 20000, 24 queues, mq, part 5). */
void tsg_config_default(tsg_config* cfg);
tsg_status tsg_config_validate(const tsg_config* cfg);

/* Lifecycle. n_gpus devices (devices may be NULL for 0..n_gpus-1). An index
 * built on a context shards its rows across the context's devices in
 * contiguous ranges; search combines the per-shard answers:
 *   - distinct devices: one NCCL communicator over them (ncclCommInitAll);
 *     per batch an ncclAllReduce(min) of the shards' seed best-so-far
 *     distances (every shard prunes against the global seed) and one
 *     ncclAllGather of the per-shard result records, merged on the device
 *     (lexicographic (distance, position) minimum = scan_nn's tie rule,
 *     src/scan.cpp:54-59);
 *   - the same device repeated (e.g. {0, 0}): the same two exchanges over
 *     device memory (local shards, for tests and over-decomposition);
 *   - any other mix: TSG_INVALID_ARGUMENT.
 * NCCL is loaded at run time (the process's libnccl.so.2, else the system's;
 * TSG_NCCL_LIB overrides); failures map to TSG_NCCL. Free every index of a
 * context before closing it. */
tsg_status tsg_open(int n_gpus, const int* devices, tsg_ctx** out);
tsg_status tsg_close(tsg_ctx* ctx);

/* One process per GPU (torchrun-style). Rank 0 creates an id, the caller
 * distributes it (any channel), every rank joins its one-device context to the
 * communicator. An index built on the context is this rank's shard (pass its
 * first global row as position_offset); tsg_search / tsg_search_device /
 * tsg_search_measure on it are COLLECTIVE: every rank calls them with the same
 * nq, and every rank receives the global answers (seed-BSF allreduce inside
 * the query pipeline, result all-gather + device merge after it). */
typedef struct tsg_comm_id {
    uint8_t internal[128];
} tsg_comm_id;
tsg_status tsg_comm_unique_id(tsg_comm_id* id);
tsg_status tsg_comm_init(tsg_ctx* ctx, int nranks, int rank, const tsg_comm_id* id);
enum { TSG_TRANSPORT_NONE = 0, TSG_TRANSPORT_LOCAL = 1, TSG_TRANSPORT_NCCL = 2 };
/* transport of the context, its number of shards / ranks, and this process's rank. */
tsg_status tsg_comm_info(const tsg_ctx* ctx, int* transport, int* nranks, int* rank);

/* Build from HOST rows (count x length float32, row-major). The library
 * copies the rows into HBM; the caller keeps ownership of its buffer.
 * position_offset is added to every returned position (a shard's first
 * global row when one process builds one shard of a larger dataset). */
tsg_status tsg_index_build(tsg_ctx* ctx, const float* host_rows, uint64_t count,
                           uint64_t length, const tsg_config* cfg, uint64_t position_offset,
                           tsg_index** out, tsg_build_stats* stats);

/* Build from rows already resident in device memory on the context's first
 * device. The index borrows them: they must stay valid until tsg_index_free.
 * Single-device contexts only. Ordering: the library reads device inputs on its
 * own non-blocking stream, so every write to them (on any stream) must have
 * completed before the call — synchronise the producing stream first (the
 * Python mirror synchronises torch's current stream of the tensor's device). */
tsg_status tsg_index_build_device(tsg_ctx* ctx, const float* dev_rows, uint64_t count,
                                  uint64_t length, const tsg_config* cfg,
                                  uint64_t position_offset, tsg_index** out,
                                  tsg_build_stats* stats);

/* Build straight from a headerless float32 file (count x length, row-major)
 * <- tsidx::load_dataset(path, length) (src/dataset.cpp:87-117) followed by
 * tsidx::build_index (src/index.cpp:258-318). The series count comes from the
 * file size (load_dataset's checks and messages: TSG_INVALID_ARGUMENT for
 * length 0, TSG_RUNTIME for a missing file or a size that is not a positive
 * multiple of length * 4). Each device reads its range of the file in
 * ~128 MB chunks through pinned buffers while K1 summarises the chunks that
 * already arrived (disk, PCIe and K1 overlap); no host copy of the dataset
 * is kept. stats->h2d_ns = wall time of the streaming phase. */
tsg_status tsg_index_build_file(tsg_ctx* ctx, const char* path, uint64_t length,
                                const tsg_config* cfg, uint64_t position_offset,
                                tsg_index** out, tsg_build_stats* stats);

tsg_status tsg_index_free(tsg_index* index);

/* tsidx::Measure (include/tsidx/query.hpp): Euclidean, or DTW under a
 * Sakoe-Chiba band of half-width `window` (0 <= window < n; the device path
 * supports window <= 255). */
enum { TSG_MEASURE_ED = 0, TSG_MEASURE_DTW = 1 };
typedef struct tsg_measure {
    int32_t kind;
    int32_t window;
} tsg_measure;

/* exact_search / approximate_search with a Measure (query.hpp:133-151) for nq
 * queries (host, or device when queries_on_device != 0). DTW follows
 * calculate_real_distance_leaf's DTW branch (src/query.cpp:138-145): envelope
 * bound on nodes and entries (mindist_envelope_isax), LB_Keogh, then banded DTW
 * with abandonment; answers equal scan_nn(Measure::dtw(window)) with ties to the
 * lowest position. Invalid window -> TSG_INVALID_ARGUMENT ("dtw window must be
 * in [0, n)"). */
tsg_status tsg_search_measure(tsg_index* index, const float* queries, int queries_on_device, uint32_t nq,
                              const tsg_measure* measure, int approximate, tsg_result* out);

tsg_status tsg_index_info(const tsg_index* index, uint64_t* count, uint64_t* length,
                          tsg_config* cfg, tsg_build_stats* stats);

/* Exact 1-NN of nq HOST queries (nq x length float32). out[nq] on the host. */
tsg_status tsg_search(tsg_index* index, const float* host_queries, uint32_t nq,
                      tsg_result* out);

/* Same for queries already in device memory (first device of the index).
 * out is a HOST array. The same ordering rule as tsg_index_build_device: the
 * queries must be complete (producing stream synchronised) when called. */
tsg_status tsg_search_device(tsg_index* index, const float* dev_queries, uint32_t nq,
                             tsg_result* out);

/* Approximate answer: the best series inside the query's closest leaf. */
tsg_status tsg_approximate_search(tsg_index* index, const float* host_query, tsg_result* out);

/* ---- kernel-level entry points (parity tests, benchmarks) ---------------- */

/* K1 alone over device rows: words[count][word_stride] (left-aligned
 * symbols, segment order, zero padded) and root keys[count]. word_stride is
 * 16 for w <= 16, else 32. stream may be NULL (legacy default stream). */
tsg_status tsg_summarise(const float* dev_rows, uint64_t count, uint64_t length, int w,
                         int bits, uint8_t* dev_words, uint32_t* dev_root_keys, void* stream);

/* The symbol thresholds of cardinality 2^bits: out[256] receives the 2^bits - 1
 * breakpoints of tsidx::breakpoints_for(2^bits) (src/breakpoints.cpp:65-114,
 * Acklam + one Newton step, lower half mirrored) followed by +inf padding, as
 * computed on the host for upload (no GPU needed). */
tsg_status tsg_breakpoints(int bits, double* out256);

/* The threshold table the index's summarisation and query kernels read, copied
 * back from HBM (first device): 256 doubles in the layout of tsg_breakpoints. */
tsg_status tsg_index_thresholds(const tsg_index* index, double* out256);

/* tsidx::ValidationReport (include/tsidx/index.hpp:180-196) of the flat index.
 * Device meaning: nodes = leaves + inner (split) nodes; the audit checks every
 * position stored exactly once, every stored word equal to the word recomputed
 * from its series, key / position order, one root key per leaf, leaf capacity
 * (overflow leaves only where no key bit can split), page tiling and the exact
 * min / max of every page / run / quad box (group and top boxes containing
 * their children), and the fine summary against a recomputation. */
typedef struct tsg_validation_report {
    uint64_t nodes;
    uint64_t inner_nodes;
    uint64_t leaves;
    uint64_t empty_leaves;
    uint64_t overflow_leaves;
    uint64_t max_depth;
    uint64_t total_entries;
    uint64_t leaf_fill_histogram[11]; /* 10% buckets of leaf_capacity, then overflow leaves */
    uint64_t violation_count;
    uint32_t n_violations;            /* messages below (the first 20 kinds found) */
    uint32_t reserved;
    char violations[20][160];
    /* device extension */
    uint64_t pages;
    uint64_t checked_boxes;
} tsg_validation_report;

/* <- tsidx::validate_index(const Index&) (src/index.cpp:332-484). */
tsg_status tsg_index_validate(tsg_index* index, tsg_validation_report* out);

/* Test hook: overwrite n bytes at byte offset `offset` of one of the index's
 * device arrays (first shard): 0 words, 1 positions, 2 leaf offsets, 3 page
 * min boxes, 4 quad boxes ((min, max) pairs of 2 x word stride bytes, from the
 * first min), 5 fine summary, 6 run boxes (pairs, from the first max), 7
 * group min boxes. Lets tests prove the audit catches each kind of corruption. */
tsg_status tsg_index_debug_poke(tsg_index* index, int array, uint64_t offset, const void* bytes, uint64_t n);

/* Word stride used by the device layout for a given w. */
int tsg_word_stride(int w);

/* Copy the index's flat SoA back to the host (single-device index):
 * words[count][word_stride] in index order, positions[count] (global),
 * leaf_offsets[leaves+1], page_offsets[pages+1] and the per-page symbol
 * boxes page_lo/page_hi[pages][word_stride]. Any pointer may be NULL. */
tsg_status tsg_index_export(const tsg_index* index, uint8_t* words, uint32_t* positions,
                            uint32_t* leaf_offsets, uint32_t* page_offsets, uint8_t* page_lo,
                            uint8_t* page_hi);

/* The fine summary (device extension, a second lower bound in front of
 * refinement): *fine_width = 2w half-segment symbols per series (0 when the
 * index has none: 2w > 64, n % 2w != 0, or TSG_NO_FINE at build time) and,
 * if fine is not NULL, fine[count][stride] in dataset order, stride = the
 * fine width rounded up to 16 bytes. Symbol = the FP64 mean of the half
 * segment (the same sums as summarisation) quantised uniformly over
 * [-2.5, 2.5) in 256 steps (0 / 255 open-ended). */
tsg_status tsg_index_export_fine(const tsg_index* index, uint32_t* fine_width, uint8_t* fine);

/* Device data generator: rows [begin, begin+count) of the reference's
 * generate_random_walk(., length, seed) (src/dataset.cpp:22-68), optionally
 * z-normalised the CLI way (degenerate -> zeros, tools/main.cpp:128-139),
 * written to dev_rows. Input-setup utility, not part of the timed path. */
tsg_status tsg_generate_random_walk(float* dev_rows, uint64_t begin, uint64_t count,
                                    uint64_t length, uint64_t seed, int znorm, void* stream);

/* Device generators for the BASELINE workloads (input setup, not timed):
 * kind 0 = random walk (as tsg_generate_random_walk), 3 = config 3 (AR(1) +
 * sinusoid), 4 = config 4 (1024-component Gaussian mixture), 5 = config 5
 * queries: rows [begin, begin+count) of query stream `seed`, each a
 * z-normalised random-walk row of (data_seed, data_count) chosen by the
 * stream plus N(0, noise^2), re-z-normalised. Definitions and their CPU
 * restatement: oracle/tsidx_oracle.cpp. */
tsg_status tsg_generate_series(int kind, float* dev_rows, uint64_t begin, uint64_t count, uint64_t length,
                               uint64_t seed, int znorm, double noise, uint64_t data_count,
                               uint64_t data_seed, void* stream);

/* Number of kernel launches this process issued through the library. */
uint64_t tsg_launch_count(void);

/* Per-kernel device timing of the search pipeline (CUDA events recorded on
 * the index's stream around every launch; the pipeline then runs without its
 * CUDA graph). Slots: 0 unused, 1 groups + bound (both page waves), 2 prepare +
 * seed, 3 refine wave A (fine bound + rows), 4 lbscan (both waves), 5 refine
 * wave B, 6 finalize, 7 cross-shard seed-BSF exchange. ms[8] (max over the
 * index's shards) and launches[8] (query-launches, summed) accumulate until
 * reset. */
tsg_status tsg_profile_enable(tsg_index* index, int enable);
tsg_status tsg_profile_read(tsg_index* index, double* ms, uint64_t* launches, int reset);

#ifdef __cplusplus
}
#endif

#endif /* TSGPU_H */
