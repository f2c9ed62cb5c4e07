// tsidx C++ API — drop-in for the reference's build/search surface, backed
// by the B200 device path (libtsgpu.so, C ABI in include/tsgpu.h).
//
// Mirrors, name for name (paths relative to /root/reference/proj/core):
//   IndexConfig, QueueMode           include/tsidx/config.hpp:10-32
//   Dataset, generate_random_walk,
//   znormalize, load_dataset,
//   save_dataset,
//   pad_to_segment_multiple          include/tsidx/dataset.hpp:14-47
//   Measure, MeasureKind, kAbandoned include/tsidx/metrics.hpp:15-27
//   BuildStats, Index, build_index   include/tsidx/index.hpp:121-158
//   SearchStats, SearchOptions,
//   SearchResult, ApproxResult,
//   exact_search, approximate_search include/tsidx/query.hpp:17-151
//   ValidationReport, validate_index include/tsidx/index.hpp:180-202
//
// Error contract as in the reference: std::invalid_argument for bad
// configs/inputs, std::logic_error, std::runtime_error for device failures.
// Differences: Measure::dtw is answered on the device for windows
// <= 255 (larger windows: std::invalid_argument, no CPU fallback),
// workers/queues/mode options are accepted and ignored, w <= 32.
#pragma once

#include <cstddef>
#include <array>
#include <cstdint>
#include <filesystem>
#include <limits>
#include <memory>
#include <optional>
#include <span>
#include <string>
#include <vector>

#include "../tsgpu.h"

namespace tsidx {

enum class QueueMode { single, multi };

struct IndexConfig {
    std::size_t n = 256;
    int w = 16;
    int max_card_bits = 8;
    std::size_t leaf_capacity = 2000;
    std::size_t chunk_size = 20000;
    unsigned n_index_workers = 0;
    unsigned n_search_workers = 0;
    unsigned n_queues = 24;
    QueueMode queue_mode = QueueMode::multi;
    std::size_t initial_buffer_part_size = 5;

    static unsigned default_workers();
    std::size_t segment_length() const { return n / static_cast<std::size_t>(w); }
    unsigned index_workers() const;
    unsigned search_workers() const;
    void validate() const;  // throws std::invalid_argument naming the field
};

struct Dataset {
    std::size_t count = 0;
    std::size_t length = 0;
    std::size_t source_length = 0;
    std::vector<float> values;

    std::span<const float> series(std::size_t i) const { return {values.data() + i * length, length}; }
    std::span<float> series_mut(std::size_t i) { return {values.data() + i * length, length}; }
};

// Same seeded generator as the reference (bit-identical), run on the GPU.
Dataset generate_random_walk(std::size_t count, std::size_t length, std::uint64_t seed);
bool znormalize(std::span<float> series);
Dataset load_dataset(const std::filesystem::path& path, std::size_t length);
void save_dataset(const std::filesystem::path& path, const Dataset& dataset);
Dataset pad_to_segment_multiple(Dataset dataset, int w);

inline constexpr double kAbandoned = std::numeric_limits<double>::infinity();
enum class MeasureKind { euclidean, dtw };
struct Measure {
    MeasureKind kind = MeasureKind::euclidean;
    int window = 0;
    static Measure ed() { return {MeasureKind::euclidean, 0}; }
    static Measure dtw(int window) { return {MeasureKind::dtw, window}; }
};

struct BuildStats {
    std::uint64_t build_ns = 0;
    std::size_t series = 0;
    std::size_t nodes = 0;
    std::size_t inner_nodes = 0;
    std::size_t leaves = 0;
    std::size_t empty_leaves = 0;
    std::size_t overflow_leaves = 0;
    std::size_t max_depth = 0;
    std::string kv_line() const;
};

struct SearchStats {
    std::uint64_t lb_node_calcs = 0;
    std::uint64_t lb_entry_calcs = 0;
    std::uint64_t real_dist_calcs = 0;
    std::uint64_t bsf_updates = 0;
    std::uint64_t pruned_subtrees = 0;
    std::uint64_t queue_insertions = 0;
    SearchStats& operator+=(const SearchStats& other);
    std::string kv_line() const;
};

struct SearchOptions {
    unsigned workers = 0;
    unsigned queues = 0;
    std::optional<QueueMode> mode;
};

struct SearchResult {
    double distance = 0.0;
    std::uint32_t position = 0;
    SearchStats stats;
};

struct ApproxResult {
    double distance = 0.0;
    std::uint32_t position = 0;
};

// Owns the host Dataset (like the reference Index) and the device index.
class Index {
  public:
    Index(Dataset dataset, IndexConfig config, tsg_index* handle, BuildStats stats);
    Index(Index&&) noexcept;
    Index& operator=(Index&&) noexcept;
    ~Index();

    const IndexConfig& config() const { return config_; }
    const Dataset& data() const { return data_; }
    std::span<const float> series(std::uint32_t position) const { return data_.series(position); }
    const BuildStats& build_stats() const { return stats_; }
    tsg_index* handle() const { return handle_; }

  private:
    Dataset data_;
    IndexConfig config_;
    tsg_index* handle_ = nullptr;
    BuildStats stats_;
};

Index build_index(Dataset dataset, IndexConfig config);

SearchResult exact_search(const Index& index, std::span<const float> query, Measure measure = Measure::ed(),
                          SearchOptions options = {});

// Batched form: one device call for many queries (queries.size() == k * n).
std::vector<SearchResult> exact_search_batch(const Index& index, std::span<const float> queries,
                                             Measure measure = Measure::ed());

ApproxResult approximate_search(const Index& index, std::span<const float> query,
                                Measure measure = Measure::ed());

// <- tsidx::ValidationReport / validate_index (include/tsidx/index.hpp:180-202):
// the device audit of the flat index (tsg_index_validate, see include/tsgpu.h).
struct ValidationReport {
    std::size_t nodes = 0;
    std::size_t inner_nodes = 0;
    std::size_t leaves = 0;
    std::size_t empty_leaves = 0;
    std::size_t overflow_leaves = 0;
    std::size_t max_depth = 0;
    std::size_t total_entries = 0;
    std::array<std::size_t, 11> leaf_fill_histogram{};
    std::vector<std::string> violations;  // first few, see violation_count
    std::size_t violation_count = 0;

    bool ok() const { return violation_count == 0; }
    std::string summary() const;
};

ValidationReport validate_index(const Index& index);

}  // namespace tsidx
