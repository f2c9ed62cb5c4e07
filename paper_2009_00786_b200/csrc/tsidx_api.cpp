// tsidx C++ API (include/tsidx/tsidx.hpp) over the C ABI (include/tsgpu.h).
//
// Same names, argument meaning and error behaviour as the reference's
// public interface (paths relative to /root/reference/proj/core):
// IndexConfig::validate (src/config.cpp:22-35), build_index
// (src/index.cpp:258-318), exact_search (src/query.cpp:258-298),
// approximate_search (src/query.cpp:250-256), dataset utilities
// (src/dataset.cpp:41-137). Compute goes to the GPU; the host code here only
// converts types, owns the host Dataset and maps status codes back to the
// reference's exception types.
#include "../../include/tsidx/tsidx.hpp"

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>

namespace tsidx {

namespace {

void throw_status(tsg_status s) {
    if (s == TSG_OK) return;
    const std::string msg = tsg_last_error();
    switch (s) {
        case TSG_INVALID_ARGUMENT: throw std::invalid_argument(msg);
        case TSG_LOGIC: throw std::logic_error(msg);
        case TSG_OOM: throw std::bad_alloc();
        default: throw std::runtime_error("tsgpu: " + msg);
    }
}

tsg_config to_c(const IndexConfig& c) {
    tsg_config o{};
    o.n = c.n;
    o.w = c.w;
    o.max_card_bits = c.max_card_bits;
    o.leaf_capacity = c.leaf_capacity;
    o.chunk_size = c.chunk_size;
    o.n_index_workers = c.n_index_workers;
    o.n_search_workers = c.n_search_workers;
    o.n_queues = c.n_queues;
    o.queue_mode = c.queue_mode == QueueMode::single ? 0 : 1;
    o.initial_buffer_part_size = c.initial_buffer_part_size;
    return o;
}

tsg_ctx* default_context() {
    static std::once_flag once;
    static tsg_ctx* ctx = nullptr;
    static tsg_status status = TSG_OK;
    static std::string error;
    std::call_once(once, [] {
        status = tsg_open(1, nullptr, &ctx);
        if (status != TSG_OK) error = tsg_last_error();
    });
    if (status != TSG_OK) throw std::runtime_error("tsgpu: " + error);
    return ctx;
}

void check_measure(const Measure& m, std::size_t n) {
    if (m.kind == MeasureKind::dtw && (m.window < 0 || static_cast<std::size_t>(m.window) >= n))
        throw std::invalid_argument("dtw window must be in [0, n)");
}

tsg_measure measure_of(const Measure& m) {
    tsg_measure c{};
    c.kind = m.kind == MeasureKind::dtw ? TSG_MEASURE_DTW : TSG_MEASURE_ED;
    c.window = m.window;
    return c;
}

SearchStats stats_of(const tsg_search_stats& s) {
    SearchStats o;
    o.lb_node_calcs = s.lb_node_calcs;
    o.lb_entry_calcs = s.lb_entry_calcs;
    o.real_dist_calcs = s.real_dist_calcs;
    o.bsf_updates = s.bsf_updates;
    o.pruned_subtrees = s.pruned_subtrees;
    o.queue_insertions = s.queue_insertions;
    return o;
}

}  // namespace

unsigned IndexConfig::default_workers() {
    const unsigned hw = std::thread::hardware_concurrency();
    return hw == 0 ? 1 : hw;
}

unsigned IndexConfig::index_workers() const { return n_index_workers == 0 ? default_workers() : n_index_workers; }
unsigned IndexConfig::search_workers() const { return n_search_workers == 0 ? default_workers() : n_search_workers; }

void IndexConfig::validate() const {
    const tsg_config c = to_c(*this);
    throw_status(tsg_config_validate(&c));
}

Dataset generate_random_walk(std::size_t count, std::size_t length, std::uint64_t seed) {
    if (count == 0 || length == 0)
        throw std::invalid_argument("generate_random_walk: count and length must be positive");
    default_context();
    Dataset ds;
    ds.count = count;
    ds.length = length;
    ds.source_length = length;
    ds.values.resize(count * length);
    // Bit-identical to the reference generator; produced on the GPU in chunks.
    const std::size_t chunk = std::max<std::size_t>(1, (std::size_t{1} << 28) / (length * sizeof(float)));
    float* dev = nullptr;
    if (cudaMalloc(&dev, std::min(chunk, count) * length * sizeof(float)) != cudaSuccess)
        throw std::runtime_error("generate_random_walk: device allocation failed");
    try {
        for (std::size_t b = 0; b < count; b += chunk) {
            const std::size_t c = std::min(chunk, count - b);
            throw_status(tsg_generate_random_walk(dev, b, c, length, seed, 0, nullptr));
            if (cudaMemcpy(ds.values.data() + b * length, dev, c * length * sizeof(float), cudaMemcpyDeviceToHost) !=
                cudaSuccess)
                throw std::runtime_error("generate_random_walk: copy failed");
        }
    } catch (...) {
        cudaFree(dev);
        throw;
    }
    cudaFree(dev);
    return ds;
}

// ---- dataset utilities (input preparation, not the indexed path) ----------
// The arithmetic of znormalize must equal the reference's bit for bit
// (src/dataset.cpp:70-85): FP64 sums taken left to right, population standard
// deviation, untouched and false at std <= 1e-12. The file helpers keep the
// reference's checks and error messages (src/dataset.cpp:87-137), which are
// part of the drop-in contract.
namespace {

struct Moments {
    double mean;
    double stddev;
};

Moments moments_of(std::span<const float> x) {
    const double n = static_cast<double>(x.size());
    double acc = 0.0;
    for (std::size_t i = 0; i < x.size(); ++i) acc += x[i];
    const double mean = acc / n;
    double dev2 = 0.0;
    for (std::size_t i = 0; i < x.size(); ++i) {
        const double d = x[i] - mean;
        dev2 += d * d;
    }
    return {mean, std::sqrt(dev2 / n)};
}

std::uint64_t checked_file_series(const std::filesystem::path& path, std::size_t length) {
    std::error_code ec;
    const std::uint64_t size = std::filesystem::file_size(path, ec);
    if (ec) throw std::runtime_error("load_dataset: cannot stat " + path.string() + ": " + ec.message());
    const std::uint64_t row = length * sizeof(float);
    if (size == 0 || size % row != 0)
        throw std::runtime_error("load_dataset: " + path.string() + " holds " + std::to_string(size) +
                                 " bytes, not a positive multiple of " + std::to_string(row) + " (length " +
                                 std::to_string(length) + " * 4)");
    return size / row;
}

struct FileCloser {
    void operator()(std::FILE* f) const {
        if (f) std::fclose(f);
    }
};
using File = std::unique_ptr<std::FILE, FileCloser>;

}  // namespace

bool znormalize(std::span<float> series) {
    if (series.empty()) throw std::invalid_argument("znormalize: empty series");
    const Moments m = moments_of(series);
    if (m.stddev <= 1e-12) return false;
    std::transform(series.begin(), series.end(), series.begin(),
                   [&](float v) { return static_cast<float>((v - m.mean) / m.stddev); });
    return true;
}

Dataset load_dataset(const std::filesystem::path& path, std::size_t length) {
    if (length == 0) throw std::invalid_argument("load_dataset: length must be positive");
    const std::uint64_t rows = checked_file_series(path, length);
    Dataset ds;
    ds.count = rows;
    ds.length = ds.source_length = length;
    ds.values.resize(rows * length);
    File f(std::fopen(path.c_str(), "rb"));
    if (!f) throw std::runtime_error("load_dataset: cannot open " + path.string());
    if (std::fread(ds.values.data(), sizeof(float), ds.values.size(), f.get()) != ds.values.size())
        throw std::runtime_error("load_dataset: short read from " + path.string());
    return ds;
}

void save_dataset(const std::filesystem::path& path, const Dataset& dataset) {
    File f(std::fopen(path.c_str(), "wb"));
    if (!f) throw std::runtime_error("save_dataset: cannot open " + path.string());
    const std::size_t n = dataset.values.size();
    if (std::fwrite(dataset.values.data(), sizeof(float), n, f.get()) != n || std::fflush(f.get()) != 0)
        throw std::runtime_error("save_dataset: short write to " + path.string());
}

Dataset pad_to_segment_multiple(Dataset dataset, int w) {
    if (w < 1) throw std::invalid_argument("pad_to_segment_multiple: w must be at least 1");
    const std::size_t seg = static_cast<std::size_t>(w);
    const std::size_t target = (dataset.length + seg - 1) / seg * seg;  // next multiple of w
    if (target == dataset.length) return dataset;
    Dataset padded;
    padded.count = dataset.count;
    padded.length = target;
    padded.source_length = dataset.length;
    padded.values.assign(dataset.count * target, 0.f);
    // each row keeps its values and repeats its last one up to the new length
    for (std::size_t r = 0; r < dataset.count; ++r) {
        const float* from = dataset.values.data() + r * dataset.length;
        float* to = padded.values.data() + r * target;
        std::copy_n(from, dataset.length, to);
        std::fill(to + dataset.length, to + target, from[dataset.length - 1]);
    }
    return padded;
}

std::string BuildStats::kv_line() const {
    char buf[256];
    std::snprintf(buf, sizeof(buf),
                  "build series=%zu time_ns=%llu nodes=%zu inner=%zu leaves=%zu empty_leaves=%zu "
                  "overflow_leaves=%zu max_depth=%zu",
                  series, static_cast<unsigned long long>(build_ns), nodes, inner_nodes, leaves, empty_leaves,
                  overflow_leaves, max_depth);
    return buf;
}

SearchStats& SearchStats::operator+=(const SearchStats& o) {
    lb_node_calcs += o.lb_node_calcs;
    lb_entry_calcs += o.lb_entry_calcs;
    real_dist_calcs += o.real_dist_calcs;
    bsf_updates += o.bsf_updates;
    pruned_subtrees += o.pruned_subtrees;
    queue_insertions += o.queue_insertions;
    return *this;
}

std::string SearchStats::kv_line() const {
    char buf[256];
    std::snprintf(buf, sizeof(buf),
                  "lb_node=%llu lb_entry=%llu real_dist=%llu bsf_updates=%llu pruned_subtrees=%llu "
                  "queue_insertions=%llu",
                  static_cast<unsigned long long>(lb_node_calcs), static_cast<unsigned long long>(lb_entry_calcs),
                  static_cast<unsigned long long>(real_dist_calcs), static_cast<unsigned long long>(bsf_updates),
                  static_cast<unsigned long long>(pruned_subtrees), static_cast<unsigned long long>(queue_insertions));
    return buf;
}

Index::Index(Dataset dataset, IndexConfig config, tsg_index* handle, BuildStats stats)
    : data_(std::move(dataset)), config_(config), handle_(handle), stats_(stats) {}

Index::Index(Index&& o) noexcept
    : data_(std::move(o.data_)), config_(o.config_), handle_(o.handle_), stats_(o.stats_) {
    o.handle_ = nullptr;
}

Index& Index::operator=(Index&& o) noexcept {
    if (this != &o) {
        if (handle_) tsg_index_free(handle_);
        data_ = std::move(o.data_);
        config_ = o.config_;
        handle_ = o.handle_;
        stats_ = o.stats_;
        o.handle_ = nullptr;
    }
    return *this;
}

Index::~Index() {
    if (handle_) tsg_index_free(handle_);
}

Index build_index(Dataset dataset, IndexConfig config) {
    const tsg_config c = to_c(config);
    throw_status(tsg_config_validate(&c));
    if (dataset.count == 0) throw std::invalid_argument("build_index: empty dataset");
    tsg_index* h = nullptr;
    tsg_build_stats st{};
    throw_status(tsg_index_build(default_context(), dataset.values.data(), dataset.count, dataset.length, &c, 0, &h,
                                 &st));
    BuildStats bs;
    bs.build_ns = st.build_ns;
    bs.series = st.series;
    bs.nodes = st.nodes;
    bs.inner_nodes = st.inner_nodes;
    bs.leaves = st.leaves;
    bs.empty_leaves = st.empty_leaves;
    bs.overflow_leaves = st.overflow_leaves;
    bs.max_depth = st.max_depth;
    return Index(std::move(dataset), config, h, bs);
}

SearchResult exact_search(const Index& index, std::span<const float> query, Measure measure, SearchOptions) {
    check_measure(measure, index.config().n);
    if (query.size() != index.config().n)
        throw std::invalid_argument("query length " + std::to_string(query.size()) +
                                    " does not match the index series length " + std::to_string(index.config().n));
    tsg_result r{};
    const tsg_measure m = measure_of(measure);
    throw_status(tsg_search_measure(index.handle(), query.data(), 0, 1, &m, 0, &r));
    return {r.distance, r.position, stats_of(r.stats)};
}

std::vector<SearchResult> exact_search_batch(const Index& index, std::span<const float> queries, Measure measure) {
    check_measure(measure, index.config().n);
    const std::size_t n = index.config().n;
    if (queries.size() % n != 0)
        throw std::invalid_argument("exact_search_batch: queries are not a whole number of series of length " +
                                    std::to_string(n));
    const std::size_t nq = queries.size() / n;
    std::vector<tsg_result> raw(nq);
    const tsg_measure m = measure_of(measure);
    if (nq) throw_status(tsg_search_measure(index.handle(), queries.data(), 0, static_cast<uint32_t>(nq), &m, 0, raw.data()));
    std::vector<SearchResult> out;
    out.reserve(nq);
    for (const auto& r : raw) out.push_back({r.distance, r.position, stats_of(r.stats)});
    return out;
}

ApproxResult approximate_search(const Index& index, std::span<const float> query, Measure measure) {
    check_measure(measure, index.config().n);
    if (query.size() != index.config().n)
        throw std::invalid_argument("query length " + std::to_string(query.size()) +
                                    " does not match the index series length " + std::to_string(index.config().n));
    tsg_result r{};
    const tsg_measure m = measure_of(measure);
    throw_status(tsg_search_measure(index.handle(), query.data(), 0, 1, &m, 1, &r));
    return {r.distance, r.position};
}

ValidationReport validate_index(const Index& index) {
    tsg_validation_report r{};
    throw_status(tsg_index_validate(index.handle(), &r));
    ValidationReport out;
    out.nodes = r.nodes;
    out.inner_nodes = r.inner_nodes;
    out.leaves = r.leaves;
    out.empty_leaves = r.empty_leaves;
    out.overflow_leaves = r.overflow_leaves;
    out.max_depth = r.max_depth;
    out.total_entries = r.total_entries;
    for (int i = 0; i < 11; ++i) out.leaf_fill_histogram[i] = r.leaf_fill_histogram[i];
    out.violation_count = r.violation_count;
    for (uint32_t i = 0; i < r.n_violations; ++i) out.violations.emplace_back(r.violations[i]);
    return out;
}

std::string ValidationReport::summary() const {
    char buf[256];
    std::snprintf(buf, sizeof(buf),
                  "validate nodes=%zu inner=%zu leaves=%zu empty_leaves=%zu overflow_leaves=%zu max_depth=%zu "
                  "entries=%zu violations=%zu",
                  nodes, inner_nodes, leaves, empty_leaves, overflow_leaves, max_depth, total_entries,
                  violation_count);
    return buf;
}

}  // namespace tsidx
