// TEST INFRASTRUCTURE ONLY — never linked into the product path.
//
// extern "C" shims over the UNMODIFIED reference core (compiled from
// /root/reference/proj/core/src/*.cpp by oracle/Makefile with
// -Dtsidx=tsidx_ref, outputs under oracle/_ref/). Only tests/, bench.py's
// cpu_baseline / --impl reference legs and __graft_entry__.smoke() load the
// resulting library, and only as the checker or the timed CPU baseline.
//
// Each shim names the reference entry point it forwards to.

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <span>
#include <string>
#include <thread>
#include <vector>

#include "tsidx/breakpoints.hpp"
#include "tsidx/config.hpp"
#include "tsidx/dataset.hpp"
#include "tsidx/index.hpp"
#include "tsidx/metrics.hpp"
#include "tsidx/query.hpp"
#include "tsidx/sax.hpp"
#include "tsidx/scan.hpp"

namespace {
thread_local std::string g_err;

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::logic_error& e) {
        g_err = e.what();
        return 3;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 2;
    }
}

tsidx_ref::IndexConfig make_config(std::uint64_t n, int w, int bits, std::uint64_t leaf,
                                   std::uint64_t chunk, unsigned workers) {
    tsidx_ref::IndexConfig c;
    c.n = n;
    c.w = w;
    c.max_card_bits = bits;
    c.leaf_capacity = leaf;
    c.chunk_size = chunk;
    c.n_index_workers = workers;
    c.n_search_workers = workers;
    return c;
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

unsigned ref_hardware_concurrency() { return tsidx_ref::IndexConfig::default_workers(); }

// tsidx::generate_random_walk (src/dataset.cpp:41-68)
int ref_generate_random_walk(std::uint64_t count, std::uint64_t length, std::uint64_t seed,
                             float* out) {
    return guarded([&] {
        auto ds = tsidx_ref::generate_random_walk(count, length, seed);
        std::memcpy(out, ds.values.data(), ds.values.size() * sizeof(float));
    });
}

// tsidx::znormalize (src/dataset.cpp:70-85); returns 1 if normalized, 0 if degenerate.
int ref_znormalize(float* series, std::uint64_t n) {
    int ok = 0;
    int rc = guarded([&] { ok = tsidx_ref::znormalize({series, n}) ? 1 : 0; });
    return rc == 0 ? ok : -rc;
}

// The CLI's `generate --znorm` path (tools/main.cpp:125-146): degenerate
// series become all zeros. Parallel over series (per-series independent).
int ref_znormalize_rows(float* rows, std::uint64_t count, std::uint64_t n, unsigned threads,
                        std::uint64_t* degenerate) {
    return guarded([&] {
        if (threads == 0) threads = tsidx_ref::IndexConfig::default_workers();
        std::vector<std::uint64_t> deg(threads, 0);
        std::vector<std::thread> pool;
        for (unsigned t = 0; t < threads; ++t)
            pool.emplace_back([&, t] {
                std::uint64_t b = count * t / threads, e = count * (t + 1) / threads;
                for (std::uint64_t i = b; i < e; ++i) {
                    std::span<float> s{rows + i * n, n};
                    if (!tsidx_ref::znormalize(s)) {
                        std::fill(s.begin(), s.end(), 0.f);
                        deg[t] += 1;
                    }
                }
            });
        for (auto& th : pool) th.join();
        if (degenerate) {
            *degenerate = 0;
            for (auto d : deg) *degenerate += d;
        }
    });
}

// tsidx::breakpoints_for (src/breakpoints.cpp:112-114): card-1 thresholds.
int ref_breakpoints(unsigned cardinality, double* out) {
    return guarded([&] {
        auto thr = tsidx_ref::breakpoints_for(cardinality);
        std::copy(thr.begin(), thr.end(), out);
    });
}

double ref_inverse_normal_cdf(double p) { return tsidx_ref::inverse_normal_cdf(p); }
double ref_normal_cdf(double x) { return tsidx_ref::normal_cdf(x); }

// tsidx::paa_into (src/sax.cpp:10-25)
int ref_paa(const float* series, std::uint64_t n, int w, double* out) {
    return guarded([&] { tsidx_ref::paa_into({series, n}, w, {out, static_cast<std::size_t>(w)}); });
}

unsigned ref_symbol_for_value(double v, unsigned cardinality) {
    return tsidx_ref::symbol_for_value(v, cardinality);
}

// paa_into + symbols_from_paa per series, exactly the summarization hot loop
// (src/index.cpp:162-166). Parallel over series.
int ref_summarise(const float* rows, std::uint64_t count, std::uint64_t n, int w, int bits,
                  unsigned threads, std::uint8_t* words) {
    return guarded([&] {
        if (threads == 0) threads = tsidx_ref::IndexConfig::default_workers();
        threads = static_cast<unsigned>(std::min<std::uint64_t>(threads, std::max<std::uint64_t>(count, 1)));
        std::vector<std::thread> pool;
        std::vector<std::exception_ptr> errs(threads);
        for (unsigned t = 0; t < threads; ++t)
            pool.emplace_back([&, t] {
                try {
                    std::vector<double> means(static_cast<std::size_t>(w));
                    std::uint64_t b = count * t / threads, e = count * (t + 1) / threads;
                    for (std::uint64_t i = b; i < e; ++i) {
                        tsidx_ref::paa_into({rows + i * n, n}, w, means);
                        tsidx_ref::symbols_from_paa(
                            means, bits, {words + i * static_cast<std::uint64_t>(w), static_cast<std::size_t>(w)});
                    }
                } catch (...) {
                    errs[t] = std::current_exception();
                }
            });
        for (auto& th : pool) th.join();
        for (auto& e : errs)
            if (e) std::rethrow_exception(e);
    });
}

std::uint64_t ref_root_key(const std::uint8_t* symbols, int w) {
    return tsidx_ref::root_key_from_symbols({symbols, static_cast<std::size_t>(w)});
}

// tsidx::mindist_paa_isax (src/metrics.cpp:106-108)
int ref_mindist_paa_isax(const double* qpaa, const std::uint8_t* symbols,
                         const std::uint8_t* card_bits, int w, std::uint64_t n, double* out) {
    return guarded([&] {
        tsidx_ref::SaxWordView view{{symbols, static_cast<std::size_t>(w)},
                                    {card_bits, static_cast<std::size_t>(w)}};
        *out = tsidx_ref::mindist_paa_isax({qpaa, static_cast<std::size_t>(w)}, view, n);
    });
}

// tsidx::euclidean (src/metrics.cpp:95-104); cutoff < 0 means the plain kernel.
int ref_euclidean(const float* a, const float* b, std::uint64_t n, double cutoff, double* out) {
    return guarded([&] {
        *out = cutoff < 0 ? tsidx_ref::euclidean({a, n}, {b, n})
                          : tsidx_ref::euclidean({a, n}, {b, n}, cutoff);
    });
}

// tsidx::scan_nn (src/scan.cpp:31-60), Euclidean. The dataset is borrowed:
// it is copied into a Dataset because scan_nn takes one by reference.
struct RefData {
    tsidx_ref::Dataset ds;
};

void* ref_dataset_new(const float* rows, std::uint64_t count, std::uint64_t n) {
    auto* d = new RefData;
    d->ds.count = count;
    d->ds.length = n;
    d->ds.source_length = n;
    d->ds.values.assign(rows, rows + count * n);
    return d;
}

void ref_dataset_free(void* d) { delete static_cast<RefData*>(d); }

int ref_scan_nn(void* data, const float* query, unsigned threads, double* dist,
                std::uint32_t* pos) {
    return guarded([&] {
        auto& ds = static_cast<RefData*>(data)->ds;
        auto r = tsidx_ref::scan_nn(ds, {query, ds.length}, tsidx_ref::Measure::ed(), threads);
        *dist = r.distance;
        *pos = r.position;
    });
}

// tsidx::build_index (src/index.cpp:258-318) over a copy of the rows.
struct RefIndex {
    std::unique_ptr<tsidx_ref::Index> index;
};

int ref_build_index(const float* rows, std::uint64_t count, std::uint64_t n, int w, int bits,
                    std::uint64_t leaf_capacity, std::uint64_t chunk, unsigned workers,
                    void** out, std::uint64_t* stats /* 8 fields, BuildStats order */) {
    return guarded([&] {
        tsidx_ref::Dataset ds;
        ds.count = count;
        ds.length = n;
        ds.source_length = n;
        if (count) ds.values.assign(rows, rows + count * n);
        auto cfg = make_config(n, w, bits, leaf_capacity, chunk, workers);
        auto idx = std::make_unique<tsidx_ref::Index>(tsidx_ref::build_index(std::move(ds), cfg));
        const auto& s = idx->build_stats();
        if (stats) {
            stats[0] = s.build_ns;
            stats[1] = s.series;
            stats[2] = s.nodes;
            stats[3] = s.inner_nodes;
            stats[4] = s.leaves;
            stats[5] = s.empty_leaves;
            stats[6] = s.overflow_leaves;
            stats[7] = s.max_depth;
        }
        auto* h = new RefIndex;
        h->index = std::move(idx);
        *out = h;
    });
}

void ref_index_free(void* h) { delete static_cast<RefIndex*>(h); }

// The CLI's `generate --znorm` followed by build_index, without any host
// copy of the rows (a 100M x 256 dataset is 102 GB): generate_random_walk
// (src/dataset.cpp:41-68) + per-series znormalize (degenerate -> zeros,
// tools/main.cpp:128-139) + build_index(std::move(ds)). gen_ns / build_ns
// report the two phases separately.
int ref_build_generated(std::uint64_t count, std::uint64_t n, std::uint64_t seed, int znorm, int w,
                        int bits, std::uint64_t leaf_capacity, std::uint64_t chunk, unsigned workers,
                        void** out, std::uint64_t* stats, std::uint64_t* gen_ns) {
    return guarded([&] {
        auto t0 = std::chrono::steady_clock::now();
        tsidx_ref::Dataset ds = tsidx_ref::generate_random_walk(count, n, seed);
        if (znorm) {
            unsigned threads = workers ? workers : tsidx_ref::IndexConfig::default_workers();
            std::vector<std::thread> pool;
            for (unsigned t = 0; t < threads; ++t)
                pool.emplace_back([&, t] {
                    std::uint64_t b = count * t / threads, e = count * (t + 1) / threads;
                    for (std::uint64_t i = b; i < e; ++i) {
                        auto s = ds.series_mut(i);
                        if (!tsidx_ref::znormalize(s)) std::fill(s.begin(), s.end(), 0.f);
                    }
                });
            for (auto& th : pool) th.join();
        }
        auto t1 = std::chrono::steady_clock::now();
        if (gen_ns)
            *gen_ns = static_cast<std::uint64_t>(
                std::chrono::duration_cast<std::chrono::nanoseconds>(t1 - t0).count());
        auto cfg = make_config(n, w, bits, leaf_capacity, chunk, workers);
        auto idx = std::make_unique<tsidx_ref::Index>(tsidx_ref::build_index(std::move(ds), cfg));
        const auto& s = idx->build_stats();
        if (stats) {
            stats[0] = s.build_ns;
            stats[1] = s.series;
            stats[2] = s.nodes;
            stats[3] = s.inner_nodes;
            stats[4] = s.leaves;
            stats[5] = s.empty_leaves;
            stats[6] = s.overflow_leaves;
            stats[7] = s.max_depth;
        }
        auto* h = new RefIndex;
        h->index = std::move(idx);
        *out = h;
    });
}

// Rows [begin, begin+count) of generate_random_walk(., n, seed) +
// z-normalisation, for queries (the generator seeds per series, so a window
// is generated directly; identical to the corresponding full-call rows).
int ref_series_window(std::uint64_t begin, std::uint64_t count, std::uint64_t n, std::uint64_t seed,
                      int znorm, float* out) {
    return guarded([&] {
        auto ds = tsidx_ref::generate_random_walk(begin + count, n, seed);
        for (std::uint64_t i = 0; i < count; ++i) {
            auto s = ds.series_mut(begin + i);
            if (znorm && !tsidx_ref::znormalize(s)) std::fill(s.begin(), s.end(), 0.f);
            std::copy(s.begin(), s.end(), out + i * n);
        }
    });
}

// tsidx::exact_search (src/query.cpp:258-298), ED. mode: 0 single, 1 multi.
int ref_exact_search(void* h, const float* query, unsigned workers, unsigned queues, int mode,
                     double* dist, std::uint32_t* pos, std::uint64_t* stats /* 6 */,
                     std::uint64_t* time_ns) {
    return guarded([&] {
        auto& idx = *static_cast<RefIndex*>(h)->index;
        tsidx_ref::SearchOptions opt;
        opt.workers = workers;
        opt.queues = queues;
        if (mode >= 0) opt.mode = mode == 0 ? tsidx_ref::QueueMode::single : tsidx_ref::QueueMode::multi;
        auto t0 = std::chrono::steady_clock::now();
        auto r = tsidx_ref::exact_search(idx, {query, idx.config().n}, tsidx_ref::Measure::ed(), opt);
        auto t1 = std::chrono::steady_clock::now();
        if (time_ns)
            *time_ns = static_cast<std::uint64_t>(
                std::chrono::duration_cast<std::chrono::nanoseconds>(t1 - t0).count());
        *dist = r.distance;
        *pos = r.position;
        if (stats) {
            stats[0] = r.stats.lb_node_calcs;
            stats[1] = r.stats.lb_entry_calcs;
            stats[2] = r.stats.real_dist_calcs;
            stats[3] = r.stats.bsf_updates;
            stats[4] = r.stats.pruned_subtrees;
            stats[5] = r.stats.queue_insertions;
        }
    });
}

// tsidx::approximate_search (src/query.cpp:250-256)
int ref_approximate_search(void* h, const float* query, double* dist, std::uint32_t* pos) {
    return guarded([&] {
        auto& idx = *static_cast<RefIndex*>(h)->index;
        auto r = tsidx_ref::approximate_search(idx, {query, idx.config().n});
        *dist = r.distance;
        *pos = r.position;
    });
}


// ---- DTW: dtw, keogh_envelope, lb_keogh, mindist_envelope_isax
// (src/metrics.cpp:112-202) and the DTW forms of scan_nn / exact_search.
int ref_dtw(const float* a, const float* b, std::uint64_t n, int window, double cutoff, double* out) {
    return guarded([&] {
        *out = cutoff < 0 ? tsidx_ref::dtw({a, n}, {b, n}, window) : tsidx_ref::dtw({a, n}, {b, n}, window, cutoff);
    });
}

int ref_keogh_envelope(const float* q, std::uint64_t n, int window, int w, float* upper, float* lower,
                       double* upper_paa, double* lower_paa) {
    return guarded([&] {
        auto env = tsidx_ref::keogh_envelope({q, n}, window, w);
        std::copy(env.upper.begin(), env.upper.end(), upper);
        std::copy(env.lower.begin(), env.lower.end(), lower);
        std::copy(env.upper_paa.begin(), env.upper_paa.end(), upper_paa);
        std::copy(env.lower_paa.begin(), env.lower_paa.end(), lower_paa);
    });
}

int ref_lb_keogh(const float* q, std::uint64_t n, int window, int w, const float* candidate, double* out) {
    return guarded([&] {
        auto env = tsidx_ref::keogh_envelope({q, n}, window, w);
        *out = tsidx_ref::lb_keogh(env, {candidate, n});
    });
}

int ref_mindist_envelope_isax(const float* q, std::uint64_t n, int window, int w, const std::uint8_t* symbols,
                              int bits, double* out) {
    return guarded([&] {
        auto env = tsidx_ref::keogh_envelope({q, n}, window, w);
        std::vector<std::uint8_t> cb(static_cast<std::size_t>(w), static_cast<std::uint8_t>(bits));
        tsidx_ref::SaxWordView view{{symbols, static_cast<std::size_t>(w)}, cb};
        *out = tsidx_ref::mindist_envelope_isax(env, view, n);
    });
}

int ref_scan_nn_dtw(void* data, const float* query, int window, unsigned threads, double* dist,
                    std::uint32_t* pos) {
    return guarded([&] {
        auto& ds = static_cast<RefData*>(data)->ds;
        auto r = tsidx_ref::scan_nn(ds, {query, ds.length}, tsidx_ref::Measure::dtw(window), threads);
        *dist = r.distance;
        *pos = r.position;
    });
}

int ref_exact_search_dtw(void* h, const float* query, int window, double* dist, std::uint32_t* pos) {
    return guarded([&] {
        auto& idx = *static_cast<RefIndex*>(h)->index;
        auto r = tsidx_ref::exact_search(idx, {query, idx.config().n}, tsidx_ref::Measure::dtw(window), {});
        *dist = r.distance;
        *pos = r.position;
    });
}

}  // extern "C"
