// C++ API test: the reference's own call pattern (tools/main.cpp:169-213,
// tests/test_query.cpp) against include/tsidx/tsidx.hpp + libtsgpu.so.
// Exhaustive scan below is test infrastructure (the checker), written here
// from the reference's definition (src/metrics.cpp:17-40, src/scan.cpp:54-59).
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <filesystem>
#include <limits>
#include <stdexcept>
#include <string>

#include "tsidx/tsidx.hpp"

namespace {

int failures = 0;

#define CHECK(cond)                                                              \
    do {                                                                         \
        if (!(cond)) {                                                           \
            std::fprintf(stderr, "CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #cond); \
            ++failures;                                                          \
        }                                                                        \
    } while (0)

template <typename E, typename F>
bool throws(F&& f) {
    try {
        f();
    } catch (const E&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

double blocked_sq(std::span<const float> a, std::span<const float> b) {
    double sum = 0.0;
    for (std::size_t i = 0; i < a.size(); i += 8) {
        double blk = 0.0;
        for (std::size_t j = i; j < std::min(i + 8, a.size()); ++j) {
            const double d = static_cast<double>(a[j]) - static_cast<double>(b[j]);
            blk += d * d;
        }
        sum += blk;
    }
    return sum;
}

std::pair<double, std::uint32_t> scan(const tsidx::Dataset& ds, std::span<const float> q) {
    double best = std::numeric_limits<double>::infinity();
    std::uint32_t pos = 0;
    for (std::size_t i = 0; i < ds.count; ++i) {
        const double d = std::sqrt(blocked_sq(ds.series(i), q));
        if (d < best) {
            best = d;
            pos = static_cast<std::uint32_t>(i);
        }
    }
    return {best, pos};
}

}  // namespace

int main() {
    using namespace tsidx;
    // generate --znorm (tools/main.cpp:125-146)
    Dataset data = generate_random_walk(20000, 256, 1);
    for (std::size_t i = 0; i < data.count; ++i) {
        auto s = data.series_mut(i);
        if (!znormalize(s)) std::fill(s.begin(), s.end(), 0.f);
    }
    Dataset queries = generate_random_walk(10, 256, 2);
    for (std::size_t i = 0; i < queries.count; ++i) znormalize(queries.series_mut(i));

    IndexConfig cfg;  // defaults: n=256, w=16, 8 bits, leaf 2000
    Index index = build_index(Dataset(data), cfg);
    const BuildStats& bs = index.build_stats();
    CHECK(bs.series == 20000);
    CHECK(bs.leaves >= 1 && bs.nodes >= bs.leaves);
    std::printf("%s\n", bs.kv_line().c_str());
    // validate_index (tools/main.cpp:305-316): the audit passes and agrees with the build
    const ValidationReport vr = validate_index(index);
    std::printf("%s\n", vr.summary().c_str());
    CHECK(vr.ok());
    CHECK(vr.total_entries == 20000 && vr.leaves == bs.leaves && vr.nodes == bs.nodes);

    for (std::size_t k = 0; k < queries.count; ++k) {
        const auto q = queries.series(k);
        const auto want = scan(data, q);
        const SearchResult got = exact_search(index, q, Measure::ed(), {});
        CHECK(got.position == want.second);
        CHECK(got.distance == want.first);
        CHECK(got.stats.real_dist_calcs >= 1);
        const ApproxResult ap = approximate_search(index, q);
        CHECK(ap.distance >= got.distance);
    }
    const auto batch = exact_search_batch(index, {queries.values.data(), queries.values.size()});
    CHECK(batch.size() == queries.count);
    for (std::size_t k = 0; k < batch.size(); ++k) CHECK(batch[k].position == scan(data, queries.series(k)).second);

    // members come back at distance zero at their own position (tests/test_query.cpp:190-198)
    for (std::uint32_t m : {17u, 655u, 19999u}) {
        const SearchResult r = exact_search(index, index.series(m));
        CHECK(r.distance == 0.0 && r.position == m);
    }

    // error contracts (tests/test_index.cpp:388-399, tests/test_query.cpp:231-238)
    IndexConfig bad = cfg;
    bad.w = 0;
    CHECK(throws<std::invalid_argument>([&] { bad.validate(); }));
    CHECK(throws<std::invalid_argument>([&] { build_index(Dataset{}, cfg); }));
    std::vector<float> wrong(255, 0.f);
    CHECK(throws<std::invalid_argument>([&] { exact_search(index, wrong); }));
    std::vector<float> zq(256, 0.f);
    CHECK(throws<std::invalid_argument>([&] { exact_search(index, zq, Measure::dtw(300)); }));
    // DTW: the banded DTW distance never exceeds the Euclidean one
    // (the diagonal is a warping path); window 0 is the sequentially summed ED.
    for (std::size_t k = 0; k < 3; ++k) {
        const auto q = queries.series(k);
        const SearchResult ed = exact_search(index, q);
        const SearchResult d10 = exact_search(index, q, Measure::dtw(10));
        const SearchResult d0 = exact_search(index, q, Measure::dtw(0));
        CHECK(d10.distance <= ed.distance * (1 + 1e-12));
        CHECK(std::abs(d0.distance - ed.distance) <= 1e-9 * ed.distance);
    }

    // dataset file round trip + padding (src/dataset.cpp:87-137)
    const auto path = std::filesystem::temp_directory_path() / "tsidx_b200_roundtrip.f32";
    save_dataset(path, queries);
    const Dataset back = load_dataset(path, 256);
    CHECK(back.count == queries.count && back.values == queries.values);
    std::filesystem::remove(path);
    const Dataset padded = pad_to_segment_multiple(generate_random_walk(3, 30, 9), 8);
    CHECK(padded.length == 32 && padded.source_length == 30);

    std::printf("%s: %d failures\n", failures ? "FAIL" : "OK", failures);
    return failures ? 1 : 0;
}
