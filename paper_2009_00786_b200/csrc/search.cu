// Exact Euclidean 1-NN over the flat SoA index (one device shard).
//
// Replaces exact_search (src/query.cpp:258-298) and its pieces. Per query,
// six kernels on the index's stream:
//   seed      approximate_search_state (src/query.cpp:226-238): the leaf the
//             query's own iSAX word descends to (binary search of its
//             plane-major key over the page keys) is refined exhaustively
//             and seeds the best-so-far (BSF).
//   bound     node_lower_bound over every page box (src/query.cpp:102-107)
//             + the pruning test (src/query.cpp:159): pages whose bound is
//             within the BSF survive (block-aggregated compaction).
//   lbscan    the entry-level filter of calculate_real_distance_leaf
//             (src/query.cpp:129-134): words of surviving pages are bounded
//             with one table lookup per segment and compacted with warp
//             ballot + prefix popcount into two LB-ordered candidate waves.
//   refine x2 euclidean (src/metrics.cpp:17-40, 95-104), wave 0 (bounds up
//             to `split` x the scan bound) then wave 1, the GPU analog of
//             MESSI's LB-ordered priority queues (src/query.cpp:173-184): an
//             8-lane group per candidate row, 256-bit loads of 8-float
//             blocks, FP64 block sums without FMA, added left to right
//             exactly like squared_l2; the BSF is an atomicMin on the double
//             bit pattern (non-negative doubles order as unsigned integers),
//             the SharedBsf analog (src/query.cpp:35-42); a candidate whose
//             bound exceeds the live BSF is skipped (`LB >= cutoff -> skip`).
//   finalize  result = min over refined candidates of (sqrt(sum), position):
//             ties resolve to the lowest position exactly as scan_nn does
//             (src/scan.cpp:54-59); the last block writes the result and
//             resets the scratch for the next query.
// Every kernel computes the query PAA in FP64 reference order, the query
// symbols and, where needed, a [w][256] table of per-segment squared region
// gaps (mindist_bands, src/metrics.cpp:47-70) scaled by n/w and rounded DOWN
// to float, so every float bound here is <= the exact FP64 bound. Pruning
// keeps ties: an entry is dropped only when its bound is strictly above the
// BSF widened by 1e-9 relative (covering FP64 rounding of the sums).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <utility>
#include <vector>

#include "common.cuh"
#include "kernels.cuh"

namespace tsg {

namespace {

constexpr unsigned long long kInfBits = 0x7FF0000000000000ull;
constexpr double kSlack = 1.0 + 1e-9;
constexpr int kThreads = 256;
constexpr int kRowLanes = 8;  // lanes per candidate row in the refine kernels

enum Stat { kLbNode = 0, kLbEntry, kRealDist, kBsfUpd, kPruned, kQueueIns };

__device__ __forceinline__ double bsf_of(unsigned long long bits) {
    return __longlong_as_double(static_cast<long long>(bits));
}

__device__ __forceinline__ float bound_from_bits(unsigned long long bits) {
    return __double2float_ru(bsf_of(bits) * kSlack);
}

__device__ __forceinline__ uint32_t word32(const uint4& v, int i) {
    return i == 0 ? v.x : i == 1 ? v.y : i == 2 ? v.z : v.w;
}

__device__ __forceinline__ uint32_t byte_of(const uint4& v, int s) { return (word32(v, s >> 2) >> (8 * (s & 3))) & 255u; }

struct QueryShared {
    double thr[kThrPad];
    double qpaa[kMaxW];
    unsigned char qsym[kMaxW];
};

// The [w][256] table: per segment s and symbol byte v, the squared gap
// between the query's PAA mean and v's region, times n/w, rounded down.
__device__ __forceinline__ void fill_lut(const QueryShared& qs, int n, int w, int bits, float* out) {
    const unsigned card = 1u << bits;
    const double scale = static_cast<double>(n) / static_cast<double>(w);
    for (int idx = threadIdx.x; idx < w * 256; idx += blockDim.x) {
        const int s = idx >> 8, v = idx & 255;
        const unsigned prefix = static_cast<unsigned>(v) >> (8 - bits);
        const double lo = prefix == 0 ? -INFINITY : qs.thr[prefix - 1];
        const double hi = prefix == card - 1 ? INFINITY : qs.thr[prefix];
        const double x = qs.qpaa[s];
        double gap = 0.0;
        if (x < lo) gap = lo - x;
        else if (x > hi) gap = x - hi;
        out[idx] = __double2float_rd(__dmul_rn(__dmul_rn(gap, gap), scale));
    }
}

// Block-local query preparation: PAA (FP64, reference order) and symbols;
// with lut != nullptr also the [w][256] squared-gap table.
__device__ void prepare_query(const float* __restrict__ q, int n, int w, int bits, const double* __restrict__ thr_g,
                              QueryShared& qs, float* s_lut) {
    for (int i = threadIdx.x; i < kThrPad; i += blockDim.x) qs.thr[i] = thr_g[i];
    __syncthreads();
    const int seg = n / w;
    if (threadIdx.x < w) {
        const int g = threadIdx.x;
        double sum = 0.0;
        for (int j = 0; j < seg; ++j) sum = __dadd_rn(sum, static_cast<double>(q[g * seg + j]));
        const double mean = __ddiv_rn(sum, static_cast<double>(seg));
        qs.qpaa[g] = mean;
        qs.qsym[g] = static_cast<unsigned char>(symbol_of(qs.thr, bits, mean) << (8 - bits));
    }
    __syncthreads();
    if (!s_lut) return;
    fill_lut(qs, n, w, bits, s_lut);
    __syncthreads();
}

// Loads the table and the query symbols the seed kernel prepared for this
// query (one 16 KB L2 read per block instead of recomputing 4K FP64 gaps).
__device__ __forceinline__ void load_prepared(const float* __restrict__ lut_g, const QueryWork* wk, int w,
                                              float* s_lut, unsigned char* qsym) {
    const float4* src = reinterpret_cast<const float4*>(lut_g);
    float4* dst = reinterpret_cast<float4*>(s_lut);
    for (int i = threadIdx.x; i < w * 64; i += blockDim.x) dst[i] = src[i];
    for (int i = threadIdx.x; i < kMaxW; i += blockDim.x) qsym[i] = i < w ? wk->qsym[i] : 0;
    __syncthreads();
}

// Bound of one word: sum over segments of the table entry of its symbol.
// W16: compile-time w = 16 (fully unrolled); otherwise runtime w.
template <bool W16>
__device__ __forceinline__ float word_bound(const float* s_lut, const uint4* v, int w) {
    float lb = 0.f;
    if (W16) {
#pragma unroll
        for (int s = 0; s < 16; ++s) lb = __fadd_rd(lb, s_lut[s * 256 + byte_of(v[0], s)]);
    } else {
        for (int s = 0; s < w; ++s) lb = __fadd_rd(lb, s_lut[s * 256 + byte_of(v[s >> 4], s & 15)]);
    }
    return lb;
}

__device__ __forceinline__ void reset_work(QueryWork* wk) {
    wk->bsf_bits = kInfBits;
    wk->seed_key = ~0ull;
    wk->ncand = 0;
    wk->nseed = 0;
    wk->nhigh = 0;
    wk->work_next = 0;
    wk->best_pos = 0xFFFFFFFFu;
    wk->nsurv = 0;
    wk->nsurv_hi = 0;
    wk->ngroups = 0;
    for (int i = 0; i < 6; ++i) wk->stats[i] = 0;
}

__global__ void k_reset(QueryWork* wk) {
    reset_work(wk);
    wk->done_blocks = 0;
}

// ---------------------------------------------------- row refinement
struct F8 {
    float v[8];
};

__device__ __forceinline__ F8 ld256(const float* p) {
    F8 r;
    asm volatile("ld.global.nc.L1::no_allocate.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(r.v[0]), "=f"(r.v[1]), "=f"(r.v[2]), "=f"(r.v[3]), "=f"(r.v[4]), "=f"(r.v[5]),
                   "=f"(r.v[6]), "=f"(r.v[7])
                 : "l"(p));
    return r;
}

__device__ __forceinline__ double block_sq(const float* x, const float* q, int cnt) {
    double blk = 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k)
        if (k < cnt) {
            const double d = __dsub_rn(static_cast<double>(x[k]), static_cast<double>(q[k]));
            blk = __dadd_rn(blk, __dmul_rn(d, d));
        }
    return blk;
}

// Squared distance of a row computed by an 8-lane group: lane j owns blocks
// j, j+8, j+16, j+24 of each 32-block round (the 8 lanes read 256 contiguous
// bytes per load); the group leader then adds the block sums left to right,
// squared_l2's order. Rows longer than 256 take several rounds; after each
// round the running sum is checked against the live BSF (strict), the
// reference's abandonment (metrics.cpp:28). Group-local: only the group's 8
// lanes take part (shuffles use the group mask), so groups of a warp work on
// different candidates independently. Every lane of the group returns the
// sum, +inf if abandoned.
template <bool VEC>
__device__ __forceinline__ double group_row_sq(const float* __restrict__ row, const float* __restrict__ s_q, int n,
                                               const unsigned long long* bsf) {
    const int lane = threadIdx.x & 31, j = lane & (kRowLanes - 1), base = lane & ~(kRowLanes - 1);
    const unsigned gmask = 0xFFu << base;
    const int nb = (n + 7) >> 3;
    double sum = 0.0;
    for (int r0 = 0; r0 < nb; r0 += 32) {
        double blk[4] = {0.0, 0.0, 0.0, 0.0};
        if (VEC) {
            F8 x[4];
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                const int b = r0 + j + kRowLanes * t;
                if (b < nb) x[t] = ld256(row + 8 * b);
            }
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                const int b = r0 + j + kRowLanes * t;
                if (b < nb) blk[t] = block_sq(x[t].v, s_q + 8 * b, 8);
            }
        } else {
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                const int b = r0 + j + kRowLanes * t;
                if (b < nb) {
                    const int cnt = min(8, n - 8 * b);
                    float x[8];
#pragma unroll
                    for (int k = 0; k < 8; ++k) x[k] = k < cnt ? row[8 * b + k] : 0.f;
                    blk[t] = block_sq(x, s_q + 8 * b, cnt);
                }
            }
        }
        // Left-to-right over the round's blocks: block r0 + 8t + i lives in
        // lane base+i, slot t.
#pragma unroll
        for (int t = 0; t < 4; ++t)
#pragma unroll
            for (int i = 0; i < kRowLanes; ++i) {
                const double v = __shfl_sync(gmask, blk[t], base + i);
                if (r0 + kRowLanes * t + i < nb) sum = __dadd_rn(sum, v);
            }
        if (r0 + 32 < nb && bsf && sum > bsf_of(ld_volatile_u64(bsf)) * kSlack) return INFINITY;
    }
    return sum;
}

// Publishes a finished sum: candidate record, BSF atomicMin only when it can
// improve, strict-improvement count. *seen receives the BSF observed (an
// upper bound of the current BSF, for the caller's cached pruning bound).
__device__ __forceinline__ unsigned long long publish(QueryWork* wk, double s, uint64_t c, double* cand_sq,
                                                      unsigned long long* seen = nullptr) {
    cand_sq[c] = s;
    const unsigned long long cur = ld_volatile_u64(&wk->bsf_bits);
    if (seen) *seen = cur;
    if (!(s < INFINITY)) return 0;
    const unsigned long long sb = static_cast<unsigned long long>(__double_as_longlong(s));
    if (sb >= cur) return 0;
    if (seen) *seen = sb;
    return atomicMin(&wk->bsf_bits, sb) > sb ? 1 : 0;
}

__device__ __forceinline__ void load_query(float* s_q, const float* q, int n) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) s_q[i] = q[i];
    __syncthreads();
}

// The page the query's own key falls into: the largest p with
// page_key[p] <= key (0 if none), i.e. where the query's iSAX word would be
// stored. Two parallel rounds instead of a serial binary search: the block
// counts the directory entries (every 256th page key) <= key, then counts
// the keys <= key inside that 256-page window. blockDim.x must be 256.
__device__ __forceinline__ uint32_t locate_page(const uint64_t* __restrict__ page_key,
                                                const uint64_t* __restrict__ page_dir, uint64_t P, uint64_t key) {
    __shared__ unsigned s_part[kThreads / 32];
    const uint64_t nd = (P + 255) / 256;
    unsigned c = 0;
    for (uint64_t i = threadIdx.x; i < nd; i += blockDim.x) c += page_dir[i] <= key ? 1u : 0u;
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xFFFFFFFFu, c, o);
    if ((threadIdx.x & 31) == 0) s_part[threadIdx.x >> 5] = c;
    __syncthreads();
    unsigned dirs = 0;
    for (int i = 0; i < kThreads / 32; ++i) dirs += s_part[i];
    const uint64_t w0 = dirs == 0 ? 0 : static_cast<uint64_t>(dirs - 1) * 256;
    const uint64_t p = w0 + threadIdx.x;
    const int cnt = __syncthreads_count(p < P && page_key[p] <= key);
    return static_cast<uint32_t>(cnt == 0 ? 0 : w0 + cnt - 1);
}

// Plane-major 64-bit key of the query word (same layout as the index keys).
__device__ __forceinline__ uint64_t query_key(const unsigned char* qsym, int w) {
    uint64_t k = 0;
    int left = 64;
    for (int p = 0; p < 8 && left > 0; ++p)
        for (int g = 0; g < w && left > 0; ++g, --left) k = (k << 1) | ((qsym[g] >> (7 - p)) & 1u);
    return left >= 64 ? 0 : k << left;
}

// -------------------------------------------------------------- seed
// The leaf the query's own iSAX word descends to; an overflow leaf larger
// than seed_cap is replaced by that page alone. Every entry is refined.
template <bool VEC>
__global__ void __launch_bounds__(kThreads)
    k_seed(const float* __restrict__ rows, int n, int w, int bits, const double* __restrict__ thr_g,
           const float* __restrict__ query, const uint32_t* __restrict__ leaf_off,
           const uint32_t* __restrict__ page_off, const uint32_t* __restrict__ page_leaf,
           const uint64_t* __restrict__ page_key, const uint64_t* __restrict__ page_dir, uint64_t P,
           const uint32_t* __restrict__ pos, uint32_t seed_cap, QueryWork* wk, uint32_t* __restrict__ cand_pos,
           double* __restrict__ cand_sq, float* __restrict__ lut_out) {
    extern __shared__ float s_q[];
    __shared__ QueryShared qs;
    __shared__ uint32_t s_range[2];
    load_query(s_q, query, n);
    prepare_query(s_q, n, w, bits, thr_g, qs, nullptr);
    if (blockIdx.x == gridDim.x - 1) {  // one block publishes the query's table and symbols
        fill_lut(qs, n, w, bits, lut_out);
        if (threadIdx.x < w) wk->qsym[threadIdx.x] = qs.qsym[threadIdx.x];
    }
    const uint32_t page = locate_page(page_key, page_dir, P, query_key(qs.qsym, w));
    if (threadIdx.x == 0) {
        const uint32_t leaf = page_leaf[page];
        uint32_t a = leaf_off[leaf], b = leaf_off[leaf + 1];
        if (b - a > seed_cap) {
            a = page_off[page];
            b = page_off[page + 1];
        }
        s_range[0] = a;
        s_range[1] = b;
        if (blockIdx.x == 0) {
            wk->seed_key = page;
            wk->nseed = b - a;
            wk->ncand = b - a;
            wk->seed_begin = a;
            wk->seed_end = b;
            wk->stats[kRealDist] += b - a;
        }
    }
    __syncthreads();
    const uint32_t a = s_range[0], b = s_range[1];
    const int lane = threadIdx.x & 31;
    const uint64_t group = (blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x) / kRowLanes;
    const uint64_t ngroups = static_cast<uint64_t>(gridDim.x) * blockDim.x / kRowLanes;
    unsigned long long updates = 0;
    for (uint64_t e = a + group; e < b; e += ngroups) {  // groups run independently
        const uint32_t p = pos[e];
        const double s = group_row_sq<VEC>(rows + static_cast<uint64_t>(p) * n, s_q, n, &wk->bsf_bits);
        if ((lane & (kRowLanes - 1)) == 0) {
            cand_pos[e - a] = static_cast<uint32_t>(e);  // index-order entry (finalize maps via pos[])
            updates += publish(wk, s, e - a, cand_sq);
        }
    }
    if (updates) atomicAdd(&wk->stats[kBsfUpd], updates);
}

// ------------------------------------------------------- bound + filter
// Box bound: per segment the table entry of the query symbol clamped into the
// box [lo, hi] (0 when the query symbol is inside) — node_lower_bound's
// region gap (src/query.cpp:102-107) over a box of iSAX words.
template <int H, bool W16>
__device__ __forceinline__ float box_bound(const float* s_lut, const uint4* q4, const uint4* lo, const uint4* hi, int w) {
    uint4 c[H];
#pragma unroll
    for (int h = 0; h < H; ++h)
        c[h] = make_uint4(__vminu4(__vmaxu4(q4[h].x, lo[h].x), hi[h].x), __vminu4(__vmaxu4(q4[h].y, lo[h].y), hi[h].y),
                          __vminu4(__vmaxu4(q4[h].z, lo[h].z), hi[h].z), __vminu4(__vmaxu4(q4[h].w, lo[h].w), hi[h].w));
    return word_bound<W16>(s_lut, c, w);
}

// Block-wide slot reservation: each thread brings two counts (< 2^16 per
// block); returns its first slot in each of two global lists, with one
// atomicAdd per list per block. All threads of the block must call it.
__device__ __forceinline__ uint2 block_reserve(unsigned c0, unsigned c1, unsigned* ctr0, unsigned* ctr1) {
    __shared__ uint32_t s_cnt[kThreads / 32];
    __shared__ uint32_t s_base[2];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t mine = c0 | (c1 << 16);
    uint32_t incl = mine;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if (lane >= o) incl += t;
    }
    if (lane == 31) s_cnt[warp] = incl;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t tot = 0;
        for (int i = 0; i < kThreads / 32; ++i) {
            const uint32_t c = s_cnt[i];
            s_cnt[i] = tot;
            tot += c;
        }
        s_base[0] = (tot & 0xFFFFu) ? atomicAdd(ctr0, tot & 0xFFFFu) : 0u;
        s_base[1] = (tot >> 16) && ctr1 ? atomicAdd(ctr1, tot >> 16) : 0u;
    }
    __syncthreads();
    const uint32_t before = s_cnt[warp] + (incl - mine);
    const uint2 r = make_uint2(s_base[0] + (before & 0xFFFFu), s_base[1] + (before >> 16));
    __syncthreads();  // s_cnt / s_base are reused by the next call
    return r;
}

// Level 1, the flat analog of the tree's internal nodes: one box per group
// of kGroup consecutive pages. Surviving groups are listed (block-aggregated)
// for the page level, which then runs balanced over them.
constexpr int kGP = 4;  // groups / pages per thread per round

template <int WS, bool W16>
__global__ void __launch_bounds__(kThreads)
    k_groups(const float* __restrict__ lut_g, int w, const uint8_t* __restrict__ glo, const uint8_t* __restrict__ ghi,
             uint64_t NG, QueryWork* wk, uint32_t* __restrict__ gsurv) {
    constexpr int H = WS / 16;
    extern __shared__ float s_lut[];
    __shared__ __align__(16) unsigned char qsym[kMaxW];
    load_prepared(lut_g, wk, w, s_lut, qsym);
    uint4 q4[H];
#pragma unroll
    for (int h = 0; h < H; ++h) q4[h] = *reinterpret_cast<const uint4*>(qsym + 16 * h);
    const float bound = bound_from_bits(wk->bsf_bits);
    if (blockIdx.x == 0 && threadIdx.x == 0) wk->scan_bound = bound;
    unsigned long long pruned = 0;
    constexpr uint64_t kRound = static_cast<uint64_t>(kThreads) * kGP;
    for (uint64_t base = static_cast<uint64_t>(blockIdx.x) * kRound; base < NG;
         base += static_cast<uint64_t>(gridDim.x) * kRound) {
        uint4 bl[kGP][H], bh[kGP][H];
#pragma unroll
        for (int k = 0; k < kGP; ++k) {
            const uint64_t g = base + threadIdx.x + static_cast<uint64_t>(kThreads) * k;
#pragma unroll
            for (int h = 0; h < H; ++h) {
                bl[k][h] = g < NG ? ld_stream_u4(glo + g * WS + 16 * h) : make_uint4(0, 0, 0, 0);
                bh[k][h] = g < NG ? ld_stream_u4(ghi + g * WS + 16 * h) : make_uint4(0, 0, 0, 0);
            }
        }
        unsigned keep = 0;
#pragma unroll
        for (int k = 0; k < kGP; ++k) {
            const uint64_t g = base + threadIdx.x + static_cast<uint64_t>(kThreads) * k;
            if (g >= NG) continue;
            if (box_bound<H, W16>(s_lut, q4, bl[k], bh[k], w) <= bound) keep |= 1u << k;
            else pruned += 1;
        }
        uint32_t at = block_reserve(__popc(keep), 0, &wk->ngroups, nullptr).x;
#pragma unroll
        for (int k = 0; k < kGP; ++k)
            if (keep & (1u << k)) gsurv[at++] = static_cast<uint32_t>(base + threadIdx.x + static_cast<uint64_t>(kThreads) * k);
    }
    for (int o = 16; o > 0; o >>= 1) pruned += __shfl_xor_sync(0xFFFFFFFFu, pruned, o);
    if ((threadIdx.x & 31) == 0 && pruned) atomicAdd(&wk->stats[kPruned], pruned);
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(&wk->stats[kLbNode], NG);
}

// Level 2: the pages of the surviving groups, kGP per thread per round.
// Pages whose bound is within the BSF (and outside the seed range) survive,
// split into page wave 0 (bound <= split x BSF, front of surv) and wave 1
// (back of surv); one atomic pair per block and round reserves the slots.
template <int WS, bool W16>
__global__ void __launch_bounds__(kThreads)
    k_bound(const float* __restrict__ lut_g, int w, const uint32_t* __restrict__ gsurv,
            const uint8_t* __restrict__ lo, const uint8_t* __restrict__ hi, const uint32_t* __restrict__ page_off,
            uint64_t P, QueryWork* wk, float split, uint2* __restrict__ surv, float* __restrict__ surv_lb) {
    constexpr int H = WS / 16;
    extern __shared__ float s_lut[];
    __shared__ __align__(16) unsigned char qsym[kMaxW];
    load_prepared(lut_g, wk, w, s_lut, qsym);
    uint4 q4[H];
#pragma unroll
    for (int h = 0; h < H; ++h) q4[h] = *reinterpret_cast<const uint4*>(qsym + 16 * h);
    const float bound = wk->scan_bound;
    const uint32_t sa = wk->seed_begin, sb = wk->seed_end;
    const float cut = bound * split;  // wave 0: the most promising pages
    const uint64_t nitems = static_cast<uint64_t>(wk->ngroups) * kGroup;
    unsigned long long pruned = 0, nodes = 0;
    constexpr uint64_t kRound = static_cast<uint64_t>(kThreads) * kGP;
    for (uint64_t base = static_cast<uint64_t>(blockIdx.x) * kRound; base < nitems;
         base += static_cast<uint64_t>(gridDim.x) * kRound) {
        uint4 bl[kGP][H], bh[kGP][H];
        uint32_t ea[kGP], eb[kGP];
        bool valid[kGP];
#pragma unroll
        for (int k = 0; k < kGP; ++k) {
            const uint64_t i = base + threadIdx.x + static_cast<uint64_t>(kThreads) * k;
            const uint64_t p = i < nitems ? static_cast<uint64_t>(gsurv[i / kGroup]) * kGroup + i % kGroup : P;
            valid[k] = p < P;
#pragma unroll
            for (int h = 0; h < H; ++h) {
                bl[k][h] = valid[k] ? ld_stream_u4(lo + p * WS + 16 * h) : make_uint4(0, 0, 0, 0);
                bh[k][h] = valid[k] ? ld_stream_u4(hi + p * WS + 16 * h) : make_uint4(0, 0, 0, 0);
            }
            ea[k] = valid[k] ? page_off[p] : 0u;
            eb[k] = valid[k] ? page_off[p + 1] : 0u;
        }
        unsigned lowmask = 0, highmask = 0;
        float lbs[kGP];
#pragma unroll
        for (int k = 0; k < kGP; ++k) {
            lbs[k] = 0.f;
            if (!valid[k]) continue;
            nodes += 1;
            const float lb = box_bound<H, W16>(s_lut, q4, bl[k], bh[k], w);
            lbs[k] = lb;
            const bool seeded = ea[k] >= sa && eb[k] <= sb;
            const bool keep = !seeded && lb <= bound;
            lowmask |= (keep && lb <= cut) ? (1u << k) : 0u;
            highmask |= (keep && lb > cut) ? (1u << k) : 0u;
            pruned += (!keep && !seeded) ? 1 : 0;
        }
        const uint2 at0 = block_reserve(__popc(lowmask), __popc(highmask), &wk->nsurv, &wk->nsurv_hi);
        uint32_t at = at0.x, at_hi = at0.y;
#pragma unroll
        for (int k = 0; k < kGP; ++k) {
            if (lowmask & (1u << k)) {
                surv_lb[at] = lbs[k];
                surv[at++] = make_uint2(ea[k], eb[k]);
            } else if (highmask & (1u << k)) {
                const uint64_t slot = P - 1 - at_hi++;
                surv_lb[slot] = lbs[k];
                surv[slot] = make_uint2(ea[k], eb[k]);
            }
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        pruned += __shfl_xor_sync(0xFFFFFFFFu, pruned, o);
        nodes += __shfl_xor_sync(0xFFFFFFFFu, nodes, o);
    }
    if ((threadIdx.x & 31) == 0) {
        if (pruned) atomicAdd(&wk->stats[kPruned], pruned);
        if (nodes) atomicAdd(&wk->stats[kLbNode], nodes);
    }
}

// ------------------------------------------------------------ lbscan
constexpr int kStageCap = 256;

// Writes a warp's staged candidates: refinement wave A (bound <= cut) grows
// upward from ncand, wave B downward from the top of the candidate arrays
// (nhigh). cut = +inf sends everything to A, cut < 0 everything to B.
__device__ __forceinline__ void flush_stage(QueryWork* wk, const uint32_t* s_pos, const float* s_lb, int cnt, int lane,
                                            float cut, uint64_t cap, uint32_t* __restrict__ cand_pos,
                                            float* __restrict__ cand_lb) {
    for (int i0 = 0; i0 < cnt; i0 += 32) {
        const int i = i0 + lane;
        const bool valid = i < cnt;
        const float lb = valid ? s_lb[i] : 0.f;
        const bool low = valid && lb <= cut;
        const unsigned ml = __ballot_sync(0xFFFFFFFFu, low), mh = __ballot_sync(0xFFFFFFFFu, valid && !low);
        uint32_t bl = 0, bh = 0;
        if (lane == 0) {
            if (ml) bl = atomicAdd(&wk->ncand, static_cast<unsigned>(__popc(ml)));
            if (mh) bh = atomicAdd(&wk->nhigh, static_cast<unsigned>(__popc(mh)));
        }
        bl = __shfl_sync(0xFFFFFFFFu, bl, 0);
        bh = __shfl_sync(0xFFFFFFFFu, bh, 0);
        const unsigned below = (1u << lane) - 1u;
        if (low) {
            const uint64_t at = bl + __popc(ml & below);
            cand_pos[at] = s_pos[i];
            cand_lb[at] = lb;
        } else if (valid) {
            const uint64_t at = cap - 1 - (bh + __popc(mh & below));
            cand_pos[at] = s_pos[i];
            cand_lb[at] = lb;
        }
    }
    __syncwarp();
}

// One page wave: wave 0 scans the pages whose box bound is within `split`
// of the seed bound (surv[0, nsurv)), wave 1 the rest (surv[P - nsurv_hi, P)),
// re-filtered against the BSF that wave 0's refinement tightened — MESSI's
// LB-ordered leaf processing (src/query.cpp:173-184) at page granularity.
// Below the page sits one more box level: aligned kRun-entry runs. A warp
// takes three surviving pages at a time; lane 10j + t bounds run t of page j
// (a <= 128-entry page touches at most 9 runs) with the same clamped-symbol
// box bound as the page filter, surviving runs (clipped to their page) queue
// in shared memory, and the queue drains four runs per step: each half-warp
// bounds one run's words, one entry per lane. Words of pruned runs are never
// read. The next triple's ranges and run boxes are in flight while the
// current one is bounded.
template <int WS, bool W16>
__global__ void __launch_bounds__(kThreads)
    k_lbscan(const float* __restrict__ lut_g, int w, const uint8_t* __restrict__ words,
             const uint8_t* __restrict__ run_lo, const uint8_t* __restrict__ run_hi,
             const uint2* __restrict__ surv, const float* __restrict__ surv_lb,
             uint64_t P, QueryWork* wk,
             int wave, float split, uint64_t cap, uint32_t* __restrict__ cand_pos, float* __restrict__ cand_lb) {
    constexpr int kRunQ = 40;
    extern __shared__ float s_lut[];
    __shared__ __align__(16) unsigned char qsym[kMaxW];
    __shared__ uint32_t s_pos[kThreads / 32][kStageCap];
    __shared__ float s_lb[kThreads / 32][kStageCap];
    __shared__ uint2 s_runq[kThreads / 32][kRunQ];
    load_prepared(lut_g, wk, w, s_lut, qsym);
    constexpr int H = WS / 16;
    uint4 q4[H];
#pragma unroll
    for (int h = 0; h < H; ++h) q4[h] = *reinterpret_cast<const uint4*>(qsym + 16 * h);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const unsigned below = (1u << lane) - 1u;
    const int grp = lane / 10, t = lane - 10 * grp;  // page of the triple, run of the page (lanes 30, 31 idle)
    const float bound = bound_from_bits(wk->bsf_bits);
    // Page wave 0 splits its candidates into refinement waves A and B by their
    // own bound; page wave 1 (scanned after wave A is refined) feeds wave B.
    const float cut = wave == 0 ? wk->scan_bound * split : -1.f;
    const uint32_t nsurv = wave == 0 ? wk->nsurv : wk->nsurv_hi;
    const uint64_t ntrip = (static_cast<uint64_t>(nsurv) + 2) / 3;
    const uint64_t gwarp = (blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x) >> 5;
    const uint64_t nwarps = static_cast<uint64_t>(gridDim.x) * (blockDim.x >> 5);
    int cnt = 0, qn = 0;
    unsigned long long scanned = 0, pruned = 0;

    auto stage = [&](bool pass, uint32_t e, float lb) {
        const unsigned m = __ballot_sync(0xFFFFFFFFu, pass);
        if (!m) return;
        if (pass) {
            const int slot = cnt + __popc(m & below);
            s_pos[warp][slot] = e;  // refine gathers pos[e] off this kernel's path
            s_lb[warp][slot] = lb;
        }
        cnt += __popc(m);
        __syncwarp();
        if (cnt > kStageCap - 32) {
            flush_stage(wk, s_pos[warp], s_lb[warp], cnt, lane, cut, cap, cand_pos, cand_lb);
            cnt = 0;
        }
    };
    // Bounds the words of the first min(qn, 4) queued runs, then shifts the queue.
    auto drain = [&]() {
        const int take = min(qn, 4);
        uint4 wv[2][H];
        uint32_t e[2];
        bool ok[2];
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            const int q = 2 * k + (lane >> 4);
            ok[k] = false;
            e[k] = 0;
            if (q < take) {
                const uint2 rr = s_runq[warp][q];
                e[k] = rr.x + (lane & 15);
                ok[k] = e[k] < rr.y;
            }
#pragma unroll
            for (int h = 0; h < H; ++h)
                wv[k][h] = ok[k] ? ld_stream_u4(words + static_cast<uint64_t>(e[k]) * WS + 16 * h) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            const float lb = word_bound<W16>(s_lut, wv[k], w);
            scanned += ok[k] ? 1 : 0;
            stage(ok[k] && lb <= bound, e[k], lb);
        }
        const int rest = qn - take;
        uint2 v = make_uint2(0, 0);
        if (lane < rest) v = s_runq[warp][take + lane];
        __syncwarp();
        if (lane < rest) s_runq[warp][lane] = v;
        __syncwarp();
        qn = rest;
    };

    uint32_t na = 0, nb = 0, nrun = 0;
    bool nvalid = false;
    uint4 nbl[H], nbh[H];
    auto fetch = [&](uint64_t T) {
        uint32_t a = 0, b = 0;
        if (lane < 3) {
            const uint64_t i = 3 * T + lane;
            if (i < nsurv) {
                const uint64_t slot = wave == 0 ? i : P - 1 - i;
                if (wave == 0 || surv_lb[slot] <= bound) {
                    const uint2 r = surv[slot];
                    a = r.x;
                    b = r.y;
                } else {
                    pruned += 1;
                }
            }
        }
        na = __shfl_sync(0xFFFFFFFFu, a, min(grp, 2));
        nb = __shfl_sync(0xFFFFFFFFu, b, min(grp, 2));
        nrun = na / kRun + t;
        nvalid = grp < 3 && na < nb && nrun * kRun < nb;
#pragma unroll
        for (int h = 0; h < H; ++h) {
            nbl[h] = nvalid ? ld_stream_u4(run_lo + static_cast<uint64_t>(nrun) * WS + 16 * h) : make_uint4(0, 0, 0, 0);
            nbh[h] = nvalid ? ld_stream_u4(run_hi + static_cast<uint64_t>(nrun) * WS + 16 * h) : make_uint4(0, 0, 0, 0);
        }
    };
    if (gwarp < ntrip) fetch(gwarp);
    for (uint64_t T = gwarp; T < ntrip; T += nwarps) {
        const uint32_t a = na, b = nb, r = nrun;
        const bool valid = nvalid;
        uint4 c[H];
#pragma unroll
        for (int h = 0; h < H; ++h)
            c[h] = make_uint4(__vminu4(__vmaxu4(q4[h].x, nbl[h].x), nbh[h].x),
                              __vminu4(__vmaxu4(q4[h].y, nbl[h].y), nbh[h].y),
                              __vminu4(__vmaxu4(q4[h].z, nbl[h].z), nbh[h].z),
                              __vminu4(__vmaxu4(q4[h].w, nbl[h].w), nbh[h].w));
        if (T + nwarps < ntrip) fetch(T + nwarps);
        bool pass = false;
        if (valid) pass = word_bound<W16>(s_lut, c, w) <= bound;
        pruned += valid && !pass ? 1 : 0;
        const unsigned m = __ballot_sync(0xFFFFFFFFu, pass);
        if (pass) s_runq[warp][qn + __popc(m & below)] = make_uint2(max(a, r * kRun), min(b, r * kRun + kRun));
        qn += __popc(m);
        __syncwarp();
        while (qn >= 4) drain();
    }
    while (qn > 0) drain();
    for (int o = 16; o > 0; o >>= 1) {
        scanned += __shfl_xor_sync(0xFFFFFFFFu, scanned, o);
        pruned += __shfl_xor_sync(0xFFFFFFFFu, pruned, o);
    }
    // Final flush, one atomic pair per block instead of one per warp.
    __shared__ uint32_t s_wcnt[kThreads / 32], s_wbase[2];
    int lo_cnt = 0;
    for (int i = lane; i < cnt; i += 32) lo_cnt += s_lb[warp][i] <= cut ? 1 : 0;
    for (int o = 16; o > 0; o >>= 1) lo_cnt += __shfl_xor_sync(0xFFFFFFFFu, lo_cnt, o);
    if (lane == 0) s_wcnt[warp] = static_cast<uint32_t>(lo_cnt) | (static_cast<uint32_t>(cnt - lo_cnt) << 16);
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t tot = 0;
        for (int i = 0; i < kThreads / 32; ++i) {
            const uint32_t c2 = s_wcnt[i];
            s_wcnt[i] = tot;
            tot += c2;
        }
        s_wbase[0] = (tot & 0xFFFFu) ? atomicAdd(&wk->ncand, tot & 0xFFFFu) : 0u;
        s_wbase[1] = (tot >> 16) ? atomicAdd(&wk->nhigh, tot >> 16) : 0u;
    }
    __syncthreads();
    {
        uint32_t at_lo = s_wbase[0] + (s_wcnt[warp] & 0xFFFFu), at_hi = s_wbase[1] + (s_wcnt[warp] >> 16);
        for (int i0 = 0; i0 < cnt; i0 += 32) {
            const int i = i0 + lane;
            const bool valid = i < cnt;
            const float lb = valid ? s_lb[warp][i] : 0.f;
            const bool low = valid && lb <= cut;
            const unsigned ml = __ballot_sync(0xFFFFFFFFu, low), mh = __ballot_sync(0xFFFFFFFFu, valid && !low);
            const unsigned below = (1u << lane) - 1u;
            if (low) {
                const uint64_t at = at_lo + __popc(ml & below);
                cand_pos[at] = s_pos[warp][i];
                cand_lb[at] = lb;
            } else if (valid) {
                const uint64_t at = cap - 1 - (at_hi + __popc(mh & below));
                cand_pos[at] = s_pos[warp][i];
                cand_lb[at] = lb;
            }
            at_lo += __popc(ml);
            at_hi += __popc(mh);
        }
    }
    if (lane == 0 && scanned) atomicAdd(&wk->stats[kLbEntry], scanned);
    if (lane == 0 && pruned) atomicAdd(&wk->stats[kPruned], pruned);
}

// ------------------------------------------------------------ refine
// One wave: wave 0 = [nseed, ncand), wave 1 = [cap - nhigh, cap).
template <bool VEC>
__global__ void __launch_bounds__(kThreads)
    k_refine(const float* __restrict__ rows, int n, const float* __restrict__ query, const uint32_t* __restrict__ pos,
             QueryWork* wk,
             const uint32_t* __restrict__ cand_pos, const float* __restrict__ cand_lb,
             double* __restrict__ cand_sq, int wave, uint64_t cap) {
    extern __shared__ float s_q[];
    load_query(s_q, query, n);
    const uint64_t begin = wave == 0 ? wk->nseed : cap - wk->nhigh;
    const uint64_t end = wave == 0 ? wk->ncand : cap;
    const int lane = threadIdx.x & 31;
    const bool leader = (lane & (kRowLanes - 1)) == 0;
    unsigned long long refined = 0, updates = 0;
    // Each 8-lane group walks its own candidates (group-stride), the next
    // candidate's record prefetched while the current row is refined; a
    // candidate whose bound exceeds the live BSF costs one check.
    const uint64_t group = (blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x) / kRowLanes;
    const uint64_t ngroups = static_cast<uint64_t>(gridDim.x) * blockDim.x / kRowLanes;
    uint64_t c = begin + group;
    float nlb = c < end ? cand_lb[c] : 0.f;
    uint32_t np = c < end ? pos[cand_pos[c]] : 0u;  // candidate records hold index-order entries
    // Cached pruning bound: refreshed from the BSF each publish observes, so a
    // skipped candidate costs no memory access (a stale bound only refines more).
    float bnd = bound_from_bits(ld_volatile_u64(&wk->bsf_bits));
    for (; c < end; c += ngroups) {
        const float lb = nlb;
        const uint32_t p = np;
        if (c + ngroups < end) {
            nlb = cand_lb[c + ngroups];
            np = pos[cand_pos[c + ngroups]];
        }
        if (lb > bnd) {
            if (leader) cand_sq[c] = INFINITY;
            continue;
        }
        // read the BSF for the next candidate's bound while this row is in flight
        const unsigned long long seen = ld_volatile_u64(&wk->bsf_bits);
        const double s = group_row_sq<VEC>(rows + static_cast<uint64_t>(p) * n, s_q, n, &wk->bsf_bits);
        if (leader) {
            refined += 1;
            updates += publish(wk, s, c, cand_sq);
        }
        bnd = bound_from_bits(min(seen, static_cast<unsigned long long>(__double_as_longlong(s < INFINITY ? s : INFINITY))));
    }
    if (leader) {
        if (refined) atomicAdd(&wk->stats[kRealDist], refined);
        if (updates) atomicAdd(&wk->stats[kBsfUpd], updates);
    }
}

// ----------------------------------------------------------- finalize
// Lowest position among the candidates whose sqrt(sum) equals the best
// distance; the last block to finish writes the result and resets `wk`.
__global__ void __launch_bounds__(kThreads)
    k_finalize(QueryWork* wk, const uint32_t* __restrict__ pos, const uint32_t* __restrict__ cand_pos,
               const double* __restrict__ cand_sq, int seed_only,
               uint64_t cap, DevResult* out, uint64_t P, uint64_t pos_offset) {
    const double best = bsf_of(wk->bsf_bits);
    const double dist = sqrt(best);
    const double lim = best * kSlack;
    const uint64_t lo_end = seed_only ? wk->nseed : wk->ncand;
    const uint64_t hi_n = seed_only ? 0 : wk->nhigh;
    uint32_t mine = 0xFFFFFFFFu;
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < lo_end + hi_n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint64_t c = i < lo_end ? i : cap - 1 - (i - lo_end);
        const double s = cand_sq[c];
        if (s <= lim && sqrt(s) == dist) mine = min(mine, pos[cand_pos[c]]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mine = min(mine, __shfl_xor_sync(0xFFFFFFFFu, mine, o));
    if ((threadIdx.x & 31) == 0 && mine != 0xFFFFFFFFu) atomicMin(&wk->best_pos, mine);
    __threadfence();
    __syncthreads();
    __shared__ bool last;
    if (threadIdx.x == 0) last = atomicAdd(&wk->done_blocks, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!last || threadIdx.x != 0) return;
    __threadfence();
    const unsigned best_pos = atomicAdd(&wk->best_pos, 0u);
    out->distance = dist;
    out->position = static_cast<uint32_t>(best_pos + pos_offset);
    out->reserved = 0;
    out->stats[kLbNode] = wk->stats[kLbNode];
    out->stats[kLbEntry] = wk->stats[kLbEntry] + wk->nseed;
    out->stats[kRealDist] = wk->stats[kRealDist];
    out->stats[kBsfUpd] = wk->stats[kBsfUpd];
    out->stats[kPruned] = wk->stats[kPruned];
    out->stats[kQueueIns] = wk->ncand - wk->nseed + wk->nhigh;
    reset_work(wk);  // for the next query on this stream
    __threadfence();
    wk->done_blocks = 0;
}

unsigned cap_grid(uint64_t want, int sms, int per_sm) {
    return static_cast<unsigned>(std::max<uint64_t>(1, std::min<uint64_t>(want, static_cast<uint64_t>(sms) * per_sm)));
}

template <typename K>
int blocks_per_sm(K kernel, size_t smem) {
    int b = 0;
    TSG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kernel, kThreads, smem));
    return std::max(b, 1);
}

}  // namespace

void search_batch(DevIndex& ix, const float* d_queries, uint32_t nq, bool approximate) {
    cudaStream_t st = ix.stream;
    const int n = ix.n, w = ix.w;
    const size_t lut_bytes = static_cast<size_t>(w) * 256 * sizeof(float);
    const size_t q_bytes = static_cast<size_t>(n) * sizeof(float);
    const bool vec = (n % 8) == 0 && (reinterpret_cast<uintptr_t>(ix.rows) % 32) == 0;
    const bool w16 = w == 16;
    auto refine = vec ? k_refine<true> : k_refine<false>;
    auto seed = vec ? k_seed<true> : k_seed<false>;
    auto lbscan = ix.ws == 16 ? (w16 ? k_lbscan<16, true> : k_lbscan<16, false>) : k_lbscan<32, false>;
    auto bound = ix.ws == 16 ? (w16 ? k_bound<16, true> : k_bound<16, false>) : k_bound<32, false>;
    auto groups = ix.ws == 16 ? (w16 ? k_groups<16, true> : k_groups<16, false>) : k_groups<32, false>;
    TSG_CUDA(cudaFuncSetAttribute(groups, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024));
    // Per-device function attributes (cheap; set on every call so each device is covered).
    TSG_CUDA(cudaFuncSetAttribute(refine, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024));
    TSG_CUDA(cudaFuncSetAttribute(seed, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024));
    TSG_CUDA(cudaFuncSetAttribute(lbscan, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024));
    TSG_CUDA(cudaFuncSetAttribute(bound, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024));
    const uint32_t seed_cap = static_cast<uint32_t>(std::min<uint64_t>(2 * ix.leaf_cap, 1u << 20));
    // With several query lanes, each kernel gets a share of the GPU so kernels
    // of different queries co-reside (TSG_GRID_SHARE: 1/share of the
    // resident-block capacity; default 2 when lanes run concurrently).
    const int share_env = std::getenv("TSG_GRID_SHARE") ? std::atoi(std::getenv("TSG_GRID_SHARE")) : 0;
    const int share = std::max(1, share_env > 0 ? share_env : (ix.nlanes > 1 && !ix.profile ? 2 : 1));
    const unsigned group_grid = cap_grid((ix.NG + kThreads * kGP - 1) / (kThreads * kGP), ix.sms,
                                         std::max(1, std::min(6, blocks_per_sm(groups, lut_bytes)) / share));
    // (the page level's size is only known on the device: a resident-capacity grid)
    const unsigned bound_grid = cap_grid((ix.P + kThreads * kGP - 1) / (kThreads * kGP), ix.sms,
                                         std::max(1, std::min(6, blocks_per_sm(bound, lut_bytes)) / share));
    const unsigned seed_grid = cap_grid((std::min<uint64_t>(seed_cap, ix.N) * kRowLanes + kThreads - 1) / kThreads,
                                        ix.sms, blocks_per_sm(seed, q_bytes));
    const unsigned scan_grid = static_cast<unsigned>(std::max(ix.sms, ix.sms * blocks_per_sm(lbscan, lut_bytes) / share));
    const unsigned refine_grid = static_cast<unsigned>(std::max(ix.sms, ix.sms * blocks_per_sm(refine, q_bytes) / share));
    const uint64_t cap = ix.cand_cap;
    // Profiling runs one lane so per-kernel times are not overlapped.
    const int nl = ix.profile ? 1 : std::max(1, std::min<int>(ix.nlanes, static_cast<int>(nq)));

    // Optional per-kernel timing: events around every launch, summed after the batch.
    std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> marks;
    auto mark = [&](cudaStream_t ls, int slot, auto&& launch) {
        if (!ix.profile) {
            launch();
            return;
        }
        cudaEvent_t a, b;
        TSG_CUDA(cudaEventCreate(&a));
        TSG_CUDA(cudaEventCreate(&b));
        TSG_CUDA(cudaEventRecord(a, ls));
        launch();
        TSG_CUDA(cudaEventRecord(b, ls));
        marks.push_back({slot, {a, b}});
    };

    // Fork (every lane starts after the work already queued on the index
    // stream), the queries round-robin over the lanes, join.
    auto enqueue = [&]() {
        TSG_CUDA(cudaEventRecord(ix.lanes[0].done, st));
        for (int k = 0; k < nl; ++k) {
            DevIndex::Lane& L = ix.lanes[k];
            if (k > 0) TSG_CUDA(cudaStreamWaitEvent(L.stream, ix.lanes[0].done, 0));
            k_reset<<<1, 1, 0, L.stream>>>(L.work);
            TSG_LAUNCHED();
        }
        for (uint32_t qi = 0; qi < nq; ++qi) {
            const DevIndex::Lane& L = ix.lanes[qi % nl];
            cudaStream_t ls = L.stream;
            const float* q = d_queries + static_cast<uint64_t>(qi) * n;
            mark(ls, 2, [&] {
                seed<<<seed_grid, kThreads, q_bytes, ls>>>(ix.rows, n, w, ix.bits, ix.thr, q, ix.leaf_off, ix.page_off,
                                                           ix.page_leaf, ix.page_key, ix.page_dir, ix.P, ix.pos, seed_cap,
                                                           L.work, L.cand_pos, L.cand_sq, L.lut);
            });
            TSG_LAUNCHED();
            if (!approximate) {
                mark(ls, 1, [&] {
                    groups<<<group_grid, kThreads, lut_bytes, ls>>>(L.lut, w, ix.group_lo, ix.group_hi, ix.NG, L.work,
                                                                    L.gsurv);
                    TSG_LAUNCHED();
                    bound<<<bound_grid, kThreads, lut_bytes, ls>>>(L.lut, w, L.gsurv, ix.page_lo, ix.page_hi, ix.page_off,
                                                                   ix.P, L.work, ix.refine_split, L.surv, L.surv_lb);
                });
                TSG_LAUNCHED();
                for (int wave = 0; wave < 2; ++wave) {
                    mark(ls, 4, [&] {
                        lbscan<<<scan_grid, kThreads, lut_bytes, ls>>>(L.lut, w, ix.words, ix.run_lo, ix.run_hi, L.surv, L.surv_lb,
                                                                       ix.P, L.work, wave, ix.refine_split, cap, L.cand_pos,
                                                                       L.cand_lb);
                    });
                    TSG_LAUNCHED();
                    mark(ls, wave == 0 ? 3 : 5, [&] {
                        refine<<<refine_grid, kThreads, q_bytes, ls>>>(ix.rows, n, q, ix.pos, L.work, L.cand_pos, L.cand_lb,
                                                                       L.cand_sq, wave, cap);
                    });
                    TSG_LAUNCHED();
                }
            }
            mark(ls, 6, [&] {
                k_finalize<<<ix.sms, kThreads, 0, ls>>>(L.work, ix.pos, L.cand_pos, L.cand_sq, approximate ? 1 : 0, cap,
                                                        ix.results + qi, ix.P, ix.pos_offset);
            });
            TSG_LAUNCHED();
        }
        // Join: the index stream waits for every lane.
        for (int k = 1; k < nl; ++k) {
            TSG_CUDA(cudaEventRecord(ix.lanes[k].done, ix.lanes[k].stream));
            TSG_CUDA(cudaStreamWaitEvent(st, ix.lanes[k].done, 0));
        }
    };

    // TSG_GRAPHS=1: the batch is captured into a CUDA graph (~7 kernels per
    // query over the lanes' streams as one launch, replayed while the batch
    // shape and buffers repeat). Measured no faster than direct launches on
    // c2 (the host enqueue overlaps the GPU), so off by default; it lets ncu
    // (--graph-profiling graph) measure a whole concurrent batch.
    const char* genv = std::getenv("TSG_GRAPHS");
    const bool graph = !ix.profile && genv && genv[0] == '1';
    if (!graph) {
        enqueue();
    } else if (ix.graph && ix.graph_key.queries == d_queries && ix.graph_key.nq == nq &&
               ix.graph_key.approximate == approximate && ix.graph_key.nlanes == nl) {
        // Same batch shape and buffers as the captured graph: replay it.
        TSG_CUDA(cudaGraphLaunch(ix.graph, st));
        note_launch(ix.graph_key.kernels);
    } else {
        TSG_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
        try {
            enqueue();
        } catch (...) {
            cudaGraph_t g = nullptr;
            cudaStreamEndCapture(st, &g);
            if (g) cudaGraphDestroy(g);
            throw;
        }
        cudaGraph_t g = nullptr;
        TSG_CUDA(cudaStreamEndCapture(st, &g));
        if (ix.graph) {
            TSG_CUDA(cudaStreamSynchronize(st));  // the previous batch's graph may still run
            TSG_CUDA(cudaGraphExecDestroy(ix.graph));
            ix.graph = nullptr;
        }
        TSG_CUDA(cudaGraphInstantiate(&ix.graph, g, 0));
        TSG_CUDA(cudaGraphDestroy(g));
        ix.graph_key = {d_queries, nq, approximate, nl, nl + static_cast<int>(nq) * (approximate ? 2 : 8)};
        TSG_CUDA(cudaGraphLaunch(ix.graph, st));
    }
    if (!marks.empty()) {
        TSG_CUDA(cudaStreamSynchronize(st));
        for (auto& m : marks) {
            float ms = 0.f;
            TSG_CUDA(cudaEventElapsedTime(&ms, m.second.first, m.second.second));
            ix.prof_ms[m.first] += ms;
            ix.prof_launches[m.first] += 1;
            cudaEventDestroy(m.second.first);
            cudaEventDestroy(m.second.second);
        }
    }
}

}  // namespace tsg
