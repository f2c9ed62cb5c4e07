// Exact Euclidean 1-NN over the flat SoA index (one device shard), a batch
// of queries at a time.
//
// Replaces exact_search (src/query.cpp:258-298) and its pieces. A batch of up
// to batch_max queries runs through nine kernels, each launched ONCE for the
// whole batch; every query owns a slot of scratch (QueryWork, table, page
// lists, candidate records):
//   prepare   per query: PAA (FP64, reference order), symbols, the [w][256]
//             table of squared region gaps, and the leaf its own iSAX word
//             descends to (approximate_search_state, src/query.cpp:226-238).
//   seed      that leaf's rows refined exhaustively: the first best-so-far.
//   groups    node_lower_bound (src/query.cpp:102-107) over the page-group
//             boxes + the pruning test (src/query.cpp:159).
//   bound     the same over the pages of surviving groups; surviving pages
//             split into page wave 0 (bound <= split x BSF) and wave 1.
//   lbscan x2 the entry filter of calculate_real_distance_leaf
//             (src/query.cpp:129-134) over run boxes, quad boxes and words of
//             the surviving pages, compacted with warp ballot + prefix
//             popcount into candidate waves A (front) and B (back).
//   refine x2 euclidean (src/metrics.cpp:17-40, 95-104): an 8-lane group per
//             candidate row, 256-bit loads, FP64 block sums without FMA added
//             left to right like squared_l2; the BSF is an atomicMin on the
//             double bit pattern (the SharedBsf analog, src/query.cpp:35-42).
//   finalize  (sqrt(min sum), lowest position among equal distances), the
//             tie rule of scan_nn (src/scan.cpp:54-59).
// page wave 1 runs after refinement wave A tightened the BSF: MESSI's
// LB-ordered priority-queue processing (src/query.cpp:173-184) in two steps.
// bound / lbscan / refine are persistent grids fed from per-query chunk
// counters with block-to-query affinity: a block drains the chunks of one
// query (whose table or row stays in shared memory), then moves on to the next
// query with work left, so easy and hard queries of a batch share the GPU
// without per-query launches or tails.
// Soundness: the table is rounded DOWN to float and bounds are summed with
// __fadd_rd, so every float bound is <= the exact FP64 bound; the BSF bound
// is rounded up and widened by 1e-9 relative; pruning is strict, so ties
// reach the exact FP64 comparison.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <tuple>
#include <stdexcept>
#include <utility>
#include <vector>

#include <cuda_fp16.h>

#include "common.cuh"
#include "exchange.cuh"
#include "kernels.cuh"

namespace tsg {

namespace {

constexpr unsigned long long kInfBits = 0x7FF0000000000000ull;
constexpr double kSlack = 1.0 + 1e-9;
constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kRowLanes = 8;  // lanes per candidate row in the refine kernels

enum Stat { kLbNode = 0, kLbEntry, kRealDist, kBsfUpd, kPruned, kQueueIns };

// Resident blocks per SM the persistent kernels are compiled for (register
// caps; -D overrides for tuning runs).
#ifndef TSG_MINB_LBSCAN
#define TSG_MINB_LBSCAN 4  // 5 until the block-wide query selection: with the switch stalls gone the kernel is issue-bound and 64 registers beat 40 warps (12.55 -> 12.11 us/query)
#endif
#ifndef TSG_MINB_REFINE
#define TSG_MINB_REFINE 4
#endif
#ifndef TSG_MINB_BOUND
#define TSG_MINB_BOUND 4  // 5 while bound was latency-bound (round 2a); 4 since the block-wide query selection (7.17 -> 6.89 us/query)
#endif
// w = 16 box bounds clamp with the native u16x2 min/max (0: byte-SIMD __vmaxu4 / __vminu4)
#ifndef TSG_BOX_U16
#define TSG_BOX_U16 1
#endif

// ---------------------------------------------------------------- views
// Kernel-side views of the index and of a slot set (passed by value).
struct IndexView {
    const float* rows;
    int n, w, bits;
    const double* thr;
    const uint8_t* words;
    const uint32_t* pos;
    const uint32_t* leaf_off;
    const uint32_t* page_off;
    const uint32_t* page_leaf;
    const uint64_t* page_key;
    const uint64_t* page_dir;
    uint64_t P;
    const uint8_t *page_lo, *page_hi, *group_lo, *group_hi, *top_lo, *top_hi;
    uint64_t NG, NT;
    const uint8_t *run_lo, *run_hi, *quad_lo, *quad_hi;
    uint32_t seed_cap;
    float split;
    uint64_t pos_offset;
    int window;  // < 0: Euclidean; >= 0: DTW with this Sakoe-Chiba window
    int rev_keogh;  // DTW refinement also tests the reversed LB_Keogh (per-warp scratch in shared memory)
    const uint8_t* fine;       // [N][fws] fine summary (index order); null: none
    int fw, fws;
};

struct SlotView {
    QueryWork* work;
    float* lut;
    uint32_t* gsurv;
    uint2* surv;
    float* surv_lb;
    uint32_t* cand_pos;
    float* cand_lb;
    double* cand_sq;
    float* env;  // [slots][2][n] DTW envelopes (upper, lower)
    uint64_t cap, P, NG;
    int lut_len;
    uint64_t rcap;  // run-list capacity per slot
    uint2* dpage;   // [slots][P] pages deferred to the second bound pass
    float* dpage_lb;
    float* fine_lut;  // [slots][fw][256] fine-summary tables
    int fine_lut_len;
};

__device__ __forceinline__ double bsf_of(unsigned long long bits) {
    return __longlong_as_double(static_cast<long long>(bits));
}

__device__ __forceinline__ float bound_from_bits(unsigned long long bits) {
    return __double2float_ru(bsf_of(bits) * kSlack);
}

__device__ __forceinline__ uint64_t u64min(uint64_t a, uint64_t b) { return a < b ? a : b; }

__device__ __forceinline__ unsigned ld_volatile_u32(const unsigned* p) { return *reinterpret_cast<const volatile unsigned*>(p); }

__device__ __forceinline__ uint32_t word32(const uint4& v, int i) {
    return i == 0 ? v.x : i == 1 ? v.y : i == 2 ? v.z : v.w;
}

__device__ __forceinline__ uint32_t byte_of(const uint4& v, int s) { return (word32(v, s >> 2) >> (8 * (s & 3))) & 255u; }

// ------------------------------------------------------ query prepare
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

// The fine summary's table: per fine segment s (2w half segments of n / fw
// points) and symbol v, the squared gap between the query's fine mean (FP64,
// the same sums as K1) and v's region (fine_quant) widened by kFineSlack,
// times n / fw, rounded down. Every entry is <= the exact PAA term, so a sum
// of entries (rounded down) never exceeds the squared Euclidean distance —
// the PAA lower-bounding lemma behind mindist_paa_isax (src/metrics.cpp:47-70)
// at twice the segments.
__device__ __forceinline__ void fill_fine_lut(const float* s_q, int n, int fw, float* out) {
    __shared__ double s_fm[kMaxFine];
    const int h = n / fw;
    if (threadIdx.x < fw) {
        double sum = 0.0;
        for (int j = 0; j < h; ++j) sum = __dadd_rn(sum, static_cast<double>(s_q[threadIdx.x * h + j]));
        s_fm[threadIdx.x] = __ddiv_rn(sum, static_cast<double>(h));
    }
    __syncthreads();
    const double scale = static_cast<double>(h);
    for (int idx = threadIdx.x; idx < fw * 256; idx += blockDim.x) {
        const int s = idx >> 8, v = idx & 255;
        const double lo = v == 0 ? -INFINITY : kFineLo + v * kFineStep - kFineSlack;
        const double hi = v == 255 ? INFINITY : kFineLo + (v + 1) * kFineStep + kFineSlack;
        const double x = s_fm[s];
        double gap = 0.0;  // a NaN mean keeps 0: never prunes
        if (x < lo) gap = lo - x;
        else if (x > hi) gap = x - hi;
        out[idx] = __double2float_rd(__dmul_rn(__dmul_rn(gap, gap), scale));
    }
}

// DTW: the same table for the envelope band [lower_paa, upper_paa]
// (mindist_envelope_isax, src/metrics.cpp:48-70,194-196): per segment the
// squared gap from the band to each symbol's region, times n/w, rounded down.
// It is zero exactly on the symbols between those of lower_paa and
// upper_paa, so box bounds clamp the lower_paa symbol into the box.
__device__ __forceinline__ void fill_lut_band(const double* thr, const double* lo_paa, const double* hi_paa, int n,
                                              int w, int bits, float* out) {
    const unsigned card = 1u << bits;
    const double scale = static_cast<double>(n) / static_cast<double>(w);
    for (int idx = threadIdx.x; idx < w * 256; idx += blockDim.x) {
        const int s = idx >> 8, v = idx & 255;
        const unsigned prefix = static_cast<unsigned>(v) >> (8 - bits);
        const double lo = prefix == 0 ? -INFINITY : thr[prefix - 1];
        const double hi = prefix == card - 1 ? INFINITY : thr[prefix];
        double gap = 0.0;
        if (hi_paa[s] < lo) gap = lo - hi_paa[s];
        else if (lo_paa[s] > hi) gap = lo_paa[s] - hi;
        out[idx] = __double2float_rd(__dmul_rn(__dmul_rn(gap, gap), scale));
    }
}

// Block-local query preparation: PAA (FP64, reference order) and symbols.
__device__ void prepare_query(const float* __restrict__ q, int n, int w, int bits, const double* __restrict__ thr_g,
                              QueryShared& qs) {
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
}

// Loads a query's table and symbols (prepared once per query by k_prepare)
// into shared memory. Callers synchronise before overwriting a previous one.
__device__ __forceinline__ void load_prepared(const float* __restrict__ lut_g, const QueryWork* wk, int w,
                                              float* s_lut, unsigned char* qsym) {
    const float4* src = reinterpret_cast<const float4*>(lut_g);
    float4* dst = reinterpret_cast<float4*>(s_lut);
    for (int i = threadIdx.x; i < w * 64; i += blockDim.x) dst[i] = src[i];
    for (int i = threadIdx.x; i < kMaxW; i += blockDim.x) qsym[i] = i < w ? wk->qsym[i] : 0;
    __syncthreads();
}

__device__ __forceinline__ void load_query(float* s_q, const float* q, int n) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) s_q[i] = q[i];
    __syncthreads();
}

// The query widened to double once per block (the refinement subtracts in FP64).
__device__ __forceinline__ void load_query_f64(double* s_q, const float* q, int n) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) s_q[i] = static_cast<double>(q[i]);
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

// Box bound: per segment the table entry of the query symbol clamped into the
// box [lo, hi] (0 when the query symbol is inside) — node_lower_bound's region
// gap (src/query.cpp:102-107) over a box of iSAX words.
__device__ __forceinline__ uint32_t vmax_u16x2(uint32_t a, uint32_t b) {
    uint32_t r;
    asm("max.u16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
    return r;
}
__device__ __forceinline__ uint32_t vmin_u16x2(uint32_t a, uint32_t b) {
    uint32_t r;
    asm("min.u16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
    return r;
}

// Four segments of a w = 16 box: the even and odd symbols spread into 16-bit
// lanes (one LOP3 / PRMT each) are clamped with the native u16x2 min/max
// (one VIMNMX per two segments; __vmaxu4 / __vminu4 are emulated in about
// seven instructions each), then read back as table byte offsets.
__device__ __forceinline__ void box_quad16(const float* s_lut, int s0, uint32_t q, uint32_t lo, uint32_t hi, float* t) {
    const uint32_t ce = vmin_u16x2(vmax_u16x2(q & 0x00FF00FFu, lo & 0x00FF00FFu), hi & 0x00FF00FFu);
    const uint32_t co = vmin_u16x2(vmax_u16x2(__byte_perm(q, 0, 0x4341), __byte_perm(lo, 0, 0x4341)),
                                   __byte_perm(hi, 0, 0x4341));
    const char* b = reinterpret_cast<const char*>(s_lut);
    // lanes hold symbols <= 255, so the upper lane shifted right by 14 is its
    // byte offset (the lower lane's bits 14-15 are zero)
    t[0] = *reinterpret_cast<const float*>(b + (s0 + 0) * 1024 + ((ce << 2) & 0x3FCu));
    t[1] = *reinterpret_cast<const float*>(b + (s0 + 1) * 1024 + ((co << 2) & 0x3FCu));
    t[2] = *reinterpret_cast<const float*>(b + (s0 + 2) * 1024 + (ce >> 14));
    t[3] = *reinterpret_cast<const float*>(b + (s0 + 3) * 1024 + (co >> 14));
}

template <int H, bool W16>
__device__ __forceinline__ float box_bound(const float* s_lut, const uint4* q4, const uint4* lo, const uint4* hi, int w) {
    if constexpr (W16 && TSG_BOX_U16) {
        float t[16];
        box_quad16(s_lut, 0, q4[0].x, lo[0].x, hi[0].x, t + 0);
        box_quad16(s_lut, 4, q4[0].y, lo[0].y, hi[0].y, t + 4);
        box_quad16(s_lut, 8, q4[0].z, lo[0].z, hi[0].z, t + 8);
        box_quad16(s_lut, 12, q4[0].w, lo[0].w, hi[0].w, t + 12);
        float lb = 0.f;
#pragma unroll
        for (int s = 0; s < 16; ++s) lb = __fadd_rd(lb, t[s]);  // segment order, as word_bound
        return lb;
    }
    uint4 c[H];
#pragma unroll
    for (int h = 0; h < H; ++h)
        c[h] = make_uint4(__vminu4(__vmaxu4(q4[h].x, lo[h].x), hi[h].x), __vminu4(__vmaxu4(q4[h].y, lo[h].y), hi[h].y),
                          __vminu4(__vmaxu4(q4[h].z, lo[h].z), hi[h].z), __vminu4(__vmaxu4(q4[h].w, lo[h].w), hi[h].w));
    return word_bound<W16>(s_lut, c, w);
}

// ------------------------------------------------ scheduling switches
// the refinement kernels' blocks start at queries in proportion to the queries' chunk counts (bound and
// lbscan measured slower with it: 7.18 -> 7.43 and 12.53 -> 13.14 us/query on c2)
#ifndef TSG_WEIGHTED_START
#define TSG_WEIGHTED_START 1
#endif

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

__device__ __forceinline__ double block_sq(const float* x, const double* q, int cnt) {
    double blk = 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k)
        if (k < cnt) {
            const double d = __dsub_rn(static_cast<double>(x[k]), q[k]);
            blk = __dadd_rn(blk, __dmul_rn(d, d));
        }
    return blk;
}

// Squared distance of a row computed by an 8-lane group: lane j owns blocks
// j, j+8, j+16, j+24 of each 32-block round (the 8 lanes read 256 contiguous
// bytes per load); the group then adds the block sums left to right,
// squared_l2's order. Rows longer than 256 take several rounds; after each
// round the running sum is checked against the live BSF (strict), the
// reference's abandonment (metrics.cpp:28). Group-local: only the group's 8
// lanes take part (shuffles use the group mask), so groups of a warp work on
// different candidates independently. Every lane of the group returns the
// sum, +inf if abandoned.
template <bool VEC>
__device__ __forceinline__ double group_row_sq(const float* __restrict__ row, const double* __restrict__ s_q, int n,
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
// improve, strict-improvement count.
// A finished row whose sum is within the BSF it was compared with (which is
// >= the final BSF) joins the query's tie list: the answer and every row
// whose sqrt equals it are always in the list.
__device__ __forceinline__ void note_tie(QueryWork* wk, double s, uint32_t row, unsigned long long seen) {
    if (!(s <= bsf_of(seen) * kSlack)) return;
    const unsigned i = atomicAdd(&wk->nties, 1u);
    if (i < kTieCap) {
        wk->tie_sq[i] = s;
        wk->tie_row[i] = row;
    }
}

// row = ~0u: not noted (the seed range, which finalize scans itself).
__device__ __forceinline__ unsigned long long publish(QueryWork* wk, double s, uint64_t c, double* cand_sq,
                                                      uint32_t row) {
    cand_sq[c] = s;
    const unsigned long long cur = ld_volatile_u64(&wk->bsf_bits);
    if (!(s < INFINITY)) return 0;
    if (row != ~0u) note_tie(wk, s, row, cur);
    const unsigned long long sb = static_cast<unsigned long long>(__double_as_longlong(s));
    if (sb >= cur) return 0;
    return atomicMin(&wk->bsf_bits, sb) > sb ? 1 : 0;
}

// A (min, max) box pair of a w <= 16 word, or a 32-byte fine row (32 contiguous bytes, 32-byte
// aligned), in one 256-bit load: one request per lane instead of two, half the L1 wavefronts of
// those loads (the box filters are bound by the L1/LSU data pipe).
__device__ __forceinline__ void ld_box_pair(const uint8_t* p, uint4& lo, uint4& hi) {
    asm volatile("ld.global.nc.L1::no_allocate.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(lo.x), "=r"(lo.y), "=r"(lo.z), "=r"(lo.w), "=r"(hi.x), "=r"(hi.y), "=r"(hi.z), "=r"(hi.w)
                 : "l"(p));
}

// Shared-memory accesses through a 32-bit shared address kept in a register. The address of a
// per-warp shared array costs ~10 instructions each time the compiler re-derives it (thread id,
// cluster CTA rank, window base, shifts, masks), which it does at every use in the persistent
// kernels' hot loops; an address passed through an empty asm statement is opaque and stays put.
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(p));
    asm volatile("" : "+r"(a));
    return a;
}
__device__ __forceinline__ uint2 lds_u2(uint32_t a) {
    uint2 v;
    asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ float lds_f32(uint32_t a) {
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ uint32_t lds_u32(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ void sts_u2(uint32_t a, uint2 v) {
    asm volatile("st.shared.v2.u32 [%0], {%1,%2};" ::"r"(a), "r"(v.x), "r"(v.y) : "memory");
}
__device__ __forceinline__ void sts_u32(uint32_t a, uint32_t v) {
    asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ void sts_f32(uint32_t a, float v) {
    asm volatile("st.shared.f32 [%0], %1;" ::"r"(a), "f"(v) : "memory");
}

// L2 prefetch of boxes / words a few steps before they are read (the box
// filters are bound by load latency; TSG_PREFETCH=0 for A/B builds).
#ifndef TSG_PREFETCH
#define TSG_PREFETCH 1
#endif
__device__ __forceinline__ void prefetch_l2(const void* p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }
// Prefetch of exactly `bytes` (a multiple of 16, 16-byte aligned) into L2 with the bulk-copy unit:
// unlike prefetch.global.L2 it does not pull the neighbouring sectors of the line.
__device__ __forceinline__ void prefetch_l2_bytes(const void* p, unsigned bytes) {
#if TSG_PREFETCH == 2
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
#else
    (void)bytes;
    prefetch_l2(p);
#endif
}

// -------------------------------------------------------- scheduling
// Block-level work distribution with query affinity. Each query has a chunk
// counter per kernel (`k`); a block drains chunks of its current query and,
// when that query has none left, moves on to the next query with work. The
// claim of a block's next chunk is issued (by thread 0) when the current
// chunk starts and read when it ends, so the atomic's latency hides behind
// the chunk's work. A claim returns the query (-1 when every query is
// exhausted) and the chunk; it begins with a barrier, so the previous
// chunk's shared state is free to reuse.
template <typename NChunks>
__device__ __forceinline__ int claim_search(QueryWork* work, int nq, int k, int q, uint32_t& c, NChunks nchunks) {
    for (int tries = 0; tries < nq; ++tries) {
        QueryWork* wk = work + q;
        const uint32_t n = nchunks(wk);
        if (ld_volatile_u32(&wk->next[k]) < n) {
            c = atomicAdd(&wk->next[k], 1u);
            if (c < n) return q;
        }
        q = q + 1 == nq ? 0 : q + 1;
    }
    return -1;
}

// `pre`: thread 0's claim issued at the start of the current chunk of query
// `q` (or ~0u for none, e.g. before the first chunk).
template <typename NChunks>
__device__ __forceinline__ int claim(QueryWork* work, int nq, int k, int& cur, uint32_t& chunk, uint32_t pre, int q,
                                     NChunks nchunks) {
    __shared__ int s_q;
    __shared__ uint32_t s_c;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t c = 0;
        int res;
        if (q >= 0 && pre < nchunks(work + q)) {
            res = q;
            c = pre;
        } else {
            res = claim_search(work, nq, k, q >= 0 ? q : cur, c, nchunks);
        }
        s_q = res;
        s_c = c;
    }
    __syncthreads();
    const int r = s_q;
    if (r >= 0) cur = r;
    chunk = s_c;
    return r;
}

// The block's next query: the first from `cur` on (circular) whose chunk counter `k` has work
// left, -1 if none; it takes no chunk (the block's warps claim their own). The whole block
// chooses at once: every thread tests one query (nq <= the batch slots). A serial scan by thread 0
// costs up to nq dependent L2 round trips per query switch - tens of microseconds at the end of
// every launch, when each block finds every query exhausted. Begins with a barrier (the previous
// query's shared state is free afterwards) and returns the same query in every thread.
template <typename NChunks>
__device__ __forceinline__ int select_query_block(QueryWork* work, int nq, int k, int cur, NChunks nchunks) {
    __shared__ int s_first;
    __syncthreads();
    if (threadIdx.x == 0) s_first = 0x7FFFFFFF;
    __syncthreads();
    for (int t = threadIdx.x; t < nq; t += blockDim.x) {
        const int q = cur + t >= nq ? cur + t - nq : cur + t;
        QueryWork* wk = work + q;
        if (ld_volatile_u32(&wk->next[k]) < nchunks(wk)) atomicMin(&s_first, t);
    }
    __syncthreads();
    const int t = s_first;
    if (t == 0x7FFFFFFF) return -1;
    return cur + t >= nq ? cur + t - nq : cur + t;
}

__device__ __forceinline__ unsigned long long warp_sum(unsigned long long v) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
    return v;
}

// Blocks a launch needs: with little work in the batch (one easy query: a few chunks) a full
// persistent grid only costs - every block loads the query's table and polls the same counters -
// so a launch with fewer chunks than kMinChunks per block retires its surplus blocks at once
// (c5 sigma 0.01 / 0.1: batch 1 10.1K -> 10.9K / 6.6K -> 7.3K q/s, batch 8 55.6K -> 62.3K / 36K;
// 8 chunks per block was slower from batch 8 up). Returns the number of active blocks (0 in a
// surplus block, which returns at once) and sets the uniform start query over the active blocks.
// Ends with a barrier.
#ifndef TSG_MIN_CHUNKS
#define TSG_MIN_CHUNKS 1
#endif
constexpr unsigned kMinChunks = TSG_MIN_CHUNKS;  // chunks per active block
template <typename NChunks>
__device__ __forceinline__ unsigned active_blocks(const QueryWork* work, int nq, NChunks nchunks, int& cur) {
    __shared__ unsigned long long s_total;
    if (threadIdx.x == 0) s_total = 0;
    __syncthreads();
    unsigned long long mine = 0;
    for (int t = threadIdx.x; t < nq; t += blockDim.x) mine += nchunks(work + t);
    mine = warp_sum(mine);
    if ((threadIdx.x & 31) == 0 && mine) atomicAdd(&s_total, mine);
    __syncthreads();
    const unsigned long long want = (s_total + kMinChunks - 1) / kMinChunks;
    const unsigned active = static_cast<unsigned>(min(static_cast<unsigned long long>(gridDim.x), max(want, 1ull)));
    if (blockIdx.x >= active) return 0;
    cur = static_cast<int>(static_cast<uint64_t>(blockIdx.x) * nq / active);
    return active;
}

// A block's first query, weighted by the queries' chunk counts: block b starts at the query
// where the running chunk total crosses (b + 1/2) / active blocks of all chunks, so every query gets
// blocks in proportion to its work and most blocks stay with one query for the whole launch
// (a uniform start leaves the blocks of easy queries switching through the batch). Up to
// kWeightedMax queries (else `fallback`). Ends with a barrier.
constexpr int kWeightedMax = 256;
template <typename NChunks>
__device__ __forceinline__ int weighted_start(const QueryWork* work, int nq, int fallback, unsigned active,
                                              NChunks nchunks) {
    __shared__ uint32_t s_w[kWeightedMax];
    __shared__ int s_start;
    if (nq < 2 || nq > kWeightedMax || nq > static_cast<int>(blockDim.x)) return fallback;
    if (static_cast<int>(threadIdx.x) < nq) s_w[threadIdx.x] = nchunks(work + threadIdx.x);
    __syncthreads();
    if (threadIdx.x < 32) {
        const int lane = threadIdx.x, per = (nq + 31) / 32, b = lane * per;
        unsigned long long mine = 0;
        for (int i = b; i < min(b + per, nq); ++i) mine += s_w[i];
        unsigned long long incl = mine;
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long v = __shfl_up_sync(0xFFFFFFFFu, incl, o);
            if (lane >= o) incl += v;
        }
        const unsigned long long total = __shfl_sync(0xFFFFFFFFu, incl, 31);
        // the first query whose inclusive prefix exceeds the block's target
        const unsigned long long target = total * (2ull * blockIdx.x + 1) / (2ull * active);
        const bool here = total > 0 && incl > target && incl - mine <= target;
        if (lane == 0) s_start = fallback;
        __syncwarp();
        if (here) {
            unsigned long long run = incl - mine;
            int q = b;
            for (int i = b; i < min(b + per, nq); ++i) {
                run += s_w[i];
                if (run > target) {
                    q = i;
                    break;
                }
            }
            s_start = q;
        }
    }
    __syncthreads();
    return s_start;
}

// Thread 0 reserves the block's next chunk of query q (read by the next claim).
__device__ __forceinline__ uint32_t claim_ahead(QueryWork* work, int q, int k) {
    return threadIdx.x == 0 ? atomicAdd(&work[q].next[k], 1u) : ~0u;
}

// ----------------------------------------------------------- prepare
// The page the query's own key falls into: the largest p with
// page_key[p] <= key (0 if none), i.e. where the query's iSAX word would be
// stored. Two parallel rounds instead of a serial binary search: the block
// counts the directory entries (every 256th page key) <= key, then counts
// the keys <= key inside that 256-page window. blockDim.x must be 256.
__device__ __forceinline__ uint32_t locate_page(const uint64_t* __restrict__ page_key,
                                                const uint64_t* __restrict__ page_dir, uint64_t P, uint64_t key) {
    __shared__ unsigned s_part[kWarps];
    const uint64_t nd = (P + 255) / 256;
    unsigned c = 0;
    for (uint64_t i = threadIdx.x; i < nd; i += blockDim.x) c += page_dir[i] <= key ? 1u : 0u;
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xFFFFFFFFu, c, o);
    if ((threadIdx.x & 31) == 0) s_part[threadIdx.x >> 5] = c;
    __syncthreads();
    unsigned dirs = 0;
    for (int i = 0; i < kWarps; ++i) dirs += s_part[i];
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

// One block per query: resets the slot, prepares the query (PAA, symbols,
// table) and picks the seed range: the leaf the query's own iSAX word
// descends to, replaced by that page alone when the leaf is an overflow leaf
// larger than seed_cap.
__global__ void __launch_bounds__(kThreads)
    k_prepare(IndexView ix, SlotView S, const float* __restrict__ queries) {
    extern __shared__ float s_q[];
    __shared__ QueryShared qs;
    const int q = blockIdx.x;
    QueryWork* wk = S.work + q;
    load_query(s_q, queries + static_cast<uint64_t>(q) * ix.n, ix.n);
    prepare_query(s_q, ix.n, ix.w, ix.bits, ix.thr, qs);
    if (ix.window < 0) {
        fill_lut(qs, ix.n, ix.w, ix.bits, S.lut + static_cast<uint64_t>(q) * S.lut_len);
        if (threadIdx.x < kMaxW) wk->qsym[threadIdx.x] = threadIdx.x < ix.w ? qs.qsym[threadIdx.x] : 0;
        if (ix.fw) fill_fine_lut(s_q, ix.n, ix.fw, S.fine_lut + static_cast<uint64_t>(q) * S.fine_lut_len);
    } else {
        // keogh_envelope (src/metrics.cpp:72-91,167-177): window max / min (exact,
        // so a direct scan equals the reference's deque), then the bands' PAA.
        float* up = s_q + ix.n;
        float* lo = s_q + 2 * ix.n;
        float* env = S.env + static_cast<uint64_t>(q) * 2 * ix.n;
        const int r = ix.window;
        for (int i = threadIdx.x; i < ix.n; i += blockDim.x) {
            const int a = max(0, i - r), b = min(ix.n - 1, i + r);
            float hi = s_q[a], lw = s_q[a];
            for (int j = a + 1; j <= b; ++j) {
                hi = fmaxf(hi, s_q[j]);
                lw = fminf(lw, s_q[j]);
            }
            up[i] = hi;
            lo[i] = lw;
            env[i] = hi;
            env[ix.n + i] = lw;
        }
        __syncthreads();
        __shared__ double s_bpaa[2][kMaxW];
        const int seg = ix.n / ix.w;
        if (threadIdx.x < 2 * ix.w) {
            const int g = threadIdx.x % ix.w, which = threadIdx.x / ix.w;  // 0: upper, 1: lower
            const float* src = which == 0 ? up : lo;
            double sum = 0.0;
            for (int j = 0; j < seg; ++j) sum = __dadd_rn(sum, static_cast<double>(src[g * seg + j]));
            s_bpaa[which][g] = __ddiv_rn(sum, static_cast<double>(seg));
        }
        __syncthreads();
        fill_lut_band(qs.thr, s_bpaa[1], s_bpaa[0], ix.n, ix.w, ix.bits, S.lut + static_cast<uint64_t>(q) * S.lut_len);
        // box bounds clamp the symbol of lower_paa (the band's first zero-gap symbol)
        if (threadIdx.x < kMaxW)
            wk->qsym[threadIdx.x] = threadIdx.x < ix.w
                ? static_cast<unsigned char>(symbol_of(qs.thr, ix.bits, s_bpaa[1][threadIdx.x]) << (8 - ix.bits))
                : 0;
    }
    const uint32_t page = locate_page(ix.page_key, ix.page_dir, ix.P, query_key(qs.qsym, ix.w));
    if (threadIdx.x == 0) {
        const uint32_t leaf = ix.page_leaf[page];
        uint32_t a = ix.leaf_off[leaf], b = ix.leaf_off[leaf + 1];
        // DTW seeds with the query's page only: every seed row is a full DTW
        // (nothing to prune against yet), the rest of the leaf goes through the filters.
        if (b - a > ix.seed_cap || ix.window >= 0) {
            a = ix.page_off[page];
            b = ix.page_off[page + 1];
        }
        wk->bsf_bits = kInfBits;
        wk->cand = b - a;
        wk->nseed = b - a;
        wk->seed_begin = a;
        wk->seed_end = b;
        wk->ngroups = 0;
        wk->runs = 0;
        wk->ndefer = 0;
        for (int k = 0; k < kNextCount; ++k) wk->next[k] = 0;
        wk->done_blocks = 0;
        wk->best_pos = 0xFFFFFFFFu;
        wk->overflow = (b - a) > S.cap ? 1u : 0u;
        wk->scan_bound = 0.f;
        wk->boxes = 0;
        wk->fine_calcs = 0;
        wk->nties = 0;
        for (int k = 0; k < 6; ++k) wk->stats[k] = 0;
        wk->stats[kRealDist] = 0;  // the seed kernels count the rows they refine
    }
}

// -------------------------------------------------------------- seed
// Grid (x, query): every entry of the seed range is refined; 32 row groups
// per block.
template <bool VEC>
__global__ void __launch_bounds__(kThreads)
    k_seed(IndexView ix, SlotView S, const float* __restrict__ queries) {
    extern __shared__ double s_qd[];
    const int q = blockIdx.y;
    QueryWork* wk = S.work + q;
    const uint32_t a = wk->seed_begin, b = wk->seed_end;
    constexpr int kGroups = kThreads / kRowLanes;
    if (wk->overflow || a + static_cast<uint64_t>(blockIdx.x) * kGroups >= b) return;
    load_query_f64(s_qd, queries + static_cast<uint64_t>(q) * ix.n, ix.n);
    uint32_t* cand_pos = S.cand_pos + q * S.cap;
    double* cand_sq = S.cand_sq + q * S.cap;
    const int lane = threadIdx.x & 31;
    const uint64_t group = static_cast<uint64_t>(blockIdx.x) * kGroups + threadIdx.x / kRowLanes;
    const uint64_t ngroups = static_cast<uint64_t>(gridDim.x) * kGroups;
    unsigned long long updates = 0, refined = 0;
    // With the fine summary (Euclidean) the seed runs on few blocks per query: rows of the later
    // rounds first take their fine bound (the query's table read through L1) against the BSF
    // the earlier rounds found, and most are never read.
    const bool fine = ix.fine != nullptr && ix.window < 0;
    const float* flut = fine ? S.fine_lut + static_cast<uint64_t>(q) * S.fine_lut_len : nullptr;
    const int j8 = lane & (kRowLanes - 1);
    const unsigned gmask = 0xFFu << (lane & ~(kRowLanes - 1));
    // The next row's position and (32-wide fine summary) its four fine bytes of this lane are
    // loaded one row ahead: the per-row chain position -> fine bytes -> table -> row was serial.
    const bool fine32 = fine && ix.fw == 32;
    uint64_t e = a + group;
    uint32_t p = e < b ? ix.pos[e] : 0u;
    uint32_t fb = fine32 && e < b ? *reinterpret_cast<const uint32_t*>(ix.fine + e * ix.fws + 4 * j8) : 0u;
    for (; e < b; e += ngroups) {  // groups run independently
        const uint64_t en = e + ngroups;
        const uint32_t p_cur = p, fb_cur = fb;
        if (en < b) {
            p = ix.pos[en];
            if (fine32) fb = *reinterpret_cast<const uint32_t*>(ix.fine + en * ix.fws + 4 * j8);
        }
        if (fine && e >= a + ngroups) {
            const uint8_t* f = ix.fine + e * ix.fws;  // fine rows are in index order
            float acc = 0.f;
            if (fine32) {
#pragma unroll
                for (int i = 0; i < 4; ++i)
                    acc = __fadd_rd(acc, __ldg(flut + (4 * j8 + i) * 256 + ((fb_cur >> (8 * i)) & 255u)));
            } else {
                for (int sg = j8; sg < ix.fw; sg += kRowLanes) acc = __fadd_rd(acc, __ldg(flut + sg * 256 + f[sg]));
            }
#pragma unroll
            for (int o = kRowLanes / 2; o > 0; o >>= 1) acc = __fadd_rd(acc, __shfl_xor_sync(gmask, acc, o));
            if (acc > bound_from_bits(ld_volatile_u64(&wk->bsf_bits))) {
                if (j8 == 0) {
                    cand_pos[e - a] = static_cast<uint32_t>(e);
                    cand_sq[e - a] = INFINITY;
                }
                continue;
            }
        }
        const double s = group_row_sq<VEC>(ix.rows + static_cast<uint64_t>(p_cur) * ix.n, s_qd, ix.n, &wk->bsf_bits);
        if (j8 == 0) {
            cand_pos[e - a] = static_cast<uint32_t>(e);  // candidate records hold index entries
            updates += publish(wk, s, e - a, cand_sq, ~0u);
            refined += 1;
        }
    }
    if (updates) atomicAdd(&wk->stats[kBsfUpd], updates);
    if (refined) atomicAdd(&wk->stats[kRealDist], refined);
}

// ------------------------------------------------------------ groups
// Levels 1 and 0 of the box filter, the flat analog of the tree's internal
// nodes: one box per group of kGroup consecutive pages, and one per "top" of
// kGroup consecutive groups. Grid (x, query); per round a block bounds kGP
// tops per thread, lists the surviving tops in shared memory, then bounds
// their groups (one per thread); surviving groups are listed per query
// (block-aggregated) for the page level.
constexpr int kGP = 4;  // tops per thread per round

template <int WS, bool W16>
__global__ void __launch_bounds__(kThreads)
    k_groups(IndexView ix, SlotView S) {
    constexpr int H = WS / 16;
    extern __shared__ float s_lut[];
    __shared__ __align__(16) unsigned char qsym[kMaxW];
    __shared__ uint32_t s_top[kThreads * kGP];
    __shared__ unsigned s_ntop;
    const int q = blockIdx.y;
    QueryWork* wk = S.work + q;
    if (wk->overflow) return;
    load_prepared(S.lut + static_cast<uint64_t>(q) * S.lut_len, wk, ix.w, s_lut, qsym);
    uint4 q4[H];
#pragma unroll
    for (int h = 0; h < H; ++h) q4[h] = *reinterpret_cast<const uint4*>(qsym + 16 * h);
    const float bound = bound_from_bits(wk->bsf_bits);
    if (blockIdx.x == 0 && threadIdx.x == 0) wk->scan_bound = bound;
    uint32_t* gsurv = S.gsurv + q * S.NG;
    unsigned long long pruned = 0, nodes = 0;
    constexpr uint64_t kRound = static_cast<uint64_t>(kThreads) * kGP;
    for (uint64_t base = static_cast<uint64_t>(blockIdx.x) * kRound; base < ix.NT;
         base += static_cast<uint64_t>(gridDim.x) * kRound) {
        if (threadIdx.x == 0) s_ntop = 0;
        __syncthreads();
        // tops: kGP per thread, loads first
        uint4 bl[kGP][H], bh[kGP][H];
#pragma unroll
        for (int k = 0; k < kGP; ++k) {
            const uint64_t t = base + threadIdx.x + static_cast<uint64_t>(kThreads) * k;
#pragma unroll
            for (int h = 0; h < H; ++h) {
                bl[k][h] = t < ix.NT ? ld_stream_u4(ix.top_lo + t * WS + 16 * h) : make_uint4(0, 0, 0, 0);
                bh[k][h] = t < ix.NT ? ld_stream_u4(ix.top_hi + t * WS + 16 * h) : make_uint4(0, 0, 0, 0);
            }
        }
#pragma unroll
        for (int k = 0; k < kGP; ++k) {
            const uint64_t t = base + threadIdx.x + static_cast<uint64_t>(kThreads) * k;
            if (t >= ix.NT) continue;
            nodes += 1;
            if (box_bound<H, W16>(s_lut, q4, bl[k], bh[k], ix.w) <= bound) s_top[atomicAdd(&s_ntop, 1u)] = static_cast<uint32_t>(t);
            else pruned += 1;
        }
        __syncthreads();
        // groups of the surviving tops: kGP per thread per step, loads first, and one warp-
        // aggregated reservation per step (one item per step was a dependent chain of a box load
        // and an atomic's round trip: groups + bound 6.60 -> 6.31 us per c2 query)
        const unsigned items = s_ntop * kGroup;
        const unsigned lane = threadIdx.x & 31, below = (1u << lane) - 1u;
        for (unsigned i0 = 0; i0 < items; i0 += kThreads * kGP) {
            uint64_t g[kGP];
            uint4 gl[kGP][H], gh[kGP][H];
#pragma unroll
            for (int k = 0; k < kGP; ++k) {
                const unsigned i = i0 + k * kThreads + threadIdx.x;
                g[k] = i < items ? static_cast<uint64_t>(s_top[i / kGroup]) * kGroup + i % kGroup : ix.NG;
#pragma unroll
                for (int h = 0; h < H; ++h) {
                    gl[k][h] = g[k] < ix.NG ? ld_stream_u4(ix.group_lo + g[k] * WS + 16 * h) : make_uint4(0, 0, 0, 0);
                    gh[k][h] = g[k] < ix.NG ? ld_stream_u4(ix.group_hi + g[k] * WS + 16 * h) : make_uint4(0, 0, 0, 0);
                }
            }
            unsigned m[kGP], total = 0;
            bool keep[kGP];
#pragma unroll
            for (int k = 0; k < kGP; ++k) {
                keep[k] = false;
                if (g[k] < ix.NG) {
                    nodes += 1;
                    keep[k] = box_bound<H, W16>(s_lut, q4, gl[k], gh[k], ix.w) <= bound;
                    pruned += keep[k] ? 0 : 1;
                }
                m[k] = __ballot_sync(0xFFFFFFFFu, keep[k]);
                total += __popc(m[k]);
            }
            uint32_t at = 0;
            if (lane == 0 && total) at = atomicAdd(&wk->ngroups, total);
            at = __shfl_sync(0xFFFFFFFFu, at, 0);
#pragma unroll
            for (int k = 0; k < kGP; ++k) {
                if (keep[k]) gsurv[at + __popc(m[k] & below)] = static_cast<uint32_t>(g[k]);
                at += __popc(m[k]);
            }
        }
    }
    pruned = warp_sum(pruned);
    nodes = warp_sum(nodes);
    if ((threadIdx.x & 31) == 0) {
        if (pruned) atomicAdd(&wk->stats[kPruned], pruned);
        if (nodes) atomicAdd(&wk->stats[kLbNode], nodes);
    }
}

// ------------------------------------------------------------- bound
// Levels 2 and 3: the pages of the surviving groups, then the aligned
// kRun-entry runs of the surviving pages (persistent, affinity chunks of
// kThreads x kGP pages). A page survives when its bound is within the BSF
// (and it is not inside the seed range); its runs are then bounded by all
// threads of the block at once (the chunk's surviving pages are compacted in
// shared memory and each thread takes (page, run) items), and every run within
// the BSF is listed, clipped to its page: run wave 0 (bound <= split x BSF,
// front of the slot's run list) or wave 1 (back). Survivors are staged per
// warp and written with one 64-bit atomic per flush (both waves' counts).
// Pages are cut on run boundaries inside a leaf and the first page of a leaf ends at the kPage-th
// entry from the start of its first run (build.cu first_page_end): every page lies within kPage /
// kRun aligned runs (an arbitrary 128-entry window would touch 9).
constexpr int kRunsPerPage = kPage / kRun;
#ifndef TSG_RUN_STAGE
#define TSG_RUN_STAGE 256  // 128 until round 2e: half the flushes (each an atomic round trip), bound 5.77 -> 5.66 us/query; 64: 6.06
#endif
constexpr int kRunStage = TSG_RUN_STAGE;  // staged surviving runs per warp
#ifndef TSG_BOUND_PL
#define TSG_BOUND_PL 2
#endif
constexpr int kBoundPL = TSG_BOUND_PL;  // pages per lane per bound chunk

__device__ __forceinline__ void flush_runs(QueryWork* wk, uint32_t a_r, uint32_t a_l, int cnt, int lo_cnt, int lane,
                                           float cut, uint32_t rcap, uint2* __restrict__ surv,
                                           float* __restrict__ surv_lb) {
    // one 64-bit atomic reserves both waves' slots for the whole stage (lo_cnt: the staged runs
    // with bound <= cut, counted while staging)
    unsigned long long old = 0;
    if (lane == 0) {
        old = atomicAdd(&wk->runs, static_cast<unsigned long long>(lo_cnt) |
                                       (static_cast<unsigned long long>(cnt - lo_cnt) << 32));
        if ((old & 0xFFFFFFFFull) + (old >> 32) + cnt > rcap)
            atomicExch(&wk->overflow, 1u);  // cannot happen with rcap = R + P; never write out of range
    }
    old = __shfl_sync(0xFFFFFFFFu, old, 0);
    uint32_t at_lo = static_cast<uint32_t>(old), at_hi = static_cast<uint32_t>(old >> 32);
    const unsigned below = (1u << lane) - 1u;
    for (int i0 = 0; i0 < cnt; i0 += 32) {
        const int i = i0 + lane;
        const bool valid = i < cnt;
        const float lb = valid ? lds_f32(a_l + 4u * i) : 0.f;
        const uint2 r = valid ? lds_u2(a_r + 8u * i) : make_uint2(0, 0);
        const bool low = valid && lb <= cut;
        const unsigned ml = __ballot_sync(0xFFFFFFFFu, low), mh = __ballot_sync(0xFFFFFFFFu, valid && !low);
        if (low) {
            const uint32_t at = at_lo + __popc(ml & below);
            if (at < rcap) {
                surv[at] = r;
                surv_lb[at] = lb;
            }
        } else if (valid) {
            const uint32_t off = at_hi + __popc(mh & below);
            if (off < rcap) {
                surv[rcap - 1 - off] = r;
                surv_lb[rcap - 1 - off] = lb;
            }
        }
        at_lo += __popc(ml);
        at_hi += __popc(mh);
    }
    __syncwarp();
}

template <int WS, bool W16>
__global__ void __launch_bounds__(kThreads, TSG_MINB_BOUND)
    k_bound(IndexView ix, SlotView S, int nq, int pass) {
    constexpr int H = WS / 16;
    constexpr uint32_t kWChunk = 32 * kBoundPL;  // pages per warp chunk (kBoundPL per lane)
    const int k_next = pass == 0 ? kNextBound : kNextBound1;
    extern __shared__ float s_lut[];
    __shared__ __align__(16) unsigned char qsym[kMaxW];
    __shared__ uint2 s_pg[kWarps][kWChunk];      // the warp chunk's surviving pages
    __shared__ uint2 s_r[kWarps][kRunStage];     // staged surviving runs
    __shared__ float s_l[kWarps][kRunStage];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t a_pg = smem_addr(&s_pg[warp][0]), a_r = smem_addr(&s_r[warp][0]), a_l = smem_addr(&s_l[warp][0]);
    const unsigned below = (1u << lane) - 1u;
    int cur = static_cast<int>(static_cast<uint64_t>(blockIdx.x) * nq / gridDim.x);
    uint4 q4[H];
    uint32_t pruned = 0, nodes = 0;  // per lane and query
    int cnt = 0, cnt_lo = 0;         // staged runs, and those of them for wave 0 (bound <= cut)
    auto nchunks = [pass](const QueryWork* wk) -> uint32_t {
        if (wk->overflow) return 0;
        const uint32_t items = pass == 0 ? wk->ngroups * static_cast<uint32_t>(kGroup) : wk->ndefer;
        return (items + kWChunk - 1) / kWChunk;
    };
    if (!active_blocks(S.work, nq, nchunks, cur)) return;
    for (;;) {
        // Query loop (block level; the only barriers): pick a query with
        // chunks left and load its table; the warps then claim chunks of it
        // on their own until it is exhausted.
        const int q = select_query_block(S.work, nq, k_next, cur, nchunks);
        if (q < 0) break;
        cur = q;
        QueryWork* wk = S.work + q;
        load_prepared(S.lut + static_cast<uint64_t>(q) * S.lut_len, wk, ix.w, s_lut, qsym);
#pragma unroll
        for (int h = 0; h < H; ++h) q4[h] = *reinterpret_cast<const uint4*>(qsym + 16 * h);
        // pass 0: the seed bound; pass 1 (after refinement wave A): the tightened BSF
        const float bound = pass == 0 ? wk->scan_bound : bound_from_bits(ld_volatile_u64(&wk->bsf_bits));
        const float cut = pass == 0 ? bound * ix.split : -1.f;  // wave 0: the most promising runs
        const uint32_t sa = wk->seed_begin, sb = wk->seed_end;
        const uint32_t* gsurv = S.gsurv + q * S.NG;
        uint2* surv = S.surv + q * S.rcap;
        float* surv_lb = S.surv_lb + q * S.rcap;
        uint2* dpage = S.dpage + q * S.P;
        float* dpage_lb = S.dpage_lb + q * S.P;
        const uint64_t items = pass == 0 ? static_cast<uint64_t>(wk->ngroups) * kGroup : wk->ndefer;
        const uint32_t nch = nchunks(wk);
        uint32_t chunk = 0;
        if (lane == 0) chunk = atomicAdd(&wk->next[k_next], 1u);
        chunk = __shfl_sync(0xFFFFFFFFu, chunk, 0);
        while (chunk < nch) {
            uint32_t pre = 0;
            if (lane == 0) pre = atomicAdd(&wk->next[k_next], 1u);  // read after this chunk
            // pages: two per lane
            bool keep[kBoundPL], defer[kBoundPL];
            uint32_t ea[kBoundPL], eb[kBoundPL];
            float plb[kBoundPL];
            if (pass == 0) {
                uint4 bl[kBoundPL][H], bh[kBoundPL][H];
                bool valid[kBoundPL];
#pragma unroll
                for (int k = 0; k < kBoundPL; ++k) {
                    const uint64_t i = static_cast<uint64_t>(chunk) * kWChunk + 32 * k + lane;
                    const uint64_t p = i < items ? static_cast<uint64_t>(gsurv[i / kGroup]) * kGroup + i % kGroup : ix.P;
                    valid[k] = p < ix.P;
#pragma unroll
                    for (int h = 0; h < H; ++h) {
                        bl[k][h] = valid[k] ? ld_stream_u4(ix.page_lo + p * WS + 16 * h) : make_uint4(0, 0, 0, 0);
                        bh[k][h] = valid[k] ? ld_stream_u4(ix.page_hi + p * WS + 16 * h) : make_uint4(0, 0, 0, 0);
                    }
                    ea[k] = valid[k] ? ix.page_off[p] : 0u;
                    eb[k] = valid[k] ? ix.page_off[p + 1] : 0u;
                }
#pragma unroll
                for (int k = 0; k < kBoundPL; ++k) {
                    keep[k] = defer[k] = false;
                    plb[k] = 0.f;
                    if (!valid[k]) continue;
                    nodes += 1;
                    const float lb = box_bound<H, W16>(s_lut, q4, bl[k], bh[k], ix.w);
                    plb[k] = lb;
                    const bool seeded = ea[k] >= sa && eb[k] <= sb;
                    keep[k] = !seeded && lb <= cut;
                    defer[k] = !seeded && lb > cut && lb <= bound;
                    pruned += !seeded && lb > bound ? 1 : 0;
                }
                // pages beyond split x bound wait for pass 1 (one atomic per warp and chunk)
                unsigned dm[kBoundPL], dtotal = 0;
#pragma unroll
                for (int k = 0; k < kBoundPL; ++k) {
                    dm[k] = __ballot_sync(0xFFFFFFFFu, defer[k]);
                    dtotal += __popc(dm[k]);
                }
                uint32_t base = 0;
                if (lane == 0 && dtotal) base = atomicAdd(&wk->ndefer, dtotal);
                base = __shfl_sync(0xFFFFFFFFu, base, 0);
#pragma unroll
                for (int k = 0; k < kBoundPL; ++k) {
                    if (defer[k]) {
                        const uint32_t at = base + __popc(dm[k] & below);
                        dpage[at] = make_uint2(ea[k], eb[k]);
                        dpage_lb[at] = plb[k];
                    }
                    base += __popc(dm[k]);
                }
            } else {
                // the deferred pages, re-tested against the tightened BSF
#pragma unroll
                for (int k = 0; k < kBoundPL; ++k) {
                    const uint64_t i = static_cast<uint64_t>(chunk) * kWChunk + 32 * k + lane;
                    const bool in = i < items;
                    const uint2 r = in ? dpage[i] : make_uint2(0, 0);
                    ea[k] = r.x;
                    eb[k] = r.y;
                    keep[k] = in && dpage_lb[i] <= bound;
                    defer[k] = false;
                    pruned += in && !keep[k] ? 1 : 0;
                }
            }
            // the warp's surviving pages, then their runs (kRunsPerPage items per page)
            uint32_t np = 0;
#pragma unroll
            for (int k = 0; k < kBoundPL; ++k) {
                const unsigned m = __ballot_sync(0xFFFFFFFFu, keep[k]);
                if (keep[k]) sts_u2(a_pg + 8u * (np + __popc(m & below)), make_uint2(ea[k], eb[k]));
                np += __popc(m);
            }
            __syncwarp();
            const uint32_t nri = np * kRunsPerPage;
            for (uint32_t j0 = 0; j0 < nri; j0 += 64) {
                bool ok[2];
                uint32_t e0[2], e1[2];
                uint4 rl[2][H], rh[2][H];
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    const uint32_t j = j0 + 32 * u + lane;
                    ok[u] = false;
                    e0[u] = e1[u] = 0;
                    uint64_t r = 0;
                    if (j < nri) {
                        const uint2 pg = lds_u2(a_pg + 8u * (j / kRunsPerPage));
                        r = pg.x / kRun + j % kRunsPerPage;
                        e0[u] = max(pg.x, static_cast<uint32_t>(r * kRun));
                        e1[u] = min(pg.y, static_cast<uint32_t>(r * kRun + kRun));
                        ok[u] = e0[u] < e1[u];
                    }
                    if constexpr (H == 1) {
                        rl[u][0] = rh[u][0] = make_uint4(0, 0, 0, 0);
                        if (ok[u]) ld_box_pair(ix.run_lo + r * 2 * WS, rl[u][0], rh[u][0]);
                    } else {
#pragma unroll
                        for (int h = 0; h < H; ++h) {
                            rl[u][h] = ok[u] ? ld_stream_u4(ix.run_lo + r * 2 * WS + 16 * h) : make_uint4(0, 0, 0, 0);
                            rh[u][h] = ok[u] ? ld_stream_u4(ix.run_hi + r * 2 * WS + 16 * h) : make_uint4(0, 0, 0, 0);
                        }
                    }
                }
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    const float lb = ok[u] ? box_bound<H, W16>(s_lut, q4, rl[u], rh[u], ix.w) : INFINITY;
                    const bool pass_ = ok[u] && lb <= bound;
                    nodes += ok[u] ? 1 : 0;  // run boxes are node bounds (box_calcs counts quads)
                    pruned += ok[u] && !pass_ ? 1 : 0;
                    const unsigned m = __ballot_sync(0xFFFFFFFFu, pass_);
                    if (pass_) {
                        const int slot = cnt + __popc(m & below);
                        sts_u2(a_r + 8u * slot, make_uint2(e0[u], e1[u]));
                        sts_f32(a_l + 4u * slot, lb);
                    }
                    cnt += __popc(m);
                    if (pass == 0) cnt_lo += __popc(__ballot_sync(0xFFFFFFFFu, pass_ && lb <= cut));
                    __syncwarp();
                    if (cnt > kRunStage - 32) {
                        flush_runs(wk, a_r, a_l, cnt, cnt_lo, lane, cut, static_cast<uint32_t>(S.rcap), surv, surv_lb);
                        cnt = cnt_lo = 0;
                    }
                }
            }
            chunk = __shfl_sync(0xFFFFFFFFu, pre, 0);
        }
        // leave the query: the stage and the counters
        if (cnt) flush_runs(wk, a_r, a_l, cnt, cnt_lo, lane, cut, static_cast<uint32_t>(S.rcap), surv, surv_lb);
        cnt = cnt_lo = 0;
        const unsigned long long pr = warp_sum(static_cast<unsigned long long>(pruned));
        const unsigned long long nd = warp_sum(static_cast<unsigned long long>(nodes));
        if (lane == 0) {
            if (pr) atomicAdd(&wk->stats[kPruned], pr);
            if (nd) atomicAdd(&wk->stats[kLbNode], nd);
        }
        pruned = nodes = 0;
    }
}

// ------------------------------------------------------------ lbscan

#ifndef TSG_STAGE_CAP
#define TSG_STAGE_CAP 256  // 512 costs lbscan a block per SM (11.85 -> 13.4 us/query)
#endif
constexpr int kStageCap = TSG_STAGE_CAP;  // staged candidates per warp
#ifndef TSG_SCAN_QK
#define TSG_SCAN_QK 2
#endif

// Writes a warp's staged candidates: refinement wave A (bound <= cut) grows
// upward after the seed range, wave B downward from the top of the slot's
// candidate arrays; both counts are reserved with one 64-bit atomic so a
// slot that would overflow is detected exactly (the query is then flagged
// and rerun with a full-size slot; nothing is written out of range).
// cut = +inf sends everything to A, cut < 0 everything to B.
__device__ __forceinline__ void flush_stage(QueryWork* wk, uint32_t a_pos, uint32_t a_lb, int cnt, int lo_cnt, int lane,
                                            float cut, uint64_t cap, uint32_t* __restrict__ cand_pos,
                                            float* __restrict__ cand_lb) {
    // one 64-bit atomic reserves both waves' records for the whole stage (per 32
    // records it contended on c4, where every warp queues millions per query);
    // lo_cnt: the staged records with bound <= cut, counted while staging
    unsigned long long old = 0;
    if (lane == 0) {
        old = atomicAdd(&wk->cand, static_cast<unsigned long long>(lo_cnt) |
                                       (static_cast<unsigned long long>(cnt - lo_cnt) << 32));
        if ((old & 0xFFFFFFFFull) + (old >> 32) + cnt > cap) atomicExch(&wk->overflow, 1u);
    }
    old = __shfl_sync(0xFFFFFFFFu, old, 0);
    uint64_t bl = old & 0xFFFFFFFFull, bh = old >> 32;
    const unsigned below = (1u << lane) - 1u;
    for (int i0 = 0; i0 < cnt; i0 += 32) {
        const int i = i0 + lane;
        const bool valid = i < cnt;
        const float lb = valid ? lds_f32(a_lb + 4u * i) : 0.f;
        const bool low = valid && lb <= cut;
        const uint32_t row = valid ? lds_u32(a_pos + 4u * i) : 0u;  // index entries (mapped to rows only when refined)
        const unsigned ml = __ballot_sync(0xFFFFFFFFu, low), mh = __ballot_sync(0xFFFFFFFFu, valid && !low);
        if (low) {
            const uint64_t at = bl + __popc(ml & below);
            if (at < cap) {
                cand_pos[at] = row;
                cand_lb[at] = lb;
            }
        } else if (valid) {
            const uint64_t off = bh + __popc(mh & below);
            if (off < cap) {
                cand_pos[cap - 1 - off] = row;
                cand_lb[cap - 1 - off] = lb;
            }
        }
        bl += __popc(ml);
        bh += __popc(mh);
    }
    __syncwarp();
}

// One run wave (persistent; warps claim chunks of 32 listed runs): wave 0
// scans the front of the slot's run list, wave 1 the back, re-filtered
// against the BSF that refinement wave A tightened. Below the run sit the
// aligned kQuad-entry quads, bounded like the other boxes:
//   runs:  a lane takes one listed run (clipped to its page); those still
//          within the BSF queue in shared memory;
//   quads: eight queued runs at a time, lane 4k + u bounds quad u of run k;
//          surviving quads queue likewise;
//   words: sixteen queued quads at a time, each lane bounds the words of
//          entry u of two queued quads.
// Only the words of surviving quads are read. Candidates are staged per warp
// and flushed when the stage fills or the block moves to another query.
template <int WS, bool W16>
__global__ void __launch_bounds__(kThreads, TSG_MINB_LBSCAN)
    k_lbscan(IndexView ix, SlotView S, int nq, int wave) {
    constexpr int kRing = 64;  // per-warp ring queues (entry ranges), power of two
    constexpr int kQK = TSG_SCAN_QK;  // words per lane per drain (at most 8 kQK - 1 + 32 quads queue: kQK <= 4)
    constexpr int H = WS / 16;
    extern __shared__ float s_lut[];
    __shared__ __align__(16) unsigned char qsym[kMaxW];
    __shared__ uint32_t s_pos[kWarps][kStageCap];
    __shared__ float s_lb[kWarps][kStageCap];
    __shared__ uint2 s_rq[kWarps][kRing];  // surviving runs
    __shared__ uint2 s_qq[kWarps][kRing];  // surviving quads
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t a_rq = smem_addr(&s_rq[warp][0]), a_qq = smem_addr(&s_qq[warp][0]);
    const uint32_t a_pos = smem_addr(&s_pos[warp][0]), a_lb = smem_addr(&s_lb[warp][0]);
    const unsigned below = (1u << lane) - 1u;
    int cur = static_cast<int>(static_cast<uint64_t>(blockIdx.x) * nq / gridDim.x);
    uint4 q4[H];
    float bound = 0.f, cut = 0.f;
    QueryWork* wk = nullptr;
    uint32_t* cand_pos = nullptr;
    float* cand_lb = nullptr;
    const uint2* surv = nullptr;
    const float* surv_lb = nullptr;
    int cnt = 0, cnt_lo = 0;                  // staged candidates, and those of them for wave A (bound <= cut)
    uint32_t rh = 0, rt = 0, qh = 0, qt = 0;  // ring heads / tails (warp-uniform)
    uint32_t scanned = 0, pruned = 0, boxes = 0;  // per lane and query (32-bit: one add per count in the hot loops)
    const int k_next = wave == 0 ? kNextScan0 : kNextScan1;
    auto nchunks = [wave](const QueryWork* w) -> uint32_t {
        if (w->overflow) return 0;
        const unsigned long long r = w->runs;
        const uint32_t ns = static_cast<uint32_t>(wave == 0 ? (r & 0xFFFFFFFFull) : (r >> 32));
        return (ns + 31) / 32;
    };
    auto leave_query = [&]() {  // flush this warp's stage and counters to the loaded query
        if (cnt) flush_stage(wk, a_pos, a_lb, cnt, cnt_lo, lane, cut, S.cap, cand_pos, cand_lb);
        cnt = cnt_lo = 0;
        const unsigned long long sc = warp_sum(static_cast<unsigned long long>(scanned));
        const unsigned long long pr = warp_sum(static_cast<unsigned long long>(pruned));
        const unsigned long long bx = warp_sum(static_cast<unsigned long long>(boxes));
        if (lane == 0) {
            if (sc) atomicAdd(&wk->stats[kLbEntry], sc);
            if (pr) atomicAdd(&wk->stats[kPruned], pr);
            if (bx) atomicAdd(&wk->boxes, bx);
        }
        scanned = pruned = boxes = 0;
    };

    auto stage = [&](bool pass, uint32_t e, float lb) {
        const unsigned m = __ballot_sync(0xFFFFFFFFu, pass);
        if (!m) return;
        if (pass) {
            const int slot = cnt + __popc(m & below);
            sts_u32(a_pos + 4u * slot, e);  // the flush maps entries to dataset rows
            sts_f32(a_lb + 4u * slot, lb);
        }
        cnt += __popc(m);
        if (wave == 0) cnt_lo += __popc(__ballot_sync(0xFFFFFFFFu, pass && lb <= cut));
        __syncwarp();
        if (cnt > kStageCap - 32) {
            flush_stage(wk, a_pos, a_lb, cnt, cnt_lo, lane, cut, S.cap, cand_pos, cand_lb);
            cnt = cnt_lo = 0;
        }
    };
    // Words of up to 8 kQK queued quads: lane 4j + u takes entry u of quads j, j + 8, ...
    auto drain_quads = [&]() {
        const uint32_t take = min(qt - qh, 8u * kQK);
        uint4 wv[kQK][H];
        uint32_t e[kQK];
        bool ok[kQK];
#pragma unroll
        for (int k = 0; k < kQK; ++k) {
            const uint32_t qi = 8 * k + (lane >> 2);
            ok[k] = false;
            e[k] = 0;
            if (qi < take) {
                const uint2 rr = lds_u2(a_qq + 8u * ((qh + qi) & (kRing - 1)));
                e[k] = rr.x + (lane & 3);
                ok[k] = e[k] < rr.y;
            }
#pragma unroll
            for (int h = 0; h < H; ++h)
                wv[k][h] = ok[k] ? ld_stream_u4(ix.words + static_cast<uint64_t>(e[k]) * WS + 16 * h)
                                 : make_uint4(0, 0, 0, 0);
        }
        qh += take;
#pragma unroll
        for (int k = 0; k < kQK; ++k) {
            const float lb = word_bound<W16>(s_lut, wv[k], ix.w);
            scanned += ok[k] ? 1 : 0;
            stage(ok[k] && lb <= bound, e[k], lb);
        }
    };
    // Quads of up to 8 queued runs: lane 4k + u bounds quad u of run k.
    auto drain_runs = [&]() {
        const uint32_t take = min(rt - rh, 8u);
        const uint32_t k = lane >> 2, u = lane & 3;
        bool ok = false;
        uint32_t e0 = 0, e1 = 0, qd = 0;
        if (k < take) {
            const uint2 rr = lds_u2(a_rq + 8u * ((rh + k) & (kRing - 1)));
            qd = (rr.x / kRun) * (kRun / kQuad) + u;  // the run's aligned quads
            e0 = max(rr.x, qd * kQuad);
            e1 = min(rr.y, qd * kQuad + kQuad);
            ok = e0 < e1;
        }
        uint4 bl[H], bh[H];
        if constexpr (H == 1) {
            bl[0] = bh[0] = make_uint4(0, 0, 0, 0);
            if (ok) ld_box_pair(ix.quad_lo + static_cast<uint64_t>(qd) * 2 * WS, bl[0], bh[0]);
        } else {
#pragma unroll
            for (int h = 0; h < H; ++h) {
                bl[h] = ok ? ld_stream_u4(ix.quad_lo + static_cast<uint64_t>(qd) * 2 * WS + 16 * h) : make_uint4(0, 0, 0, 0);
                bh[h] = ok ? ld_stream_u4(ix.quad_hi + static_cast<uint64_t>(qd) * 2 * WS + 16 * h) : make_uint4(0, 0, 0, 0);
            }
        }
        rh += take;
        const bool pass = ok && box_bound<H, W16>(s_lut, q4, bl, bh, ix.w) <= bound;
        pruned += ok && !pass ? 1 : 0;
        boxes += ok ? 1 : 0;
        const unsigned m = __ballot_sync(0xFFFFFFFFu, pass);
        if (pass) {
            sts_u2(a_qq + 8u * ((qt + __popc(m & below)) & (kRing - 1)), make_uint2(e0, e1));
            if (TSG_PREFETCH) prefetch_l2_bytes(ix.words + static_cast<uint64_t>(e0) * WS, (e1 - e0) * WS);  // read when 16 quads queue
        }
        qt += __popc(m);
        __syncwarp();
        while (qt - qh >= 8u * kQK) drain_quads();
    };

    // Query loop (block level; the only barriers): pick a query with chunks
    // left, load its table; then every warp claims chunks of it on its own
    // (lane 0, the next claim issued while the current chunk runs) until it
    // is exhausted, drains its queues and flushes its stage.
    if (!active_blocks(S.work, nq, nchunks, cur)) return;
    for (;;) {
        const int q = select_query_block(S.work, nq, k_next, cur, nchunks);
        if (q < 0) break;
        cur = q;
        wk = S.work + q;
        bound = bound_from_bits(wk->bsf_bits);
        load_prepared(S.lut + static_cast<uint64_t>(q) * S.lut_len, wk, ix.w, s_lut, qsym);
#pragma unroll
        for (int h = 0; h < H; ++h) q4[h] = *reinterpret_cast<const uint4*>(qsym + 16 * h);
        // Page wave 0 splits its candidates into refinement waves A and B by
        // their own bound; page wave 1 (scanned after wave A is refined)
        // feeds wave B.
        cut = wave == 0 ? wk->scan_bound * ix.split : -1.f;
        const unsigned long long rr = wk->runs;
        const uint64_t nruns = wave == 0 ? (rr & 0xFFFFFFFFull) : (rr >> 32);
        cand_pos = S.cand_pos + q * S.cap;
        cand_lb = S.cand_lb + q * S.cap;
        surv = S.surv + q * S.rcap;
        surv_lb = S.surv_lb + q * S.rcap;
        const uint32_t nch = nchunks(wk);
        uint32_t chunk = 0;
        if (lane == 0) chunk = atomicAdd(&wk->next[k_next], 1u);
        chunk = __shfl_sync(0xFFFFFFFFu, chunk, 0);
        while (chunk < nch) {
            uint32_t pre = 0;
            if (lane == 0) pre = atomicAdd(&wk->next[k_next], 1u);  // read after this chunk
            const uint64_t i = static_cast<uint64_t>(chunk) * 32 + lane;
            bool pass = false;
            uint2 run = make_uint2(0, 0);
            if (i < nruns) {
                const uint64_t slot = wave == 0 ? i : S.rcap - 1 - i;
                run = surv[slot];
                pass = wave == 0 || surv_lb[slot] <= bound;  // wave 1: re-filtered with the tightened BSF
                pruned += pass ? 0 : 1;
            }
            const unsigned m = __ballot_sync(0xFFFFFFFFu, pass);
            if (pass) {
                sts_u2(a_rq + 8u * ((rt + __popc(m & below)) & (kRing - 1)), run);
                if (TSG_PREFETCH) {  // the run's quad boxes are read a few drains later
                    const uint64_t qd0 = static_cast<uint64_t>(run.x / kRun) * (kRun / kQuad);
                    prefetch_l2_bytes(ix.quad_lo + qd0 * 2 * WS, (kRun / kQuad) * 2 * WS);  // the run's 128-byte line
                }
            }
            rt += __popc(m);
            __syncwarp();
            while (rt - rh >= 8) drain_runs();
            chunk = __shfl_sync(0xFFFFFFFFu, pre, 0);
        }
        while (rt != rh) drain_runs();
        while (qt != qh) drain_quads();
        leave_query();
    }
}

// ------------------------------------------------- fine table in shared memory
// The fine summary's [fw][256] table as the TMA refinement kernel keeps it:
// the float table (default), or half precision rounded DOWN from it
// (TSG_FINE_LUT_HALF=1: entries stay <= the exact terms, sums stay lower
// bounds, half the shared memory). Measured on c2 (profiles/ab_refine3.sh):
// three blocks per SM with the half table and 64- or 128-record chunks are
// 2-3% slower than two blocks per SM with the float table - the refinement
// waits on gathered rows, not on occupancy.
#ifndef TSG_FINE_LUT_HALF
#define TSG_FINE_LUT_HALF 0
#endif
#if TSG_FINE_LUT_HALF
using FineLutT = __half;
__device__ __forceinline__ void store_fine_lut4(FineLutT* d, float4 v) {
    d[0] = __float2half_rd(v.x);
    d[1] = __float2half_rd(v.y);
    d[2] = __float2half_rd(v.z);
    d[3] = __float2half_rd(v.w);
}
__device__ __forceinline__ float fine_lut_at(const FineLutT* t, int i) { return __half2float(t[i]); }
#else
using FineLutT = float;
__device__ __forceinline__ void store_fine_lut4(FineLutT* d, float4 v) { *reinterpret_cast<float4*>(d) = v; }
__device__ __forceinline__ float fine_lut_at(const FineLutT* t, int i) { return t[i]; }
#endif

// ------------------------------------------------- fine + refine
// One refinement wave with the fine summary (persistent, block-to-query
// affinity like lbscan; the query's [fw][256] fine table and the query row
// (FP64) in shared memory). Warps claim chunks of 32 K candidate records:
//   1. lane per record: a record whose bound is within the BSF takes its fine
//      bound (the fine row of its series, one table entry per fine segment,
//      __fadd_rd sums) — the larger of the two bounds decides;
//   2. the survivors (ballot compaction into the warp's list) are refined by
//      the warp's four 8-lane groups: 256-bit row loads, FP64 blocks added
//      left to right like squared_l2 (src/metrics.cpp:17-40), abandoned
//      against the live BSF between 256-float rounds; the BSF is an atomicMin
//      on the double bits (SharedBsf, src/query.cpp:35-42).
// Every record gets its squared distance or +inf in cand_sq (finalize).
#ifndef TSG_FINE_K
#define TSG_FINE_K 4
#endif
constexpr int kFineK = TSG_FINE_K;  // candidate records per lane per chunk
#ifndef TSG_MINB_FINE
#define TSG_MINB_FINE 2
#endif
template <int FW, int K, bool VEC>
__global__ void __launch_bounds__(kThreads, TSG_MINB_FINE)
    k_fine_refine(IndexView ix, SlotView S, const float* __restrict__ queries, int nq, int wave) {
    extern __shared__ __align__(128) unsigned char s_dyn[];
    const int fw = FW > 0 ? FW : ix.fw;
    float* s_flut = reinterpret_cast<float*>(s_dyn);                                         // [fw][256]
    double* s_qd = reinterpret_cast<double*>(s_dyn + static_cast<size_t>(fw) * 256 * 4);    // [n]
    __shared__ uint16_t s_c[kWarps][32 * K];  // kept records: offset in the chunk
    __shared__ uint32_t s_p[kWarps][32 * K];  // and their dataset rows (pos of the entry)
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int wg = lane / kRowLanes;
    const bool leader = (lane & (kRowLanes - 1)) == 0;
    int cur = static_cast<int>(static_cast<uint64_t>(blockIdx.x) * nq / gridDim.x);
    const int k_next = wave == 0 ? kNextFine0 : kNextFine1;
    auto range = [wave, &S](const QueryWork* w, uint64_t& begin, uint64_t& end) {
        const unsigned long long c = w->cand;
        if (wave == 0) {
            begin = w->nseed;
            end = c & 0xFFFFFFFFull;
        } else {
            begin = S.cap - (c >> 32);
            end = S.cap;
        }
    };
    auto nchunks = [&](const QueryWork* w) -> uint32_t {
        if (w->overflow) return 0;
        uint64_t b, e;
        range(w, b, e);
        return static_cast<uint32_t>((e - b + 32 * K - 1) / (32 * K));
    };
    unsigned long long calcs = 0, refined = 0, updates = 0;
    const unsigned active = active_blocks(S.work, nq, nchunks, cur);
    if (!active) return;
#if TSG_WEIGHTED_START
    cur = weighted_start(S.work, nq, cur, active, nchunks);
#endif
    for (;;) {
        const int q = select_query_block(S.work, nq, k_next, cur, nchunks);
        if (q < 0) break;
        cur = q;
        QueryWork* wk = S.work + q;
        {
            const float4* src = reinterpret_cast<const float4*>(S.fine_lut + static_cast<uint64_t>(q) * S.fine_lut_len);
            float4* dst = reinterpret_cast<float4*>(s_flut);
            for (int i = threadIdx.x; i < fw * 64; i += blockDim.x) dst[i] = src[i];
        }
        load_query_f64(s_qd, queries + static_cast<uint64_t>(q) * ix.n, ix.n);  // syncs
        const uint32_t* cand_pos = S.cand_pos + q * S.cap;
        const float* cand_lb = S.cand_lb + q * S.cap;
        double* cand_sq = S.cand_sq + q * S.cap;
        uint64_t begin, end;
        range(wk, begin, end);
        const uint32_t nch = nchunks(wk);
        for (;;) {
            uint32_t chunk = 0;
            if (lane == 0) chunk = atomicAdd(&wk->next[k_next], 1u);
            chunk = __shfl_sync(0xFFFFFFFFu, chunk, 0);
            if (chunk >= nch) break;
            const uint64_t c0 = begin + static_cast<uint64_t>(chunk) * (32 * K);
            float bnd = bound_from_bits(ld_volatile_u64(&wk->bsf_bits));
            bool live[K];
            uint32_t row[K];
#pragma unroll
            for (int k = 0; k < K; ++k) {
                const uint64_t c = c0 + 32 * k + lane;
                live[k] = c < end && cand_lb[c] <= bnd;
            }
#pragma unroll
            for (int k = 0; k < K; ++k) row[k] = live[k] ? cand_pos[c0 + 32 * k + lane] : 0u;  // index entries
            float acc[K];
#pragma unroll
            for (int k = 0; k < K; ++k) acc[k] = 0.f;
            for (int h = 0; 16 * h < fw; ++h) {
                uint4 v[K];
#pragma unroll
                for (int k = 0; k < K; ++k)
                    v[k] = live[k] ? ld_stream_u4(ix.fine + static_cast<uint64_t>(row[k]) * ix.fws + 16 * h)
                                   : make_uint4(0, 0, 0, 0);
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    const int sg = 16 * h + i;
                    if (FW > 0 || sg < fw) {
#pragma unroll
                        for (int k = 0; k < K; ++k) acc[k] = __fadd_rd(acc[k], s_flut[sg * 256 + byte_of(v[k], i)]);
                    }
                }
            }
            bnd = bound_from_bits(ld_volatile_u64(&wk->bsf_bits));
            uint32_t m = 0;
#pragma unroll
            for (int k = 0; k < K; ++k) {
                calcs += live[k] ? 1 : 0;
                const bool keep = live[k] && acc[k] <= bnd;
                const uint64_t c = c0 + 32 * k + lane;
                if (c < end && !keep) cand_sq[c] = INFINITY;
                const unsigned mk = __ballot_sync(0xFFFFFFFFu, keep);
                if (keep) {
                    const uint32_t slot = m + __popc(mk & ((1u << lane) - 1u));
                    s_c[warp][slot] = static_cast<uint16_t>(32 * k + lane);
                    s_p[warp][slot] = ix.pos[row[k]];
                }
                m += __popc(mk);
            }
            __syncwarp();
            for (uint32_t j = wg; j < m; j += 32 / kRowLanes) {
                const uint64_t c = c0 + s_c[warp][j];
                const double sq = group_row_sq<VEC>(ix.rows + static_cast<uint64_t>(s_p[warp][j]) * ix.n, s_qd, ix.n,
                                                    &wk->bsf_bits);
                if (leader) {
                    refined += 1;
                    updates += publish(wk, sq, c, cand_sq, s_p[warp][j]);
                }
            }
            __syncwarp();  // the warp's list is reused by the next chunk
        }
        calcs = warp_sum(calcs);
        if (lane == 0 && calcs) atomicAdd(&wk->fine_calcs, calcs);
        if (leader) {
            if (refined) atomicAdd(&wk->stats[kRealDist], refined);
            if (updates) atomicAdd(&wk->stats[kBsfUpd], updates);
        }
        calcs = refined = updates = 0;
    }
}


// ------------------------------------------------------------ refine
// One refinement wave (persistent, affinity chunks of kRefChunk candidates):
// wave 0 = records [nseed, nA), wave 1 = [cap - nB, cap). Each 8-lane group
// walks its own candidates of the chunk, the next record prefetched while the
// current row is refined; a candidate whose bound exceeds the live BSF costs
// one check.
constexpr uint32_t kRefPerGroup = 8;
constexpr uint32_t kRefChunk = (kThreads / kRowLanes) * kRefPerGroup;

template <bool VEC>
__global__ void __launch_bounds__(kThreads, TSG_MINB_REFINE)
    k_refine(IndexView ix, SlotView S, const float* __restrict__ queries, int nq, int wave) {
    extern __shared__ double s_qd[];
    constexpr uint32_t kGroups = kThreads / kRowLanes;
    const int lane = threadIdx.x & 31;
    const bool leader = (lane & (kRowLanes - 1)) == 0;
    const uint32_t g = threadIdx.x / kRowLanes;
    int cur = static_cast<int>(static_cast<uint64_t>(blockIdx.x) * nq / gridDim.x), loaded = -1;
    unsigned long long refined = 0, updates = 0;
    auto range = [wave, &S](const QueryWork* w, uint64_t& begin, uint64_t& end) {
        const unsigned long long c = w->cand;
        if (wave == 0) {
            begin = w->nseed;
            end = c & 0xFFFFFFFFull;
        } else {
            begin = S.cap - (c >> 32);
            end = S.cap;
        }
    };
    auto nchunks = [&](const QueryWork* w) -> uint32_t {
        if (w->overflow) return 0;
        uint64_t b, e;
        range(w, b, e);
        return static_cast<uint32_t>((e - b + kRefChunk - 1) / kRefChunk);
    };
    auto leave_query = [&](int q) {
        if (leader) {
            if (refined) atomicAdd(&S.work[q].stats[kRealDist], refined);
            if (updates) atomicAdd(&S.work[q].stats[kBsfUpd], updates);
        }
        refined = updates = 0;
    };
    uint32_t chunk = 0, pre = ~0u;
    const int k_next = wave == 0 ? kNextRefine0 : kNextRefine1;
    for (int q = -1;;) {
        q = claim(S.work, nq, k_next, cur, chunk, pre, q, nchunks);
        if (q < 0) break;
        pre = claim_ahead(S.work, q, k_next);
        QueryWork* wk = S.work + q;
        if (q != loaded) {
            if (loaded >= 0) leave_query(loaded);
            load_query_f64(s_qd, queries + static_cast<uint64_t>(q) * ix.n, ix.n);
            loaded = q;
        }
        const uint32_t* cand_pos = S.cand_pos + q * S.cap;
        const float* cand_lb = S.cand_lb + q * S.cap;
        double* cand_sq = S.cand_sq + q * S.cap;
        uint64_t begin, end;
        range(wk, begin, end);
        const uint64_t c0 = begin + static_cast<uint64_t>(chunk) * kRefChunk;
        const uint64_t c1 = u64min(c0 + kRefChunk, end);
        uint64_t c = c0 + g;
        float nlb = c < c1 ? cand_lb[c] : 0.f;
        uint32_t np = c < c1 ? ix.pos[cand_pos[c]] : 0u;  // candidate records hold index entries
        // Cached pruning bound: refreshed from the BSF each refinement sees,
        // so a skipped candidate costs no memory access (a stale bound only
        // refines more).
        float bnd = bound_from_bits(ld_volatile_u64(&wk->bsf_bits));
        for (; c < c1; c += kGroups) {
            const float lb = nlb;
            const uint32_t p = np;
            if (c + kGroups < c1) {
                nlb = cand_lb[c + kGroups];
                np = ix.pos[cand_pos[c + kGroups]];
            }
            if (lb > bnd) {
                if (leader) cand_sq[c] = INFINITY;
                continue;
            }
            // read the BSF for the next candidate's bound while this row is in flight
            const unsigned long long seen = ld_volatile_u64(&wk->bsf_bits);
            const double s = group_row_sq<VEC>(ix.rows + static_cast<uint64_t>(p) * ix.n, s_qd, ix.n, &wk->bsf_bits);
            if (leader) {
                refined += 1;
                updates += publish(wk, s, c, cand_sq, p);
            }
            bnd = bound_from_bits(min(seen, static_cast<unsigned long long>(__double_as_longlong(s < INFINITY ? s : INFINITY))));
        }
    }
    if (loaded >= 0) leave_query(loaded);
}

// Refinement with TMA row staging (n % 8 == 0, n in {64, 96, 128, 256, 512}).
// Blocks pick a query (barriers only when switching); each warp then claims
// chunks of kTmaChunk candidate records of it on its own: lanes keep the
// records whose bound is within the BSF (ballot compaction into the warp's
// list, row positions gathered by all 32 lanes at once), and the warp's four
// 8-lane groups walk the kept rows with two shared-memory row buffers each:
// while a group sums row j from one buffer, a 1-D bulk copy (cp.async.bulk,
// mbarrier-tracked) brings its next row into the other, so the row fetch
// overlaps the FP64 arithmetic. Sums are the blocked FP64 sums in
// squared_l2's order (whole rows: an abandoned sum only ever exceeds the
// BSF, so computing it in full changes no answer).
#ifndef TSG_TMA_CHUNK
#define TSG_TMA_CHUNK 64
#endif
constexpr uint32_t kTmaChunk = TSG_TMA_CHUNK;  // candidate records per warp chunk

// NB = n / 8 blocks per row, a compile-time constant so the row sum unrolls.
#ifndef TSG_MINB_TMA
#define TSG_MINB_TMA 4
#endif
#ifndef TSG_HALF_ROWS
#define TSG_HALF_ROWS 1
#endif
// Half-row refinement applies when a half row is a whole number of 8-block rounds.
constexpr bool tma_half_rows(int n) { return TSG_HALF_ROWS && (n / 8) % 16 == 0; }
// Floats of row buffers per 8-lane group: two whole rows, or three half rows.
constexpr int tma_group_floats(int n) { return tma_half_rows(n) ? 3 * n / 2 : 2 * n; }
#ifndef TSG_FINE_CHUNK
#define TSG_FINE_CHUNK 128
#endif
// FW > 0: the fine summary's bound (fine width FW, the query's [FW][256] table
// after the query in shared memory) filters the records in phase 1 as well;
// chunks are then 128 records and the kernel runs at two blocks per SM.
template <int NB, int FW>
#ifndef TSG_MINB_TMA_FINE
#define TSG_MINB_TMA_FINE 2
#endif
__global__ void __launch_bounds__(kThreads, FW > 0 ? TSG_MINB_TMA_FINE : TSG_MINB_TMA)
    k_refine_tma(IndexView ix, SlotView S, const float* __restrict__ queries, int nq, int wave) {
    constexpr uint32_t kChunk = FW > 0 ? static_cast<uint32_t>(TSG_FINE_CHUNK) : kTmaChunk;
    // Claims are in slices of kSlice records, up to kChunk at a time; near the end
    // of a query (fewer than kGuideTail slices left) one slice at a time, so the
    // block's warps reach the query switch together (guided scheduling).
    constexpr uint32_t kSlice = FW > 0 ? 32u : kChunk;
    constexpr uint32_t kMaxSl = kChunk / kSlice;
    constexpr uint32_t kGuideTail = 128;
    constexpr int kGroups = kThreads / kRowLanes;
    constexpr int kWarpGroups = 32 / kRowLanes;
    constexpr int n = NB * 8;
    constexpr int kTq = (NB + kRowLanes - 1) / kRowLanes;  // blocks per lane
    // half-row fetches keep the lane-ordered query layout when a half is a whole number of 8-block rounds
    constexpr bool kHalf = tma_half_rows(n);
    extern __shared__ __align__(128) unsigned char s_dyn[];
    constexpr int kGF = tma_group_floats(n);  // row buffers per group: 2 rows, or 3 half rows
    float* s_rows = reinterpret_cast<float*>(s_dyn);                                           // [kGroups][kGF]
    double* s_qd = reinterpret_cast<double*>(s_dyn + static_cast<size_t>(kGroups) * kGF * 4);  // lane-ordered query
    FineLutT* s_flut = reinterpret_cast<FineLutT*>(s_qd + 8 * 8 * kTq);                        // [FW][256]
    __shared__ __align__(8) uint64_t s_bar[kGroups][3];
    __shared__ uint32_t s_c[kWarps][kChunk], s_p[kWarps][kChunk];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = threadIdx.x / kRowLanes, j8 = lane & (kRowLanes - 1);
    const int wg = lane / kRowLanes;  // group within the warp
    const int gbase = lane & ~(kRowLanes - 1);
    const unsigned gmask = 0xFFu << gbase;
    const bool leader = j8 == 0;
    const int hsw = (j8 >> 2) & 1;
    constexpr unsigned row_bytes = static_cast<unsigned>(n) * 4u;
    for (int i = threadIdx.x; i < 3 * kGroups; i += blockDim.x) mbar_init(&s_bar[i / 3][i % 3], 1);
    if (threadIdx.x == 0) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();
    unsigned phase = 0;  // bit b: parity of this group's buffer b
    float* buf0 = s_rows + static_cast<size_t>(g) * kGF;
    int cur = static_cast<int>(static_cast<uint64_t>(blockIdx.x) * nq / gridDim.x);
    unsigned long long refined = 0, updates = 0, fine_calcs = 0;
    const int k_next = wave == 0 ? kNextRefine0 : kNextRefine1;
    auto range = [wave, &S](const QueryWork* w, uint64_t& begin, uint64_t& end) {
        const unsigned long long c = w->cand;
        if (wave == 0) {
            begin = w->nseed;
            end = c & 0xFFFFFFFFull;
        } else {
            begin = S.cap - (c >> 32);
            end = S.cap;
        }
    };
    auto nchunks = [&](const QueryWork* w) -> uint32_t {
        if (w->overflow) return 0;
        uint64_t b, e;
        range(w, b, e);
        return static_cast<uint32_t>((e - b + kSlice - 1) / kSlice);
    };
    auto issue = [&](int b, uint32_t p) {  // leader: row p -> this group's buffer b
        fence_proxy_async_smem();
        mbar_expect_tx(&s_bar[g][b], row_bytes);
        tma_copy_1d(buf0 + b * n, ix.rows + static_cast<uint64_t>(p) * n, row_bytes, &s_bar[g][b]);
    };
    // Half rows (kHalf): three half-row buffers per group at 0, n/2, n; a row's
    // first half is fetched one row ahead, its second half only if the sum of
    // the first half is still within the BSF (squared_l2's abandonment,
    // metrics.cpp:28, at half-row granularity) — most rows stop there.
    constexpr int kHB = NB / 2;                       // blocks per half row
    constexpr int kTh = (kHB + kRowLanes - 1) / kRowLanes;
    constexpr unsigned half_bytes = row_bytes / 2;
    auto hbuf = [&](int b) { return buf0 + b * (n / 2); };
    auto issue_half = [&](int b, uint32_t p, int h) {  // leader: half h of row p -> half buffer b
        fence_proxy_async_smem();
        mbar_expect_tx(&s_bar[g][b], half_bytes);
        tma_copy_1d(hbuf(b), ix.rows + static_cast<uint64_t>(p) * n + h * (n / 2), half_bytes, &s_bar[g][b]);
    };
    auto wait_buf = [&](int b) {
        mbar_wait(&s_bar[g][b], (phase >> b) & 1u);
        phase ^= 1u << b;
    };
    // Block sums of half h of a row in half buffer b, added left to right by the
    // leader onto `sum` (the leader's value is the one that counts).
    // Block sums of half h of the row in half buffer b, written back into that
    // buffer (block k at double k) for the leader's left-to-right chain.
    auto half_blocks = [&](int b, int h) {
        const float* row = hbuf(b);
        double blk[kTh];
#pragma unroll
        for (int t = 0; t < kTh; ++t) {
            const int kh = j8 + kRowLanes * t;  // block within the half
            blk[t] = 0.0;
            if (kh < kHB) {
                const float4 ua = *reinterpret_cast<const float4*>(row + 8 * kh + 4 * hsw);
                const float4 ub = *reinterpret_cast<const float4*>(row + 8 * kh + 4 * (1 - hsw));
                const float4 x0 = hsw ? ub : ua, x1 = hsw ? ua : ub;
                const float x[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
                const int tf = t + h * kTh;  // lane-ordered query block index (block j8 + 8 tf)
                double b8 = 0.0;
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const double d = __dsub_rn(static_cast<double>(x[i]), s_qd[(8 * tf + i) * 8 + j8]);
                    b8 = __dadd_rn(b8, __dmul_rn(d, d));
                }
                blk[t] = b8;
            }
        }
        double* sums = reinterpret_cast<double*>(hbuf(b));
        __syncwarp(gmask);  // every lane has read its slices
#pragma unroll
        for (int t = 0; t < kTh; ++t)
            if (j8 + kRowLanes * t < kHB) sums[j8 + kRowLanes * t] = blk[t];
    };
    auto half_sum = [&](int b, int h, double sum) -> double {
        half_blocks(b, h);
        __syncwarp(gmask);
        if (leader) {
            const double* sums = reinterpret_cast<const double*>(hbuf(b));
#pragma unroll
            for (int k = 0; k < kHB; ++k) sum = __dadd_rn(sum, sums[k]);
        }
        __syncwarp(gmask);  // the buffer is free again
        return sum;
    };
    const unsigned active = active_blocks(S.work, nq, nchunks, cur);
    if (!active) return;
#if TSG_WEIGHTED_START
    cur = weighted_start(S.work, nq, cur, active, nchunks);
#endif
    for (;;) {
        const int q = select_query_block(S.work, nq, k_next, cur, nchunks);
        if (q < 0) break;
        cur = q;
        QueryWork* wk = S.work + q;
        // The query widened to double in lane order: element i of lane j8's
        // t-th block (block j8 + 8t) at [(8t + i) * 8 + j8], so the eight
        // lanes of a group read eight consecutive doubles (no bank conflicts).
        const float* qg = queries + static_cast<uint64_t>(q) * n;
        for (int e = threadIdx.x; e < 8 * 8 * kTq; e += blockDim.x) {
            const int jj = e & 7, i = (e >> 3) & 7, t = e >> 6;
            const int k = jj + kRowLanes * t;
            s_qd[e] = k < NB ? static_cast<double>(qg[8 * k + i]) : 0.0;
        }
        if (FW > 0) {
            const float4* src = reinterpret_cast<const float4*>(S.fine_lut + static_cast<uint64_t>(q) * S.fine_lut_len);
            for (int i = threadIdx.x; i < FW * 64; i += blockDim.x) store_fine_lut4(s_flut + 4 * i, src[i]);
        }
        __syncthreads();
        const uint32_t* cand_pos = S.cand_pos + q * S.cap;
        const float* cand_lb = S.cand_lb + q * S.cap;
        double* cand_sq = S.cand_sq + q * S.cap;
        uint64_t begin, end;
        range(wk, begin, end);
        const uint32_t nch = nchunks(wk);
        // lane 0: claim the next slices; returns start | size << 32 (valid in lane 0)
        auto claim_slices = [&]() -> unsigned long long {
            const unsigned cur0 = ld_volatile_u32(&wk->next[k_next]);
            const unsigned want = kMaxSl > 1 && cur0 + kGuideTail < nch ? kMaxSl : 1u;
            const unsigned st0 = atomicAdd(&wk->next[k_next], want);
            return static_cast<unsigned long long>(st0) | (static_cast<unsigned long long>(want) << 32);
        };
        unsigned long long cl = 0;
        if (lane == 0) cl = claim_slices();
        cl = __shfl_sync(0xFFFFFFFFu, cl, 0);
        uint32_t chunk = static_cast<uint32_t>(cl), csize = static_cast<uint32_t>(cl >> 32);
        // The current chunk's records (bound, entry) are loaded one chunk ahead,
        // while the previous chunk's rows are being refined.
        constexpr int kPer = kChunk / 32;
        float rlb[kPer];
        uint32_t rcp[kPer];
        auto load_records = [&](uint32_t ch, uint32_t sz, float* lbv, uint32_t* cpv) {
#pragma unroll
            for (int k = 0; k < kPer; ++k) {
                const uint64_t c = begin + static_cast<uint64_t>(ch) * kSlice + 32 * k + lane;
                const bool in = ch < nch && 32u * k < sz * kSlice && c < end;
                lbv[k] = in ? cand_lb[c] : INFINITY;
                cpv[k] = in ? cand_pos[c] : 0u;
            }
        };
        load_records(chunk, csize, rlb, rcp);
        while (chunk < nch) {
            unsigned long long pre = 0;
            if (lane == 0) pre = claim_slices();
            const uint64_t c0 = begin + static_cast<uint64_t>(chunk) * kSlice;
            const uint64_t c1 = u64min(c0 + static_cast<uint64_t>(csize) * kSlice, end);
            // Phase 1 (warp): keep the records whose bound (then fine bound) is within the BSF.
            const float bnd = bound_from_bits(ld_volatile_u64(&wk->bsf_bits));
            bool kp[kPer];
#pragma unroll
            for (int k = 0; k < kPer; ++k) kp[k] = c0 + 32 * k + lane < c1 && rlb[k] <= bnd;
            if (FW > 0) {
                float acc[kPer];
#pragma unroll
                for (int k = 0; k < kPer; ++k) acc[k] = 0.f;
#pragma unroll
                if constexpr (FW == 32) {
                    // a 32-byte fine row (index order) in one 256-bit load: one L1 wavefront per row
                    uint4 va[kPer], vb[kPer];
#pragma unroll
                    for (int k = 0; k < kPer; ++k) {
                        va[k] = vb[k] = make_uint4(0, 0, 0, 0);
                        if (kp[k]) ld_box_pair(ix.fine + static_cast<uint64_t>(rcp[k]) * ix.fws, va[k], vb[k]);
                    }
#pragma unroll
                    for (int i = 0; i < 16; ++i)
#pragma unroll
                        for (int k = 0; k < kPer; ++k)
                            acc[k] = __fadd_rd(acc[k], fine_lut_at(s_flut, i * 256 + byte_of(va[k], i)));
#pragma unroll
                    for (int i = 0; i < 16; ++i)
#pragma unroll
                        for (int k = 0; k < kPer; ++k)
                            acc[k] = __fadd_rd(acc[k], fine_lut_at(s_flut, (16 + i) * 256 + byte_of(vb[k], i)));
                } else {
                    for (int h = 0; h < FW / 16; ++h) {
                        uint4 v[kPer];
#pragma unroll
                        for (int k = 0; k < kPer; ++k)
                            v[k] = kp[k] ? ld_stream_u4(ix.fine + static_cast<uint64_t>(rcp[k]) * ix.fws + 16 * h)  // index order
                                         : make_uint4(0, 0, 0, 0);
#pragma unroll
                        for (int i = 0; i < 16; ++i)
#pragma unroll
                            for (int k = 0; k < kPer; ++k)
                                acc[k] = __fadd_rd(acc[k], fine_lut_at(s_flut, (16 * h + i) * 256 + byte_of(v[k], i)));
                    }
                }
                const float bnd2 = bound_from_bits(ld_volatile_u64(&wk->bsf_bits));
#pragma unroll
                for (int k = 0; k < kPer; ++k) {
                    fine_calcs += kp[k] ? 1 : 0;
                    kp[k] = kp[k] && acc[k] <= bnd2;
                }
            }
            uint32_t m = 0;
#pragma unroll
            for (int k = 0; k < kPer; ++k) {
                const uint64_t c = c0 + 32 * k + lane;
                const bool in = c < c1;
                const bool keep = kp[k];
                if (in && !keep) cand_sq[c] = INFINITY;
                const unsigned mk = __ballot_sync(0xFFFFFFFFu, keep);
                if (keep) {
                    const uint32_t slot = m + __popc(mk & ((1u << lane) - 1u));
                    s_c[warp][slot] = static_cast<uint32_t>(c);
                    s_p[warp][slot] = ix.pos[rcp[k]];  // candidate records hold index entries
                }
                m += __popc(mk);
            }
            __syncwarp();
            const unsigned long long ncl = __shfl_sync(0xFFFFFFFFu, pre, 0);
            const uint32_t next = static_cast<uint32_t>(ncl), nsize = static_cast<uint32_t>(ncl >> 32);
            load_records(next, nsize, rlb, rcp);  // in flight during phase 2
            if constexpr (kHalf) {
                // Phase 2 (half rows): first halves one row ahead in buffers 0 / 1,
                // the pending second half in buffer 2, completed one row later.
                bool pending = false;
                uint32_t pend_c = 0, pend_p = 0;
                double pend_sum = 0.0;
                unsigned long long pend_seen = 0;
                if (leader && static_cast<uint32_t>(wg) < m) issue_half(0, s_p[warp][wg], 0);
                int fb = 0;
                for (uint32_t j = wg; j < m; j += kWarpGroups, fb ^= 1) {
                    if (leader && j + kWarpGroups < m) issue_half(fb ^ 1, s_p[warp][j + kWarpGroups], 0);
                    const unsigned long long seen = ld_volatile_u64(&wk->bsf_bits);
                    // this row's first half and the previous row's second half: block
                    // sums by the lanes, then the leader's two left-to-right chains
                    // interleaved (independent, so their latencies overlap)
                    wait_buf(fb);
                    half_blocks(fb, 0);
                    if (pending) {
                        wait_buf(2);
                        half_blocks(2, 1);
                    }
                    __syncwarp(gmask);
                    double part = 0.0;
                    if (leader) {
                        const double* sa = reinterpret_cast<const double*>(hbuf(fb));
                        const double* sb2 = reinterpret_cast<const double*>(hbuf(2));
                        double sum = pend_sum;
                        if (pending) {
#pragma unroll
                            for (int k = 0; k < kHB; ++k) {
                                part = __dadd_rn(part, sa[k]);
                                sum = __dadd_rn(sum, sb2[k]);
                            }
                            cand_sq[pend_c] = sum;
                            note_tie(wk, sum, pend_p, pend_seen);
                            const unsigned long long sb = static_cast<unsigned long long>(__double_as_longlong(sum));
                            if (sb < pend_seen) updates += atomicMin(&wk->bsf_bits, sb) > sb ? 1 : 0;
                        } else {
#pragma unroll
                            for (int k = 0; k < kHB; ++k) part = __dadd_rn(part, sa[k]);
                        }
                    }
                    __syncwarp(gmask);  // both buffers are free again
                    pending = false;
                    const bool cont = __shfl_sync(gmask, leader && !(part > bsf_of(seen) * kSlack), gbase);
                    if (leader) refined += 1;
                    if (cont) {
                        if (leader) issue_half(2, s_p[warp][j], 1);
                        pending = true;
                        pend_c = s_c[warp][j];
                        pend_p = s_p[warp][j];
                        pend_sum = part;
                        pend_seen = seen;
                    } else if (leader) {
                        cand_sq[s_c[warp][j]] = INFINITY;  // abandoned after its first half
                    }
                }
                if (pending) {
                    wait_buf(2);
                    const double sum = half_sum(2, 1, pend_sum);
                    if (leader) {
                        cand_sq[pend_c] = sum;
                        note_tie(wk, sum, pend_p, pend_seen);
                        const unsigned long long sb = static_cast<unsigned long long>(__double_as_longlong(sum));
                        if (sb < pend_seen) updates += atomicMin(&wk->bsf_bits, sb) > sb ? 1 : 0;
                    }
                }
                __syncwarp();  // the warp's list is reused by the next chunk
                chunk = next;
                csize = nsize;
                continue;
            }
            // Phase 2: the kept rows, double-buffered per group.
            if (leader && static_cast<uint32_t>(wg) < m) issue(0, s_p[warp][wg]);
            int b = 0;
            for (uint32_t j = wg; j < m; j += kWarpGroups, b ^= 1) {
                if (leader && j + kWarpGroups < m) issue(b ^ 1, s_p[warp][j + kWarpGroups]);
                const unsigned long long seen = ld_volatile_u64(&wk->bsf_bits);
                mbar_wait(&s_bar[g][b], (phase >> b) & 1u);
                phase ^= 1u << b;
                const float* row = buf0 + b * n;
                double blk[kTq];
#pragma unroll
                for (int t = 0; t < kTq; ++t) {
                    const int k = j8 + kRowLanes * t;
                    blk[t] = 0.0;
                    if (k < NB) {
                        // Lanes 4-7 read the halves in the other order, so the
                        // group's 16-byte reads of one instruction hit all 32 banks.
                        const float4 ua = *reinterpret_cast<const float4*>(row + 8 * k + 4 * hsw);
                        const float4 ub = *reinterpret_cast<const float4*>(row + 8 * k + 4 * (1 - hsw));
                        const float4 x0 = hsw ? ub : ua, x1 = hsw ? ua : ub;
                        const float x[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
                        double b8 = 0.0;
#pragma unroll
                        for (int i = 0; i < 8; ++i) {
                            const double d = __dsub_rn(static_cast<double>(x[i]), s_qd[(8 * t + i) * 8 + j8]);
                            b8 = __dadd_rn(b8, __dmul_rn(d, d));
                        }
                        blk[t] = b8;
                    }
                }
                // Left to right over the blocks by the group leader: the block
                // sums go through the row buffer just consumed (block k at double k).
                double* sums = reinterpret_cast<double*>(buf0 + b * n);
                __syncwarp(gmask);  // every lane has read its row slices
#pragma unroll
                for (int t = 0; t < kTq; ++t)
                    if (j8 + kRowLanes * t < NB) sums[j8 + kRowLanes * t] = blk[t];
                __syncwarp(gmask);
                if (leader) {
                    double sum = 0.0;
#pragma unroll
                    for (int k = 0; k + 1 < NB; k += 2) {
                        const double2 v = *reinterpret_cast<const double2*>(sums + k);
                        sum = __dadd_rn(__dadd_rn(sum, v.x), v.y);
                    }
                    if (NB & 1) sum = __dadd_rn(sum, sums[NB - 1]);
                    cand_sq[s_c[warp][j]] = sum;
                    note_tie(wk, sum, s_p[warp][j], seen);
                    refined += 1;
                    const unsigned long long sb = static_cast<unsigned long long>(__double_as_longlong(sum));
                    if (sb < seen) updates += atomicMin(&wk->bsf_bits, sb) > sb ? 1 : 0;
                }
                __syncwarp(gmask);  // the group is done with buffer b before it is refilled
            }
            __syncwarp();  // the warp's list is reused by the next chunk
            chunk = next;
            csize = nsize;
        }
        if (leader) {
            if (refined) atomicAdd(&wk->stats[kRealDist], refined);
            if (updates) atomicAdd(&wk->stats[kBsfUpd], updates);
        }
        if (FW > 0) {
            fine_calcs = warp_sum(fine_calcs);
            if (lane == 0 && fine_calcs) atomicAdd(&wk->fine_calcs, fine_calcs);
        }
        refined = updates = fine_calcs = 0;
    }
}

// --------------------------------------------------------------- DTW
// Banded DTW (src/metrics.cpp:112-164) by one warp along anti-diagonals: the
// cells of diagonal k = i + j inside the band |j - i| <= r are independent,
// so lane l holds band offsets u = j - i + r = 2 (l + 32 t) + p (p = parity
// of k + r, t < M slots) and each step reads its up / left neighbours from
// diagonal k - 1 by shuffles and its diagonal neighbour from k - 2 in its own
// registers. Every cell is min(up, diagonal, left) + (a_i - b_j)^2 in FP64
// (product rounded, then the sum) — the reference's recurrence, so the value
// is bit-identical (min is exact; dtw is symmetric bit for bit). Abandonment:
// every warping path meets diagonal k or k + 1 and cell values only grow
// along a path, so once both diagonals exceed cutoff_sq the distance does
// too (sound; the reference abandons per row). Returns the squared distance
// or +inf. r + 1 <= 32 M.
template <int M>
__device__ double warp_dtw_sq(const float* __restrict__ sa, const float* __restrict__ b, int n, int r,
                              double cutoff_sq) {
    const int lane = threadIdx.x & 31;
    constexpr unsigned kFull = 0xFFFFFFFFu;
    double p1[M], p2[M];
#pragma unroll
    for (int t = 0; t < M; ++t) p1[t] = p2[t] = INFINITY;
    double prev_min = INFINITY;
    for (int k = 0; k < 2 * n - 1; ++k) {
        const int p = (k + r) & 1;
        double cur[M];
        double cmin = INFINITY;
#pragma unroll
        for (int t = 0; t < M; ++t) {
            // On a diagonal of parity 0 the up neighbour is this lane's own cell
            // of diagonal k - 1 and the left one is lane - 1's; on parity 1 the
            // left one is this lane's and the up one lane + 1's (p is uniform).
            double up, left;
            if (p == 0) {
                up = p1[t];
                const double upn = __shfl_up_sync(kFull, p1[t], 1);
                const double wrap = M > 1 ? __shfl_sync(kFull, p1[t > 0 ? t - 1 : 0], 31) : INFINITY;
                left = lane == 0 ? (t > 0 ? wrap : INFINITY) : upn;
            } else {
                left = p1[t];
                const double dn = __shfl_down_sync(kFull, p1[t], 1);
                const double wrap = M > 1 ? __shfl_sync(kFull, p1[t + 1 < M ? t + 1 : t], 0) : INFINITY;
                up = lane == 31 ? (t + 1 < M ? wrap : INFINITY) : dn;
            }
            const int u = 2 * (lane + 32 * t) + p;
            const int delta = u - r;
            const int i2 = k - delta;
            const int i = i2 >> 1, j = (k + delta) >> 1;
            double cell = INFINITY;
            if (u <= 2 * r && i2 >= 0 && i < n && j >= 0 && j < n) {
                const double best = (i == 0 && j == 0) ? 0.0 : fmin(fmin(up, left), p2[t]);
                const double d = __dsub_rn(static_cast<double>(sa[i]), static_cast<double>(__ldg(b + j)));
                cell = __dadd_rn(best, __dmul_rn(d, d));
            }
            cur[t] = cell;
            cmin = fmin(cmin, cell);
        }
#pragma unroll
        for (int t = 0; t < M; ++t) {
            p2[t] = p1[t];
            p1[t] = cur[t];
        }
        if ((k & 7) == 7) {
            double m2 = fmin(cmin, prev_min);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) m2 = fmin(m2, __shfl_xor_sync(kFull, m2, o));
            if (m2 > cutoff_sq) return INFINITY;
        }
        prev_min = cmin;
    }
    // cell (n - 1, n - 1): diagonal 2n - 2, u = r
    const int idx = (r - (r & 1)) / 2;
    double v = INFINITY;
#pragma unroll
    for (int t = 0; t < M; ++t)
        if (t == (idx >> 5)) v = p1[t];
    return __shfl_sync(kFull, v, idx & 31);
}

// Two banded DTWs at once by one warp (r < 32, one band cell per lane each):
// the same recurrence as warp_dtw_sq for rows b0 and b1, interleaved so the
// two dependency chains hide each other's latency. Each abandons on its own.
__device__ void warp_dtw_sq_pair(const float* __restrict__ sa, const float* __restrict__ b0,
                                 const float* __restrict__ b1, int n, int r, double cut0, double cut1, double& out0,
                                 double& out1) {
    const int lane = threadIdx.x & 31;
    constexpr unsigned kFull = 0xFFFFFFFFu;
    double p1a = INFINITY, p2a = INFINITY, p1b = INFINITY, p2b = INFINITY;
    double prev_a = INFINITY, prev_b = INFINITY;
    bool live_a = true, live_b = true;
    for (int k = 0; k < 2 * n - 1; ++k) {
        const int p = (k + r) & 1;
        double upa, lefta, upb, leftb;
        if (p == 0) {
            upa = p1a;
            upb = p1b;
            const double la = __shfl_up_sync(kFull, p1a, 1), lb = __shfl_up_sync(kFull, p1b, 1);
            lefta = lane == 0 ? INFINITY : la;
            leftb = lane == 0 ? INFINITY : lb;
        } else {
            lefta = p1a;
            leftb = p1b;
            const double ua = __shfl_down_sync(kFull, p1a, 1), ub = __shfl_down_sync(kFull, p1b, 1);
            upa = lane == 31 ? INFINITY : ua;
            upb = lane == 31 ? INFINITY : ub;
        }
        const int u = 2 * lane + p;
        const int delta = u - r;
        const int i2 = k - delta;
        const int i = i2 >> 1, j = (k + delta) >> 1;
        double ca = INFINITY, cb = INFINITY;
        if (u <= 2 * r && i2 >= 0 && i < n && j >= 0 && j < n) {
            const double ai = static_cast<double>(sa[i]);
            const bool origin = i == 0 && j == 0;
            const double besta = origin ? 0.0 : fmin(fmin(upa, lefta), p2a);
            const double bestb = origin ? 0.0 : fmin(fmin(upb, leftb), p2b);
            const double da = __dsub_rn(ai, static_cast<double>(__ldg(b0 + j)));
            const double db = __dsub_rn(ai, static_cast<double>(__ldg(b1 + j)));
            ca = __dadd_rn(besta, __dmul_rn(da, da));
            cb = __dadd_rn(bestb, __dmul_rn(db, db));
        }
        p2a = p1a;
        p1a = ca;
        p2b = p1b;
        p1b = cb;
        if ((k & 7) == 7) {
            double ma = fmin(ca, prev_a), mb = fmin(cb, prev_b);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                ma = fmin(ma, __shfl_xor_sync(kFull, ma, o));
                mb = fmin(mb, __shfl_xor_sync(kFull, mb, o));
            }
            live_a = live_a && !(ma > cut0);
            live_b = live_b && !(mb > cut1);
            if (!live_a && !live_b) break;
        }
        prev_a = ca;
        prev_b = cb;
    }
    const int idx = (r - (r & 1)) / 2;
    const double va = __shfl_sync(kFull, p1a, idx), vb = __shfl_sync(kFull, p1b, idx);
    out0 = live_a ? va : INFINITY;
    out1 = live_b ? vb : INFINITY;
}

// LB_Keogh (src/metrics.cpp:179-192), squared, by one warp (any summation
// order: it is only a filter, compared with the same 1e-9 slack as the BSF).
__device__ __forceinline__ double warp_lb_keogh_sq(const float* __restrict__ up, const float* __restrict__ lo,
                                                   const float* __restrict__ c, int n) {
    double sum = 0.0;
    for (int i = threadIdx.x & 31; i < n; i += 32) {
        const double v = __ldg(c + i);
        double d = 0.0;
        if (v > up[i]) d = v - up[i];
        else if (v < lo[i]) d = lo[i] - v;
        sum += d * d;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xFFFFFFFFu, sum, o);
    return sum;
}

#ifndef TSG_REV_KEOGH
#define TSG_REV_KEOGH 1
#endif
constexpr bool kRevKeogh = TSG_REV_KEOGH;
// The reversed LB_Keogh (the UCR suite's second envelope bound): the query
// against the candidate's Keogh envelope (window max / min over |j - i| <= r,
// exact in float), every term from shared memory. DTW is symmetric, so this is
// a lower bound of the same DTW as the forward LB_Keogh (metrics.cpp:179-192
// with the roles swapped). w_row: the candidate row already in the warp's
// scratch; w_up / w_lo: scratch for its envelope.
__device__ __forceinline__ double warp_lb_keogh_rev_sq(const float* w_row, float* w_up, float* w_lo,
                                                       const float* s_q, int n, int r) {
    const int lane = threadIdx.x & 31;
    for (int i = lane; i < n; i += 32) {
        const int a = max(0, i - r), b = min(n - 1, i + r);
        float hi = w_row[a], lo = w_row[a];
        for (int j = a + 1; j <= b; ++j) {
            hi = fmaxf(hi, w_row[j]);
            lo = fminf(lo, w_row[j]);
        }
        w_up[i] = hi;
        w_lo[i] = lo;
    }
    __syncwarp();
    double sum = 0.0;
    for (int i = lane; i < n; i += 32) {
        const double v = s_q[i];
        double d = 0.0;
        if (v > w_up[i]) d = v - w_up[i];
        else if (v < w_lo[i]) d = w_lo[i] - v;
        sum += d * d;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xFFFFFFFFu, sum, o);
    __syncwarp();  // the scratch is free again
    return sum;
}

// LB_Keogh of one candidate row by an 8-lane group (lane j: elements j, j + 8,
// ...: each step reads 32 contiguous bytes); every lane of the group returns it.
__device__ __forceinline__ double group_lb_keogh_sq(const float* __restrict__ up, const float* __restrict__ lo,
                                                    const float* __restrict__ c, int n) {
    const int lane = threadIdx.x & 31, j = lane & (kRowLanes - 1), base = lane & ~(kRowLanes - 1);
    const unsigned gmask = 0xFFu << base;
    double sum = 0.0;
    for (int i = j; i < n; i += kRowLanes) {
        const double v = __ldg(c + i);
        double d = 0.0;
        if (v > up[i]) d = v - up[i];
        else if (v < lo[i]) d = lo[i] - v;
        sum += d * d;
    }
#pragma unroll
    for (int o = kRowLanes / 2; o > 0; o >>= 1) sum += __shfl_xor_sync(gmask, sum, o);
    return sum;
}

// One candidate row under DTW by a warp: LB_Keogh against the live BSF, then
// the banded DTW abandoning at it (calculate_real_distance_leaf's DTW branch,
// src/query.cpp:138-145). Returns the squared distance or +inf; `refined`
// tells whether the DTW ran.
template <int M>
__device__ double warp_dtw_candidate(const float* s_q, const float* s_up, const float* s_lo, const float* row, int n,
                                     int r, const QueryWork* wk, bool& refined) {
    const double cut = bsf_of(ld_volatile_u64(&wk->bsf_bits)) * kSlack;
    refined = false;
    if (warp_lb_keogh_sq(s_up, s_lo, row, n) > cut) return INFINITY;
    refined = true;
    return warp_dtw_sq<M>(s_q, row, n, r, cut);
}

// Query + envelope into shared memory: [query | upper | lower], n floats each.
__device__ __forceinline__ void load_query_env(float* s, const float* q, const float* env, int n) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        s[i] = q[i];
        s[n + i] = env[i];
        s[2 * n + i] = env[n + i];
    }
    __syncthreads();
}

// DTW seed: every row of the seed range, one warp per row. Grid (x, query).
template <int M>
__global__ void __launch_bounds__(kThreads)
    k_seed_dtw(IndexView ix, SlotView S, const float* __restrict__ queries) {
    extern __shared__ float s_qe[];
    const int q = blockIdx.y;
    QueryWork* wk = S.work + q;
    const uint32_t a = wk->seed_begin, b = wk->seed_end;
    if (wk->overflow || a + static_cast<uint64_t>(blockIdx.x) * kWarps >= b) return;
    const int n = ix.n;
    load_query_env(s_qe, queries + static_cast<uint64_t>(q) * n, S.env + static_cast<uint64_t>(q) * 2 * n, n);
    uint32_t* cand_pos = S.cand_pos + q * S.cap;
    double* cand_sq = S.cand_sq + q * S.cap;
    const int lane = threadIdx.x & 31;
    unsigned long long updates = 0, refined = 0;
    for (uint64_t e = a + static_cast<uint64_t>(blockIdx.x) * kWarps + (threadIdx.x >> 5); e < b;
         e += static_cast<uint64_t>(gridDim.x) * kWarps) {
        const uint32_t p = ix.pos[e];
        bool ran;
        const double sq = warp_dtw_candidate<M>(s_qe, s_qe + n, s_qe + 2 * n, ix.rows + static_cast<uint64_t>(p) * n,
                                                n, ix.window, wk, ran);
        if (lane == 0) {
            cand_pos[e - a] = static_cast<uint32_t>(e);
            updates += publish(wk, sq, e - a, cand_sq, ~0u);
            refined += ran ? 1 : 0;
        }
    }
    if (lane == 0) {
        if (updates) atomicAdd(&wk->stats[kBsfUpd], updates);
        if (refined) atomicAdd(&wk->stats[kRealDist], refined);
    }
}

// DTW refinement wave: blocks pick a query (barriers only when switching),
// warps claim chunks of 32 candidate records, keep those whose word bound is
// within the BSF, and refine them one at a time (LB_Keogh, then DTW).
template <int M>
__global__ void __launch_bounds__(kThreads)
    k_refine_dtw(IndexView ix, SlotView S, const float* __restrict__ queries, int nq, int wave) {
    extern __shared__ float s_qe[];
    const int n = ix.n;
    const int lane = threadIdx.x & 31;
    int cur = static_cast<int>(static_cast<uint64_t>(blockIdx.x) * nq / gridDim.x);
    const int k_next = wave == 0 ? kNextRefine0 : kNextRefine1;
    auto range = [wave, &S](const QueryWork* w, uint64_t& begin, uint64_t& end) {
        const unsigned long long c = w->cand;
        if (wave == 0) {
            begin = w->nseed;
            end = c & 0xFFFFFFFFull;
        } else {
            begin = S.cap - (c >> 32);
            end = S.cap;
        }
    };
    auto nchunks = [&](const QueryWork* w) -> uint32_t {
        if (w->overflow) return 0;
        uint64_t b, e;
        range(w, b, e);
        return static_cast<uint32_t>((e - b + 31) / 32);
    };
    unsigned long long refined = 0, updates = 0;
    const unsigned active = active_blocks(S.work, nq, nchunks, cur);
    if (!active) return;
#if TSG_WEIGHTED_START
    cur = weighted_start(S.work, nq, cur, active, nchunks);
#endif
    for (;;) {
        const int q = select_query_block(S.work, nq, k_next, cur, nchunks);
        if (q < 0) break;
        cur = q;
        QueryWork* wk = S.work + q;
        load_query_env(s_qe, queries + static_cast<uint64_t>(q) * n, S.env + static_cast<uint64_t>(q) * 2 * n, n);
        const uint32_t* cand_pos = S.cand_pos + q * S.cap;
        const float* cand_lb = S.cand_lb + q * S.cap;
        double* cand_sq = S.cand_sq + q * S.cap;
        uint64_t begin, end;
        range(wk, begin, end);
        const uint32_t nch = nchunks(wk);
        for (;;) {
            uint32_t chunk = 0;
            if (lane == 0) chunk = atomicAdd(&wk->next[k_next], 1u);
            chunk = __shfl_sync(0xFFFFFFFFu, chunk, 0);
            if (chunk >= nch) break;
            const uint64_t c = begin + static_cast<uint64_t>(chunk) * 32 + lane;
            const float bnd = bound_from_bits(ld_volatile_u64(&wk->bsf_bits));
            const bool in = c < end;
            const bool keep = in && cand_lb[c] <= bnd;
            if (in && !keep) cand_sq[c] = INFINITY;
            const uint32_t p = keep ? ix.pos[cand_pos[c]] : 0u;
            unsigned m = __ballot_sync(0xFFFFFFFFu, keep);
            if constexpr (M == 1) {
                // LB_Keogh first, four candidates at a time (one per 8-lane group); the
                // reversed LB_Keogh; the survivors two at a time through the paired DTW
                unsigned fwd = 0;
                {
                    const int wgi = lane / kRowLanes;
                    const bool gl = (lane & (kRowLanes - 1)) == 0;
                    while (m) {
                        unsigned t = m;
                        for (int k = 0; k < wgi && t; ++k) t &= t - 1;
                        const int srcg = t ? __ffs(t) - 1 : -1;
                        for (int k = 0; k < 32 / kRowLanes && m; ++k) m &= m - 1;
                        const uint32_t pg = __shfl_sync(0xFFFFFFFFu, p, srcg >= 0 ? srcg : 0);
                        const double cut = bsf_of(ld_volatile_u64(&wk->bsf_bits)) * kSlack;
                        const double lbf = group_lb_keogh_sq(s_qe + n, s_qe + 2 * n, ix.rows + static_cast<uint64_t>(pg) * n, n);
                        const unsigned bit = gl && srcg >= 0 && lbf <= cut ? 1u << srcg : 0u;
                        const unsigned drop_bit = gl && srcg >= 0 && !(lbf <= cut) ? 1u << srcg : 0u;
                        fwd |= __reduce_or_sync(0xFFFFFFFFu, bit);
                        const unsigned dropped = __reduce_or_sync(0xFFFFFFFFu, drop_bit);
                        if (dropped >> lane & 1u) cand_sq[c] = INFINITY;
                    }
                }
                unsigned live = 0;
                while (fwd) {
                    const int src = __ffs(fwd) - 1;
                    fwd &= fwd - 1;
                    const uint32_t pp = __shfl_sync(0xFFFFFFFFu, p, src);
                    const uint64_t cc = __shfl_sync(0xFFFFFFFFu, c, src);
                    const double cut = bsf_of(ld_volatile_u64(&wk->bsf_bits)) * kSlack;
                    bool drop = false;
                    if (ix.rev_keogh) {  // the query against the candidate's envelope
                        float* w_row = s_qe + 3 * n + (threadIdx.x >> 5) * 3 * n;
                        const float* row = ix.rows + static_cast<uint64_t>(pp) * n;
                        for (int i = lane; i < n; i += 32) w_row[i] = __ldg(row + i);
                        __syncwarp();
                        drop = warp_lb_keogh_rev_sq(w_row, w_row + n, w_row + 2 * n, s_qe, n, ix.window) > cut;
                    }
                    if (drop) {
                        if (lane == 0) cand_sq[cc] = INFINITY;
                    } else {
                        live |= 1u << src;
                    }
                }
                while (live) {
                    const int s0 = __ffs(live) - 1;
                    live &= live - 1;
                    const int s1 = live ? __ffs(live) - 1 : -1;
                    if (s1 >= 0) live &= live - 1;
                    const uint32_t p0 = __shfl_sync(0xFFFFFFFFu, p, s0);
                    const uint64_t c0 = __shfl_sync(0xFFFFFFFFu, c, s0);
                    const uint32_t p1 = __shfl_sync(0xFFFFFFFFu, p, s1 >= 0 ? s1 : s0);
                    const uint64_t c1 = __shfl_sync(0xFFFFFFFFu, c, s1 >= 0 ? s1 : s0);
                    const double cut = bsf_of(ld_volatile_u64(&wk->bsf_bits)) * kSlack;
                    double d0, d1 = INFINITY;
                    if (s1 >= 0) {
                        warp_dtw_sq_pair(s_qe, ix.rows + static_cast<uint64_t>(p0) * n,
                                         ix.rows + static_cast<uint64_t>(p1) * n, n, ix.window, cut, cut, d0, d1);
                    } else {
                        d0 = warp_dtw_sq<1>(s_qe, ix.rows + static_cast<uint64_t>(p0) * n, n, ix.window, cut);
                    }
                    if (lane == 0) {
                        refined += s1 >= 0 ? 2 : 1;
                        updates += publish(wk, d0, c0, cand_sq, p0);
                        if (s1 >= 0) updates += publish(wk, d1, c1, cand_sq, p1);
                    }
                }
            } else {
                while (m) {
                    const int src = __ffs(m) - 1;
                    m &= m - 1;
                    const uint32_t pp = __shfl_sync(0xFFFFFFFFu, p, src);
                    const uint64_t cc = __shfl_sync(0xFFFFFFFFu, c, src);
                    bool ran;
                    const double sq = warp_dtw_candidate<M>(s_qe, s_qe + n, s_qe + 2 * n,
                                                            ix.rows + static_cast<uint64_t>(pp) * n, n, ix.window, wk,
                                                            ran);
                    if (lane == 0) {
                        refined += ran ? 1 : 0;
                        updates += publish(wk, sq, cc, cand_sq, pp);
                    }
                }
            }
        }
        if (lane == 0) {
            if (refined) atomicAdd(&wk->stats[kRealDist], refined);
            if (updates) atomicAdd(&wk->stats[kBsfUpd], updates);
        }
        refined = updates = 0;
    }
}

// ----------------------------------------------------------- finalize
__device__ __forceinline__ void write_result(const IndexView& ix, const QueryWork* wk, DevResult* out, double dist,
                                             unsigned best_pos, bool overflow, unsigned long long cand) {
    // No row of this shard reaches the BSF (it was imported from another
    // shard, exchange.cuh): +inf / 0xFFFFFFFF, which loses every merge.
    const bool none = best_pos == 0xFFFFFFFFu;
    out->distance = none ? INFINITY : dist;
    out->position = none ? 0xFFFFFFFFu : static_cast<uint32_t>(best_pos + ix.pos_offset);
    out->flags = overflow ? kResultOverflow : 0u;
    out->stats[kLbNode] = wk->stats[kLbNode];
    out->stats[kLbEntry] = wk->stats[kLbEntry] + wk->nseed;
    out->stats[kRealDist] = wk->stats[kRealDist];
    out->stats[kBsfUpd] = wk->stats[kBsfUpd];
    out->stats[kPruned] = wk->stats[kPruned];
    out->stats[kQueueIns] = (cand & 0xFFFFFFFFull) - wk->nseed + (cand >> 32);
    out->boxes = wk->boxes;
    out->fine_calcs = wk->fine_calcs;
}

// Grid (x, query): lowest position among the candidates whose sqrt(sum)
// equals the best distance; the last block of a query writes its result
// (flagged when the slot overflowed).
__global__ void __launch_bounds__(kThreads)
    k_finalize(IndexView ix, SlotView S, int seed_only, DevResult* __restrict__ results) {
    const int q = blockIdx.y;
    QueryWork* wk = S.work + q;
    const double best = bsf_of(wk->bsf_bits);
    const double dist = sqrt(best);
    const double lim = best * kSlack;
    const bool overflow = wk->overflow != 0;
    const unsigned long long cand = wk->cand;
    const uint64_t lo_end = seed_only ? wk->nseed : (cand & 0xFFFFFFFFull);
    const uint64_t hi_n = seed_only ? 0 : (cand >> 32);
    const uint32_t* cand_pos = S.cand_pos + q * S.cap;
    const double* cand_sq = S.cand_sq + q * S.cap;
    uint32_t mine = 0xFFFFFFFFu;
    const unsigned nties = wk->nties;
    if (!overflow && nties <= kTieCap) {
        // every row that can be the answer is in the seed range or the tie list: block 0 decides
        if (blockIdx.x != 0) return;
        // four records per thread per step, loads first (a dependent-load chain per step otherwise)
        const unsigned ns = wk->nseed, total = ns + nties;
        for (unsigned i0 = threadIdx.x; i0 < total; i0 += 4 * blockDim.x) {
            double sv[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const unsigned i = i0 + u * blockDim.x;
                sv[u] = i >= total ? INFINITY : i < ns ? cand_sq[i] : wk->tie_sq[i - ns];
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const unsigned i = i0 + u * blockDim.x;
                if (sv[u] <= lim && sqrt(sv[u]) == dist)
                    mine = min(mine, i < ns ? ix.pos[cand_pos[i]] : wk->tie_row[i - ns]);
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) mine = min(mine, __shfl_xor_sync(0xFFFFFFFFu, mine, o));
        __shared__ unsigned s_min[kWarps];
        if ((threadIdx.x & 31) == 0) s_min[threadIdx.x >> 5] = mine;
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int i = 1; i < kWarps; ++i) mine = min(mine, s_min[i]);
            write_result(ix, wk, results + q, dist, mine, false, cand);
        }
        return;
    }
    if (!overflow) {
        // four records per thread per step, loads first (the scan is latency-bound)
        const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x, total = lo_end + hi_n;
        for (uint64_t i0 = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i0 < total; i0 += 4 * stride) {
            double sv[4];
            uint64_t cv[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const uint64_t i = i0 + u * stride;
                cv[u] = i < lo_end ? i : S.cap - 1 - (i - lo_end);
                sv[u] = i < total ? cand_sq[cv[u]] : INFINITY;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (sv[u] <= lim && sqrt(sv[u]) == dist) mine = min(mine, ix.pos[cand_pos[cv[u]]]);
        }
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
    write_result(ix, wk, results + q, dist, atomicAdd(&wk->best_pos, 0u), overflow, cand);
}

template <typename K>
int blocks_per_sm(K kernel, size_t smem) {
    // cached per (device, kernel, shared memory): the driver query costs
    // microseconds, which a one-query batch would pay on every call
    static std::mutex mu;
    static std::map<std::tuple<int, const void*, size_t>, int> cache;
    int dev = 0;
    TSG_CUDA(cudaGetDevice(&dev));
    const auto key = std::make_tuple(dev, reinterpret_cast<const void*>(kernel), smem);
    {
        std::lock_guard<std::mutex> lk(mu);
        const auto it = cache.find(key);
        if (it != cache.end()) return it->second;
    }
    int b = 0;
    TSG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kernel, kThreads, smem));
    b = std::max(b, 1);
    std::lock_guard<std::mutex> lk(mu);
    cache[key] = b;
    return b;
}

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (device, kernel, bytes).
void set_max_smem(const void* f, int bytes) {
    static std::mutex mu;
    static std::map<std::tuple<int, const void*, int>, bool> done;
    int dev = 0;
    TSG_CUDA(cudaGetDevice(&dev));
    const auto key = std::make_tuple(dev, f, bytes);
    std::lock_guard<std::mutex> lk(mu);
    if (done.count(key)) return;
    TSG_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    done[key] = true;
}

// The batch pipeline (prepare .. finalize, nine launches, no host round trip)
// as CUDA graphs, one per batch shape: a one-query batch otherwise pays every
// launch's latency in series. The graph reads the queries from its own
// staging rows, filled by its first node (a device copy whose source is
// re-pointed before each launch), so the caller's query pointer is not part
// of the key.
struct SearchGraph {
    cudaGraph_t graph = nullptr;  // kept: the copy nodes belong to it
    cudaGraphExec_t exec = nullptr;
    cudaGraphNode_t copy = nullptr;     // caller's queries -> staging rows (source re-pointed per launch)
    cudaGraphNode_t copy_out = nullptr; // graph-owned results -> caller's results (destination re-pointed)
    uint64_t launches = 0;  // kernel launches per replay (gpu_launches)
};
// (slot arrays, slot sizes, batch size, mode, window, seed cap, split, seed exchange); the index's
// own arrays are fixed for the cache's lifetime (it is freed with the shard). The caller's query
// and result buffers are not part of the key: copy nodes at both ends are re-pointed per launch.
using GraphKey = std::tuple<const void*, const void*, const void*, const void*, uint64_t, uint64_t, uint32_t, int,
                            int, uint32_t, float, int>;
struct GraphCache {
    std::map<GraphKey, SearchGraph> graphs;
    float* staging = nullptr;      // [staging_rows][n]
    DevResult* results = nullptr;  // [staging_rows]
    uint32_t staging_rows = 0;
};
constexpr size_t kMaxGraphs = 32;

// Ends a capture that an exception interrupted: the stream leaves capture
// mode, the partial graph is destroyed and the capture's sticky error cleared,
// so later searches on the shard still work.
struct CaptureGuard {
    cudaStream_t st;
    bool active = true;
    ~CaptureGuard() {
        if (!active) return;
        cudaGraph_t g = nullptr;
        cudaStreamEndCapture(st, &g);
        if (g) cudaGraphDestroy(g);
        cudaGetLastError();
    }
};

void clear_graphs(GraphCache& gc) {
    for (auto& kv : gc.graphs) {
        cudaGraphExecDestroy(kv.second.exec);
        cudaGraphDestroy(kv.second.graph);
    }
    gc.graphs.clear();
}

}  // namespace

void free_search_graphs(DevIndex& ix) {
    auto* gc = static_cast<GraphCache*>(ix.graphs);
    if (!gc) return;
    clear_graphs(*gc);
    cudaFree(gc->staging);
    cudaFree(gc->results);
    delete gc;
    ix.graphs = nullptr;
}

void search_batch(DevIndex& ix, const DevIndex::Slots& slots, const float* d_queries, uint32_t nq, bool approximate,
                  DevResult* results, int window, bool exchange) {
    if (nq == 0) return;
    // the seed-BSF exchange with the other shards (exchange.cuh); TSG_NO_SEED_EXCHANGE=1 for A/B runs
    static const bool no_seed_x = std::getenv("TSG_NO_SEED_EXCHANGE") != nullptr;
    Exchange* xc = exchange && !approximate && !no_seed_x ? ix.xchg : nullptr;
    if (xc) xc->reserve(nq);
    if (nq > slots.n) throw std::logic_error("search_batch: batch larger than its slots");
    cudaStream_t st = ix.stream;
    const int n = ix.n, w = ix.w;
    const size_t lut_bytes = static_cast<size_t>(w) * 256 * sizeof(float);
    const size_t q_bytes = static_cast<size_t>(n) * sizeof(float);
    const size_t qd_bytes = static_cast<size_t>(n) * sizeof(double);
    const bool vec = (n % 8) == 0 && (reinterpret_cast<uintptr_t>(ix.rows) % 32) == 0;
    const bool w16 = w == 16;
    auto refine = vec ? k_refine<true> : k_refine<false>;
    auto seed = vec ? k_seed<true> : k_seed<false>;
    auto lbscan = ix.ws == 16 ? (w16 ? k_lbscan<16, true> : k_lbscan<16, false>) : k_lbscan<32, false>;
    auto bound = ix.ws == 16 ? (w16 ? k_bound<16, true> : k_bound<16, false>) : k_bound<32, false>;
    auto groups = ix.ws == 16 ? (w16 ? k_groups<16, true> : k_groups<16, false>) : k_groups<32, false>;
    // Per-device function attributes (cheap; set on every call so each device is covered).
    // TMA-staged refinement for the row lengths it is instantiated for.
    auto refine_tma = n == 256 ? k_refine_tma<32, 0> : n == 128 ? k_refine_tma<16, 0> : n == 96 ? k_refine_tma<12, 0>
                    : n == 64 ? k_refine_tma<8, 0> : n == 512 ? k_refine_tma<64, 0> : nullptr;
    const bool tma = vec && refine_tma && !std::getenv("TSG_NO_TMA_REFINE");
    const size_t tma_bytes = static_cast<size_t>(kThreads / kRowLanes) * tma_group_floats(n) * 4 +
                             static_cast<size_t>((n / 8 + kRowLanes - 1) / kRowLanes) * 64 * 8;
    if (tma) set_max_smem(reinterpret_cast<const void*>(refine_tma), 150 * 1024);
    for (const void* f : {reinterpret_cast<const void*>(refine), reinterpret_cast<const void*>(seed),
                          reinterpret_cast<const void*>(lbscan), reinterpret_cast<const void*>(bound),
                          reinterpret_cast<const void*>(groups), reinterpret_cast<const void*>(k_prepare)})
        set_max_smem(f, 100 * 1024);

    IndexView iv{};
    iv.rows = ix.rows;
    iv.n = n;
    iv.w = w;
    iv.bits = ix.bits;
    iv.thr = ix.thr;
    iv.words = ix.words;
    iv.pos = ix.pos;
    iv.leaf_off = ix.leaf_off;
    iv.page_off = ix.page_off;
    iv.page_leaf = ix.page_leaf;
    iv.page_key = ix.page_key;
    iv.page_dir = ix.page_dir;
    iv.P = ix.P;
    iv.page_lo = ix.page_lo;
    iv.page_hi = ix.page_hi;
    iv.group_lo = ix.group_lo;
    iv.group_hi = ix.group_hi;
    iv.NG = ix.NG;
    iv.top_lo = ix.top_lo;
    iv.top_hi = ix.top_hi;
    iv.NT = ix.NT;
    iv.run_lo = ix.run_lo;
    iv.run_hi = ix.run_hi;
    iv.quad_lo = ix.quad_lo;
    iv.quad_hi = ix.quad_hi;
    iv.seed_cap = static_cast<uint32_t>(std::min<uint64_t>(2 * ix.leaf_cap, 1u << 20));
    if (const char* e = std::getenv("TSG_SEED_CAP")) iv.seed_cap = static_cast<uint32_t>(std::atoll(e));  // A/B runs
    iv.split = ix.refine_split;
    iv.pos_offset = ix.pos_offset;
    iv.window = window;
    const bool fine = ix.fw > 0 && window < 0;  // the fine bound is Euclidean
    iv.fine = fine ? ix.fine : nullptr;
    iv.fw = ix.fw;
    iv.fws = ix.fws;
    SlotView sv{slots.work, slots.lut, slots.gsurv, slots.surv, slots.surv_lb, slots.cand_pos, slots.cand_lb,
                slots.cand_sq, slots.env, slots.cap, ix.P, ix.NG, w * 256, slots.rcap, slots.dpage, slots.dpage_lb,
                slots.fine_lut, ix.fw * 256};
    // DTW kernels, by band-diagonal registers per lane (window <= 32 M - 1).
    const bool dtw = window >= 0;
    if (window > kMaxDtwWindow) throw std::invalid_argument("exact_search: dtw window above the device limit");
    const int dtw_m = window < 32 ? 1 : window < 64 ? 2 : window < 128 ? 4 : 8;
    auto seed_dtw = dtw_m == 1 ? k_seed_dtw<1> : dtw_m == 2 ? k_seed_dtw<2> : dtw_m == 4 ? k_seed_dtw<4> : k_seed_dtw<8>;
    auto refine_dtw = dtw_m == 1 ? k_refine_dtw<1> : dtw_m == 2 ? k_refine_dtw<2> : dtw_m == 4 ? k_refine_dtw<4>
                                                                                     : k_refine_dtw<8>;
    const size_t qe_bytes = 3ull * n * sizeof(float);

    const int sms = ix.sms;
    const unsigned seed_x = (iv.seed_cap + kThreads / kRowLanes - 1) / (kThreads / kRowLanes);
    // Seed blocks per query with the fine summary: 8 (best from batch 64 up), or one wave of
    // blocks over the batch when it is small (batch 1: 8.8K -> 9.9K q/s at c5 sigma 0.01,
    // profiles/ab_seed_blocks.sh); TSG_SEED_BLOCKS overrides.
    static const int seed_env = [] {
        const char* e = std::getenv("TSG_SEED_BLOCKS");
        return e ? std::max(1, std::atoi(e)) : 0;
    }();
    const unsigned seed_fine_x = seed_env ? static_cast<unsigned>(seed_env)
                                          : std::max(8u, static_cast<unsigned>(ix.sms) / nq);
    // Two waves of group blocks over the batch (c2: groups + bound 6.31 -> 6.19 us/query against one
    // wave; three are no better); TSG_GROUP_WAVES overrides (A/B runs).
    static const int group_waves = [] {
        const char* e = std::getenv("TSG_GROUP_WAVES");
        return e ? std::max(1, std::atoi(e)) : 2;
    }();
    const unsigned group_x = static_cast<unsigned>(std::max<uint64_t>(
        1, std::min<uint64_t>((ix.NT + kThreads * kGP - 1) / (kThreads * kGP),
                              static_cast<uint64_t>(group_waves) * sms * blocks_per_sm(groups, lut_bytes) / nq)));
    // TSG_GRID_CAP (A/B runs): blocks per SM of the persistent kernels
    static const int grid_cap = [] {
        const char* e = std::getenv("TSG_GRID_CAP");
        return e ? std::max(1, std::atoi(e)) : 1 << 20;
    }();
    auto capped = [&](int b) { return static_cast<unsigned>(sms * std::min(b, grid_cap)); };
    const unsigned bound_grid = capped(blocks_per_sm(bound, lut_bytes));
    const unsigned scan_grid = capped(blocks_per_sm(lbscan, lut_bytes));
    const unsigned refine_grid = tma ? static_cast<unsigned>(sms * blocks_per_sm(refine_tma, tma_bytes))
                                     : static_cast<unsigned>(sms * blocks_per_sm(refine, qd_bytes));
    const unsigned fin_x = std::max(1u, std::min(256u, static_cast<unsigned>(sms * 32 / nq)));
    auto fine_k = vec ? (ix.fw == 32 ? k_fine_refine<32, kFineK, true> : ix.fw == 64 ? k_fine_refine<64, kFineK, true>
                                                                          : k_fine_refine<0, kFineK, true>)
                      : (ix.fw == 32 ? k_fine_refine<32, kFineK, false> : ix.fw == 64 ? k_fine_refine<64, kFineK, false>
                                                                           : k_fine_refine<0, kFineK, false>);
    const size_t fine_bytes = static_cast<size_t>(ix.fw) * 256 * sizeof(float) + qd_bytes;
    // With a 32-wide fine summary and a TMA row length, the fine bound runs inside the
    // TMA-staged refinement (half-row abandonment, double-buffered rows); TSG_FINE_FUSED=1
    // selects the simpler fused kernel instead.
    auto refine_tma_fine = ix.fw != 32 ? nullptr : n == 256 ? k_refine_tma<32, 32> : n == 128 ? k_refine_tma<16, 32>
                         : n == 96 ? k_refine_tma<12, 32> : n == 64 ? k_refine_tma<8, 32> : n == 512 ? k_refine_tma<64, 32>
                                                                                      : nullptr;
    const bool tma_fine = fine && tma && refine_tma_fine && !std::getenv("TSG_FINE_FUSED");
    const size_t tma_fine_bytes = tma_bytes + 32 * 256 * sizeof(FineLutT);
    unsigned tma_fine_grid = 0;
    if (tma_fine) {
        set_max_smem(reinterpret_cast<const void*>(refine_tma_fine), 180 * 1024);
        tma_fine_grid = capped(blocks_per_sm(refine_tma_fine, tma_fine_bytes));
    }
    unsigned fine_grid = 0;
    if (fine) {
        set_max_smem(reinterpret_cast<const void*>(fine_k), 100 * 1024);
        fine_grid = static_cast<unsigned>(sms * blocks_per_sm(fine_k, fine_bytes));
    }
    if (dtw) {
        set_max_smem(reinterpret_cast<const void*>(seed_dtw), 100 * 1024);
        set_max_smem(reinterpret_cast<const void*>(refine_dtw), 100 * 1024);
    }
    const unsigned seed_dtw_x = (iv.seed_cap + kWarps - 1) / kWarps;
    // refine_dtw: query + envelope, then per-warp scratch for a candidate row and its envelope
    iv.rev_keogh = kRevKeogh && static_cast<size_t>(kWarps + 1) * qe_bytes <= 96 * 1024 ? 1 : 0;
    const size_t rdtw_bytes = qe_bytes + (iv.rev_keogh ? static_cast<size_t>(kWarps) * qe_bytes : 0);
    const unsigned refine_dtw_grid = dtw ? static_cast<unsigned>(sms * blocks_per_sm(refine_dtw, rdtw_bytes)) : 0u;

    // Optional per-kernel timing: events around every launch, summed after the batch.
    std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> marks;
    auto mark = [&](int slot, auto&& launch) {
        if (!ix.profile) {
            launch();
            return;
        }
        cudaEvent_t a, b;
        TSG_CUDA(cudaEventCreate(&a));
        TSG_CUDA(cudaEventCreate(&b));
        TSG_CUDA(cudaEventRecord(a, st));
        launch();
        TSG_CUDA(cudaEventRecord(b, st));
        marks.push_back({slot, {a, b}});
    };
    const int inq = static_cast<int>(nq);
    auto pipeline = [&](const float* qsrc, DevResult* res) {
        mark(2, [&] {
            k_prepare<<<nq, kThreads, dtw ? qe_bytes : q_bytes, st>>>(iv, sv, qsrc);
            TSG_LAUNCHED();
            if (dtw) seed_dtw<<<dim3(seed_dtw_x, nq), kThreads, qe_bytes, st>>>(iv, sv, qsrc);
            else seed<<<dim3(fine ? std::min(seed_x, seed_fine_x) : seed_x, nq), kThreads, qd_bytes, st>>>(iv, sv, qsrc);
            TSG_LAUNCHED();
        });
        if (xc) mark(7, [&] { xc->seed_bsf(sv.work, nq, st); });
        if (!approximate) {
            mark(1, [&] {
                groups<<<dim3(group_x, nq), kThreads, lut_bytes, st>>>(iv, sv);
                TSG_LAUNCHED();
                bound<<<bound_grid, kThreads, lut_bytes, st>>>(iv, sv, inq, 0);
                TSG_LAUNCHED();
            });
            for (int wave = 0; wave < 2; ++wave) {
                if (wave == 1)
                    mark(1, [&] {  // runs of the deferred pages, against the BSF refinement wave A tightened
                        bound<<<bound_grid, kThreads, lut_bytes, st>>>(iv, sv, inq, 1);
                        TSG_LAUNCHED();
                    });
                mark(4, [&] {
                    lbscan<<<scan_grid, kThreads, lut_bytes, st>>>(iv, sv, inq, wave);
                    TSG_LAUNCHED();
                });
                mark(wave == 0 ? 3 : 5, [&] {
                    if (tma_fine)
                        refine_tma_fine<<<tma_fine_grid, kThreads, tma_fine_bytes, st>>>(iv, sv, qsrc, inq, wave);
                    else if (fine) fine_k<<<fine_grid, kThreads, fine_bytes, st>>>(iv, sv, qsrc, inq, wave);
                    else if (dtw) refine_dtw<<<refine_dtw_grid, kThreads, rdtw_bytes, st>>>(iv, sv, qsrc, inq, wave);
                    else if (tma) refine_tma<<<refine_grid, kThreads, tma_bytes, st>>>(iv, sv, qsrc, inq, wave);
                    else refine<<<refine_grid, kThreads, qd_bytes, st>>>(iv, sv, qsrc, inq, wave);
                    TSG_LAUNCHED();
                });
            }
        }
        mark(6, [&] {
            k_finalize<<<dim3(fin_x, nq), kThreads, 0, st>>>(iv, sv, approximate ? 1 : 0, res);
            TSG_LAUNCHED();
        });
    };
    static const bool no_graph = std::getenv("TSG_NO_GRAPH") != nullptr;  // A/B: plain stream launches
    if (ix.profile || no_graph || (xc && !xc->capturable())) {
        pipeline(d_queries, results);
    } else {
        if (!ix.graphs) ix.graphs = new GraphCache;
        GraphCache& gc = *static_cast<GraphCache*>(ix.graphs);
        const size_t qbytes = static_cast<size_t>(nq) * n * sizeof(float);
        if (gc.staging_rows < nq) {  // graphs point at the old staging rows
            TSG_CUDA(cudaStreamSynchronize(st));
            clear_graphs(gc);
            cudaFree(gc.staging);
            cudaFree(gc.results);
            gc.staging = nullptr;
            gc.results = nullptr;
            gc.staging_rows = std::max(nq, ix.batch_max);
            TSG_CUDA(cudaMalloc(&gc.staging, static_cast<size_t>(gc.staging_rows) * n * sizeof(float)));
            TSG_CUDA(cudaMalloc(&gc.results, static_cast<size_t>(gc.staging_rows) * sizeof(DevResult)));
        }
        const GraphKey key{slots.work, slots.cand_pos, slots.surv, slots.fine_lut, slots.cap, slots.rcap, nq,
                           approximate ? 1 : 0, window, iv.seed_cap, iv.split, xc ? 1 : 0};
        auto it = gc.graphs.find(key);
        if (it == gc.graphs.end()) {
            if (gc.graphs.size() >= kMaxGraphs) clear_graphs(gc);
            SearchGraph sg;
            const uint64_t l0 = launch_count_thread();
            TSG_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
            CaptureGuard guard{st};
            TSG_CUDA(cudaMemcpyAsync(gc.staging, d_queries, qbytes, cudaMemcpyDeviceToDevice, st));
            pipeline(gc.staging, gc.results);
            TSG_CUDA(cudaMemcpyAsync(results, gc.results, nq * sizeof(DevResult), cudaMemcpyDeviceToDevice, st));
            cudaGraph_t g = nullptr;
            guard.active = false;
            TSG_CUDA(cudaStreamEndCapture(st, &g));
            sg.graph = g;
            sg.launches = launch_count_thread() - l0;  // this thread's launches: the pipeline's own
            size_t count = 0;
            TSG_CUDA(cudaGraphGetNodes(g, nullptr, &count));
            std::vector<cudaGraphNode_t> nodes(count);
            TSG_CUDA(cudaGraphGetNodes(g, nodes.data(), &count));
            for (cudaGraphNode_t nd : nodes) {
                cudaGraphNodeType t;
                TSG_CUDA(cudaGraphNodeGetType(nd, &t));
                if (t != cudaGraphNodeTypeMemcpy) continue;
                cudaMemcpy3DParms p{};
                TSG_CUDA(cudaGraphMemcpyNodeGetParams(nd, &p));
                if (p.dstPtr.ptr == gc.staging) sg.copy = nd;
                else if (p.srcPtr.ptr == gc.results) sg.copy_out = nd;
            }
            if (!sg.copy || !sg.copy_out) {
                cudaGraphDestroy(g);
                throw std::runtime_error("search_batch: captured graph lacks its query / result copy node");
            }
            const cudaError_t ie = cudaGraphInstantiate(&sg.exec, g, 0);
            if (ie != cudaSuccess) {
                cudaGraphDestroy(g);
                TSG_CUDA(ie);
            }
            it = gc.graphs.emplace(key, sg).first;
        } else {
            note_launch(static_cast<int>(it->second.launches));  // a capture counts its launches once
        }
        TSG_CUDA(cudaGraphExecMemcpyNodeSetParams1D(it->second.exec, it->second.copy, gc.staging, d_queries, qbytes,
                                                    cudaMemcpyDeviceToDevice));
        TSG_CUDA(cudaGraphExecMemcpyNodeSetParams1D(it->second.exec, it->second.copy_out, results, gc.results,
                                                    nq * sizeof(DevResult), cudaMemcpyDeviceToDevice));
        TSG_CUDA(cudaGraphLaunch(it->second.exec, st));
    }
    if (!marks.empty()) {
        TSG_CUDA(cudaStreamSynchronize(st));
        for (auto& m : marks) {
            float ms = 0.f;
            TSG_CUDA(cudaEventElapsedTime(&ms, m.second.first, m.second.second));
            ix.prof_ms[m.first] += ms;
            ix.prof_launches[m.first] += nq;
            cudaEventDestroy(m.second.first);
            cudaEventDestroy(m.second.second);
        }
    }
}

}  // namespace tsg
