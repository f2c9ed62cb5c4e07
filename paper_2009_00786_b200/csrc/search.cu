// Exact Euclidean 1-NN over the flat SoA index (one device shard).
//
// Replaces exact_search (src/query.cpp:258-298) and its pieces. Per query,
// five kernels on the index's stream:
//   bound     QueryState (src/query.cpp:81-100) + node_lower_bound
//             (src/query.cpp:102-107): every block computes the query PAA in
//             FP64 reference order, the query symbols and a [w][256] table of
//             per-segment squared region gaps (mindist_bands,
//             src/metrics.cpp:47-70) rounded DOWN to float, so every float
//             bound here is <= the exact FP64 bound (sound pruning); then the
//             bound of every page box, and the argmin page.
//   seed      approximate_search_state (src/query.cpp:226-238): the leaf of
//             the argmin page is refined exhaustively and seeds the BSF.
//   filter    traverse_root_subtree's pruning (src/query.cpp:154-171) at page
//             granularity: pages whose box bound exceeds the BSF are dropped;
//             survivors are compacted (block-aggregated).
//   lbscan    the entry-level filter of calculate_real_distance_leaf
//             (src/query.cpp:129-134): words of surviving pages are bounded
//             with 16 table lookups and compacted with warp ballot + prefix
//             popcount into the candidate list.
//   refine    euclidean (src/metrics.cpp:17-40, 95-104): one thread per
//             candidate row, 256-bit loads of 8-float blocks, FP64 block sums
//             without FMA added left to right exactly like squared_l2, early
//             abandonment when the running sum exceeds the live best-so-far
//             (strict, so ties survive); the BSF is an atomicMin on the double
//             bit pattern (non-negative doubles order as unsigned integers),
//             the SharedBsf analog (src/query.cpp:35-42). A candidate whose
//             bound exceeds the live BSF is skipped (`LB >= cutoff -> skip`).
//   finalize  result = min over refined candidates of (sqrt(sum), position):
//             ties resolve to the lowest position exactly as scan_nn does
//             (src/scan.cpp:54-59); the last block writes the result and
//             resets the scratch for the next query.
// Pruning keeps ties: a candidate is dropped only when its bound (or partial
// sum) is strictly above the best-so-far widened by 1e-9 relative (covering
// FP64 rounding of the distance sums), so the exact answer is never lost.
#include <algorithm>
#include <cmath>
#include <utility>
#include <vector>

#include "common.cuh"
#include "kernels.cuh"

namespace tsg {

namespace {

constexpr unsigned long long kInfBits = 0x7FF0000000000000ull;
constexpr double kSlack = 1.0 + 1e-9;
constexpr int kThreads = 256;

enum Stat { kLbNode = 0, kLbEntry, kRealDist, kBsfUpd, kPruned, kQueueIns };

__device__ __forceinline__ double bsf_of(unsigned long long bits) {
    return __longlong_as_double(static_cast<long long>(bits));
}

__device__ __forceinline__ float bound_from_bits(unsigned long long bits) {
    return __double2float_ru(bsf_of(bits) * kSlack);
}

__device__ __forceinline__ uint8_t byte_of(const uint4& v, int s) {
    const uint32_t word = s < 4 ? v.x : s < 8 ? v.y : s < 12 ? v.z : v.w;
    return static_cast<uint8_t>(word >> (8 * (s & 3)));
}

struct QueryShared {
    double thr[kThrPad];
    double qpaa[kMaxW];
    unsigned char qsym[kMaxW];
};

// Block-local query preparation: PAA (FP64, reference order), symbols, and
// the [w][256] squared-gap table (scaled by n/w, rounded down).
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
        s_lut[idx] = __double2float_rd(__dmul_rn(__dmul_rn(gap, gap), scale));
    }
    __syncthreads();
}

__device__ __forceinline__ void reset_work(QueryWork* wk) {
    wk->bsf_bits = kInfBits;
    wk->seed_key = ~0ull;
    wk->ncand = 0;
    wk->nseed = 0;
    wk->work_next = 0;
    wk->best_pos = 0xFFFFFFFFu;
    wk->nsurv = 0;
    for (int i = 0; i < 6; ++i) wk->stats[i] = 0;
}

__global__ void k_reset(QueryWork* wk) {
    reset_work(wk);
    wk->done_blocks = 0;
}

// ------------------------------------------------------------ bound
__global__ void __launch_bounds__(kThreads)
    k_bound(const float* __restrict__ q, int n, int w, int bits, const double* __restrict__ thr_g,
            const uint8_t* __restrict__ lo, const uint8_t* __restrict__ hi, uint64_t P, int ws, QueryWork* wk,
            float* __restrict__ page_lb) {
    extern __shared__ float s_lut[];
    __shared__ QueryShared qs;
    prepare_query(q, n, w, bits, thr_g, qs, s_lut);
    unsigned long long best = ~0ull;
    for (uint64_t p = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; p < P;
         p += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        float lb = 0.f;
        for (int h = 0; h < ws / 16; ++h) {
            const uint4 a = ld_stream_u4(lo + p * ws + 16 * h);
            const uint4 b = ld_stream_u4(hi + p * ws + 16 * h);
            const int smax = min(16, w - 16 * h);
            for (int s = 0; s < smax; ++s) {
                const int g = 16 * h + s;
                const uint8_t ql = qs.qsym[g], bl = byte_of(a, s), bh = byte_of(b, s);
                const float gv = ql < bl ? s_lut[g * 256 + bl] : (ql > bh ? s_lut[g * 256 + bh] : 0.f);
                lb = __fadd_rd(lb, gv);
            }
        }
        page_lb[p] = lb;
        best = min(best, (static_cast<unsigned long long>(__float_as_uint(lb)) << 32) | p);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) best = min(best, __shfl_xor_sync(0xFFFFFFFFu, best, o));
    if ((threadIdx.x & 31) == 0 && best != ~0ull) atomicMin(&wk->seed_key, best);
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

constexpr int kGroup = 4;  // blocks of 8 floats in flight per thread

// Squared Euclidean distance of one row to the query in squared_l2's exact
// order; returns +inf as soon as the running sum exceeds the live bound
// (re-read from `bsf` every kGroup blocks). VEC: n % 8 == 0, 32-byte aligned.
template <bool VEC>
__device__ __forceinline__ double row_sq(const float* __restrict__ row, const float* __restrict__ s_q, int n,
                                         const unsigned long long* bsf) {
    const int nb = (n + 7) >> 3;
    double sum = 0.0;
    for (int b0 = 0; b0 < nb; b0 += kGroup) {
        if (VEC) {
            F8 x[kGroup];
#pragma unroll
            for (int j = 0; j < kGroup; ++j)
                if (b0 + j < nb) x[j] = ld256(row + 8 * (b0 + j));
#pragma unroll
            for (int j = 0; j < kGroup; ++j)
                if (b0 + j < nb) sum = __dadd_rn(sum, block_sq(x[j].v, s_q + 8 * (b0 + j), 8));
        } else {
#pragma unroll
            for (int j = 0; j < kGroup; ++j) {
                const int b = b0 + j;
                if (b >= nb) break;
                const int cnt = min(8, n - 8 * b);
                float x[8];
#pragma unroll
                for (int k = 0; k < 8; ++k) x[k] = k < cnt ? row[8 * b + k] : 0.f;
                sum = __dadd_rn(sum, block_sq(x, s_q + 8 * b, cnt));
            }
        }
        if (bsf && sum > bsf_of(ld_volatile_u64(bsf)) * kSlack) return INFINITY;
    }
    return sum;
}

__device__ __forceinline__ void seed_range(const uint32_t* leaf_off, const uint32_t* page_off,
                                           const uint32_t* page_leaf, uint32_t seed_cap, unsigned long long key,
                                           uint32_t& a, uint32_t& b) {
    const uint32_t page = static_cast<uint32_t>(key & 0xFFFFFFFFull);
    const uint32_t leaf = page_leaf[page];
    a = leaf_off[leaf];
    b = leaf_off[leaf + 1];
    if (b - a > seed_cap) {
        a = page_off[page];
        b = page_off[page + 1];
    }
}

__device__ __forceinline__ void load_query(float* s_q, const float* q, int n) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) s_q[i] = q[i];
    __syncthreads();
}

// Publishes a finished sum: candidate record, BSF atomicMin only when it can
// improve, strict-improvement count.
__device__ __forceinline__ unsigned long long publish(QueryWork* wk, double s, uint64_t c, double* cand_sq) {
    cand_sq[c] = s;
    if (!(s < INFINITY)) return 0;
    const unsigned long long sb = static_cast<unsigned long long>(__double_as_longlong(s));
    if (sb >= ld_volatile_u64(&wk->bsf_bits)) return 0;
    return atomicMin(&wk->bsf_bits, sb) > sb ? 1 : 0;
}

// -------------------------------------------------------------- seed
// The leaf holding the best page (the leaf the reference's approximate
// search descends to); an overflow leaf larger than seed_cap is replaced by
// that page alone. Every entry is refined against the running seed BSF.
template <bool VEC>
__global__ void __launch_bounds__(128)
    k_seed(const float* __restrict__ rows, int n, const float* __restrict__ query,
           const uint32_t* __restrict__ leaf_off, const uint32_t* __restrict__ page_off,
           const uint32_t* __restrict__ page_leaf, const uint32_t* __restrict__ pos, uint32_t seed_cap,
           QueryWork* wk, uint32_t* __restrict__ cand_pos, double* __restrict__ cand_sq) {
    extern __shared__ float s_q[];
    load_query(s_q, query, n);
    uint32_t a, b;
    seed_range(leaf_off, page_off, page_leaf, seed_cap, wk->seed_key, a, b);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        wk->nseed = b - a;
        wk->ncand = b - a;
        wk->seed_begin = a;
        wk->seed_end = b;
        wk->stats[kRealDist] += b - a;
    }
    unsigned long long updates = 0;
    for (uint32_t e = a + blockIdx.x * blockDim.x + threadIdx.x; e < b; e += gridDim.x * blockDim.x) {
        const uint32_t p = pos[e];
        cand_pos[e - a] = p;
        const double s = row_sq<VEC>(rows + static_cast<uint64_t>(p) * n, s_q, n, &wk->bsf_bits);
        updates += publish(wk, s, e - a, cand_sq);
    }
    for (int o = 16; o > 0; o >>= 1) updates += __shfl_xor_sync(0xFFFFFFFFu, updates, o);
    if ((threadIdx.x & 31) == 0 && updates) atomicAdd(&wk->stats[kBsfUpd], updates);
}

// ------------------------------------------------------------ filter
// Pages with bound <= BSF (and outside the seed range) survive; one atomic
// per block reserves their slots in the survivor list.
__global__ void __launch_bounds__(kThreads)
    k_filter(const float* __restrict__ page_lb, const uint32_t* __restrict__ page_off, uint64_t P, QueryWork* wk,
             uint32_t* __restrict__ surv) {
    __shared__ uint32_t s_cnt[kThreads / 32];
    __shared__ uint32_t s_base;
    const float bound = bound_from_bits(wk->bsf_bits);
    const uint32_t sa = wk->seed_begin, sb = wk->seed_end;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    unsigned long long pruned = 0;
    for (uint64_t base = static_cast<uint64_t>(blockIdx.x) * blockDim.x; base < P;
         base += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint64_t p = base + threadIdx.x;
        bool keep = false;
        if (p < P) {
            const uint32_t a = page_off[p], b = page_off[p + 1];
            const bool seeded = a >= sa && b <= sb;
            keep = !seeded && page_lb[p] <= bound;
            pruned += (!keep && !seeded) ? 1 : 0;
        }
        const unsigned m = __ballot_sync(0xFFFFFFFFu, keep);
        if (lane == 0) s_cnt[warp] = __popc(m);
        __syncthreads();
        if (threadIdx.x == 0) {
            uint32_t tot = 0;
            for (int i = 0; i < kThreads / 32; ++i) {
                const uint32_t c = s_cnt[i];
                s_cnt[i] = tot;
                tot += c;
            }
            s_base = tot ? atomicAdd(&wk->nsurv, tot) : 0u;
        }
        __syncthreads();
        if (keep) surv[s_base + s_cnt[warp] + __popc(m & ((1u << lane) - 1u))] = static_cast<uint32_t>(p);
        __syncthreads();
    }
    for (int o = 16; o > 0; o >>= 1) pruned += __shfl_xor_sync(0xFFFFFFFFu, pruned, o);
    if (lane == 0 && pruned) atomicAdd(&wk->stats[kPruned], pruned);
}

// ------------------------------------------------------------ lbscan
constexpr int kStageCap = 256;

__device__ __forceinline__ void flush_stage(QueryWork* wk, const uint32_t* s_pos, const float* s_lb, int cnt, int lane,
                                            uint32_t* __restrict__ cand_pos, float* __restrict__ cand_lb) {
    uint32_t base = 0;
    if (lane == 0) base = atomicAdd(&wk->ncand, static_cast<unsigned>(cnt));
    base = __shfl_sync(0xFFFFFFFFu, base, 0);
    for (int i = lane; i < cnt; i += 32) {
        cand_pos[base + i] = s_pos[i];
        cand_lb[base + i] = s_lb[i];
    }
    __syncwarp();
}

// Surviving pages round-robin over warps (each page <= kPage entries, so
// work units are bounded); a lane bounds entries lane, lane+32, ... of the
// page with all of its loads in flight at once.
template <int WS>
__global__ void __launch_bounds__(kThreads)
    k_lbscan(const float* __restrict__ q, int n, int w, int bits, const double* __restrict__ thr_g,
             const uint8_t* __restrict__ words, const uint32_t* __restrict__ pos,
             const uint32_t* __restrict__ page_off, const uint32_t* __restrict__ surv, QueryWork* wk,
             uint32_t* __restrict__ cand_pos, float* __restrict__ cand_lb) {
    extern __shared__ float s_lut[];
    __shared__ QueryShared qs;
    __shared__ uint32_t s_pos[kThreads / 32][kStageCap];
    __shared__ float s_lb[kThreads / 32][kStageCap];
    prepare_query(q, n, w, bits, thr_g, qs, s_lut);
    constexpr int H = WS / 16;
    constexpr int K = kPage / 32;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const float bound = bound_from_bits(wk->bsf_bits);
    const uint32_t nsurv = wk->nsurv;
    const uint64_t gwarp = (blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x) >> 5;
    const uint64_t nwarps = static_cast<uint64_t>(gridDim.x) * (blockDim.x >> 5);
    int cnt = 0;
    unsigned long long scanned = 0;
    for (uint64_t i = gwarp; i < nsurv; i += nwarps) {
        const uint32_t page = surv[i];
        const uint32_t a = page_off[page], b = page_off[page + 1];
        scanned += b - a;
        uint4 wv[K][H];
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const uint32_t e = a + lane + 32 * k;
#pragma unroll
            for (int h = 0; h < H; ++h)
                wv[k][h] = e < b ? ld_stream_u4(words + static_cast<uint64_t>(e) * WS + 16 * h) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const uint32_t e = a + lane + 32 * k;
            float lb = 0.f;
#pragma unroll
            for (int h = 0; h < H; ++h) {
                const int smax = min(16, w - 16 * h);
#pragma unroll
                for (int s = 0; s < 16; ++s)
                    if (s < smax) lb = __fadd_rd(lb, s_lut[(16 * h + s) * 256 + byte_of(wv[k][h], s)]);
            }
            const bool pass = e < b && lb <= bound;
            const unsigned m = __ballot_sync(0xFFFFFFFFu, pass);
            if (m) {
                if (pass) {
                    const int slot = cnt + __popc(m & ((1u << lane) - 1u));
                    s_pos[warp][slot] = pos[e];
                    s_lb[warp][slot] = lb;
                }
                cnt += __popc(m);
                __syncwarp();
                if (cnt > kStageCap - 32) {
                    flush_stage(wk, s_pos[warp], s_lb[warp], cnt, lane, cand_pos, cand_lb);
                    cnt = 0;
                }
            }
        }
    }
    if (cnt) flush_stage(wk, s_pos[warp], s_lb[warp], cnt, lane, cand_pos, cand_lb);
    if (lane == 0 && scanned) atomicAdd(&wk->stats[kLbEntry], scanned);
}

// ------------------------------------------------------------ refine
template <bool VEC>
__global__ void __launch_bounds__(kThreads)
    k_refine(const float* __restrict__ rows, int n, const float* __restrict__ query, QueryWork* wk,
             const uint32_t* __restrict__ cand_pos, const float* __restrict__ cand_lb,
             double* __restrict__ cand_sq) {
    extern __shared__ float s_q[];
    load_query(s_q, query, n);
    const uint32_t begin = wk->nseed, end = wk->ncand;
    unsigned long long refined = 0, updates = 0;
    for (uint64_t c = begin + blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; c < end;
         c += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const float lb = cand_lb[c];
        const uint32_t p = cand_pos[c];
        if (lb > bound_from_bits(ld_volatile_u64(&wk->bsf_bits))) {
            cand_sq[c] = INFINITY;
            continue;
        }
        refined += 1;
        const double s = row_sq<VEC>(rows + static_cast<uint64_t>(p) * n, s_q, n, &wk->bsf_bits);
        updates += publish(wk, s, c, cand_sq);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        refined += __shfl_xor_sync(0xFFFFFFFFu, refined, o);
        updates += __shfl_xor_sync(0xFFFFFFFFu, updates, o);
    }
    if ((threadIdx.x & 31) == 0) {
        if (refined) atomicAdd(&wk->stats[kRealDist], refined);
        if (updates) atomicAdd(&wk->stats[kBsfUpd], updates);
    }
}

// ----------------------------------------------------------- finalize
// Lowest position among the candidates whose sqrt(sum) equals the best
// distance; the last block to finish writes the result and resets `wk`.
__global__ void __launch_bounds__(kThreads)
    k_finalize(QueryWork* wk, const uint32_t* __restrict__ cand_pos, const double* __restrict__ cand_sq, int seed_only,
               DevResult* out, uint64_t P, uint64_t pos_offset) {
    const double best = bsf_of(wk->bsf_bits);
    const double dist = sqrt(best);
    const double lim = best * kSlack;
    const uint32_t end = seed_only ? wk->nseed : wk->ncand;
    uint32_t mine = 0xFFFFFFFFu;
    for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < end; c += gridDim.x * blockDim.x) {
        const double s = cand_sq[c];
        if (s <= lim && sqrt(s) == dist) mine = min(mine, cand_pos[c]);
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
    out->stats[kLbNode] = P;
    out->stats[kLbEntry] = wk->stats[kLbEntry] + wk->nseed;
    out->stats[kRealDist] = wk->stats[kRealDist];
    out->stats[kBsfUpd] = wk->stats[kBsfUpd];
    out->stats[kPruned] = wk->stats[kPruned];
    out->stats[kQueueIns] = wk->ncand - wk->nseed;
    reset_work(wk);  // for the next query on this stream
    __threadfence();
    wk->done_blocks = 0;
}

unsigned cap_grid(uint64_t want, int sms, int per_sm) {
    return static_cast<unsigned>(std::max<uint64_t>(1, std::min<uint64_t>(want, static_cast<uint64_t>(sms) * per_sm)));
}

}  // namespace

void search_batch(DevIndex& ix, const float* d_queries, uint32_t nq, bool approximate) {
    cudaStream_t st = ix.stream;
    const int n = ix.n, w = ix.w;
    const size_t lut_bytes = static_cast<size_t>(w) * 256 * sizeof(float);
    const size_t q_bytes = static_cast<size_t>(n) * sizeof(float);
    const bool vec = (n % 8) == 0 && (reinterpret_cast<uintptr_t>(ix.rows) % 32) == 0;
    auto refine = vec ? k_refine<true> : k_refine<false>;
    auto seed = vec ? k_seed<true> : k_seed<false>;
    auto lbscan = ix.ws == 16 ? k_lbscan<16> : k_lbscan<32>;
    // Per-device function attributes (cheap; set on every call so each device is covered).
    TSG_CUDA(cudaFuncSetAttribute(refine, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024));
    TSG_CUDA(cudaFuncSetAttribute(seed, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024));
    TSG_CUDA(cudaFuncSetAttribute(lbscan, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024));
    TSG_CUDA(cudaFuncSetAttribute(k_bound, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024));
    const uint32_t seed_cap = static_cast<uint32_t>(std::min<uint64_t>(2 * ix.leaf_cap, 1u << 20));
    const unsigned bound_grid = cap_grid((ix.P + kThreads - 1) / kThreads, ix.sms, 4);
    const unsigned filter_grid = cap_grid((ix.P + kThreads - 1) / kThreads, ix.sms, 8);
    const unsigned seed_grid = cap_grid((std::min<uint64_t>(seed_cap, ix.N) + 127) / 128, ix.sms, 2);

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

    k_reset<<<1, 1, 0, st>>>(ix.work);
    TSG_LAUNCHED();
    for (uint32_t qi = 0; qi < nq; ++qi) {
        const float* q = d_queries + static_cast<uint64_t>(qi) * n;
        mark(1, [&] {
            k_bound<<<bound_grid, kThreads, lut_bytes, st>>>(q, n, w, ix.bits, ix.thr, ix.page_lo, ix.page_hi, ix.P,
                                                             ix.ws, ix.work, ix.page_lb);
        });
        TSG_LAUNCHED();
        mark(2, [&] {
            seed<<<seed_grid, 128, q_bytes, st>>>(ix.rows, n, q, ix.leaf_off, ix.page_off, ix.page_leaf, ix.pos,
                                                  seed_cap, ix.work, ix.cand_pos, ix.cand_sq);
        });
        TSG_LAUNCHED();
        if (!approximate) {
            mark(3, [&] { k_filter<<<filter_grid, kThreads, 0, st>>>(ix.page_lb, ix.page_off, ix.P, ix.work, ix.surv); });
            TSG_LAUNCHED();
            mark(4, [&] {
                lbscan<<<ix.sms * 4, kThreads, lut_bytes, st>>>(q, n, w, ix.bits, ix.thr, ix.words, ix.pos,
                                                                ix.page_off, ix.surv, ix.work, ix.cand_pos,
                                                                ix.cand_lb);
            });
            TSG_LAUNCHED();
            mark(5, [&] {
                refine<<<ix.sms * 8, kThreads, q_bytes, st>>>(ix.rows, n, q, ix.work, ix.cand_pos, ix.cand_lb,
                                                              ix.cand_sq);
            });
            TSG_LAUNCHED();
        }
        mark(6, [&] {
            k_finalize<<<ix.sms, kThreads, 0, st>>>(ix.work, ix.cand_pos, ix.cand_sq, approximate ? 1 : 0,
                                                    ix.results + qi, ix.P, ix.pos_offset);
        });
        TSG_LAUNCHED();
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
