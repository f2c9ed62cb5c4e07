// Exact Euclidean 1-NN over the flat SoA index (one device shard).
//
// Replaces exact_search (src/query.cpp:258-298) and its pieces:
//   prep      QueryState (src/query.cpp:81-100): query PAA in FP64 reference
//             order, query symbols, and a [w][256] table of per-segment
//             squared region gaps (mindist_bands, src/metrics.cpp:47-70)
//             rounded DOWN to float, so every float lower bound below is <=
//             the exact FP64 bound (sound pruning).
//   leaf LB   node_lower_bound over every leaf box (src/query.cpp:102-107);
//             the argmin leaf seeds the best-so-far, the analog of
//             approximate_search_state (src/query.cpp:226-238).
//   refine    calculate_real_distance_leaf + euclidean (src/query.cpp:121-152,
//             src/metrics.cpp:17-40): one warp per candidate row, lane j owns
//             the j-th block of 8 floats, FP64 block sums without FMA, then
//             the block sums are added left to right exactly like
//             squared_l2; best-so-far = atomicMin on the double bit pattern
//             (non-negative doubles order as unsigned integers), the
//             SharedBsf analog (src/query.cpp:35-42).
//   lbscan    traverse_root_subtree + the entry-level LB filter
//             (src/query.cpp:129-134,154-171): leaves whose box bound exceeds
//             the BSF are skipped whole; words of surviving leaves are
//             bounded with 16 table lookups and compacted with warp ballot +
//             prefix popcount into a candidate list.
//   finalize  result = min over refined candidates of (sqrt(sum), position):
//             ties resolve to the lowest position exactly as scan_nn does
//             (src/scan.cpp:54-59).
// Pruning keeps ties: a candidate is dropped only when its bound is strictly
// above the best-so-far widened by 1e-9 relative (covering FP64 rounding of
// the distance sums), so the exact answer is never lost.
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

enum Stat { kLbNode = 0, kLbEntry, kRealDist, kBsfUpd, kPruned, kQueueIns };

__device__ __forceinline__ float bound_from_bits(unsigned long long bits) {
    const double s = __longlong_as_double(static_cast<long long>(bits));
    return __double2float_ru(s * kSlack);
}

// ---------------------------------------------------------------- prep
__global__ void k_query_prep(const float* __restrict__ q, int n, int w, int bits,
                             const double* __restrict__ thr_g, QueryWork* wk, float* __restrict__ lut) {
    __shared__ double thr[kThrPad];
    __shared__ double qpaa[kMaxW];
    for (int i = threadIdx.x; i < kThrPad; i += blockDim.x) thr[i] = thr_g[i];
    __syncthreads();
    const int seg = n / w;
    if (threadIdx.x < w) {
        const int g = threadIdx.x;
        double sum = 0.0;
        for (int j = 0; j < seg; ++j) sum = __dadd_rn(sum, static_cast<double>(q[g * seg + j]));
        const double mean = __ddiv_rn(sum, static_cast<double>(seg));
        qpaa[g] = mean;
        wk->qpaa[g] = mean;
        wk->qsym[g] = static_cast<unsigned char>(symbol_of(thr, bits, mean) << (8 - bits));
    }
    if (threadIdx.x == 0) {
        wk->bsf_bits = kInfBits;
        wk->seed_key = ~0ull;
        wk->ncand = 0;
        wk->nseed = 0;
        wk->work_next = 0;
        wk->best_pos = 0xFFFFFFFFu;
        for (int i = 0; i < 6; ++i) wk->stats[i] = 0;
    }
    __syncthreads();
    const unsigned card = 1u << bits;
    const double scale = static_cast<double>(n) / static_cast<double>(w);
    for (int idx = threadIdx.x; idx < w * 256; idx += blockDim.x) {
        const int s = idx >> 8, v = idx & 255;
        const unsigned prefix = static_cast<unsigned>(v) >> (8 - bits);
        const double lo = prefix == 0 ? -INFINITY : thr[prefix - 1];
        const double hi = prefix == card - 1 ? INFINITY : thr[prefix];
        const double x = qpaa[s];
        double gap = 0.0;
        if (x < lo) gap = lo - x;
        else if (x > hi) gap = x - hi;
        lut[idx] = __double2float_rd(__dmul_rn(__dmul_rn(gap, gap), scale));
    }
}

// Loads the [w][256] table and the query symbols into shared memory.
__device__ __forceinline__ void load_lut(float* s_lut, unsigned char* s_qsym, const float* lut,
                                         const QueryWork* wk, int w) {
    for (int i = threadIdx.x; i < w * 256; i += blockDim.x) s_lut[i] = lut[i];
    for (int i = threadIdx.x; i < w; i += blockDim.x) s_qsym[i] = wk->qsym[i];
}

__device__ __forceinline__ uint8_t byte_of(const uint4& v, int s) {
    const uint32_t word = s < 4 ? v.x : s < 8 ? v.y : s < 12 ? v.z : v.w;
    return static_cast<uint8_t>(word >> (8 * (s & 3)));
}

// ------------------------------------------------------------- page LB
// Lower bound of every page box (the node bound of src/query.cpp:102-107 at
// page granularity); the argmin page seeds the best-so-far.
__global__ void k_page_lb(const uint8_t* __restrict__ lo, const uint8_t* __restrict__ hi, uint64_t L, int w,
                          int ws, const float* __restrict__ lut, QueryWork* wk, float* __restrict__ leaf_lb) {
    extern __shared__ float s_lut[];
    __shared__ unsigned char s_qsym[kMaxW];
    load_lut(s_lut, s_qsym, lut, wk, w);
    __syncthreads();
    unsigned long long best = ~0ull;
    for (uint64_t l = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; l < L;
         l += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        float lb = 0.f;
        for (int h = 0; h < ws / 16; ++h) {
            const uint4 a = *reinterpret_cast<const uint4*>(lo + l * ws + 16 * h);
            const uint4 b = *reinterpret_cast<const uint4*>(hi + l * ws + 16 * h);
            const int smax = min(16, w - 16 * h);
            for (int s = 0; s < smax; ++s) {
                const int g = 16 * h + s;
                const uint8_t ql = s_qsym[g], bl = byte_of(a, s), bh = byte_of(b, s);
                const float gv = ql < bl ? s_lut[g * 256 + bl] : (ql > bh ? s_lut[g * 256 + bh] : 0.f);
                lb = __fadd_rd(lb, gv);
            }
        }
        leaf_lb[l] = lb;
        const unsigned long long key = (static_cast<unsigned long long>(__float_as_uint(lb)) << 32) | l;
        best = min(best, key);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) best = min(best, __shfl_xor_sync(0xFFFFFFFFu, best, o));
    if ((threadIdx.x & 31) == 0 && best != ~0ull) atomicMin(&wk->seed_key, best);
}

// ---------------------------------------------------------- seed leaf
// The seed is the leaf holding the best page (the analog of the leaf the
// reference's approximate search descends to); an overflow leaf larger than
// seed_cap is replaced by the page alone.
__global__ void k_seed(const uint32_t* __restrict__ leaf_off, const uint32_t* __restrict__ page_off,
                       const uint32_t* __restrict__ page_leaf, const uint32_t* __restrict__ pos, uint32_t seed_cap,
                       QueryWork* wk, uint32_t* __restrict__ cand_pos, float* __restrict__ cand_lb) {
    const uint32_t page = static_cast<uint32_t>(wk->seed_key & 0xFFFFFFFFull);
    const uint32_t leaf = page_leaf[page];
    uint32_t a = leaf_off[leaf], b = leaf_off[leaf + 1];
    if (b - a > seed_cap) {
        a = page_off[page];
        b = page_off[page + 1];
    }
    for (uint32_t e = a + blockIdx.x * blockDim.x + threadIdx.x; e < b; e += gridDim.x * blockDim.x) {
        cand_pos[e - a] = pos[e];
        cand_lb[e - a] = 0.f;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        wk->nseed = b - a;
        wk->ncand = b - a;
        wk->seed_begin = a;
        wk->seed_end = b;
    }
}

// -------------------------------------------------------------- refine
// UNROLL candidates per warp iteration for memory-level parallelism.
template <int UNROLL, bool VEC>
__global__ void __launch_bounds__(256)
    k_refine(const float* __restrict__ rows, int n, const float* __restrict__ query, QueryWork* wk,
             const uint32_t* __restrict__ cand_pos, const float* __restrict__ cand_lb,
             double* __restrict__ cand_sq, int seed_phase) {
    extern __shared__ unsigned char smem[];
    const int nb = (n + 7) >> 3;
    float* s_q = reinterpret_cast<float*>(smem);
    double* s_blk = reinterpret_cast<double*>(smem + ((n * 4 + 15) & ~15));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double* wblk = s_blk + static_cast<size_t>(warp) * UNROLL * nb;
    for (int i = threadIdx.x; i < n; i += blockDim.x) s_q[i] = query[i];
    __syncthreads();

    const uint32_t begin = seed_phase ? 0u : wk->nseed;
    const uint32_t end = seed_phase ? wk->nseed : wk->ncand;
    const uint64_t gwarp = (blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x) >> 5;
    const uint64_t nwarps = static_cast<uint64_t>(gridDim.x) * (blockDim.x >> 5);
    unsigned long long refined = 0, updates = 0;

    for (uint64_t c0 = begin + gwarp * UNROLL; c0 < end; c0 += nwarps * UNROLL) {
        const float bound = seed_phase ? INFINITY : bound_from_bits(ld_volatile_u64(&wk->bsf_bits));
        bool live[UNROLL];
        const float* rp[UNROLL];
#pragma unroll
        for (int u = 0; u < UNROLL; ++u) {
            const uint64_t c = c0 + u;
            live[u] = c < end && cand_lb[c] <= bound;
            rp[u] = live[u] ? rows + static_cast<uint64_t>(cand_pos[c]) * n : nullptr;
        }
        for (int b0 = 0; b0 < nb; b0 += 32) {
            const int b = b0 + lane;
            if (b < nb) {
                const int j0 = b * 8;
                if (VEC) {
                    const float4 q0 = *reinterpret_cast<const float4*>(s_q + j0);
                    const float4 q1 = *reinterpret_cast<const float4*>(s_q + j0 + 4);
                    float4 x0[UNROLL], x1[UNROLL];
#pragma unroll
                    for (int u = 0; u < UNROLL; ++u)
                        if (live[u]) {
                            x0[u] = ld_stream_f4(rp[u] + j0);
                            x1[u] = ld_stream_f4(rp[u] + j0 + 4);
                        }
#pragma unroll
                    for (int u = 0; u < UNROLL; ++u) {
                        if (!live[u]) continue;
                        const float xs[8] = {x0[u].x, x0[u].y, x0[u].z, x0[u].w, x1[u].x, x1[u].y, x1[u].z, x1[u].w};
                        const float qs[8] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w};
                        double blk = 0.0;
#pragma unroll
                        for (int k = 0; k < 8; ++k) {
                            const double d = __dsub_rn(static_cast<double>(xs[k]), static_cast<double>(qs[k]));
                            blk = __dadd_rn(blk, __dmul_rn(d, d));
                        }
                        wblk[u * nb + b] = blk;
                    }
                } else {
                    const int j1 = min(j0 + 8, n);
#pragma unroll
                    for (int u = 0; u < UNROLL; ++u) {
                        if (!live[u]) continue;
                        double blk = 0.0;
                        for (int j = j0; j < j1; ++j) {
                            const double d = __dsub_rn(static_cast<double>(rp[u][j]), static_cast<double>(s_q[j]));
                            blk = __dadd_rn(blk, __dmul_rn(d, d));
                        }
                        wblk[u * nb + b] = blk;
                    }
                }
            }
        }
        __syncwarp();
        if (lane < UNROLL) {
            const uint64_t c = c0 + lane;
            bool mine = false;
#pragma unroll
            for (int u = 0; u < UNROLL; ++u)
                if (u == lane) mine = live[u];
            if (c < end) {
                if (mine) {
                    double s = 0.0;
                    const double* bl = wblk + lane * nb;
                    for (int b = 0; b < nb; ++b) s = __dadd_rn(s, bl[b]);
                    cand_sq[c] = s;
                    const unsigned long long sb = static_cast<unsigned long long>(__double_as_longlong(s));
                    const unsigned long long old = atomicMin(&wk->bsf_bits, sb);
                    refined += 1;
                    updates += old > sb ? 1 : 0;
                } else {
                    cand_sq[c] = INFINITY;
                }
            }
        }
        __syncwarp();
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        refined += __shfl_xor_sync(0xFFFFFFFFu, refined, o);
        updates += __shfl_xor_sync(0xFFFFFFFFu, updates, o);
    }
    if (lane == 0) {
        if (refined) atomicAdd(&wk->stats[kRealDist], refined);
        if (updates) atomicAdd(&wk->stats[kBsfUpd], updates);
    }
}

// -------------------------------------------------------------- lbscan
constexpr int kStageCap = 256;

__device__ __forceinline__ void flush_stage(QueryWork* wk, uint32_t* s_pos, float* s_lb, int cnt, int lane,
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

// Warps pull batches of 32 pages (<= kPage entries each, so work units are
// bounded); surviving pages' entries are packed across the warp's lanes
// (prefix sums of page sizes), so small pages do not idle lanes. Pages of the
// seed range were already refined and are skipped.
__global__ void __launch_bounds__(256)
    k_lbscan(const uint8_t* __restrict__ words, const uint32_t* __restrict__ pos,
             const uint32_t* __restrict__ leaf_off, const float* __restrict__ leaf_lb, uint64_t L, int w, int ws,
             const float* __restrict__ lut, QueryWork* wk, uint32_t* __restrict__ cand_pos,
             float* __restrict__ cand_lb) {
    extern __shared__ float s_lut[];
    __shared__ unsigned char s_qsym[kMaxW];
    __shared__ uint32_t s_pos[8][kStageCap];
    __shared__ float s_lb[8][kStageCap];
    load_lut(s_lut, s_qsym, lut, wk, w);
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const float bound = bound_from_bits(wk->bsf_bits);
    const uint32_t seed_begin = wk->seed_begin, seed_end = wk->seed_end;
    const uint64_t nbatch = (L + 31) / 32;
    int cnt = 0;
    unsigned long long scanned = 0, pruned = 0;
    while (true) {
        uint32_t batch = 0;
        if (lane == 0) batch = atomicAdd(&wk->work_next, 1u);
        batch = __shfl_sync(0xFFFFFFFFu, batch, 0);
        if (batch >= nbatch) break;
        const uint64_t l = static_cast<uint64_t>(batch) * 32 + lane;
        const bool valid = l < L;
        const uint32_t pa = valid ? leaf_off[l] : 0u;
        const uint32_t pb = valid ? leaf_off[l + 1] : 0u;
        const bool seeded = valid && pa >= seed_begin && pb <= seed_end;
        const bool keep = valid && !seeded && leaf_lb[l] <= bound;
        pruned += __popc(__ballot_sync(0xFFFFFFFFu, valid && !keep && !seeded));
        const uint32_t start = keep ? pa : 0u;
        const uint32_t size = keep ? pb - pa : 0u;
        uint32_t incl = size;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, incl, o);
            if (lane >= o) incl += t;
        }
        const uint32_t total = __shfl_sync(0xFFFFFFFFu, incl, 31);
        scanned += total;
        for (uint32_t g = 0; g < total; g += 32) {
            const uint32_t v = g + lane;
            const bool active = v < total;
            // owner leaf slot: smallest i with incl_i > v (binary search across lanes)
            int lo = 0;
#pragma unroll
            for (int step = 16; step > 0; step >>= 1) {
                const uint32_t probe = __shfl_sync(0xFFFFFFFFu, incl, lo + step - 1);
                if (probe <= v) lo += step;
            }
            const uint32_t i_incl = __shfl_sync(0xFFFFFFFFu, incl, lo);
            const uint32_t i_size = __shfl_sync(0xFFFFFFFFu, size, lo);
            const uint32_t i_start = __shfl_sync(0xFFFFFFFFu, start, lo);
            bool pass = false;
            float lb = 0.f;
            uint32_t e = 0;
            if (active) {
                e = i_start + (v - (i_incl - i_size));
                const uint8_t* wp = words + static_cast<uint64_t>(e) * ws;
                for (int h = 0; h < ws / 16; ++h) {
                    const uint4 wv = ld_stream_u4(wp + 16 * h);
                    const int smax = min(16, w - 16 * h);
                    for (int s = 0; s < smax; ++s)
                        lb = __fadd_rd(lb, s_lut[(16 * h + s) * 256 + byte_of(wv, s)]);
                }
                pass = lb <= bound;
            }
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
    if (lane == 0) {
        atomicAdd(&wk->stats[kLbEntry], scanned);
        atomicAdd(&wk->stats[kPruned], pruned);
    }
}

// ------------------------------------------------------------ finalize
__global__ void k_finalize(QueryWork* wk, const uint32_t* __restrict__ cand_pos, const double* __restrict__ cand_sq,
                           int seed_only) {
    const double best = __longlong_as_double(static_cast<long long>(wk->bsf_bits));
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
}

__global__ void k_result(const QueryWork* wk, DevResult* out, uint64_t L, uint64_t pos_offset) {
    const double best = __longlong_as_double(static_cast<long long>(wk->bsf_bits));
    out->distance = sqrt(best);
    out->position = static_cast<uint32_t>(wk->best_pos + pos_offset);
    out->reserved = 0;
    out->stats[kLbNode] = L;
    out->stats[kLbEntry] = wk->stats[kLbEntry] + wk->nseed;
    out->stats[kRealDist] = wk->stats[kRealDist];
    out->stats[kBsfUpd] = wk->stats[kBsfUpd];
    out->stats[kPruned] = wk->stats[kPruned];
    out->stats[kQueueIns] = wk->ncand - wk->nseed;
}

unsigned cap_grid(uint64_t want, int sms, int per_sm) {
    return static_cast<unsigned>(std::max<uint64_t>(1, std::min<uint64_t>(want, static_cast<uint64_t>(sms) * per_sm)));
}

}  // namespace

void search_batch(DevIndex& ix, const float* d_queries, uint32_t nq, bool approximate) {
    cudaStream_t st = ix.stream;
    const int n = ix.n, w = ix.w;
    const size_t lut_bytes = static_cast<size_t>(w) * 256 * sizeof(float);
    const int nb = (n + 7) / 8;
    constexpr int kUnroll = 4;
    const bool vec = (n % 8) == 0 && (reinterpret_cast<uintptr_t>(ix.rows) % 16) == 0;
    const size_t refine_smem = ((static_cast<size_t>(n) * 4 + 15) & ~size_t(15)) +
                               static_cast<size_t>(8) * kUnroll * nb * sizeof(double);
    auto refine = vec ? k_refine<kUnroll, true> : k_refine<kUnroll, false>;
    // Per-device function attributes (cheap; set on every call so each device is covered).
    TSG_CUDA(cudaFuncSetAttribute(refine, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    TSG_CUDA(cudaFuncSetAttribute(k_lbscan, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024));
    if (refine_smem > 200 * 1024) throw InvalidArgument("series length too large for the device refine kernel");
    const uint32_t seed_cap = static_cast<uint32_t>(std::min<uint64_t>(2 * ix.leaf_cap, 1u << 20));

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

    for (uint32_t qi = 0; qi < nq; ++qi) {
        const float* q = d_queries + static_cast<uint64_t>(qi) * n;
        mark(0, [&] { k_query_prep<<<1, 256, 0, st>>>(q, n, w, ix.bits, ix.thr, ix.work, ix.lut); });
        TSG_LAUNCHED();
        mark(1, [&] {
            k_page_lb<<<cap_grid((ix.P + 255) / 256, ix.sms, 4), 256, lut_bytes, st>>>(
                ix.page_lo, ix.page_hi, ix.P, w, ix.ws, ix.lut, ix.work, ix.page_lb);
        });
        TSG_LAUNCHED();
        mark(2, [&] {
            k_seed<<<32, 256, 0, st>>>(ix.leaf_off, ix.page_off, ix.page_leaf, ix.pos, seed_cap, ix.work,
                                       ix.cand_pos, ix.cand_lb);
        });
        TSG_LAUNCHED();
        mark(3, [&] {
            refine<<<ix.sms * 2, 256, refine_smem, st>>>(ix.rows, n, q, ix.work, ix.cand_pos, ix.cand_lb,
                                                         ix.cand_sq, 1);
        });
        TSG_LAUNCHED();
        if (!approximate) {
            mark(4, [&] {
                k_lbscan<<<ix.sms * 4, 256, lut_bytes, st>>>(ix.words, ix.pos, ix.page_off, ix.page_lb, ix.P, w,
                                                             ix.ws, ix.lut, ix.work, ix.cand_pos, ix.cand_lb);
            });
            TSG_LAUNCHED();
            mark(5, [&] {
                refine<<<ix.sms * 4, 256, refine_smem, st>>>(ix.rows, n, q, ix.work, ix.cand_pos, ix.cand_lb,
                                                             ix.cand_sq, 0);
            });
            TSG_LAUNCHED();
        }
        mark(6, [&] { k_finalize<<<ix.sms, 256, 0, st>>>(ix.work, ix.cand_pos, ix.cand_sq, approximate ? 1 : 0); });
        TSG_LAUNCHED();
        mark(7, [&] { k_result<<<1, 1, 0, st>>>(ix.work, ix.results + qi, ix.P, ix.pos_offset); });
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
