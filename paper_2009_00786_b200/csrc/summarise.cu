// K1 summarise: float32 rows -> iSAX words + root keys + sort keys.
//
// Replaces the summarization hot loop of the reference build
// (src/index.cpp:162-167): paa_into (src/sax.cpp:10-25) + symbols_from_paa
// (src/sax.cpp:39-47) + root_key_from_symbols (src/sax.cpp:59-63).
//
// Bit-exactness: every PAA segment is summed in FP64, sequentially from 0.0
// in the reference's order, then divided by the segment length (IEEE
// division); the symbol is the number of FP64 thresholds <= mean.
//
// Data movement (B200): a persistent grid, one producer warp per CTA issues
// 2-D TMA loads (cp.async.bulk.tensor) of R whole series (R*n*4 bytes, 32 KB
// for n=256) into a STAGES-deep shared-memory ring with the 128-byte
// swizzle; 8 consumer warps read their segments back conflict-free (the
// swizzle XOR spreads the 8 lanes of an LDS.128 phase over all 32 banks),
// then one thread per series writes the 16-byte word and its keys.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>

#include "common.cuh"
#include "kernels.cuh"

namespace tsg {

namespace {

constexpr int kConsumerWarps = 8;
constexpr int kConsumers = kConsumerWarps * 32;
constexpr int kSumThreads = kConsumers + 32;  // + one producer warp

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1,
                                            uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
        "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}

// Swizzle-128B address of byte offset a inside a 1024-aligned tile.
__device__ __forceinline__ uint32_t swz(uint32_t a) { return a ^ (((a >> 7) & 7u) << 4); }

struct SumArgs {
    uint64_t count;     // series in this launch
    uint64_t out_base;  // output index of this launch's first series
    int n, w, bits, seg, R, ws;
    uint8_t* words;
    uint32_t* root_keys;  // may be null
    uint64_t* sort_keys;  // may be null
    uint8_t* fine;        // may be null: fine summary rows (fws bytes each)
    int fw, fws;
    int wst, fst;         // output strides of words / fine rows (bytes): ws / fws, or a shared record stride
    int pad_after_fine;   // record layout: zero bytes written after each fine row (the record's tail), so
                          // the record's last 32-byte sector is written whole (a partial sector costs a
                          // DRAM read-modify-write: profiles/micro/dram_granularity.cu)
    uint64_t key_mask;    // sort keys keep these bits (the sorted key width)
};

// Sort key: the first 64 bits of the plane-major bit string of the word
// (plane 0 = top bit of every segment = the root key, segment 0 first;
// then the second bit of every segment, ...). Sorting by it makes root
// subtrees contiguous and orders entries inside them the way the iSAX
// refinement bits split them.
__device__ __forceinline__ void word_keys(const uint8_t* sym, int w, uint32_t& root, uint64_t& sk) {
    uint32_t r = 0;
    for (int g = 0; g < w; ++g) r = (r << 1) | (sym[g] >> 7);
    root = r;
    uint64_t k = 0;
    int left = 64;
    for (int p = 0; p < 8 && left > 0; ++p)
        for (int g = 0; g < w && left > 0; ++g, --left) k = (k << 1) | ((sym[g] >> (7 - p)) & 1u);
    sk = left >= 64 ? 0 : k << left;
}

__device__ __forceinline__ void emit_word(const SumArgs& a, uint64_t idx, const uint8_t* wrow) {
    uint4* dst = reinterpret_cast<uint4*>(a.words + idx * static_cast<uint64_t>(a.wst));
    const uint4* src = reinterpret_cast<const uint4*>(wrow);
    dst[0] = src[0];
    if (a.ws == 32) dst[1] = src[1];
    if (a.root_keys || a.sort_keys) {
        uint32_t root;
        uint64_t sk;
        word_keys(wrow, a.w, root, sk);
        if (a.root_keys) a.root_keys[idx] = root;
        if (a.sort_keys) a.sort_keys[idx] = sk & a.key_mask;
    }
}

// SEG > 0: compile-time segment length of the w = 16 path (n = 16 SEG);
// VEC: segments are whole float4s.
template <int STAGES, int SEG, bool VEC, bool FINE>
__global__ void __launch_bounds__(kSumThreads, 2)
    k_summarise_tma(const __grid_constant__ CUtensorMap tmap, SumArgs a,
                    const double* __restrict__ thr_g) {
    extern __shared__ unsigned char smem_raw[];
    // (offset arithmetic on the shared array keeps the shared address space: LDS, not generic loads)
    unsigned char* stages = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    const uint32_t tile_bytes = static_cast<uint32_t>(a.R) * a.n * 4u;
    const uint32_t stage_stride = (tile_bytes + 1023u) & ~1023u;
    uint64_t* full = reinterpret_cast<uint64_t*>(stages + STAGES * stage_stride);
    uint64_t* empty = full + STAGES;
    double* thr = reinterpret_cast<double*>(empty + STAGES);
    unsigned char* bins = reinterpret_cast<unsigned char*>(thr + kThrPad);
    uint8_t* wbuf = bins + kBins;

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kConsumerWarps);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    for (int i = tid; i < kThrPad; i += blockDim.x) thr[i] = thr_g[i];
    {
        const unsigned char* bins_g = reinterpret_cast<const unsigned char*>(thr_g + kThrPad);
        for (int i = tid; i < kBins; i += blockDim.x) bins[i] = bins_g[i];
    }
    for (int i = tid; i < 2 * a.R * a.ws; i += blockDim.x) wbuf[i] = 0;
    __syncthreads();

    const uint64_t ntiles = (a.count + a.R - 1) / a.R;
    const int rows_per_tile = a.R * (a.n / 32);

    if (warp == kConsumerWarps) {  // producer warp
        if (lane == 0) {
            int it = 0;
            for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
                const int s = it % STAGES;
                if (it >= STAGES) mbar_wait(&empty[s], ((it / STAGES) - 1) & 1);
                mbar_expect_tx(&full[s], tile_bytes);
                tma_load_2d(stages + s * stage_stride, &tmap, 0, static_cast<int>(t * rows_per_tile),
                            &full[s]);
            }
        }
        return;
    }

    // Segment mean: sum / seg. For a power-of-two seg, multiplying by the exact
    // reciprocal is the same IEEE result as the division (pure exponent
    // shift, identical rounding), and far cheaper than DDIV's sequence.
    const int segl = SEG > 0 ? SEG : a.seg;
    const bool pow2 = (segl & (segl - 1)) == 0;
    const double inv_seg = 1.0 / static_cast<double>(segl);
    // FINE: the same pass also yields the two half-segment sums (the first
    // half is a prefix of the reference-order sum; the second half is summed
    // from 0.0 in its own chain) -> two fine symbols packed in *fine2.
    const int half = segl >> 1;
    const bool pow2h = (half & (half - 1)) == 0;
    const double inv_half = 1.0 / static_cast<double>(half);
    auto segment_symbol = [&](const unsigned char* tile, int ser, int g, unsigned* fine2) -> unsigned {
        const uint32_t f0 = static_cast<uint32_t>(ser * (SEG > 0 ? 16 * SEG : a.n) + g * segl);
        double sum = 0.0, sa = 0.0, sb = 0.0;
        if (VEC) {
            const int nq = segl >> 2, nqh = half >> 2;  // FINE && VEC: seg % 8 == 0
#pragma unroll
            for (int q = 0; q < nq; ++q) {
                const float4 v = *reinterpret_cast<const float4*>(tile + swz((f0 + 4u * q) * 4u));
                sum = __dadd_rn(sum, static_cast<double>(v.x));
                sum = __dadd_rn(sum, static_cast<double>(v.y));
                sum = __dadd_rn(sum, static_cast<double>(v.z));
                sum = __dadd_rn(sum, static_cast<double>(v.w));
                if (FINE) {
                    if (q >= nqh) {
                        sb = __dadd_rn(sb, static_cast<double>(v.x));
                        sb = __dadd_rn(sb, static_cast<double>(v.y));
                        sb = __dadd_rn(sb, static_cast<double>(v.z));
                        sb = __dadd_rn(sb, static_cast<double>(v.w));
                    }
                    if (q == nqh - 1) sa = sum;
                }
            }
        } else {
#pragma unroll
            for (int j = 0; j < segl; ++j) {
                const float v = *reinterpret_cast<const float*>(tile + swz((f0 + j) * 4u));
                sum = __dadd_rn(sum, static_cast<double>(v));
                if (FINE) {
                    if (j >= half) sb = __dadd_rn(sb, static_cast<double>(v));
                    if (j == half - 1) sa = sum;
                }
            }
        }
        if (FINE) {
            const double ma = pow2h ? __dmul_rn(sa, inv_half) : __ddiv_rn(sa, static_cast<double>(half));
            const double mb = pow2h ? __dmul_rn(sb, inv_half) : __ddiv_rn(sb, static_cast<double>(half));
            *fine2 = fine_quant(ma) | (fine_quant(mb) << 8);
        }
        const double mean = pow2 ? __dmul_rn(sum, inv_seg) : __ddiv_rn(sum, static_cast<double>(segl));
        return symbol_step(thr, bins, a.bits, mean) << (8 - a.bits);
    };

    int it = 0;
    if (a.w == 16) {
        // w = 16: a warp owns two whole series per step (lane = 16*half +
        // segment). Keys come from four warp ballots (planes 0..3, segment 0
        // = MSB), the word from three shuffles; no block barrier at all.
        for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
            const int s = it % STAGES;
            mbar_wait(&full[s], (it / STAGES) & 1);
            const unsigned char* tile = stages + s * stage_stride;
            const uint64_t first = t * a.R;
            const int valid = static_cast<int>(min(static_cast<uint64_t>(a.R), a.count - first));
            const int half = lane >> 4, g = lane & 15;
            for (int pair = warp; 2 * pair < valid; pair += kConsumerWarps) {
                const int ser = 2 * pair + half;
                const bool ok = ser < valid;
                unsigned f2 = 0;
                const unsigned sym = ok ? segment_symbol(tile, ser, g, &f2) : 0u;
                uint64_t key = 0;
#pragma unroll
                for (int p = 0; p < 4; ++p) {
                    const unsigned b = __ballot_sync(0xFFFFFFFFu, (sym >> (7 - p)) & 1u);
                    key = (key << 16) | (__brev((b >> (16 * half)) & 0xFFFFu) >> 16);
                }
                const unsigned b1 = __shfl_down_sync(0xFFFFFFFFu, sym, 1);
                const unsigned b2 = __shfl_down_sync(0xFFFFFFFFu, sym, 2);
                const unsigned b3 = __shfl_down_sync(0xFFFFFFFFu, sym, 3);
                const uint64_t idx = a.out_base + first + ser;
                if (ok && (g & 3) == 0)
                    reinterpret_cast<uint32_t*>(a.words + idx * a.wst)[g >> 2] = sym | (b1 << 8) | (b2 << 16) | (b3 << 24);
                if (ok && g == 0) {
                    if (a.sort_keys) a.sort_keys[idx] = key & a.key_mask;
                    if (a.root_keys) a.root_keys[idx] = static_cast<uint32_t>(key >> 48);
                }
                if (FINE) {  // 32 fine bytes per series: lanes g = 0, 8 store 16 each
                    const unsigned u = f2 | (__shfl_down_sync(0xFFFFFFFFu, f2, 1) << 16);
                    const unsigned u2 = __shfl_down_sync(0xFFFFFFFFu, u, 2);
                    const unsigned u4 = __shfl_down_sync(0xFFFFFFFFu, u, 4);
                    const unsigned u6 = __shfl_down_sync(0xFFFFFFFFu, u, 6);
                    if (ok && (g & 7) == 0)
                        *reinterpret_cast<uint4*>(a.fine + idx * a.fst + 2 * g) = make_uint4(u, u2, u4, u6);
                    if (ok && g == 8 && a.pad_after_fine == 16)
                        *reinterpret_cast<uint4*>(a.fine + idx * a.fst + 32) = make_uint4(0, 0, 0, 0);
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
        }
        return;
    }

    for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
        const int s = it % STAGES;
        mbar_wait(&full[s], (it / STAGES) & 1);
        const unsigned char* tile = stages + s * stage_stride;
        const uint64_t first = t * a.R;
        const int valid = static_cast<int>(min(static_cast<uint64_t>(a.R), a.count - first));
        uint8_t* wb = wbuf + (it & 1) * a.R * a.ws;
        for (int idx = tid; idx < valid * a.w; idx += kConsumers) {
            const int ser = idx / a.w, g = idx - ser * a.w;
            unsigned f2 = 0;
            wb[ser * a.ws + g] = static_cast<uint8_t>(segment_symbol(tile, ser, g, &f2));
            if (FINE)
                *reinterpret_cast<uint16_t*>(a.fine + (a.out_base + first + ser) * a.fst + 2 * g) =
                    static_cast<uint16_t>(f2);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
        asm volatile("bar.sync 1, %0;" ::"n"(kConsumers) : "memory");
        for (int ser = tid; ser < valid; ser += kConsumers)
            emit_word(a, a.out_base + first + ser, wb + ser * a.ws);
    }
}

// Shapes the TMA path cannot take (n % 32 != 0): one thread per series,
// direct loads. Same arithmetic.
__global__ void k_summarise_generic(const float* __restrict__ rows, SumArgs a,
                                    const double* __restrict__ thr_g) {
    __shared__ double thr[kThrPad];
    __shared__ unsigned char bins[kBins];
    for (int i = threadIdx.x; i < kThrPad; i += blockDim.x) thr[i] = thr_g[i];
    for (int i = threadIdx.x; i < kBins; i += blockDim.x)
        bins[i] = reinterpret_cast<const unsigned char*>(thr_g + kThrPad)[i];
    __syncthreads();
    uint8_t wrow[kMaxW] = {0};
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < a.count;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const float* r = rows + i * static_cast<uint64_t>(a.n);
        const int half = a.seg >> 1;
        for (int g = 0; g < a.w; ++g) {
            double sum = 0.0, sa = 0.0, sb = 0.0;
            for (int j = 0; j < a.seg; ++j) {
                const double v = static_cast<double>(r[g * a.seg + j]);
                sum = __dadd_rn(sum, v);
                if (j >= half) sb = __dadd_rn(sb, v);
                if (j == half - 1) sa = sum;
            }
            const double mean = __ddiv_rn(sum, static_cast<double>(a.seg));
            wrow[g] = static_cast<uint8_t>(symbol_fast(thr, bins, a.bits, mean) << (8 - a.bits));
            if (a.fine) {
                uint8_t* f = a.fine + (a.out_base + i) * a.fst + 2 * g;
                f[0] = static_cast<uint8_t>(fine_quant(__ddiv_rn(sa, static_cast<double>(half))));
                f[1] = static_cast<uint8_t>(fine_quant(__ddiv_rn(sb, static_cast<double>(half))));
            }
        }
        uint8_t buf[32] __attribute__((aligned(16)));
        for (int k = 0; k < 32; ++k) buf[k] = k < a.w ? wrow[k] : 0;
        emit_word(a, a.out_base + i, buf);
    }
}

PFN_cuTensorMapEncodeTiled_v12000 get_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    });
    if (!fn) throw CudaError("cuTensorMapEncodeTiled unavailable");
    return fn;
}

constexpr int kStages = 3;

size_t tma_smem_bytes(int R, int n, int ws) {
    const size_t stage = ((static_cast<size_t>(R) * n * 4 + 1023) / 1024) * 1024;
    return 1024 + kStages * stage + 2 * kStages * sizeof(uint64_t) + kThrBytes + 2 * static_cast<size_t>(R) * ws;
}

}  // namespace

void summarise(const float* rows, uint64_t count, int n, int w, int bits, const double* d_thr,
               uint8_t* words, uint32_t* root_keys, uint64_t* sort_keys, cudaStream_t stream, uint8_t* fine,
               int key_bits, int record_stride) {
    if (count == 0) return;
    SumArgs a{};
    a.n = n;
    a.w = w;
    a.bits = bits;
    a.seg = n / w;
    a.ws = word_stride(w);
    a.words = words;
    a.root_keys = root_keys;
    a.sort_keys = sort_keys;
    a.fw = fine_width(n, w);
    a.fws = fine_stride(a.fw);
    a.fine = a.fw ? fine : nullptr;
    a.wst = record_stride > 0 ? record_stride : a.ws;
    a.fst = record_stride > 0 ? record_stride : a.fws;
    // 64-byte records of a 16-byte word + 32-byte fine row: 16 bytes of tail
    static const bool no_pad = std::getenv("TSG_NO_RECORD_PAD") != nullptr;  // A/B
    a.pad_after_fine = !no_pad && record_stride == 64 && a.ws == 16 && a.fws == 32 && a.fine ? 16 : 0;
    a.key_mask = key_bits >= 64 ? ~0ull : key_bits <= 0 ? 0ull : ~0ull << (64 - key_bits);

    int dev = 0, sms = 0;
    TSG_CUDA(cudaGetDevice(&dev));
    TSG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));

    const bool aligned = (reinterpret_cast<uintptr_t>(rows) % 16) == 0;
    if (n % 32 != 0 || !aligned) {
        a.count = count;
        a.out_base = 0;
        const int threads = 256;
        const uint64_t blocks = std::min<uint64_t>((count + threads - 1) / threads, sms * 16ull);
        k_summarise_generic<<<static_cast<unsigned>(blocks), threads, 0, stream>>>(rows, a, d_thr);
        TSG_LAUNCHED();
        return;
    }

    // R whole series per TMA box: box outer dim (R * n/32) <= 256, tile <= 32 KB.
    const int rows_per_series = n / 32;
    int R = std::min(256 / rows_per_series, 8192 / n);
    if (R < 1) R = 1;
    a.R = R;
    const size_t smem = tma_smem_bytes(R, n, a.ws);
    const bool with_fine = a.fine != nullptr;
    const bool vec = (a.seg % 4) == 0 && (!with_fine || a.seg % 8 == 0);
    // compile-time segment lengths of the BASELINE shapes (n = 256, 128, 96 at w = 16)
    using Kern = void (*)(const CUtensorMap, SumArgs, const double*);
    Kern kern;
    if (w == 16 && a.seg == 16) kern = with_fine ? k_summarise_tma<kStages, 16, true, true> : k_summarise_tma<kStages, 16, true, false>;
    else if (w == 16 && a.seg == 8) kern = with_fine ? k_summarise_tma<kStages, 8, true, true> : k_summarise_tma<kStages, 8, true, false>;
    else if (w == 16 && a.seg == 6) kern = with_fine ? k_summarise_tma<kStages, 6, false, true> : k_summarise_tma<kStages, 6, false, false>;
    else if (with_fine) kern = vec ? k_summarise_tma<kStages, 0, true, true> : k_summarise_tma<kStages, 0, false, true>;
    else kern = vec ? k_summarise_tma<kStages, 0, true, false> : k_summarise_tma<kStages, 0, false, false>;
    TSG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem)));
    int per_sm = 0;
    TSG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kSumThreads, smem));
    per_sm = std::max(per_sm, 1);

    auto encode = get_encoder();
    // TMA coordinates are int32: launch over slices of at most ~2^31 rows.
    const uint64_t max_series =
        ((static_cast<uint64_t>(1) << 31) - 4096) / rows_per_series / R * R;
    for (uint64_t off = 0; off < count; off += max_series) {
        const uint64_t cnt = std::min(max_series, count - off);
        CUtensorMap map;
        const float* base = rows + off * static_cast<uint64_t>(n);
        cuuint64_t gdim[2] = {32, cnt * rows_per_series};
        cuuint64_t gstride[1] = {128};
        cuuint32_t box[2] = {32, static_cast<cuuint32_t>(R * rows_per_series)};
        cuuint32_t estr[2] = {1, 1};
        CUresult r = encode(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), gdim,
                            gstride, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled failed: " + std::to_string(r));
        a.count = cnt;
        a.out_base = off;
        const uint64_t tiles = (cnt + R - 1) / R;
        const unsigned grid = static_cast<unsigned>(std::min<uint64_t>(tiles, static_cast<uint64_t>(sms) * per_sm));
        kern<<<grid, kSumThreads, smem, stream>>>(map, a, d_thr);
        TSG_LAUNCHED();
    }
}

}  // namespace tsg
