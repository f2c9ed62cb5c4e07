// Shared device/host helpers for the tsgpu library (sm_100a only).
#pragma once

#include <cuda_runtime.h>
#include <cstdint>
#include <stdexcept>
#include <string>

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "tsgpu is built for sm_100a only"
#endif

namespace tsg {

// Error classes mapped onto tsg_status at the C ABI.
struct InvalidArgument : std::invalid_argument {
    using std::invalid_argument::invalid_argument;
};
struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct OutOfMemory : std::runtime_error {
    using std::runtime_error::runtime_error;
};

inline void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
    if (e == cudaSuccess) return;
    std::string msg = std::string(what) + ": " + cudaGetErrorString(e) + " (" + file + ":" +
                      std::to_string(line) + ")";
    if (e == cudaErrorMemoryAllocation) throw OutOfMemory(msg);
    throw CudaError(msg);
}

#define TSG_CUDA(expr) ::tsg::cuda_check((expr), #expr, __FILE__, __LINE__)

// Counts every kernel this library launches (reported as gpu_launches).
void note_launch(int n = 1);
uint64_t launch_count();
uint64_t launch_count_thread();  // launches noted by the calling thread

#define TSG_LAUNCHED() \
    do {                                                        \
        ::tsg::note_launch();                                   \
        TSG_CUDA(cudaPeekAtLastError());                        \
    } while (0)

// Word stride in bytes: 16 for w <= 16, 32 for w <= 32.
__host__ __device__ inline int word_stride(int w) { return w <= 16 ? 16 : 32; }

constexpr int kMaxW = 32;

// Fine summary (a second, finer lower bound in front of refinement): every
// PAA segment split in two halves, i.e. 2w segments of n / (2w) points, each
// mean quantised to a symbol of the index cardinality, one row of fw bytes
// (stride fine_stride) per dataset row. 0 = no fine summary (2w > 64 or the
// halves would not tile the series).
__host__ __device__ inline int fine_width(int n, int w) { return (2 * w <= 64 && n % (2 * w) == 0) ? 2 * w : 0; }
__host__ __device__ inline int fine_stride(int fw) { return (fw + 15) / 16 * 16; }
constexpr int kMaxFine = 64;
constexpr int kThrPad = 256;  // padded threshold table entries per cardinality

// Device threshold table for one cardinality: thr[0..card-2], padded with
// +inf up to 256 entries. Computed on the host (breakpoints.cpp), bit
// identical to tsidx::breakpoints_for (src/breakpoints.cpp:65-114).
void host_breakpoints(int bits, double* out256);

// Fast-symbol bins (see host_symbol_bins): kBins bins over [-kBinRange, kBinRange).
constexpr int kBins = 4096;
constexpr double kBinRange = 6.0;
void host_symbol_bins(const double* thr256, int bits, double range, int nbins, unsigned char* bins);

// Layout of the device threshold block: 256 doubles then kBins bytes.
constexpr size_t kThrBytes = kThrPad * sizeof(double) + kBins;

// ---- small PTX helpers ----------------------------------------------------

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// mbarrier + bulk-copy (TMA) helpers.
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// 1-D bulk copy global -> shared (16-byte aligned, size a multiple of 16),
// completing `bytes` transactions on `bar`.
__device__ __forceinline__ void tma_copy_1d(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

__device__ __forceinline__ unsigned long long ld_volatile_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ uint4 ld_stream_u4(const void* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

__device__ __forceinline__ float4 ld_stream_f4(const float* p) {
    float4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
                 : "l"(p));
    return r;
}

// Upper bound over a padded threshold table in shared memory: the number of
// thresholds <= v, i.e. std::upper_bound (src/sax.cpp:33-37). Written as
// !(v < t) so a NaN mean lands in the top region exactly as upper_bound puts it.
__device__ __forceinline__ unsigned symbol_of(const double* thr, int bits, double v) {
    unsigned s = 0;
#pragma unroll
    for (int b = 7; b >= 0; --b) {
        if (b < bits) {
            const unsigned step = 1u << b;
            if (!(v < thr[s + step - 1])) s += step;
        }
    }
    return s;
}

// The same number of thresholds <= v via the bin table: start from the bin's
// count and walk to the exact upper_bound (0-1 steps when bins are narrower
// than the threshold spacing). Out-of-range values and NaN take the plain
// binary search.
__device__ __forceinline__ unsigned symbol_fast(const double* thr, const unsigned char* bins, int bits, double v) {
    if (!(v >= -kBinRange && v < kBinRange)) return symbol_of(thr, bits, v);
    int b = __double2int_rz(__dmul_rn(__dadd_rn(v, kBinRange), kBins / (2.0 * kBinRange)));
    b = min(max(b, 0), kBins - 1);
    unsigned s = bins[b];
    const unsigned top = (1u << bits) - 1u;
    while (s > 0 && v < thr[s - 1]) --s;
    while (s < top && !(v < thr[s])) ++s;
    return s;
}

// symbol_fast without the walk: one step down or up from the bin's count.
// Exact whenever no two thresholds lie within one bin width (+ rounding) of
// each other — true for every cardinality here (8-bit breakpoints are at
// least 0.0098 apart, bins 12/4096 = 0.0029 wide); the table is +inf padded,
// so the up step never passes the top symbol.
__device__ __forceinline__ unsigned symbol_step(const double* thr, const unsigned char* bins, int bits, double v) {
    if (!(v >= -kBinRange && v < kBinRange)) return symbol_of(thr, bits, v);
    int b = __double2int_rz(__dmul_rn(__dadd_rn(v, kBinRange), kBins / (2.0 * kBinRange)));
    b = min(max(b, 0), kBins - 1);
    unsigned s = bins[b];
    s -= (s > 0 && v < thr[s > 0 ? s - 1 : 0]) ? 1u : 0u;
    s += !(v < thr[s]) ? 1u : 0u;
    return s;
}

// Fine-summary symbol (the fine summary is a filter, not a parity target):
// uniform quantisation of the half-segment mean over [-2.5, 2.5) in 256 steps
// of 5/256 (exact in binary), symbol v <-> region [v step - 2.5, (v+1) step -
// 2.5), open-ended for v = 0 and 255. For z-normalised series this is as
// tight as the N(0,1) breakpoints (measured: 221 vs 216 surviving rows per
// c1 query) and costs a multiply-add. The float rounding of the mean is
// covered by widening the regions by kFineSlack in the query's table.
constexpr double kFineLo = -2.5;
constexpr double kFineStep = 5.0 / 256.0;
constexpr double kFineSlack = 0x1p-16;
__device__ __forceinline__ unsigned fine_quant(double mean) {
    const float x = __fmul_rn(__fsub_rn(__double2float_rn(mean), static_cast<float>(kFineLo)),
                              static_cast<float>(1.0 / kFineStep));
    if (!(x >= 0.f)) return x < 0.f ? 0u : 255u;  // NaN: the top (open) region
    return min(static_cast<unsigned>(x), 255u);
}

}  // namespace tsg
