// Device input generator: the reference's seeded random walks on the GPU.
//
// Restates generate_random_walk / fill_walk / mix_seed (src/dataset.cpp:22-68)
// and the CLI's z-normalisation (src/dataset.cpp:70-85, tools/main.cpp:128-139)
// so 100M-series workloads can be created in HBM in seconds instead of
// minutes on the host. Per series: splitmix64(seed, i) seeds an MT19937-64
// (the std::mt19937_64 parameter set); uniforms are libstdc++'s
// generate_canonical<double, 53> (one draw / 2^64); normals come from the
// Marsaglia polar method with one cached deviate, in libstdc++'s order;
// the walk accumulates in FP64 and stores floats. All arithmetic is IEEE
// round-to-nearest without FMA, so the only possible difference from the
// host generator is the last bit of log() (glibc vs CUDA libdevice); the
// test suite counts mismatching series against the reference.
//
// One warp per series: the twist and the polar accept/reject run across
// lanes; the inherently serial steps (seeding recurrence, the walk, the
// z-normalisation sums) run on lane 0 in the reference order.
#include "common.cuh"
#include "kernels.cuh"

namespace tsg {

namespace {

constexpr int kMtN = 312, kMtM = 156;
constexpr int kGenWarps = 4;
constexpr int kMaxLen = 512;

__device__ __forceinline__ uint64_t mix_seed(uint64_t seed, uint64_t i) {
    uint64_t z = seed + (i + 1) * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__device__ __forceinline__ uint64_t twist_one(uint64_t xi, uint64_t xi1, uint64_t xim) {
    const uint64_t y = (xi & (~0ull << 31)) | (xi1 & ((1ull << 31) - 1));
    return xim ^ (y >> 1) ^ ((y & 1ull) ? 0xB5026F5AA96619E9ull : 0ull);
}

__device__ __forceinline__ uint64_t temper(uint64_t z) {
    z ^= (z >> 29) & 0x5555555555555555ull;
    z ^= (z << 17) & 0x71D67FFFEDA60000ull;
    z ^= (z << 37) & 0xFFF7EEE000000000ull;
    z ^= z >> 43;
    return z;
}

__device__ __forceinline__ double canonical(uint64_t x) {
    double r = __dmul_rn(__ull2double_rn(x), 5.421010862427522170037e-20);  // 2^-64, exact scaling
    if (r >= 1.0) r = 0.99999999999999988898;  // nextafter(1, 0)
    return r;
}

// In-place MT twist over the 312-word state, in the sequential order's
// dependency structure: [0,156) reads old words, [156,311) reads the new
// [0,155), and 311 reads the new word 0.
__device__ void mt_twist(uint64_t* x, int lane) {
    uint64_t v[5];
#pragma unroll
    for (int r = 0; r < 5; ++r) {
        const int i = lane + 32 * r;
        if (i < kMtM) v[r] = twist_one(x[i], x[i + 1], x[i + kMtM]);
    }
    __syncwarp();
#pragma unroll
    for (int r = 0; r < 5; ++r) {
        const int i = lane + 32 * r;
        if (i < kMtM) x[i] = v[r];
    }
    __syncwarp();
#pragma unroll
    for (int r = 0; r < 5; ++r) {
        const int i = kMtM + lane + 32 * r;
        if (i < kMtN - 1) v[r] = twist_one(x[i], x[i + 1], x[i - kMtM]);
    }
    __syncwarp();
#pragma unroll
    for (int r = 0; r < 5; ++r) {
        const int i = kMtM + lane + 32 * r;
        if (i < kMtN - 1) x[i] = v[r];
    }
    __syncwarp();
    if (lane == 0) x[kMtN - 1] = twist_one(x[kMtN - 1], x[0], x[kMtM - 1]);
    __syncwarp();
}

__global__ void __launch_bounds__(kGenWarps * 32)
    k_generate(float* __restrict__ rows, uint64_t begin, uint64_t count, int n, uint64_t seed, int znorm) {
    __shared__ uint64_t s_mt[kGenWarps][kMtN];
    __shared__ double s_norm[kGenWarps][kMaxLen + 2];
    __shared__ float s_out[kGenWarps][kMaxLen];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint64_t* mt = s_mt[warp];
    double* nrm = s_norm[warp];
    float* out = s_out[warp];
    const uint64_t gw = blockIdx.x * static_cast<uint64_t>(kGenWarps) + warp;
    const uint64_t nw = static_cast<uint64_t>(gridDim.x) * kGenWarps;
    for (uint64_t s = gw; s < count; s += nw) {
        const uint64_t idx = begin + s;
        if (lane == 0) {
            uint64_t x = mix_seed(seed, idx);
            mt[0] = x;
            for (int k = 1; k < kMtN; ++k) {
                x = 6364136223846793005ull * (x ^ (x >> 62)) + static_cast<uint64_t>(k);
                mt[k] = x;
            }
        }
        __syncwarp();
        int have = 0;  // normals produced
        while (have < n) {
            mt_twist(mt, lane);
            // 156 pairs per twist, 32 at a time, in order.
            for (int p0 = 0; p0 < kMtN / 2 && have < n; p0 += 32) {
                const int p = p0 + lane;
                bool acc = false;
                double gx = 0.0, gy = 0.0;
                if (p < kMtN / 2) {
                    const double u1 = canonical(temper(mt[2 * p]));
                    const double u2 = canonical(temper(mt[2 * p + 1]));
                    const double x = __dsub_rn(__dmul_rn(2.0, u1), 1.0);
                    const double y = __dsub_rn(__dmul_rn(2.0, u2), 1.0);
                    const double r2 = __dadd_rn(__dmul_rn(x, x), __dmul_rn(y, y));
                    acc = !(r2 > 1.0 || r2 == 0.0);
                    if (acc) {
                        const double mult = __dsqrt_rn(__ddiv_rn(__dmul_rn(-2.0, log(r2)), r2));
                        gy = __dmul_rn(y, mult);  // returned first
                        gx = __dmul_rn(x, mult);  // cached, returned second
                    }
                }
                const unsigned m = __ballot_sync(0xFFFFFFFFu, acc);
                if (acc) {
                    const int slot = have + 2 * __popc(m & ((1u << lane) - 1u));
                    if (slot < kMaxLen + 2) {
                        nrm[slot] = gy;
                        nrm[slot + 1] = gx;
                    }
                }
                have += 2 * __popc(m);
            }
            __syncwarp();
        }
        __syncwarp();
        if (lane == 0) {
            double v = 0.0;
            for (int j = 0; j < n; ++j) {
                v = __dadd_rn(v, nrm[j]);
                out[j] = __double2float_rn(v);
            }
        }
        __syncwarp();
        if (znorm) {
            __shared__ double s_ms[kGenWarps][2];
            if (lane == 0) {
                double sum = 0.0;
                for (int j = 0; j < n; ++j) sum = __dadd_rn(sum, static_cast<double>(out[j]));
                const double mean = __ddiv_rn(sum, static_cast<double>(n));
                double sq = 0.0;
                for (int j = 0; j < n; ++j) {
                    const double d = __dsub_rn(static_cast<double>(out[j]), mean);
                    sq = __dadd_rn(sq, __dmul_rn(d, d));
                }
                s_ms[warp][0] = mean;
                s_ms[warp][1] = __dsqrt_rn(__ddiv_rn(sq, static_cast<double>(n)));
            }
            __syncwarp();
            const double mean = s_ms[warp][0], sd = s_ms[warp][1];
            for (int j = lane; j < n; j += 32)
                out[j] = sd <= 1e-12 ? 0.f
                                     : __double2float_rn(__ddiv_rn(__dsub_rn(static_cast<double>(out[j]), mean), sd));
            __syncwarp();
        }
        float* dst = rows + s * static_cast<uint64_t>(n);
        for (int j = lane; j < n; j += 32) dst[j] = out[j];
        __syncwarp();
    }
}

}  // namespace

void generate_random_walk(float* rows, uint64_t begin, uint64_t count, uint64_t length, uint64_t seed, int znorm,
                          cudaStream_t stream) {
    if (length == 0 || length > static_cast<uint64_t>(kMaxLen))
        throw InvalidArgument("generate_random_walk: device generator supports 1 <= length <= 512");
    if (count == 0) return;
    int dev = 0, sms = 0;
    TSG_CUDA(cudaGetDevice(&dev));
    TSG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const uint64_t blocks = std::min<uint64_t>((count + kGenWarps - 1) / kGenWarps, static_cast<uint64_t>(sms) * 16);
    k_generate<<<static_cast<unsigned>(blocks), kGenWarps * 32, 0, stream>>>(rows, begin, count,
                                                                            static_cast<int>(length), seed, znorm);
    TSG_LAUNCHED();
}

}  // namespace tsg
