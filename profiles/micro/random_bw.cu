// Microbenchmark (round 2d): achievable HBM bandwidth of RANDOM aligned reads on B200, by read
// size (64 / 128 / 256 / 512 bytes per random location) with many independent loads in flight —
// the practical roofline of the query kernels, whose reads are random lines (quad-box lines,
// quads' words, fine rows), against the sequential-copy peak in MEASURED_PEAKS.json.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o random_bw random_bw.cu && ./random_bw
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix(uint64_t x) {
    x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull; x ^= x >> 33;
    return x;
}

// BYTES per random location; a group of BYTES / 16 lanes reads one location (16 bytes per lane);
// U independent locations per lane group in flight.
template <int BYTES, int U>
__global__ void k_rand(const uint4* __restrict__ buf, uint64_t nloc, uint64_t groups_total, unsigned* out) {
    constexpr int G = BYTES / 16;  // lanes per location
    const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint64_t nthreads = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t grp = tid / G, ngrp = nthreads / G;
    const int l = tid % G;
    unsigned acc = 0;
    for (uint64_t i = grp * U; i < groups_total; i += ngrp * U) {
        uint4 x[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            // cheap 32-bit hash -> [0, nloc) with a multiply-high (the index math must not bind)
            uint32_t h = (uint32_t)(i + u) * 2654435761u + BYTES;
            h ^= h >> 15; h *= 0x2C1B3C6Du; h ^= h >> 12; h *= 0x297A2D39u; h ^= h >> 15;
            const uint64_t loc = __umulhi(h, (uint32_t)nloc);
            const uint4* p = buf + loc * G + l;
            asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                         : "=r"(x[u].x), "=r"(x[u].y), "=r"(x[u].z), "=r"(x[u].w) : "l"(p));
        }
#pragma unroll
        for (int u = 0; u < U; ++u) acc ^= x[u].x ^ x[u].w;
    }
    if (acc == 0x12345678u) out[0] = acc;
}

__global__ void k_seq(const uint4* __restrict__ buf, uint64_t n16, unsigned* out) {
    unsigned acc = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n16; i += (uint64_t)gridDim.x * blockDim.x) {
        uint4 x;
        asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(x.x), "=r"(x.y), "=r"(x.z), "=r"(x.w) : "l"(buf + i));
        acc ^= x.x ^ x.w;
    }
    if (acc == 0x12345678u) out[0] = acc;
}

template <int BYTES, int U>
void run(const uint4* buf, uint64_t bytes, unsigned* out, int blocks) {
    const uint64_t nloc = bytes / BYTES;
    const uint64_t groups = (8ull << 30) / BYTES;  // 8 GB of useful bytes per launch
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    k_rand<BYTES, U><<<blocks, 256>>>(buf, nloc, groups, out);  // warm-up
    cudaEventRecord(a);
    k_rand<BYTES, U><<<blocks, 256>>>(buf, nloc, groups, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    std::printf("random %4d B x %d in flight, %5d blocks: %7.1f GB/s useful (%.3f ms)\n", BYTES, U, blocks,
                groups * (double)BYTES / ms / 1e6, ms);
}

int main() {
    const uint64_t bytes = 32ull << 30;  // far larger than L2
    uint4* buf;
    unsigned* out;
    if (cudaMalloc(&buf, bytes) != cudaSuccess) { std::printf("alloc failed\n"); return 1; }
    cudaMalloc(&out, 4);
    cudaMemset(buf, 1, bytes);
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    k_seq<<<148 * 8, 256>>>(buf, bytes / 16, out);
    cudaEventRecord(a);
    k_seq<<<148 * 8, 256>>>(buf, bytes / 16, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    std::printf("sequential read: %7.1f GB/s (%.3f ms)\n", bytes / ms / 1e6, ms);
    // the span of the random locations: the index arrays are 0.8 - 3.2 GB (TLB reach matters)
    for (uint64_t span : {1ull << 30, 2ull << 30, 4ull << 30, 32ull << 30}) {
        std::printf("span %llu GB\n", (unsigned long long)(span >> 30));
        for (int blocks : {148 * 4, 148 * 6}) {
            run<64, 2>(buf, span, out, blocks);
            run<64, 8>(buf, span, out, blocks);
            run<128, 2>(buf, span, out, blocks);
            run<128, 8>(buf, span, out, blocks);
            run<512, 4>(buf, span, out, blocks);
        }
    }
    std::printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
