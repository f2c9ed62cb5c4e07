// Microbenchmark (round 2): DRAM bytes moved per random read of 16 / 32 / 64 / 128 aligned bytes,
// to decide whether a 32-byte sector read costs 64 bytes of HBM traffic on B200.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dram_granularity dram_granularity.cu
//   ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum ./dram_granularity
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix(uint64_t x) {
    x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull; x ^= x >> 33;
    return x;
}

// control: each thread streams 16 bytes, coalesced
__global__ void k_seq(const uint4* __restrict__ buf, uint64_t n16, uint64_t accesses, unsigned* out) {
    unsigned acc = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < accesses; i += (uint64_t)gridDim.x * blockDim.x) {
        uint4 x;
        asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(x.x), "=r"(x.y), "=r"(x.z), "=r"(x.w) : "l"(buf + i));
        acc ^= x.x ^ x.w;
    }
    if (acc == 0x12345678u) out[0] = acc;
}

template <int BYTES>
__global__ void k_rand(const uint4* __restrict__ buf, uint64_t n16, uint64_t accesses, unsigned* out) {
    constexpr int V = BYTES / 16;
    unsigned acc = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < accesses; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t blk = mix(i * 0x9E3779B97F4A7C15ull + BYTES) % (n16 / V);
        const uint4* p = buf + blk * V;
#pragma unroll
        for (int v = 0; v < V; ++v) {
            uint4 x;
            asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(x.x), "=r"(x.y), "=r"(x.z), "=r"(x.w) : "l"(p + v));
            acc ^= x.x ^ x.w;
        }
    }
    if (acc == 0x12345678u) out[0] = acc;
}

template <int BYTES>
__global__ void k_rand_write(uint4* __restrict__ buf, uint64_t n16, uint64_t accesses, unsigned* out) {
    constexpr int V = BYTES >= 16 ? BYTES / 16 : 1;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < accesses; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t blk = mix(i * 0x9E3779B97F4A7C15ull + 7 * BYTES) % (n16 / V);
        if (BYTES < 16) {
            reinterpret_cast<unsigned*>(buf + blk)[0] = (unsigned)i;
        } else {
#pragma unroll
            for (int v = 0; v < V; ++v) buf[blk * V + v] = make_uint4((unsigned)i, v, 0, 0);
        }
    }
}

int main() {
    const uint64_t bytes = 16ull << 30;  // 16 GB: far larger than L2
    uint4* buf;
    unsigned* out;
    if (cudaMalloc(&buf, bytes) != cudaSuccess) { std::printf("alloc failed\n"); return 1; }
    cudaMalloc(&out, 4);
    cudaMemset(buf, 1, bytes);
    const uint64_t n16 = bytes / 16, acc = 1ull << 23;  // 8M random accesses per kernel
    const int grid = 148 * 8;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto run = [&](auto kernel, int size) {  // (reads and writes alike)
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(a);
            kernel<<<grid, 256>>>(buf, n16, acc, out);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms = 0;
            cudaEventElapsedTime(&ms, a, b);
            std::printf("random %3d-byte reads: %.3f ms, %.1f GB/s useful, %.1f Maccess/s\n", size, ms,
                        acc * size / (ms * 1e-3) / 1e9, acc / (ms * 1e-3) / 1e6);
        }
    };
    run(k_seq, 16);
    run(k_rand<16>, 16);
    run(k_rand<32>, 32);
    run(k_rand<64>, 64);
    run(k_rand<128>, 128);
    run(k_rand_write<4>, 4);
    run(k_rand_write<16>, 16);
    run(k_rand_write<32>, 32);
    run(k_rand_write<64>, 64);
    run(k_rand_write<128>, 128);
    cudaFree(buf);
    return 0;
}
