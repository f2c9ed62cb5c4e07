// K2 organise + K3 leaves: the flat SoA index.
//
// Replaces the reference's staging buffers and tree construction
// (SaxBuffers src/index.cpp:96-151, drain_in_position_order
// include/tsidx/index.hpp:204-231, insert_entry/split_leaf/choose_split_segment
// src/index.cpp:171-253) with:
//   K2  a stable radix sort of (32-bit plane-major key, position): entries of
//       one root key become contiguous and stay in position order inside
//       equal keys; then a gather of the 16-byte words into index order.
//   K3  leaf partition: a root bucket (run of equal root key) whose size
//       exceeds leaf_capacity is split at the first key bit on which its
//       first and last entries differ, recursively, until every range fits;
//       ranges whose 32 key bits are all equal become overflow leaves
//       (the reference's is_overflow, src/index.cpp:50-55). Then per-leaf
//       per-segment [min, max] symbol boxes for the leaf lower bound.
// The tree shape is not a parity target (north_star); the search is exact
// regardless of how entries are grouped into leaves.
#include <cub/cub.cuh>

#include <algorithm>
#include <vector>

#include "common.cuh"
#include "kernels.cuh"

namespace tsg {

namespace {

struct DevBuf {
    void* p = nullptr;
    explicit DevBuf(size_t bytes) { TSG_CUDA(cudaMalloc(&p, bytes ? bytes : 16)); }
    ~DevBuf() { cudaFree(p); }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    template <typename T>
    T* as() const { return static_cast<T*>(p); }
};

__global__ void k_iota(uint32_t* v, uint64_t n) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        v[i] = static_cast<uint32_t>(i);
}

// words[i] = words_orig[pos[i]] (16- or 32-byte rows).
__global__ void k_gather_words(const uint8_t* __restrict__ src, const uint32_t* __restrict__ pos,
                               uint8_t* __restrict__ dst, uint64_t n, int ws) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint4* s = reinterpret_cast<const uint4*>(src + static_cast<uint64_t>(pos[i]) * ws);
        uint4* d = reinterpret_cast<uint4*>(dst + i * ws);
        d[0] = s[0];
        if (ws == 32) d[1] = s[1];
    }
}

__device__ __forceinline__ uint32_t root_of(uint32_t key, int w) {
    return w >= 32 ? key : key >> (32 - w);
}

__global__ void k_bucket_flags(const uint32_t* __restrict__ keys, uint64_t n, int w,
                               uint8_t* __restrict__ flags) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        flags[i] = (i == 0 || root_of(keys[i], w) != root_of(keys[i - 1], w)) ? 1 : 0;
}

struct LeafEmit {
    uint32_t begin, end;
    int depth;
    bool overflow;
};

// Recursive split of one root bucket [a, b) (see file comment). Calls
// emit(leaf) in increasing begin order; returns the number of inner nodes.
template <typename F>
__device__ uint32_t split_bucket(const uint32_t* keys, uint32_t a, uint32_t b, uint32_t cap, F&& emit) {
    struct Item {
        uint32_t a, b;
        int d;
    } stack[40];
    int sp = 0;
    uint32_t inner = 0;
    stack[sp++] = {a, b, 1};
    while (sp > 0) {
        const Item it = stack[--sp];
        if (it.b - it.a <= cap) {
            emit(LeafEmit{it.a, it.b, it.d, false});
            continue;
        }
        const uint32_t ka = keys[it.a], kb = keys[it.b - 1];
        if (ka == kb) {
            emit(LeafEmit{it.a, it.b, it.d, true});
            continue;
        }
        const int p = __clz(ka ^ kb);  // first differing key bit (from the MSB)
        const uint32_t bit = 31 - p;
        uint32_t lo = it.a, hi = it.b - 1;  // keys[hi] has the bit set
        while (lo < hi) {
            const uint32_t mid = lo + (hi - lo) / 2;
            if ((keys[mid] >> bit) & 1u) hi = mid;
            else lo = mid + 1;
        }
        ++inner;
        stack[sp++] = {lo, it.b, it.d + 1};
        stack[sp++] = {it.a, lo, it.d + 1};
    }
    return inner;
}

struct LeafCounters {
    unsigned long long inner, overflow, max_depth;
};

__global__ void k_leaf_count(const uint32_t* __restrict__ keys, const uint32_t* __restrict__ bstart,
                             uint64_t nb, uint64_t n, uint32_t cap, uint32_t* __restrict__ count,
                             LeafCounters* ctr) {
    for (uint64_t b = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; b < nb;
         b += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint32_t lo = bstart[b];
        const uint32_t hi = b + 1 < nb ? bstart[b + 1] : static_cast<uint32_t>(n);
        uint32_t leaves = 0, over = 0;
        int depth = 0;
        const uint32_t inner = split_bucket(keys, lo, hi, cap, [&](const LeafEmit& e) {
            ++leaves;
            over += e.overflow ? 1u : 0u;
            depth = max(depth, e.depth);
        });
        count[b] = leaves;
        if (inner) atomicAdd(&ctr->inner, static_cast<unsigned long long>(inner));
        if (over) atomicAdd(&ctr->overflow, static_cast<unsigned long long>(over));
        atomicMax(&ctr->max_depth, static_cast<unsigned long long>(depth));
    }
}

__global__ void k_leaf_write(const uint32_t* __restrict__ keys, const uint32_t* __restrict__ bstart,
                             uint64_t nb, uint64_t n, uint32_t cap, const uint32_t* __restrict__ base,
                             uint32_t* __restrict__ leaf_off) {
    for (uint64_t b = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; b < nb;
         b += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint32_t lo = bstart[b];
        const uint32_t hi = b + 1 < nb ? bstart[b + 1] : static_cast<uint32_t>(n);
        uint32_t k = base[b];
        split_bucket(keys, lo, hi, cap, [&](const LeafEmit& e) { leaf_off[k++] = e.begin; });
    }
}

// One warp per leaf: bytewise min / max over the leaf's words.
__global__ void k_leaf_box(const uint8_t* __restrict__ words, const uint32_t* __restrict__ leaf_off,
                           uint64_t L, int ws, uint8_t* __restrict__ lo_out, uint8_t* __restrict__ hi_out) {
    const int lane = threadIdx.x & 31;
    const uint64_t warps = static_cast<uint64_t>(gridDim.x) * (blockDim.x >> 5);
    for (uint64_t l = (blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x) >> 5; l < L; l += warps) {
        const uint32_t a = leaf_off[l], b = leaf_off[l + 1];
        const int vecs = ws / 4;  // 32-bit lanes per word
        for (int v = 0; v < vecs; ++v) {
            uint32_t mn = 0xFFFFFFFFu, mx = 0u;
            for (uint32_t e = a + lane; e < b; e += 32) {
                const uint32_t x = reinterpret_cast<const uint32_t*>(words + static_cast<uint64_t>(e) * ws)[v];
                mn = __vminu4(mn, x);
                mx = __vmaxu4(mx, x);
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                mn = __vminu4(mn, __shfl_xor_sync(0xFFFFFFFFu, mn, o));
                mx = __vmaxu4(mx, __shfl_xor_sync(0xFFFFFFFFu, mx, o));
            }
            if (lane == 0) {
                reinterpret_cast<uint32_t*>(lo_out + l * ws)[v] = mn;
                reinterpret_cast<uint32_t*>(hi_out + l * ws)[v] = mx;
            }
        }
    }
}

unsigned grid_for(uint64_t n, int threads, int sms) {
    return static_cast<unsigned>(std::max<uint64_t>(1, std::min<uint64_t>((n + threads - 1) / threads,
                                                                          static_cast<uint64_t>(sms) * 32)));
}

}  // namespace

void build_layout(DevIndex& ix, double* ms_sum, double* ms_org, double* ms_leaf) {
    const uint64_t N = ix.N;
    cudaStream_t st = ix.stream;
    const int sms = ix.sms;
    cudaEvent_t ev[4];
    for (auto& e : ev) TSG_CUDA(cudaEventCreate(&e));

    TSG_CUDA(cudaMalloc(&ix.words, N * ix.ws));
    TSG_CUDA(cudaMalloc(&ix.pos, N * sizeof(uint32_t)));

    DevBuf words_orig(N * ix.ws), keys_in(N * 4), keys_out(N * 4), pos_in(N * 4);

    // K1 summarise
    TSG_CUDA(cudaEventRecord(ev[0], st));
    summarise(ix.rows, N, ix.n, ix.w, ix.bits, ix.thr, words_orig.as<uint8_t>(), nullptr,
              keys_in.as<uint32_t>(), st);
    TSG_CUDA(cudaEventRecord(ev[1], st));

    // K2 organise: stable sort by key, carrying positions; gather words.
    k_iota<<<grid_for(N, 256, sms), 256, 0, st>>>(pos_in.as<uint32_t>(), N);
    TSG_LAUNCHED();
    size_t temp_bytes = 0;
    TSG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, temp_bytes, keys_in.as<uint32_t>(),
                                             keys_out.as<uint32_t>(), pos_in.as<uint32_t>(), ix.pos,
                                             static_cast<int64_t>(N), 0, 32, st));
    {
        DevBuf temp(temp_bytes);
        TSG_CUDA(cub::DeviceRadixSort::SortPairs(temp.p, temp_bytes, keys_in.as<uint32_t>(),
                                                 keys_out.as<uint32_t>(), pos_in.as<uint32_t>(), ix.pos,
                                                 static_cast<int64_t>(N), 0, 32, st));
        k_gather_words<<<grid_for(N, 256, sms), 256, 0, st>>>(words_orig.as<uint8_t>(), ix.pos, ix.words, N,
                                                               ix.ws);
        TSG_LAUNCHED();
        TSG_CUDA(cudaEventRecord(ev[2], st));
    }

    // K3 leaves. Bucket starts = positions where the root key changes.
    const uint32_t* keys = keys_out.as<uint32_t>();
    DevBuf flags(N), bstart(N * 4), nsel(8);
    k_bucket_flags<<<grid_for(N, 256, sms), 256, 0, st>>>(keys, N, ix.w, flags.as<uint8_t>());
    TSG_LAUNCHED();
    {
        size_t tb = 0;
        TSG_CUDA(cub::DeviceSelect::Flagged(nullptr, tb, pos_in.as<uint32_t>(), flags.as<uint8_t>(), bstart.as<uint32_t>(),
                                            nsel.as<uint64_t>(), static_cast<int64_t>(N), st));
        DevBuf temp(tb);
        TSG_CUDA(cub::DeviceSelect::Flagged(temp.p, tb, pos_in.as<uint32_t>(), flags.as<uint8_t>(), bstart.as<uint32_t>(),
                                            nsel.as<uint64_t>(), static_cast<int64_t>(N), st));
    }
    uint64_t nb = 0;
    TSG_CUDA(cudaMemcpyAsync(&nb, nsel.p, 8, cudaMemcpyDeviceToHost, st));
    TSG_CUDA(cudaStreamSynchronize(st));
    ix.root_children = nb;

    DevBuf lcount((nb + 1) * 4), lbase((nb + 1) * 4), ctr(sizeof(LeafCounters));
    TSG_CUDA(cudaMemsetAsync(ctr.p, 0, sizeof(LeafCounters), st));
    TSG_CUDA(cudaMemsetAsync(lcount.p, 0, (nb + 1) * 4, st));
    const uint32_t cap = static_cast<uint32_t>(std::min<uint64_t>(ix.leaf_cap, 0xFFFFFFFFull));
    k_leaf_count<<<grid_for(nb, 128, sms), 128, 0, st>>>(keys, bstart.as<uint32_t>(), nb, N, cap,
                                                           lcount.as<uint32_t>(), ctr.as<LeafCounters>());
    TSG_LAUNCHED();
    {
        size_t tb = 0;
        TSG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, lcount.as<uint32_t>(), lbase.as<uint32_t>(),
                                               static_cast<int64_t>(nb + 1), st));
        DevBuf temp(tb);
        TSG_CUDA(cub::DeviceScan::ExclusiveSum(temp.p, tb, lcount.as<uint32_t>(), lbase.as<uint32_t>(),
                                               static_cast<int64_t>(nb + 1), st));
    }
    uint32_t L32 = 0;
    LeafCounters hc{};
    TSG_CUDA(cudaMemcpyAsync(&L32, lbase.as<uint32_t>() + nb, 4, cudaMemcpyDeviceToHost, st));
    TSG_CUDA(cudaMemcpyAsync(&hc, ctr.p, sizeof(hc), cudaMemcpyDeviceToHost, st));
    TSG_CUDA(cudaStreamSynchronize(st));
    ix.L = L32;
    ix.inner = hc.inner;
    ix.overflow = hc.overflow;
    ix.max_depth = hc.max_depth;

    TSG_CUDA(cudaMalloc(&ix.leaf_off, (ix.L + 1) * 4));
    TSG_CUDA(cudaMalloc(&ix.leaf_lo, ix.L * ix.ws));
    TSG_CUDA(cudaMalloc(&ix.leaf_hi, ix.L * ix.ws));
    k_leaf_write<<<grid_for(nb, 128, sms), 128, 0, st>>>(keys, bstart.as<uint32_t>(), nb, N, cap,
                                                           lbase.as<uint32_t>(), ix.leaf_off);
    TSG_LAUNCHED();
    const uint32_t n32 = static_cast<uint32_t>(N);
    TSG_CUDA(cudaMemcpyAsync(ix.leaf_off + ix.L, &n32, 4, cudaMemcpyHostToDevice, st));
    k_leaf_box<<<grid_for(ix.L * 32, 256, sms), 256, 0, st>>>(ix.words, ix.leaf_off, ix.L, ix.ws, ix.leaf_lo,
                                                               ix.leaf_hi);
    TSG_LAUNCHED();
    TSG_CUDA(cudaEventRecord(ev[3], st));
    TSG_CUDA(cudaStreamSynchronize(st));

    float t01 = 0, t12 = 0, t23 = 0;
    TSG_CUDA(cudaEventElapsedTime(&t01, ev[0], ev[1]));
    TSG_CUDA(cudaEventElapsedTime(&t12, ev[1], ev[2]));
    TSG_CUDA(cudaEventElapsedTime(&t23, ev[2], ev[3]));
    if (ms_sum) *ms_sum = t01;
    if (ms_org) *ms_org = t12;
    if (ms_leaf) *ms_leaf = t23;
    for (auto& e : ev) cudaEventDestroy(e);
}

}  // namespace tsg
