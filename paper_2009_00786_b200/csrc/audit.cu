// validate_index for the flat index: a full structural audit on the device.
//
// Replaces tsidx::validate_index / Auditor (src/index.cpp:332-484,
// include/tsidx/index.hpp:180-202). The reference walks its pointer tree
// (word/prefix consistency, leaf occupancy, subtree counts) and re-derives
// every series' word to confirm it is stored in exactly the leaf its word
// descends to. The flat layout's equivalents, one kernel per level:
//   entries  every position in range and stored exactly once; the stored word
//            equals the word recomputed from the series (K1 over the rows in
//            dataset order, the reference's paa_into + symbols_from_paa);
//            symbols carry no bits below the cardinality prefix; entries in
//            non-decreasing sort-key order with equal keys in position order
//            (the reference's position-order drain); the fine summary row of
//            every entry equals the recomputed one;
//   leaves   offsets strictly increasing and tiling [0, N); one root key per
//            leaf (a leaf never spans two root subtrees); a leaf above the
//            capacity only when it cannot be split (all sorted key bits equal:
//            the reference's is_overflow); the fill histogram;
//   pages    tile their leaves in <= kPage pieces; every page / run / quad box
//            is the exact bytewise min / max of its entries' words; group and
//            top boxes contain their children's boxes.
// Counts per violation kind plus the first offending index go back to the
// host, which words the first 20 messages like the reference's.
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/tsgpu.h"
#include "common.cuh"
#include "kernels.cuh"

namespace tsg {

namespace {

enum Violation {
    kPosRange = 0, kPosDup, kPosMissing, kWordMismatch, kSymbolBits, kOrder, kLeafShape, kLeafRoot, kLeafCap,
    kPageTile, kPageBox, kGroupBox, kRunBox, kQuadBox, kFineMismatch, kViolationKinds
};

struct AuditCounters {
    unsigned long long count[kViolationKinds];
    unsigned long long first[kViolationKinds];  // smallest offending index (entry / position / leaf / page / box)
    unsigned long long hist[11];
    unsigned long long empty_leaves, overflow_leaves, boxes;
};

__device__ __forceinline__ void report(AuditCounters* c, int kind, uint64_t where) {
    atomicAdd(&c->count[kind], 1ull);
    atomicMin(&c->first[kind], static_cast<unsigned long long>(where));
}

#define AUDIT_STRIDE(i, n)                                                                  \
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < (n); \
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x)

// Plane-major key of a stored word (the build's sort key), first key_bits bits.
__device__ __forceinline__ uint64_t sort_key(const uint8_t* word, int w, int key_bits) {
    uint64_t k = 0;
    int left = 64;
    for (int p = 0; p < 8 && left > 0; ++p)
        for (int g = 0; g < w && left > 0; ++g, --left) k = (k << 1) | ((word[g] >> (7 - p)) & 1u);
    k = left >= 64 ? 0 : k << left;
    return key_bits >= 64 ? k : k & (~0ull << (64 - key_bits));
}

__device__ __forceinline__ uint32_t root_key(const uint8_t* word, int w) {
    uint32_t r = 0;
    for (int g = 0; g < w; ++g) r = (r << 1) | (word[g] >> 7);
    return r;
}

// Structure of the entries (positions in range and counted, symbol bits, order).
__global__ void k_audit_entries(const uint8_t* __restrict__ words, const uint32_t* __restrict__ pos, uint64_t N,
                                int w, int ws, int bits, int key_bits, unsigned* __restrict__ seen, AuditCounters* c) {
    const unsigned low_mask = bits >= 8 ? 0u : (1u << (8 - bits)) - 1u;
    AUDIT_STRIDE(i, N) {
        const uint32_t p = pos[i];
        const uint8_t* wi = words + i * ws;
        if (p >= N) report(c, kPosRange, i);
        else atomicAdd(&seen[p], 1u);
        bool clean = true;
        for (int g = 0; g < w; ++g) clean = clean && (wi[g] & low_mask) == 0;
        if (!clean) report(c, kSymbolBits, i);
        if (i + 1 < N) {
            const uint64_t ka = sort_key(wi, w, key_bits), kb = sort_key(wi + ws, w, key_bits);
            if (ka > kb || (ka == kb && pos[i + 1] <= p)) report(c, kOrder, i);
        }
    }
}

// Stored words / fine rows of the entries whose series lies in [p0, p1) against
// the re-derivation of those series (one chunk of positions at a time, so the
// audit's scratch stays bounded on a 100M-series index).
__global__ void k_audit_words(const uint8_t* __restrict__ words, const uint32_t* __restrict__ pos, uint64_t N, int w,
                              int ws, uint64_t p0, uint64_t p1, const uint8_t* __restrict__ rederived,
                              const uint8_t* __restrict__ fine, const uint8_t* __restrict__ fine_rederived, int fw,
                              int fws, AuditCounters* c) {
    AUDIT_STRIDE(i, N) {
        const uint64_t p = pos[i];
        if (p < p0 || p >= p1) continue;
        const uint8_t* wi = words + i * ws;
        const uint8_t* wr = rederived + (p - p0) * ws;
        bool same = true;
        for (int g = 0; g < w; ++g) same = same && wi[g] == wr[g];
        if (!same) report(c, kWordMismatch, p);
        if (fine) {
            bool fsame = true;
            const uint8_t* fi = fine + i * fws;
            const uint8_t* fr = fine_rederived + (p - p0) * fws;
            for (int g = 0; g < fw; ++g) fsame = fsame && fi[g] == fr[g];
            if (!fsame) report(c, kFineMismatch, p);
        }
    }
}

__global__ void k_audit_seen(const unsigned* __restrict__ seen, uint64_t N, AuditCounters* c) {
    AUDIT_STRIDE(p, N) {
        if (seen[p] == 0) report(c, kPosMissing, p);
        else if (seen[p] > 1) report(c, kPosDup, p);
    }
}

__global__ void k_audit_leaves(const uint8_t* __restrict__ words, const uint32_t* __restrict__ leaf_off, uint64_t L,
                               uint64_t N, int w, int ws, int key_bits, uint64_t cap, AuditCounters* c) {
    AUDIT_STRIDE(l, L) {
        const uint32_t a = leaf_off[l], b = leaf_off[l + 1];
        if ((l == 0 && a != 0) || (l + 1 == L && b != N) || b <= a) {
            report(c, kLeafShape, l);
            if (b <= a) {
                atomicAdd(&c->empty_leaves, 1ull);
                continue;
            }
        }
        if (b > N) {
            report(c, kLeafShape, l);
            continue;
        }
        const uint8_t* wa = words + static_cast<uint64_t>(a) * ws;
        const uint8_t* wb = words + static_cast<uint64_t>(b - 1) * ws;
        if (root_key(wa, w) != root_key(wb, w)) report(c, kLeafRoot, l);
        const uint64_t fill = b - a;
        if (fill > cap) {
            if (sort_key(wa, w, key_bits) == sort_key(wb, w, key_bits)) atomicAdd(&c->overflow_leaves, 1ull);
            else report(c, kLeafCap, l);
            atomicAdd(&c->hist[10], 1ull);
        } else {
            const uint64_t bucket = fill * 10 / (cap > 0 ? cap : 1);
            atomicAdd(&c->hist[bucket < 9 ? bucket : 9], 1ull);
        }
    }
}

// Exact bytewise min / max of the words [a, b) against a stored box.
__device__ __forceinline__ bool box_exact(const uint8_t* words, int w, int ws, uint32_t a, uint32_t b,
                                          const uint8_t* lo, const uint8_t* hi) {
    bool ok = true;
    for (int g = 0; g < w; ++g) {
        unsigned mn = 255, mx = 0;
        for (uint32_t e = a; e < b; ++e) {
            const unsigned v = words[static_cast<uint64_t>(e) * ws + g];
            mn = min(mn, v);
            mx = max(mx, v);
        }
        ok = ok && lo[g] == mn && hi[g] == mx;
    }
    return ok;
}

__device__ __forceinline__ bool box_contains(int w, const uint8_t* olo, const uint8_t* ohi, const uint8_t* ilo,
                                             const uint8_t* ihi) {
    bool ok = true;
    for (int g = 0; g < w; ++g) ok = ok && olo[g] <= ilo[g] && ihi[g] <= ohi[g];
    return ok;
}

__global__ void k_audit_pages(const uint8_t* __restrict__ words, const uint32_t* __restrict__ leaf_off,
                              const uint32_t* __restrict__ page_off, const uint32_t* __restrict__ page_leaf, uint64_t P,
                              uint64_t L, uint64_t N, int w, int ws, const uint8_t* __restrict__ page_lo,
                              const uint8_t* __restrict__ page_hi, const uint8_t* __restrict__ group_lo,
                              const uint8_t* __restrict__ group_hi, AuditCounters* c) {
    AUDIT_STRIDE(p, P) {
        const uint32_t a = page_off[p], b = page_off[p + 1], l = page_leaf[p];
        // pages tile the index, at most kPage entries each, within kPage / kRun aligned runs (the bound
        // kernel's run items per page)
        bool tile = l < L && a < b && b - a <= kPage && (b - 1) / kRun - a / kRun < kPage / kRun && (p > 0 || a == 0) &&
                    (p + 1 < P || b == N);
        if (tile) {
            const uint32_t la = leaf_off[l], lb = leaf_off[l + 1];
            tile = la <= a && b <= lb && (a == la || (p > 0 && page_leaf[p - 1] == l)) &&
                   (b == lb || (p + 1 < P && page_leaf[p + 1] == l));
        }
        if (!tile) {
            report(c, kPageTile, p);
            continue;
        }
        if (!box_exact(words, w, ws, a, b, page_lo + p * ws, page_hi + p * ws)) report(c, kPageBox, p);
        const uint64_t g = p / kGroup;
        if (!box_contains(w, group_lo + g * ws, group_hi + g * ws, page_lo + p * ws, page_hi + p * ws))
            report(c, kGroupBox, p);
        atomicAdd(&c->boxes, 1ull);
    }
}

__global__ void k_audit_groups(const uint8_t* __restrict__ group_lo, const uint8_t* __restrict__ group_hi, uint64_t NG,
                               const uint8_t* __restrict__ top_lo, const uint8_t* __restrict__ top_hi, int w, int ws,
                               AuditCounters* c) {
    AUDIT_STRIDE(g, NG) {
        const uint64_t t = g / kGroup;
        if (!box_contains(w, top_lo + t * ws, top_hi + t * ws, group_lo + g * ws, group_hi + g * ws))
            report(c, kGroupBox, g);
        atomicAdd(&c->boxes, 1ull);
    }
}

// Runs and quads: aligned kRun / kQuad entry ranges of the index order.
__global__ void k_audit_small_boxes(const uint8_t* __restrict__ words, uint64_t N, int w, int ws, int span,
                                    const uint8_t* __restrict__ lo, const uint8_t* __restrict__ hi, uint64_t nbox,
                                    int kind, AuditCounters* c) {
    AUDIT_STRIDE(r, nbox) {
        const uint32_t a = static_cast<uint32_t>(r * span);
        const uint64_t end = (r + 1) * span;
        const uint32_t b = static_cast<uint32_t>(end < N ? end : N);
        if (!box_exact(words, w, ws, a, b, lo + r * 2 * ws, hi + r * 2 * ws)) report(c, kind, r);  // (min, max) pairs
        atomicAdd(&c->boxes, 1ull);
    }
}

unsigned audit_grid(uint64_t n, int sms) {
    return static_cast<unsigned>(std::max<uint64_t>(1, std::min<uint64_t>((n + 255) / 256, static_cast<uint64_t>(sms) * 16)));
}

std::string message(int kind, uint64_t where, uint64_t count) {
    const std::string at = std::to_string(where);
    std::string m;
    switch (kind) {
        case kPosRange: m = "entry " + at + ": position out of range"; break;
        case kPosDup: m = "position " + at + " stored twice"; break;
        case kPosMissing: m = "position " + at + " missing from every leaf"; break;
        case kWordMismatch: m = "stored word differs from the recomputed word at position " + at; break;
        case kSymbolBits: m = "entry " + at + ": symbol has bits set below its prefix"; break;
        case kOrder: m = "entries " + at + ", " + std::to_string(where + 1) + " out of key / position order"; break;
        case kLeafShape: m = "leaf " + at + ": offsets do not tile the index"; break;
        case kLeafRoot: m = "leaf " + at + " spans two root subtrees"; break;
        case kLeafCap: m = "leaf " + at + " above capacity but still splittable"; break;
        case kPageTile: m = "page " + at + ": does not tile its leaf"; break;
        case kPageBox: m = "page " + at + ": box is not the min / max of its words"; break;
        case kGroupBox: m = "box " + at + " not contained in its parent group / top box"; break;
        case kRunBox: m = "run " + at + ": box is not the min / max of its words"; break;
        case kQuadBox: m = "quad " + at + ": box is not the min / max of its words"; break;
        case kFineMismatch: m = "stored fine summary differs from the recomputed one at position " + at; break;
        default: m = "violation";
    }
    if (count > 1) m += " (" + std::to_string(count) + " cases)";
    return m;
}

}  // namespace

void audit_index(DevIndex& s, tsg_validation_report* out) {
    cudaStream_t st = s.stream;
    const uint64_t N = s.N;
    AuditCounters* c = nullptr;
    unsigned* seen = nullptr;
    uint8_t *rw = nullptr, *rf = nullptr;
    struct Free {
        std::vector<void*> p;
        cudaStream_t st;
        ~Free() {
            for (void* x : p) cudaFreeAsync(x, st);
            cudaStreamSynchronize(st);
        }
    } fr{{}, st};
    TSG_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&c), sizeof(AuditCounters), st));
    fr.p.push_back(c);
    TSG_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&seen), N * sizeof(unsigned), st));
    fr.p.push_back(seen);
    // re-derivation chunk: at most 8M series (128 MB of words, 256 MB of fine rows)
    const uint64_t chunk = std::min<uint64_t>(N, 8ull << 20);
    TSG_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&rw), chunk * s.ws, st));
    fr.p.push_back(rw);
    if (s.fw) {
        TSG_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&rf), chunk * s.fws, st));
        fr.p.push_back(rf);
    }
    AuditCounters init{};
    for (auto& f : init.first) f = ~0ull;
    TSG_CUDA(cudaMemcpyAsync(c, &init, sizeof(init), cudaMemcpyHostToDevice, st));
    TSG_CUDA(cudaMemsetAsync(seen, 0, N * sizeof(unsigned), st));
    const int sms = s.sms;
    // the re-derivation: K1 over the rows in dataset order, chunk by chunk
    for (uint64_t p0 = 0; p0 < N; p0 += chunk) {
        const uint64_t cnt = std::min(chunk, N - p0);
        summarise(s.rows + p0 * s.n, cnt, s.n, s.w, s.bits, s.thr, rw, nullptr, nullptr, st, rf);
        k_audit_words<<<audit_grid(N, sms), 256, 0, st>>>(s.words, s.pos, N, s.w, s.ws, p0, p0 + cnt, rw,
                                                          s.fw ? s.fine : nullptr, rf, s.fw, s.fws, c);
        TSG_LAUNCHED();
    }
    k_audit_entries<<<audit_grid(N, sms), 256, 0, st>>>(s.words, s.pos, N, s.w, s.ws, s.bits, s.key_bits, seen, c);
    TSG_LAUNCHED();
    k_audit_seen<<<audit_grid(N, sms), 256, 0, st>>>(seen, N, c);
    TSG_LAUNCHED();
    k_audit_leaves<<<audit_grid(s.L, sms), 256, 0, st>>>(s.words, s.leaf_off, s.L, N, s.w, s.ws, s.key_bits, s.leaf_cap, c);
    TSG_LAUNCHED();
    k_audit_pages<<<audit_grid(s.P, sms), 256, 0, st>>>(s.words, s.leaf_off, s.page_off, s.page_leaf, s.P, s.L, N, s.w,
                                                        s.ws, s.page_lo, s.page_hi, s.group_lo, s.group_hi, c);
    TSG_LAUNCHED();
    k_audit_groups<<<audit_grid(s.NG, sms), 256, 0, st>>>(s.group_lo, s.group_hi, s.NG, s.top_lo, s.top_hi, s.w, s.ws, c);
    TSG_LAUNCHED();
    k_audit_small_boxes<<<audit_grid(s.R, sms), 256, 0, st>>>(s.words, N, s.w, s.ws, kRun, s.run_lo, s.run_hi, s.R,
                                                              kRunBox, c);
    TSG_LAUNCHED();
    k_audit_small_boxes<<<audit_grid(s.Q, sms), 256, 0, st>>>(s.words, N, s.w, s.ws, kQuad, s.quad_lo, s.quad_hi, s.Q,
                                                              kQuadBox, c);
    TSG_LAUNCHED();
    AuditCounters h{};
    TSG_CUDA(cudaMemcpyAsync(&h, c, sizeof(h), cudaMemcpyDeviceToHost, st));
    TSG_CUDA(cudaStreamSynchronize(st));

    // aggregate into the report (several shards add up)
    out->leaves += s.L;
    out->inner_nodes += s.inner;
    out->nodes += s.L + s.inner;
    out->max_depth = std::max<uint64_t>(out->max_depth, s.max_depth);
    out->total_entries += N;
    out->empty_leaves += h.empty_leaves;
    out->overflow_leaves += h.overflow_leaves;
    out->pages += s.P;
    out->checked_boxes += h.boxes;
    for (int i = 0; i < 11; ++i) out->leaf_fill_histogram[i] += h.hist[i];
    for (int k = 0; k < kViolationKinds; ++k) {
        if (!h.count[k]) continue;
        out->violation_count += h.count[k];
        if (out->n_violations < 20) {
            const uint64_t where = h.first[k] + (k == kPosDup || k == kPosMissing || k == kWordMismatch ||
                                                         k == kFineMismatch
                                                     ? s.pos_offset
                                                     : 0);
            const std::string m = message(k, where, h.count[k]);
            std::snprintf(out->violations[out->n_violations], sizeof(out->violations[0]), "%s", m.c_str());
            out->n_violations += 1;
        }
    }
}

}  // namespace tsg
