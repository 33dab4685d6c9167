// K3 for large candidate sets (prefill: n_kv * n_q * k up to 131,072 and beyond): the
// reference's tally + vote (selection.hpp:252-286) as device-wide passes, all on the stream
// (graph-capturable) and deterministic.
//
// Bounded path -- every plan (the candidates are middle coordinates, k' <= 1024):
//   1. tally: one atomicAdd (votes) and one atomicMax (max score key) per candidate into two
//      middle-length arrays (order-independent, so deterministic);
//   2. select: one CTA per 2048 middle rows ranks its rows by (votes desc, max score desc,
//      index asc) with a shared-memory bitonic sort, keeps its best kList (>= k', a power of
//      two), and zeroes the rows it read (the arrays stay clean for the next replay); then a
//      4-ary tree of merges: the last of a node's children to arrive (a ticket) merges their
//      sorted lists (merge path: each output position found by a co-rank binary search) and
//      carries the result up; the root writes the first min(k', voted rows) winners;
//   3. spans + scope in select_kernel, as for the small vote.
// 3 launches for any size; no sort of the candidate list itself.
//
// Unbounded path -- the standalone reattn_vote / reattn_tally over arbitrary indices (no
// middle length) or k' > 1024: sort by index, run-length tally, sort by rank key.

#include "common.cuh"
#include "kernels.h"

using namespace reattn_dev;

namespace reattn_impl {

namespace {

// ---- unbounded path: a stable LSD radix sort (8-bit digits, 3 launches per pass) ----------
constexpr uint32_t kRsThreads = 256, kRsItems = 16, kRsTile = kRsThreads * kRsItems, kRsBins = 256;

size_t al(size_t x) { return (x + 255) / 256 * 256; }

uint32_t rs_tiles(uint32_t n) { return std::max(1u, (n + kRsTile - 1) / kRsTile); }

__device__ __forceinline__ uint32_t rs_digit(unsigned long long k, int shift, bool desc) {
    const uint32_t d = (uint32_t)(k >> shift) & 0xFFu;
    return desc ? 255u - d : d;
}

// per tile digit counts, digit-major: hist[d * T + tile]
__global__ void __launch_bounds__(kRsThreads) k_rs_hist(const unsigned long long* keys, uint32_t n, int shift,
                                                       bool desc, uint32_t* hist) {
    __shared__ uint32_t cnt[kRsBins];
    const uint32_t T = gridDim.x, t = blockIdx.x;
    cnt[threadIdx.x] = 0;
    __syncthreads();
    for (uint32_t r = 0; r < kRsItems; ++r) {
        const uint32_t i = t * kRsTile + r * kRsThreads + threadIdx.x;
        if (i < n) atomicAdd(&cnt[rs_digit(keys[i], shift, desc)], 1u);
    }
    __syncthreads();
    hist[threadIdx.x * T + t] = cnt[threadIdx.x];
}

// exclusive scan of m counts in place, one CTA: each thread a contiguous segment
__global__ void __launch_bounds__(1024) k_rs_scan(uint32_t* v, uint32_t m) {
    __shared__ uint32_t part[1024];
    const uint32_t seg = (m + blockDim.x - 1) / blockDim.x, b = threadIdx.x * seg, e = min(m, b + seg);
    uint32_t sum = 0;
    for (uint32_t i = b; i < e; ++i) sum += v[i];
    part[threadIdx.x] = sum;
    __syncthreads();
    for (uint32_t off = 1; off < blockDim.x; off <<= 1) {  // Hillis-Steele inclusive
        const uint32_t x = threadIdx.x >= off ? part[threadIdx.x - off] : 0u;
        __syncthreads();
        part[threadIdx.x] += x;
        __syncthreads();
    }
    uint32_t run = threadIdx.x ? part[threadIdx.x - 1] : 0u;
    for (uint32_t i = b; i < e; ++i) {
        const uint32_t x = v[i];
        v[i] = run;
        run += x;
    }
}

// stable scatter: a tile in 16 rounds of 256 consecutive items; within a round the rank of an
// item among equal digits is (earlier warps' count, then earlier lanes in its warp)
__global__ void __launch_bounds__(kRsThreads) k_rs_scatter(const unsigned long long* kin, const uint32_t* vin,
                                                          unsigned long long* kout, uint32_t* vout, uint32_t n,
                                                          int shift, bool desc, const uint32_t* hist) {
    constexpr int kW = kRsThreads / 32;
    __shared__ uint32_t base[kRsBins];
    __shared__ uint32_t wc[kW][kRsBins];
    const uint32_t T = gridDim.x, t = blockIdx.x;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    base[threadIdx.x] = hist[threadIdx.x * T + t];
#pragma unroll
    for (int j = 0; j < kW; ++j) wc[j][threadIdx.x] = 0;
    __syncthreads();
    for (uint32_t r = 0; r < kRsItems; ++r) {
        const uint32_t i = t * kRsTile + r * kRsThreads + threadIdx.x;
        const bool ok = i < n;
        unsigned long long k = 0;
        uint32_t d = kRsBins + lane;  // a lane outside the data matches no one
        if (ok) {
            k = kin[i];
            d = rs_digit(k, shift, desc);
        }
        const uint32_t peers = __match_any_sync(0xFFFFFFFFu, d);
        const uint32_t before = __popc(peers & ((1u << lane) - 1u));
        if (ok && before == 0) wc[w][d] = __popc(peers);
        __syncthreads();
        {  // per digit: exclusive prefix over the warps; the round total
            uint32_t acc = 0;
#pragma unroll
            for (int j = 0; j < kW; ++j) {
                const uint32_t x = wc[j][threadIdx.x];
                wc[j][threadIdx.x] = acc;
                acc += x;
            }
            __syncthreads();
            if (ok) {
                const uint32_t pos = base[d] + wc[w][d] + before;
                kout[pos] = k;
                if (vin) vout[pos] = vin[i];
            }
            __syncthreads();
            base[threadIdx.x] += acc;
#pragma unroll
            for (int j = 0; j < kW; ++j) wc[j][threadIdx.x] = 0;
            __syncthreads();
        }
    }
}

// sort (keys, vals) by key bits [0, bits), stable, ascending or descending; ping-pongs
// between the two buffers and returns which holds the result (0: *_a, 1: *_b)
int radix_sort(unsigned long long* ka, unsigned long long* kb, uint32_t* va, uint32_t* vb, uint32_t n,
               int bits, bool desc, uint32_t* hist, cudaStream_t s) {
    const uint32_t T = rs_tiles(n);
    int cur = 0;
    for (int shift = 0; shift < bits; shift += 8) {
        unsigned long long* kin = cur ? kb : ka;
        unsigned long long* kout = cur ? ka : kb;
        uint32_t* vin = va ? (cur ? vb : va) : nullptr;
        uint32_t* vout = va ? (cur ? va : vb) : nullptr;
        k_rs_hist<<<T, kRsThreads, 0, s>>>(kin, n, shift, desc, hist);
        k_rs_scan<<<1, 1024, 0, s>>>(hist, kRsBins * T);
        k_rs_scatter<<<T, kRsThreads, 0, s>>>(kin, vin, kout, vout, n, shift, desc, hist);
        cur ^= 1;
    }
    return cur;
}

struct SortedWs {
    unsigned long long *k0, *k1, *h0, *h1;
    uint32_t *i0, *i1, *hist;
};

SortedWs carve_sorted(void* base, uint32_t n) {
    SortedWs w;
    uint8_t* p = (uint8_t*)base;
    auto take = [&](size_t bytes) {
        void* r = p;
        p += al(bytes);
        return r;
    };
    w.k0 = (unsigned long long*)take(8ull * n);
    w.k1 = (unsigned long long*)take(8ull * n);
    w.h0 = (unsigned long long*)take(8ull * n);
    w.h1 = (unsigned long long*)take(8ull * n);
    w.i0 = (uint32_t*)take(4ull * n);
    w.i1 = (uint32_t*)take(4ull * n);
    w.hist = (uint32_t*)take(4ull * kRsBins * rs_tiles(n));
    return w;
}

size_t sorted_bytes(uint32_t n) {
    return 4 * al(8ull * n) + 2 * al(4ull * n) + al(4ull * kRsBins * rs_tiles(n)) + 256;
}

// (index << 32 | score key): sorted ascending, a run of one index ends with its max score
__global__ void k_pack(const SelectArgs a, unsigned long long* keys, uint32_t n) {
    for (uint32_t p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x) {
        const uint32_t l = p / a.list_len, j = p % a.list_len;
        const size_t src = (size_t)l * a.list_stride + j;
        keys[p] = ((unsigned long long)a.cand_idx[src] << 32) | float_key(a.cand_score[src]);
    }
}

// one rank key per run, at the run's last entry: (votes << 32 | max score key); the run's
// start by binary search for its index (no scan); other entries sort after every run
__global__ void k_runs(const unsigned long long* keys, uint32_t n, unsigned long long* hi, uint32_t* idx) {
    for (uint32_t p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x) {
        const uint32_t v = (uint32_t)(keys[p] >> 32);
        const bool last = p == n - 1 || (uint32_t)(keys[p + 1] >> 32) != v;
        if (last) {
            uint32_t lo = 0, h = p;  // first position with index v
            while (lo < h) {
                const uint32_t m = (lo + h) >> 1;
                if ((uint32_t)(keys[m] >> 32) < v) lo = m + 1;
                else h = m;
            }
            hi[p] = ((unsigned long long)(p - lo + 1) << 32) | (keys[p] & 0xFFFFFFFFull);
            idx[p] = v;
        } else {
            hi[p] = 0ull;
            idx[p] = kNoIndex;
        }
    }
}

__global__ void k_final(const unsigned long long* hi, const uint32_t* idx, uint32_t n,
                        uint32_t k_prime, uint32_t* winners, uint32_t* votes, float* score,
                        ScopeHeader* hdr) {
    __shared__ uint32_t s_nw;
    if (threadIdx.x == 0) s_nw = 0;
    __syncthreads();
    const uint32_t lim = min(k_prime, n);
    for (uint32_t j = threadIdx.x; j < lim; j += blockDim.x) {
        if (hi[j] > 0ull) {
            winners[j] = idx[j];
            if (votes) votes[j] = (uint32_t)(hi[j] >> 32);
            if (score) score[j] = key_float((uint32_t)(hi[j] & 0xFFFFFFFFull));
            atomicMax(&s_nw, j + 1);  // the positive keys form a prefix (descending sort)
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) hdr->n_winners = s_nw;
}

int grid_for(uint32_t n) { return (int)std::min<uint32_t>(148u * 8u, std::max(1u, (n + 255) / 256)); }

// ---- bounded path ---------------------------------------------------------------------
constexpr uint32_t kChunk = 2048;       // middle rows ranked per CTA
constexpr uint32_t kMaxList = 1024;     // largest kept list (k' <= kMaxList)
constexpr uint32_t kFan = 4;            // merge-tree fan-in
constexpr uint32_t kEmptyIdx = 0xFFFFFFFFu;

struct BoundedWs {
    uint32_t *votes, *maxkey;   // [middle]
    unsigned long long* lkey;   // tree node lists [nodes][kList]
    uint32_t* lidx;
    uint32_t* tickets;          // [nodes]
    uint32_t* flag;             // out-of-range candidate seen
};

uint32_t list_len_for(uint32_t k_prime) {
    uint32_t l = 128;
    while (l < k_prime) l <<= 1;
    return l;
}

// tree geometry: level 0 has G nodes (one per CTA), level L ceil(n_{L-1} / kFan) nodes
uint32_t tree_nodes(uint32_t G) {
    uint32_t total = 0, n = G;
    while (true) {
        total += n;
        if (n == 1) break;
        n = (n + kFan - 1) / kFan;
    }
    return total;
}

BoundedWs carve_bounded(void* base, uint32_t middle, uint32_t k_prime) {
    BoundedWs w;
    uint8_t* p = (uint8_t*)base;
    auto take = [&](size_t bytes) {
        void* r = p;
        p += al(bytes);
        return r;
    };
    const uint32_t G = std::max(1u, (middle + kChunk - 1) / kChunk);
    const uint32_t nodes = tree_nodes(G), L = list_len_for(k_prime);
    w.votes = (uint32_t*)take(4ull * middle);
    w.maxkey = (uint32_t*)take(4ull * middle);
    w.lkey = (unsigned long long*)take(8ull * nodes * L);
    w.lidx = (uint32_t*)take(4ull * nodes * L);
    w.tickets = (uint32_t*)take(4ull * nodes);
    w.flag = (uint32_t*)take(4);
    return w;
}

size_t bounded_bytes(uint32_t middle, uint32_t k_prime) {
    const uint32_t G = std::max(1u, (middle + kChunk - 1) / kChunk);
    const uint32_t nodes = tree_nodes(G), L = list_len_for(k_prime);
    return al(4ull * middle) * 2 + al(8ull * nodes * L) + al(4ull * nodes * L) + al(4ull * nodes) + al(4) + 256;
}

__global__ void k_tally(const SelectArgs a, BoundedWs w, uint32_t n) {
    for (uint32_t p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x) {
        const uint32_t l = p / a.list_len, j = p % a.list_len;
        const size_t src = (size_t)l * a.list_stride + j;
        const uint32_t idx = a.cand_idx[src];
        if (idx == kNoIndex) continue;
        if (idx >= a.middle_len) {
            *w.flag = 1u;
            continue;
        }
        atomicAdd(&w.votes[idx], 1u);
        atomicMax(&w.maxkey[idx], float_key(a.cand_score[src]));
    }
}

// (key desc, index asc): keys are distinct per index, so this is a total order on real rows
__device__ __forceinline__ bool ahead(unsigned long long ka, uint32_t ia, unsigned long long kb, uint32_t ib) {
    return ka > kb || (ka == kb && ia < ib);
}

// out[p] for p < L: the p-th entry of the merge of sorted lists A and B (each L long)
__device__ void merge_top(const unsigned long long* ak, const uint32_t* ai, const unsigned long long* bk,
                          const uint32_t* bi, uint32_t L, unsigned long long* ok, uint32_t* oi) {
    for (uint32_t p = threadIdx.x; p < L; p += blockDim.x) {
        // co-rank: i entries from A and p - i from B precede position p
        uint32_t lo = 0, hi = p;  // i in [0, p] (both lists are at least L > p long)
        while (lo < hi) {
            const uint32_t i = (lo + hi) >> 1;  // is A[i] ahead of B[p - 1 - i]?
            if (ahead(ak[i], ai[i], bk[p - 1 - i], bi[p - 1 - i])) lo = i + 1;
            else hi = i;
        }
        const uint32_t i = lo, j = p - i;
        const bool take_a = ahead(ak[i], ai[i], bk[j], bi[j]);
        ok[p] = take_a ? ak[i] : bk[j];
        oi[p] = take_a ? ai[i] : bi[j];
    }
}

__global__ void __launch_bounds__(1024) k_rank_tree(const SelectArgs a, BoundedWs w, uint32_t L, uint32_t G) {
    extern __shared__ unsigned long long sm[];
    unsigned long long* sk = sm;                      // [kChunk] sort keys, then list A
    unsigned long long* tk = sm + kChunk;             // [kMaxList] merge output / list B
    uint32_t* si = (uint32_t*)(sm + kChunk + kMaxList);  // [kChunk]
    uint32_t* ti = si + kChunk;                       // [kMaxList]
    __shared__ uint32_t s_last;
    const uint32_t c = blockIdx.x, base = c * kChunk, tid = threadIdx.x;
    // 1. load (and clear) this CTA's rows
    for (uint32_t r = tid; r < kChunk; r += blockDim.x) {
        const uint32_t i = base + r;
        uint32_t v = 0, m = 0;
        if (i < a.middle_len) {
            v = w.votes[i];
            m = w.maxkey[i];
            if (v) {
                w.votes[i] = 0u;
                w.maxkey[i] = 0u;
            }
        }
        sk[r] = v ? ((unsigned long long)v << 32) | m : 0ull;
        si[r] = v ? i : kEmptyIdx;
    }
    __syncthreads();
    // 2. bitonic sort, best first
    for (uint32_t k = 2; k <= kChunk; k <<= 1)
        for (uint32_t j = k >> 1; j > 0; j >>= 1) {
            for (uint32_t t = tid; t < kChunk / 2; t += blockDim.x) {
                const uint32_t i = 2 * t - (t & (j - 1)), l = i + j;
                const bool desc = (i & k) == 0;
                const bool sw = desc ? ahead(sk[l], si[l], sk[i], si[i]) : ahead(sk[i], si[i], sk[l], si[l]);
                if (sw) {
                    const unsigned long long kk = sk[i];
                    sk[i] = sk[l];
                    sk[l] = kk;
                    const uint32_t ii = si[i];
                    si[i] = si[l];
                    si[l] = ii;
                }
            }
            __syncthreads();
        }
    // 3. the merge tree: the current list is sk/si[0, L)
    uint32_t node = c, level_base = 0, n_level = G;
    while (n_level > 1) {
        unsigned long long* gk = w.lkey + (size_t)(level_base + node) * L;
        uint32_t* gi = w.lidx + (size_t)(level_base + node) * L;
        for (uint32_t r = tid; r < L; r += blockDim.x) {
            gk[r] = sk[r];
            gi[r] = si[r];
        }
        const uint32_t parent = node / kFan, first = parent * kFan;
        const uint32_t n_child = min(kFan, n_level - first);
        const uint32_t next_base = level_base + n_level;
        __threadfence();
        __syncthreads();
        if (tid == 0) {
            const uint32_t t = next_base + parent;  // ticket of the parent node
            s_last = atomicAdd(&w.tickets[t], 1u) == n_child - 1;
            if (s_last) w.tickets[t] = 0u;
        }
        __syncthreads();
        if (!s_last) return;
        __threadfence();
        for (uint32_t ch = first; ch < first + n_child; ++ch) {
            if (ch == node) continue;
            const unsigned long long* ck = w.lkey + (size_t)(level_base + ch) * L;
            const uint32_t* ci = w.lidx + (size_t)(level_base + ch) * L;
            // B := the sibling's list (into tk/ti), then merged into tk/ti via sk as A
            unsigned long long* bk = tk;
            uint32_t* bi = ti;
            for (uint32_t r = tid; r < L; r += blockDim.x) {
                bk[r] = __ldcg(ck + r);
                bi[r] = __ldcg(ci + r);
            }
            __syncthreads();
            // merged into the upper half of the sort buffer (2L <= kChunk), then copied back
            unsigned long long* ok = sk + L;
            uint32_t* oi = si + L;
            merge_top(sk, si, bk, bi, L, ok, oi);
            __syncthreads();
            for (uint32_t r = tid; r < L; r += blockDim.x) {
                sk[r] = ok[r];
                si[r] = oi[r];
            }
            __syncthreads();
        }
        node = parent;
        level_base = next_base;
        n_level = (n_level + kFan - 1) / kFan;
    }
    // 4. the root: winners
    const uint32_t kp = a.k_prime;
    if (tid == 0) s_last = 0;
    __syncthreads();
    for (uint32_t j = tid; j < min(kp, L); j += blockDim.x) {
        if (si[j] != kEmptyIdx) {
            a.winners[j] = si[j];
            if (a.rank_votes) a.rank_votes[j] = (uint32_t)(sk[j] >> 32);
            if (a.rank_score) a.rank_score[j] = key_float((uint32_t)(sk[j] & 0xFFFFFFFFull));
            atomicMax(&s_last, j + 1);  // voted rows form a prefix
        }
    }
    __syncthreads();
    if (tid == 0) {
        uint32_t nw = s_last;
        if (*w.flag) {  // a candidate outside the middle: surfaces as expand_spans' range error
            a.winners[0] = a.middle_len;
            nw = max(nw, 1u);
            *w.flag = 0u;
        }
        a.hdr->n_winners = nw;
    }
}


}  // namespace

cudaError_t launch_vote_sorted(const SelectArgs& a, void* ws, cudaStream_t s);

bool vote_bounded(uint32_t middle_len, uint32_t k_prime) { return middle_len > 0 && k_prime <= kMaxList; }

uint32_t vote_large_kernels(uint32_t n, uint32_t middle_len, uint32_t k_prime) {
    if (vote_bounded(middle_len, k_prime)) return 3;  // tally, rank tree, select
    int ib = 32, vb = 1;
    if (middle_len > 0) {
        ib = 1;
        while (ib < 32 && (1ull << ib) < (unsigned long long)middle_len) ++ib;
    }
    while (vb < 32 && (1ull << vb) <= (unsigned long long)n) ++vb;
    return 4 + 3 * (uint32_t)((32 + ib + 7) / 8 + (32 + vb + 7) / 8);  // pack, runs, final, select
}

size_t vote_large_workspace(uint32_t n, uint32_t middle_len, uint32_t k_prime) {
    if (vote_bounded(middle_len, k_prime)) return bounded_bytes(middle_len, k_prime);
    return sorted_bytes(n);
}

cudaError_t launch_vote_large(const SelectArgs& a, void* ws, cudaStream_t s) {
    const uint32_t n = a.n_lists * a.list_len;
    if (vote_bounded(a.middle_len, a.k_prime)) {
        const BoundedWs w = carve_bounded(ws, a.middle_len, a.k_prime);
        k_tally<<<grid_for(n), 256, 0, s>>>(a, w, n);
        const uint32_t G = std::max(1u, (a.middle_len + kChunk - 1) / kChunk);
        const size_t smem = (size_t)(kChunk + kMaxList) * (sizeof(unsigned long long) + sizeof(uint32_t));
        k_rank_tree<<<G, 1024, smem, s>>>(a, w, list_len_for(a.k_prime), G);
    } else {
        cudaError_t e = launch_vote_sorted(a, ws, s);
        if (e != cudaSuccess) return e;
    }
    // spans + scope from the device-resident winners (the standalone vote / tally APIs ask
    // for neither)
    if (!a.span_b) {  // the header's error field is the select's to write: clear it here
        const cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
        return cudaMemsetAsync(&a.hdr->error, 0, sizeof(a.hdr->error), s);
    }
    SelectArgs b = a;
    b.cand_idx = nullptr;
    b.cand_score = nullptr;
    b.n_lists = 0;
    b.list_len = 0;
    b.winners_in = a.winners;
    b.n_winners_in = a.k_prime;  // upper bound; the exact count is read on the device
    b.n_winners_dev = &a.hdr->n_winners;
    b.rank_votes = nullptr;
    b.rank_score = nullptr;
    return launch_select(b, s);
}

// the unbounded path: sort by (index, score key), run-length tally, sort by rank key
cudaError_t launch_vote_sorted(const SelectArgs& a, void* ws, cudaStream_t s) {
    const uint32_t n = a.n_lists * a.list_len;
    SortedWs w = carve_sorted(ws, n);
    const int g = grid_for(n);
    k_pack<<<g, 256, 0, s>>>(a, w.k0, n);
    int ib = 32;  // index bits: the middle length when known
    if (a.middle_len > 0) {
        ib = 1;
        while (ib < 32 && (1ull << ib) < (unsigned long long)a.middle_len) ++ib;
    }
    const int c1 = radix_sort(w.k0, w.k1, nullptr, nullptr, n, 32 + ib, false, w.hist, s);
    const unsigned long long* keys = c1 ? w.k1 : w.k0;
    k_runs<<<g, 256, 0, s>>>(keys, n, w.h0, w.i0);
    int vb = 1;  // votes bits
    while (vb < 32 && (1ull << vb) <= (unsigned long long)n) ++vb;
    // descending and stable: equal rank keys keep the index-ascending run order
    const int c2 = radix_sort(w.h0, w.h1, w.i0, w.i1, n, 32 + vb, true, w.hist, s);
    k_final<<<1, 1024, 0, s>>>(c2 ? w.h1 : w.h0, c2 ? w.i1 : w.i0, n, a.k_prime, a.winners, a.rank_votes,
                               a.rank_score, a.hdr);
    return cudaGetLastError();
}

}  // namespace reattn_impl
