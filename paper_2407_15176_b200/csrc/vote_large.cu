// K3 for large candidate sets (prefill: n_kv * n_q * k up to 131,072 and beyond): the
// reference's tally + vote (selection.hpp:252-286) as device-wide passes, all on the
// stream (graph-capturable), deterministic:
//   1. sort (index << 32 | score key) ascending by the index bits only (indices are middle
//      coordinates: 18 bits at 256K, 3 radix passes instead of 8) -> runs of equal index
//   2. run heads + exclusive scan -> run ids; run starts; per-run max score key (atomicMax:
//      order-independent, so deterministic)
//   3. one rank key per run: (votes << 32 | max score key), payload index
//   4. stable descending sort by rank key (runs enter in index order, so equal keys keep
//      index ascending: the reference's (votes desc, score desc, index asc))
//   5. the first min(k', runs) are the winners; spans + scope follow in select_kernel.
// The radix sorts and the scan are CUB (CUDA's header-only primitives) instantiated here.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "common.cuh"
#include "kernels.h"

using namespace reattn_dev;

namespace reattn_impl {

namespace {

struct LargeWs {
    unsigned long long *keys_in, *keys_out, *hi_in, *hi_out;
    uint32_t *heads, *runid, *rstart, *idx_in, *idx_out, *runmax;
    void* tmp;
    size_t tmp_bytes;
};

size_t al(size_t x) { return (x + 255) / 256 * 256; }

size_t cub_tmp_bytes(uint32_t n) {
    size_t a = 0, b = 0, c = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, a, (unsigned long long*)nullptr,
                                   (unsigned long long*)nullptr, (int)n);
    cub::DeviceScan::ExclusiveSum(nullptr, b, (uint32_t*)nullptr, (uint32_t*)nullptr, (int)n);
    cub::DeviceRadixSort::SortPairsDescending(nullptr, c, (unsigned long long*)nullptr,
                                              (unsigned long long*)nullptr, (uint32_t*)nullptr,
                                              (uint32_t*)nullptr, (int)n);
    return std::max(a, std::max(b, c));
}

LargeWs carve_ws(void* base, uint32_t n) {
    LargeWs w;
    uint8_t* p = (uint8_t*)base;
    auto take = [&](size_t bytes) {
        void* r = p;
        p += al(bytes);
        return r;
    };
    w.keys_in = (unsigned long long*)take(8ull * n);
    w.keys_out = (unsigned long long*)take(8ull * n);
    w.hi_in = (unsigned long long*)take(8ull * n);
    w.hi_out = (unsigned long long*)take(8ull * n);
    w.heads = (uint32_t*)take(4ull * n);
    w.runid = (uint32_t*)take(4ull * n);
    w.rstart = (uint32_t*)take(4ull * n);
    w.idx_in = (uint32_t*)take(4ull * n);
    w.idx_out = (uint32_t*)take(4ull * n);
    w.runmax = (uint32_t*)take(4ull * n);
    w.tmp_bytes = cub_tmp_bytes(n);
    w.tmp = take(w.tmp_bytes);
    return w;
}

__global__ void k_pack(const SelectArgs a, unsigned long long* keys, uint32_t n) {
    for (uint32_t p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x) {
        const uint32_t l = p / a.list_len, j = p % a.list_len;
        const size_t src = (size_t)l * a.list_stride + j;
        keys[p] = ((unsigned long long)a.cand_idx[src] << 32) | float_key(a.cand_score[src]);
    }
}

__global__ void k_heads(const unsigned long long* keys, uint32_t* heads, uint32_t n) {
    for (uint32_t p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x)
        heads[p] = (p == 0 || (keys[p] >> 32) != (keys[p - 1] >> 32)) ? 1u : 0u;
}

__global__ void k_starts(const unsigned long long* keys, const uint32_t* heads, const uint32_t* runid,
                         uint32_t* rstart, uint32_t* runmax, uint32_t n) {
    for (uint32_t p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x) {
        if (heads[p]) rstart[runid[p]] = p;
        // the sort ordered the index bits only: a run's max score key by atomicMax (the
        // run entries' order within the run is arbitrary)
        atomicMax(&runmax[runid[p] + heads[p] - 1u], (uint32_t)(keys[p] & 0xFFFFFFFFull));
    }
}

__global__ void k_rank(const unsigned long long* keys, const uint32_t* heads, const uint32_t* runid,
                       const uint32_t* rstart, const uint32_t* runmax, unsigned long long* hi,
                       uint32_t* idx, uint32_t n) {
    for (uint32_t p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x) {
        const bool last = p == n - 1 || (keys[p + 1] >> 32) != (keys[p] >> 32);
        if (last) {
            const uint32_t run = runid[p] + heads[p] - 1u;
            const uint32_t votes = p - rstart[run] + 1u;
            hi[p] = ((unsigned long long)votes << 32) | runmax[run];
            idx[p] = (uint32_t)(keys[p] >> 32);
        } else {
            hi[p] = 0ull;  // not a run end: sorts after every real run (votes >= 1)
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

}  // namespace

size_t vote_large_workspace(uint32_t n) {
    return 9 * al(8ull * n) + al(cub_tmp_bytes(n)) + 4096;
}

cudaError_t launch_vote_large(const SelectArgs& a, void* ws, cudaStream_t s) {
    const uint32_t n = a.n_lists * a.list_len;
    LargeWs w = carve_ws(ws, n);
    const int g = grid_for(n);
    k_pack<<<g, 256, 0, s>>>(a, w.keys_in, n);
    size_t tb = w.tmp_bytes;
    // index bits only (ties keep the input order: the radix sort is stable)
    int ib = 32;
    if (a.middle_len > 0) {
        ib = 1;
        while (ib < 32 && (1ull << ib) < (unsigned long long)a.middle_len) ++ib;
    }
    cudaError_t e = cub::DeviceRadixSort::SortKeys(w.tmp, tb, w.keys_in, w.keys_out, (int)n, 32,
                                                   32 + ib, s);
    if (e != cudaSuccess) return e;
    k_heads<<<g, 256, 0, s>>>(w.keys_out, w.heads, n);
    tb = w.tmp_bytes;
    e = cub::DeviceScan::ExclusiveSum(w.tmp, tb, w.heads, w.runid, (int)n, s);
    if (e != cudaSuccess) return e;
    e = cudaMemsetAsync(w.runmax, 0, 4ull * n, s);
    if (e != cudaSuccess) return e;
    k_starts<<<g, 256, 0, s>>>(w.keys_out, w.heads, w.runid, w.rstart, w.runmax, n);
    k_rank<<<g, 256, 0, s>>>(w.keys_out, w.heads, w.runid, w.rstart, w.runmax, w.hi_in, w.idx_in, n);
    tb = w.tmp_bytes;
    e = cub::DeviceRadixSort::SortPairsDescending(w.tmp, tb, w.hi_in, w.hi_out, w.idx_in,
                                                  w.idx_out, (int)n, 0, 64, s);
    if (e != cudaSuccess) return e;
    k_final<<<1, 1024, 0, s>>>(w.hi_out, w.idx_out, n, a.k_prime, a.winners, a.rank_votes,
                               a.rank_score, a.hdr);
    // spans + scope from the device-resident winners
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

}  // namespace reattn_impl
