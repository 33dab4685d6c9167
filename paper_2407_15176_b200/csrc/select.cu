// K3 — vote, span expansion and scope assembly in one single-CTA kernel.
//
// Restates (reference /root/reference/proj/include/reattn/):
//   tally_candidates + vote     selection.hpp:252-286  (votes desc, max score desc, idx asc)
//   expand_spans                selection.hpp:318-349  (aligned / centered, sorted ascending)
//   assemble_scope (indices)    scope.hpp:37-78      (global ++ spans ++ local, window check)
//   the n_q <= L' check         engine.hpp:69
// The output is a device ScopeHeader + a scope-row -> cache-row table, so the attention
// kernels run straight after it without a host round trip.  Ranking uses bitonic sorts of
// packed keys in shared memory: exact and deterministic (no atomics-order dependence).
#include <algorithm>

#include "common.cuh"
#include "kernels.h"
#include "select_small.cuh"

using namespace reattn_dev;

namespace reattn_impl {

namespace {

constexpr int kSelThreads = 1024;

__device__ __forceinline__ int pow2_at_least(int n, int lo) {
    int p = lo;
    while (p < n) p <<= 1;
    return p;
}

// ascending bitonic over (hi, lo) pairs; cmp_desc_hi: sort hi descending, lo ascending
template <bool DESC_HI>
__device__ void bitonic_pairs(unsigned long long* hi, uint32_t* lo, int n) {
    for (int k2 = 2; k2 <= n; k2 <<= 1) {
        for (int j = k2 >> 1; j > 0; j >>= 1) {
            for (int i = threadIdx.x; i < n; i += blockDim.x) {
                const int ixj = i ^ j;
                if (ixj > i) {
                    const unsigned long long xh = hi[i], yh = hi[ixj];
                    const uint32_t xl = lo ? lo[i] : 0u, yl = lo ? lo[ixj] : 0u;
                    // "x before y" in the target order
                    bool x_first;
                    if (DESC_HI)
                        x_first = xh > yh || (xh == yh && xl < yl);
                    else
                        x_first = xh < yh || (xh == yh && xl < yl);
                    const bool up = (i & k2) == 0;
                    if (up ? !x_first : x_first) {
                        hi[i] = yh;
                        hi[ixj] = xh;
                        if (lo) {
                            lo[i] = yl;
                            lo[ixj] = xl;
                        }
                    }
                }
            }
            __syncthreads();
        }
    }
}

// exclusive scan of v[0, n) in place; returns the total to every thread
__device__ uint32_t block_exclusive_scan(uint32_t* v, int n, uint32_t* warp_tot) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int per = (n + blockDim.x - 1) / blockDim.x;
    const int b0 = min(n, tid * per), b1 = min(n, b0 + per);
    uint32_t local = 0;
    for (int i = b0; i < b1; ++i) local += v[i];
    uint32_t incl = local;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, incl, off);
        if (lane >= off) incl += t;
    }
    if (lane == 31) warp_tot[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        const int nw = blockDim.x >> 5;
        uint32_t w = lane < nw ? warp_tot[lane] : 0u;
        uint32_t wi = w;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, wi, off);
            if (lane >= off) wi += t;
        }
        if (lane < nw) warp_tot[lane] = wi - w;  // exclusive warp offsets
        if (lane == nw - 1) warp_tot[32] = wi;   // total
    }
    __syncthreads();
    uint32_t run = warp_tot[warp] + incl - local;
    for (int i = b0; i < b1; ++i) {
        const uint32_t x = v[i];
        v[i] = run;
        run += x;
    }
    const uint32_t total = warp_tot[32];
    __syncthreads();
    return total;
}

// Small path: <= 32 candidates, no external winners/spans.
__global__ void __launch_bounds__(256) select_small_kernel(const SelectArgs a) {
    __shared__ SmallSelectSmem sm;
    SmallSelectIO io;
    io.k_prime = a.k_prime;
    io.span_m = a.span_m;
    io.middle_len = a.middle_len;
    io.span_mode = a.span_mode;
    io.g_end = a.g_end;
    io.l_start = a.l_start;
    io.total = a.total;
    io.window = a.build_scope ? a.window : 0xFFFFFFFFu;
    io.n_q = a.build_scope ? a.n_q : 0u;
    io.winners = a.winners;
    io.span_b = a.span_b;
    io.span_e = a.span_e;
    io.scope_src = a.build_scope ? a.scope_src : nullptr;
    io.hdr = a.hdr;
    const uint32_t n = a.n_lists * a.list_len;
    const int i = threadIdx.x;
    uint32_t ci = 0;
    float cs = 0.0f;
    const bool valid = i < (int)n;
    if (valid) {
        const size_t src = (size_t)(i / a.list_len) * a.list_stride + i % a.list_len;
        ci = a.cand_idx[src];
        cs = a.cand_score[src];
    }
    small_select_scope(io, ci, cs, valid, sm);
    if (threadIdx.x == 0 && a.hdr && !a.build_scope) a.hdr->L = 0;
}

__global__ void __launch_bounds__(kSelThreads) select_kernel(const SelectArgs a) {
    extern __shared__ unsigned long long ssm[];
    __shared__ uint32_t warp_tot[33];
    __shared__ uint32_t s_nw, s_ns, s_cov, s_err, s_L;
    const int tid = threadIdx.x;
    const uint32_t n = a.n_lists * a.list_len;
    if (tid == 0) {
        s_nw = 0;
        s_ns = 0;
        s_cov = 0;
        s_err = 0;
    }
    __syncthreads();

    uint32_t* winners = a.winners;  // global (k' entries)
    unsigned long long* spans_sm = nullptr;
    uint32_t* off_sm = nullptr;

    const bool have_spans = a.span_b_in != nullptr;
    const bool have_winners = a.winners_in != nullptr;
    if (!have_spans && !have_winners && a.k_prime > 0 && n > 0) {
        // ---- tally (selection.hpp:252-276) ----
        const int NS = pow2_at_least((int)n, 32);
        unsigned long long* key = ssm;                     // [NS]  idx<<32 | score key
        uint32_t* head = (uint32_t*)(key + NS);            // [NS]
        uint32_t* start = head + NS;                       // [NS]
        unsigned long long* rhi = (unsigned long long*)(start + NS);  // [NS]
        uint32_t* ridx = (uint32_t*)(rhi + NS);            // [NS]
        for (int p = tid; p < NS; p += blockDim.x) {
            if (p < (int)n) {
                const uint32_t l = p / a.list_len, j = p % a.list_len;
                const size_t src = (size_t)l * a.list_stride + j;
                key[p] = ((unsigned long long)a.cand_idx[src] << 32) | float_key(a.cand_score[src]);
            } else {
                key[p] = ~0ull;
            }
        }
        __syncthreads();
        bitonic_pairs<false>(key, nullptr, NS);
        for (int p = tid; p < (int)n; p += blockDim.x)
            head[p] = (p == 0 || (key[p] >> 32) != (key[p - 1] >> 32)) ? 1u : 0u;
        __syncthreads();
        // run id of a head = exclusive count of heads before it
        for (int p = tid; p < (int)n; p += blockDim.x) start[p] = head[p];
        __syncthreads();
        const uint32_t U = block_exclusive_scan(start, (int)n, warp_tot);
        // start[p] = number of heads before p, so element p belongs to run
        // start[p] + head[p] - 1.  Heads record their run's first position.
        for (int p = tid; p < (int)n; p += blockDim.x)
            if (head[p]) ridx[start[p]] = (uint32_t)p;
        __syncthreads();
        // The last element of each run carries its max score (ascending sort); it writes
        // the run's rank key (votes, max score) and replaces the start with the index.
        for (int p = tid; p < (int)n; p += blockDim.x) {
            const bool last = (p == (int)n - 1) || ((key[p + 1] >> 32) != (key[p] >> 32));
            if (last) {
                const uint32_t run = start[p] + head[p] - 1u;
                const uint32_t votes = (uint32_t)p - ridx[run] + 1u;
                rhi[run] = ((unsigned long long)votes << 32) | (uint32_t)(key[p] & 0xFFFFFFFFull);
                ridx[run] = (uint32_t)(key[p] >> 32);
            }
        }
        __syncthreads();
        const int NR = pow2_at_least((int)U, 32);
        for (int r = U + tid; r < NR; r += blockDim.x) {
            rhi[r] = 0ull;
            ridx[r] = 0xFFFFFFFFu;
        }
        __syncthreads();
        // ---- rank (selection.hpp:269-274): votes desc, score desc, index asc ----
        bitonic_pairs<true>(rhi, ridx, NR);
        const uint32_t nw = min(a.k_prime, U);
        for (uint32_t j = tid; j < nw; j += blockDim.x) {
            winners[j] = ridx[j];
            if (a.rank_votes) a.rank_votes[j] = (uint32_t)(rhi[j] >> 32);
            if (a.rank_score) a.rank_score[j] = key_float((uint32_t)(rhi[j] & 0xFFFFFFFFull));
        }
        if (tid == 0) s_nw = nw;
        __syncthreads();
    } else if (have_winners) {
        const uint32_t nwin = a.n_winners_dev ? *a.n_winners_dev : a.n_winners_in;
        if (winners != a.winners_in)
            for (uint32_t j = tid; j < nwin; j += blockDim.x) winners[j] = a.winners_in[j];
        if (tid == 0) s_nw = nwin;
        __syncthreads();
    }

    const uint32_t nw = s_nw;
    // ---- spans (selection.hpp:318-349) ----
    {
        const int NP = pow2_at_least((int)max(nw, a.n_spans_in), 32);
        spans_sm = ssm;  // reuse
        off_sm = (uint32_t*)(spans_sm + NP);
        if (have_spans) {
            for (uint32_t j = tid; j < a.n_spans_in; j += blockDim.x) {
                if (a.span_e_in[j] > a.middle_len) atomicMax(&s_err, (uint32_t)kScopeErrSpanRange);
                spans_sm[j] = ((unsigned long long)a.span_b_in[j] << 32) | a.span_e_in[j];
            }
            __syncthreads();
            if (tid == 0) s_ns = a.n_spans_in;
        } else if (nw > 0 && a.middle_len > 0) {
            for (int j = tid; j < NP; j += blockDim.x) {
                if (j < (int)nw) {
                    const uint32_t w = winners[j];
                    if (w >= a.middle_len) atomicMax(&s_err, (uint32_t)kScopeErrWinnerRange);
                    uint32_t st;
                    const uint32_t m = a.span_m;
                    if (a.span_mode == 0) {
                        st = (w / m) * m;
                    } else {
                        st = w > m / 2 ? w - m / 2 : 0u;
                        if ((uint64_t)st + m > a.middle_len) st = a.middle_len > m ? a.middle_len - m : 0u;
                    }
                    const uint32_t e = (uint32_t)min((uint64_t)st + m, (uint64_t)a.middle_len);
                    spans_sm[j] = ((unsigned long long)st << 32) | e;
                } else {
                    spans_sm[j] = ~0ull;
                }
            }
            __syncthreads();
            bitonic_pairs<false>(spans_sm, nullptr, NP);
            if (tid == 0 && s_err == 0) {
                uint32_t m = 0;
                for (uint32_t j = 0; j < nw; ++j) {
                    const uint32_t b = (uint32_t)(spans_sm[j] >> 32), e = (uint32_t)spans_sm[j];
                    if (m > 0) {
                        const uint32_t pb = (uint32_t)(spans_sm[m - 1] >> 32);
                        const uint32_t pe = (uint32_t)spans_sm[m - 1];
                        if (a.span_mode == 1 && b <= pe) {  // merge overlap (centered)
                            spans_sm[m - 1] = ((unsigned long long)pb << 32) | max(pe, e);
                            continue;
                        }
                        if (b == pb && e == pe) continue;  // aligned duplicate
                    }
                    spans_sm[m++] = ((unsigned long long)b << 32) | e;
                }
                s_ns = m;
            }
            __syncthreads();
        }
        const uint32_t ns = s_ns;
        if (tid == 0) {
            uint32_t cov = 0;
            for (uint32_t j = 0; j < ns; ++j) {
                off_sm[j] = cov;
                cov += (uint32_t)spans_sm[j] - (uint32_t)(spans_sm[j] >> 32);
            }
            s_cov = cov;
        }
        __syncthreads();
        for (uint32_t j = tid; j < ns; j += blockDim.x) {
            if (a.span_b) a.span_b[j] = (uint32_t)(spans_sm[j] >> 32);
            if (a.span_e) a.span_e[j] = (uint32_t)spans_sm[j];
        }
    }
    const uint32_t ns = s_ns, cov = s_cov;

    // ---- scope (scope.hpp:44-61, engine.hpp:69) ----
    if (a.build_scope) {
        if (tid == 0) {
            const uint64_t L = (uint64_t)a.g_end + cov + (a.total - a.l_start);
            uint32_t err = s_err;
            if (err == 0 && L > a.window) err = kScopeErrWindow;
            if (err == 0 && a.n_q > L) err = kScopeErrQueryLong;
            s_err = err;
            s_L = (uint32_t)L;
        }
        __syncthreads();
        const uint32_t L = s_L;
        if (s_err == 0 && a.scope_src) {
            const uint32_t g = a.g_end;
            for (uint32_t r = tid; r < L; r += blockDim.x) {
                uint32_t src;
                if (r < g) {
                    src = r;
                } else if (r < g + cov) {
                    const uint32_t o = r - g;
                    int lo = 0, hi = (int)ns - 1;  // last span with off <= o
                    while (lo < hi) {
                        const int mid = (lo + hi + 1) >> 1;
                        if (off_sm[mid] <= o) lo = mid;
                        else hi = mid - 1;
                    }
                    src = g + (uint32_t)(spans_sm[lo] >> 32) + (o - off_sm[lo]);
                } else {
                    src = a.l_start + (r - g - cov);
                }
                RA_ASSERT(r < a.window && src < a.total);
                a.scope_src[r] = src;
            }
        }
    }
    if (tid == 0 && a.hdr) {
        ScopeHeader h;
        h.L = a.build_scope ? s_L : 0u;
        h.n_spans = ns;
        h.coverage = cov;
        h.n_winners = nw;
        h.error = (int32_t)s_err;
        h.pad[0] = h.pad[1] = h.pad[2] = 0;
        *a.hdr = h;
    }
}

}  // namespace

size_t select_smem_bytes(uint32_t n_cand, uint32_t k_prime) {
    uint32_t NS = 32;
    while (NS < n_cand) NS <<= 1;
    uint32_t NP = 32;
    while (NP < k_prime) NP <<= 1;
    const size_t tally = (size_t)NS * (8 + 4 + 4 + 8 + 4);
    const size_t spans = (size_t)NP * (8 + 4);
    return std::max(tally, spans);
}

cudaError_t launch_select(const SelectArgs& a, cudaStream_t s) {
    const uint32_t n = a.n_lists * a.list_len;
    if (!a.winners_in && !a.span_b_in && !a.rank_votes && !a.rank_score && n <= kSmallSelectMax) {
        select_small_kernel<<<1, 256, 0, s>>>(a);
        return cudaGetLastError();
    }
    const uint32_t kp = std::max({a.k_prime, a.n_spans_in, a.n_winners_in});
    const size_t smem = select_smem_bytes(n, kp);
    static int cur = 0;
    if ((int)smem > cur) {
        cudaFuncSetAttribute(select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)std::max<size_t>(smem, 48 * 1024));
        cur = (int)std::max<size_t>(smem, 48 * 1024);
    }
    select_kernel<<<1, kSelThreads, smem, s>>>(a);
    return cudaGetLastError();
}

}  // namespace reattn_impl
