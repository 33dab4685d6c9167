// Sequence-sharded decode: merge of the per-rank candidate lists, vote +
// spans + global scope (redundantly on every rank), and the translation of the global
// scope table into this rank's local rows.
//
// Rank r holds [global | middle shard r | local] in its cache.  Its K1 scan yields, per
// (kv head, query), the exact top-k of its shard; top-k of the union of all ranks' lists
// under (score desc, index asc) is the exact global top-k (selection.hpp:81-135 ordering),
// so after an all-gather every rank merges identically and continues with the reference's
// vote / expand_spans / assemble_scope (selection.hpp:252-349, scope.hpp:37-61).
// The scope table is translated to this rank's local cache rows (replicated global and local
// rows exist on every rank; a middle row only at its owner), and the rank's share of the
// attention is written as ShardRanges: rank 0 the global rows, every rank the span rows of
// its own shard (contiguous in scope order) and a 32-row aligned 1/world slice of the local
// window -- every scope row is attended by exactly one rank, and the work is balanced.
#include "common.cuh"
#include "kernels.h"
#include "select_small.cuh"

using namespace reattn_dev;

namespace reattn_impl {

namespace {

constexpr int kMergeThreads = 1024;

__global__ void __launch_bounds__(kMergeThreads) shard_merge_select_kernel(const ShardSelectArgs a) {
    __shared__ uint32_t m_idx[kSmallSelectMax];
    __shared__ float m_score[kSmallSelectMax];
    __shared__ SmallSelectSmem ssel;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int k = a.k, kk = a.kk;
    // ---- merge: warp w handles list w (kv head); lanes load the ranks' candidates ----
    if (warp < a.n_lists) {
        float ls[8];
        uint32_t li[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            ls[j] = -INFINITY;
            li[j] = kNoIndex;
        }
        const int n = a.n_src * k;
        for (int e = lane; e < n; e += 32) {
            const int src = e / k, j = e % k;
            const size_t o = (size_t)src * a.src_stride + (size_t)warp * k + j;
            uint32_t i = a.cand_idx[o];
            const float s = a.cand_score[o];
            if (i == kNoIndex) continue;
            i += a.src_offset[src];  // shard-local middle index -> global middle index
            // bubble into the lane's sorted list (full order: score desc, index asc)
            float cs = s;
            uint32_t ci = i;
#pragma unroll
            for (int jj = 0; jj < 8; ++jj) {
                if (jj < k && better(cs, ci, ls[jj], li[jj])) {
                    const float t = ls[jj];
                    const uint32_t u = li[jj];
                    ls[jj] = cs;
                    li[jj] = ci;
                    cs = t;
                    ci = u;
                }
            }
        }
        for (int r = 0; r < kk; ++r) {
            float bs = ls[0];
            uint32_t bi = li[0];
            warp_best(bs, bi);
            if (lane == 0) {
                m_idx[warp * kk + r] = bi;
                m_score[warp * kk + r] = bs;
            }
            if (bi != kNoIndex && li[0] == bi) {
#pragma unroll
                for (int jj = 0; jj < 7; ++jj) {
                    ls[jj] = ls[jj + 1];
                    li[jj] = li[jj + 1];
                }
                ls[7] = -INFINITY;
                li[7] = kNoIndex;
            }
        }
    }
    __syncthreads();
    // ---- vote + spans + GLOBAL scope table (into scope_src) ----
    const int n = a.n_lists * kk;
    const bool valid = tid < n && m_idx[tid < n ? tid : 0] != kNoIndex;
    small_select_scope(a.sel, valid ? m_idx[tid] : 0u, valid ? m_score[tid] : 0.0f, valid, ssel);
    __syncthreads();
    // ---- translate to this rank's local rows; find the rank's span rows ----
    __shared__ uint32_t s_mb, s_me;
    if (tid == 0) {
        s_mb = 0xFFFFFFFFu;
        s_me = 0;
    }
    __syncthreads();
    if (ssel.err != 0) return;
    const uint32_t L = ssel.L;
    for (uint32_t r = tid; r < L; r += blockDim.x) {
        const uint32_t s = a.sel.scope_src[r];
        uint32_t local;
        if (s < a.sel.g_end) {
            local = s;
        } else if (s >= a.sel.l_start) {
            local = a.sel.g_end + a.shard_len + (s - a.sel.l_start);
        } else {
            const uint32_t m = s - a.sel.g_end;
            const bool mine = m >= a.shard_begin && m < a.shard_begin + a.shard_len;
            local = mine ? a.sel.g_end + (m - a.shard_begin) : kNoIndex;
            if (mine) {
                atomicMin(&s_mb, r);
                atomicMax(&s_me, r + 1);
            }
        }
        a.local_src[r] = local;
    }
    __syncthreads();
    if (tid == 0) {
        const uint32_t n_local = a.sel.total - a.sel.l_start;
        const uint32_t lb = L - n_local;
        auto cut = [&](int r) {  // 32-row aligned split of the local window
            return (uint32_t)(((uint64_t)r * n_local / (uint32_t)a.world) / 32u * 32u);
        };
        const uint32_t c0 = a.rank == 0 ? 0u : cut(a.rank);
        const uint32_t c1 = a.rank + 1 == a.world ? n_local : cut(a.rank + 1);
        ShardRanges R;
        R.n = 0;
        if (a.rank == 0 && a.sel.g_end > 0) {
            R.begin[R.n] = 0;
            R.end[R.n++] = a.sel.g_end;
        }
        if (s_mb < s_me) {
            R.begin[R.n] = s_mb;
            R.end[R.n++] = s_me;
        }
        if (c1 > c0) {
            R.begin[R.n] = lb + c0;
            R.end[R.n++] = lb + c1;
        }
        *(ShardRanges*)a.ranges = R;
    }
}

}  // namespace

cudaError_t launch_shard_merge_select(const ShardSelectArgs& a, cudaStream_t s) {
    shard_merge_select_kernel<<<1, kMergeThreads, 0, s>>>(a);
    return cudaGetLastError();
}

}  // namespace reattn_impl
