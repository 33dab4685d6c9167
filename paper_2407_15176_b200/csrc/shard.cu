// Sequence-sharded decode: merge of the per-rank candidate lists, vote +
// spans + global scope (redundantly on every rank), and the translation of the global
// scope table into this rank's local rows.
//
// Rank r holds [global | middle shard r | local] in its cache.  Its K1 scan yields, per
// (kv head, query), the exact top-k of its shard; top-k of the union of all ranks' lists
// under (score desc, index asc) is the exact global top-k (selection.hpp:81-135 ordering),
// so after an all-gather every rank merges identically and continues with the reference's
// vote / expand_spans / assemble_scope (selection.hpp:359-456, scope.hpp:248-272).
// Replicated rows (global, local) are attended by rank 0 only; a middle row by its owner;
// everything else is masked (kNoIndex) so partial attention states can be combined.
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
    // ---- translate to this rank's local rows (kNoIndex = not owned here) ----
    if (ssel.err != 0) return;
    const uint32_t L = ssel.L;
    for (uint32_t r = tid; r < L; r += blockDim.x) {
        const uint32_t s = a.sel.scope_src[r];
        uint32_t local;
        if (s < a.sel.g_end) {
            local = a.rank == 0 ? s : kNoIndex;
        } else if (s >= a.sel.l_start) {
            local = a.rank == 0 ? a.sel.g_end + a.shard_len + (s - a.sel.l_start) : kNoIndex;
        } else {
            const uint32_t m = s - a.sel.g_end;
            local = (m >= a.shard_begin && m < a.shard_begin + a.shard_len)
                        ? a.sel.g_end + (m - a.shard_begin)
                        : kNoIndex;
        }
        a.local_src[r] = local;
    }
}

}  // namespace

cudaError_t launch_shard_merge_select(const ShardSelectArgs& a, cudaStream_t s) {
    shard_merge_select_kernel<<<1, kMergeThreads, 0, s>>>(a);
    return cudaGetLastError();
}

}  // namespace reattn_impl
