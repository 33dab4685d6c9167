// Block-level vote + span expansion + scope table for <= 32 candidates (decode: n_kv*k).
//
// Same contract as select_kernel (select.cu), restating selection.hpp:252-349 and
// scope.hpp:37-78.  Every ranking is an all-pairs count, spread over the block as S = 8
// (256+ threads) or 4 (128 threads) threads per candidate (32/S comparisons each, then one
// redux.sync over the S), so each
// phase is a handful of shared-memory loads and one reduction; the phases are separated by
// __syncthreads_count / _or, which double as the block-wide counts the next phase needs.
// A single warp doing the same 32x32 compares with shuffles took 5-13 us (a chain of ~300
// dependent 36-cycle shuffles); this takes ~1 us.  The scope table is written span by span
// (one warp per span, coalesced) instead of a binary search per row.
#pragma once

#include "common.cuh"
#include "kernels.h"

namespace reattn_impl {

struct SmallSelectSmem {
    uint32_t idx[32], key[32];  // candidates; key = float_key(score)
    uint32_t votes[32], mk[32], rank[32];
    uint32_t sb[32], se[32];    // span of each candidate (winners only)
    uint32_t pb[32], pe[32];    // winners' spans sorted by (begin, end, vote rank)
    uint32_t b[32], off[32];    // kept spans: begin (middle coords), first scope row - g_end
    uint32_t vmask, repmask;
    uint32_t ns, cov, L, err;
};

// Sum / max / or over the S-lane group (S = 4 or 8, aligned): xor shuffles.  redux.sync
// with a partial mask compiles to a WARPSYNC.EXCLUSIVE loop over the groups, ~600 cycles
// each; three xor levels cost ~110.
__device__ __forceinline__ uint32_t grp_sum(uint32_t v, int S) {
    for (int o = S >> 1; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
    return v;
}
__device__ __forceinline__ uint32_t grp_max(uint32_t v, int S) {
    for (int o = S >> 1; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xFFFFFFFFu, v, o));
    return v;
}

// Candidates are in sm.idx / sm.key [0, 32) with validity sm.vmask, written by the caller
// before a __syncthreads.  Every thread of the block must call this (blockDim.x >= 128,
// a multiple of 32); it synchronises with __syncthreads.
__device__ __forceinline__ void small_select_scope_smem(const SmallSelectIO& io, SmallSelectSmem& sm,
                                                        uint64_t* trace = nullptr, bool dry = false) {
    using namespace reattn_dev;
    const int tid = threadIdx.x;
    const int S = blockDim.x >= 256 ? 8 : 4;  // threads per candidate
    const bool act = tid < 32 * S;
    const int i = (tid / S) & 31, s = tid & (S - 1);  // candidate i, comparison slice s
    const int NC = 32 / S;  // comparisons per thread
    const uint32_t vmask = io.k_prime > 0 ? sm.vmask : 0u;
    const bool vi = act && ((vmask >> i) & 1u);
    const uint32_t idx_i = sm.idx[i];
    // ---- tally: votes, max score, first occurrence (selection.hpp:252-268) ----
    uint32_t votes = 0, mk = 0, later = 0;
    if (vi) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            if (u >= NC) break;
            const int j = s + S * u;
            if (((vmask >> j) & 1u) && sm.idx[j] == idx_i) {
                ++votes;
                mk = max(mk, sm.key[j]);
                if (j < i) later = 1;
            }
        }
    }
    if (act) {
        votes = grp_sum(votes, S);
        mk = grp_max(mk, S);
        later = grp_max(later, S);
    }
    const bool rep = vi && !later;  // first occurrence of a distinct index
    if (act && s == 0) {
        sm.votes[i] = votes;
        sm.mk[i] = mk;
    }
    if (tid == 0) sm.repmask = 0u;
    __syncthreads();
    if (act && s == 0 && rep) atomicOr(&sm.repmask, 1u << i);
    const uint32_t U = (uint32_t)__syncthreads_count(act && s == 0 && rep);
    if (trace && tid == 0) trace[1030] = globaltimer();
    // ---- rank: votes desc, max score desc, index asc (selection.hpp:269-274) ----
    const uint32_t repmask = sm.repmask;
    uint32_t rank = 0;
    if (rep) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            if (u >= NC) break;
            const int j = s + S * u;
            const uint32_t vv = sm.votes[j], kk = sm.mk[j], ii = sm.idx[j];
            if (((repmask >> j) & 1u) &&
                (vv > votes || (vv == votes && (kk > mk || (kk == mk && ii < idx_i)))))
                ++rank;
        }
    }
    if (act) rank = grp_sum(rank, S);
    const uint32_t nw = min(io.k_prime, U);
    const bool win = rep && rank < nw;
    if (win && s == 0 && io.winners && !dry) io.winners[rank] = idx_i;
    // ---- spans (selection.hpp:318-349) ----
    const bool do_spans = io.middle_len > 0;
    uint32_t sb = 0, se = 0;
    bool bad = false;
    if (win && do_spans) {
        const uint32_t m = io.span_m;
        if (idx_i >= io.middle_len) bad = true;
        uint32_t st;
        if (io.span_mode == 0) {
            st = (idx_i / m) * m;
        } else {
            st = idx_i > m / 2 ? idx_i - m / 2 : 0u;
            if ((uint64_t)st + m > io.middle_len) st = io.middle_len > m ? io.middle_len - m : 0u;
        }
        sb = st;
        se = (uint32_t)min((uint64_t)st + m, (uint64_t)io.middle_len);
    }
    if (act && s == 0) {
        sm.rank[i] = win ? rank : 0xFFFFFFFFu;  // 0xFFFFFFFF: not a winner
        sm.sb[i] = sb;
        sm.se[i] = se;
    }
    const bool any_bad = __syncthreads_or(bad) != 0;
    if (trace && tid == 0) trace[1031] = globaltimer();
    // ---- position among the winners by (begin, end), ties by vote rank ----
    const bool sw = win && do_spans && !any_bad;
    uint32_t pos = 0;
    if (sw) {
        const unsigned long long skey = ((unsigned long long)sb << 32) | se;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            if (u >= NC) break;
            const int j = s + S * u;
            const uint32_t rj = sm.rank[j];
            const unsigned long long ok = ((unsigned long long)sm.sb[j] << 32) | sm.se[j];
            if (rj != 0xFFFFFFFFu && (ok < skey || (ok == skey && rj < rank))) ++pos;
        }
    }
    if (act) pos = grp_sum(pos, S);
    if (sw && s == 0) {
        sm.pb[pos] = sb;
        sm.pe[pos] = se;
    }
    const uint32_t nsw = (uint32_t)__syncthreads_count(act && sw && s == 0);
    if (trace && tid == 0) trace[1032] = globaltimer();
    // ---- merge / dedupe the sorted spans and lay them out (warp 0, lane = sorted span) ----
    if (tid < 32) {
        const uint32_t FULL = 0xFFFFFFFFu;
        const int l = tid;
        const bool have = (uint32_t)l < nsw;
        const uint32_t pb = have ? sm.pb[l] : 0u, pe = have ? sm.pe[l] : 0u;
        // inclusive prefix max of ends (the running group end of the centered merge)
        uint32_t pm = pe;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const uint32_t t = __shfl_up_sync(FULL, pm, off);
            if (l >= off) pm = max(pm, t);
        }
        const uint32_t prev_pm = __shfl_up_sync(FULL, pm, 1);
        const uint32_t prev_b = __shfl_up_sync(FULL, pb, 1);
        const uint32_t prev_e = __shfl_up_sync(FULL, pe, 1);
        bool keep;
        if (io.span_mode == 1)
            keep = have && (l == 0 || pb > prev_pm);  // merge overlapping/touching
        else
            keep = have && (l == 0 || pb != prev_b || pe != prev_e);  // drop duplicates
        const uint32_t kmask = __ballot_sync(FULL, keep);
        uint32_t gend = pe;
        if (io.span_mode == 1) {
            // group end = prefix max at the entry before the next kept entry
            const uint32_t nxt = kmask & ~((2u << l) - 1u);
            const int last_member = nxt ? (__ffs(nxt) - 2) : (int)nsw - 1;
            gend = __shfl_sync(FULL, pm, max(last_member, 0));
        }
        const uint32_t ns = __popc(kmask);
        const uint32_t outp = __popc(kmask & ((1u << l) - 1u));
        const uint32_t len = keep ? gend - pb : 0u;
        uint32_t ex = len;  // inclusive scan of kept lengths (kept order == lane order)
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const uint32_t t = __shfl_up_sync(FULL, ex, off);
            if (l >= off) ex += t;
        }
        const uint32_t cov = __shfl_sync(FULL, ex, 31);
        ex -= len;
        if (keep) {
            sm.b[outp] = pb;
            sm.off[outp] = ex;
            if (io.span_b && !dry) io.span_b[outp] = pb;
            if (io.span_e && !dry) io.span_e[outp] = gend;
        }
        if (l == 0) {
            uint32_t err = any_bad ? (uint32_t)kScopeErrWinnerRange : 0u;
            const uint64_t L = (uint64_t)io.g_end + cov + (io.total - io.l_start);
            if (err == 0 && L > io.window) err = kScopeErrWindow;
            if (err == 0 && io.n_q > L) err = kScopeErrQueryLong;
            sm.ns = any_bad ? 0u : ns;
            sm.cov = any_bad ? 0u : cov;
            sm.L = (uint32_t)L;
            sm.err = err;
            if (io.hdr && !dry) {
                ScopeHeader h;
                h.L = (uint32_t)L;
                h.n_spans = sm.ns;
                h.coverage = sm.cov;
                h.n_winners = nw;
                h.error = (int32_t)err;
                h.pad[0] = h.pad[1] = h.pad[2] = 0;
                *io.hdr = h;
            }
            if (trace) {
                trace[1029] = globaltimer();
                trace[1041] = clock64();
            }
        }
    }
    __syncthreads();
    // ---- scope table: global ++ spans ++ local (scope.hpp:54-61) ----
    // dry (instruction-cache warming, see scan_topk.cu): the same loops over few rows, stores
    // predicated off
    if ((sm.err == 0 || dry) && io.scope_src) {
        const uint32_t g = io.g_end, cov = sm.cov, ns = min(sm.ns, 32u);
        const uint32_t L = dry ? min(sm.L, g + cov + 64u) : sm.L;
        RA_ASSERT(dry || L <= io.window);
        const uint32_t nthr = blockDim.x, warp = (uint32_t)tid >> 5, lane = (uint32_t)tid & 31u;
        for (uint32_t r = tid; r < g; r += nthr)
            if (!dry) io.scope_src[r] = r;
        for (uint32_t sp = warp; sp < ns; sp += nthr >> 5) {
            const uint32_t o = sm.off[sp], e0 = sp + 1 < ns ? sm.off[sp + 1] : cov;
            const uint32_t e = dry ? min(e0, o + 32u) : e0;
            const uint32_t src0 = g + sm.b[sp];
            RA_ASSERT(dry || sm.b[sp] + (e0 - o) <= io.middle_len);
            for (uint32_t j = o + lane; j < e; j += 32)
                if (!dry) io.scope_src[g + j] = src0 + (j - o);
        }
        // local rows: 16-byte stores (when the table is 16-byte aligned) between scalar ends
        const uint32_t l0 = min(g + cov, L);
        if (!io.table_local) return;
        const bool al = ((uintptr_t)io.scope_src & 15u) == 0;
        const uint32_t v0 = al ? min(L, (l0 + 3u) & ~3u) : L, v1 = max(v0, L & ~3u);
        for (uint32_t r = l0 + tid; r < v0; r += nthr)
            if (!dry) io.scope_src[r] = io.l_start + (r - l0);
        for (uint32_t r = v1 + tid; r < L; r += nthr)
            if (!dry) io.scope_src[r] = io.l_start + (r - l0);
        for (uint32_t r = v0 + 4u * tid; r < v1; r += 4u * nthr) {
            const uint32_t x = io.l_start + (r - l0);
            if (!dry) *reinterpret_cast<uint4*>(io.scope_src + r) = make_uint4(x, x + 1, x + 2, x + 3);
        }
    }
}

// Per-thread interface: candidate i is passed by thread i (< 32) in (c_idx, c_score,
// c_valid).  Every thread of the block must call it.
__device__ __forceinline__ void small_select_scope(const SmallSelectIO& io, uint32_t c_idx,
                                                   float c_score, bool c_valid,
                                                   SmallSelectSmem& sm, uint64_t* trace = nullptr) {
    using namespace reattn_dev;
    const int tid = threadIdx.x;
    if (tid < 32) {
        sm.idx[tid] = c_valid ? c_idx : 0xFFFFFFFFu;
        sm.key[tid] = c_valid ? float_key(c_score) : 0u;
        const uint32_t vm = __ballot_sync(0xFFFFFFFFu, c_valid);
        if (tid == 0) sm.vmask = vm;
    }
    __syncthreads();
    small_select_scope_smem(io, sm, trace);
}

}  // namespace reattn_impl
