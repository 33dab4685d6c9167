// Warp-level vote + span expansion + scope table for <= 32 candidates (decode: n_kv*k).
//
// Same contract as select_kernel (select.cu), restating selection.hpp:359-456 and
// scope.hpp:248-289, but every ranking is an all-pairs count over shuffles in one warp
// (32x32 compares) instead of block-wide bitonic sorts, so it costs a few hundred cycles.
// Used by the select kernel's small path and fused into the K-scan's last CTA.  The 32-way
// shuffle loops are unrolled so their shuffles pipeline (rolled, each iteration waited on
// its own shuffle latency: ~10 us in the scan's tail).
#pragma once

#include "common.cuh"
#include "kernels.h"

namespace reattn_impl {

// Shared scratch: 32 span begins, 32 span offsets, 4 scalars.
struct SmallSelectSmem {
    uint32_t b[32];
    uint32_t off[32];
    uint32_t ns, cov, L, err;
};

// Must be called by every thread of the block (it synchronises with __syncthreads).
// Candidates (n <= 32) are passed by warp 0 lane i in (c_idx, c_score, c_valid).
__device__ __forceinline__ void small_select_scope(const SmallSelectIO& io, uint32_t c_idx,
                                                   float c_score, bool c_valid,
                                                   SmallSelectSmem& sm) {
    using namespace reattn_dev;
    const int tid = threadIdx.x;
    if (tid < 32) {
        // warp 0 is converged here: lets the compiler emit plain SHFLs instead of the
        // collective fallback it needs for shuffles in a possibly divergent region
        __syncwarp();
        const int i = tid;
        const uint32_t FULL = 0xFFFFFFFFu;
        const bool valid = c_valid && io.k_prime > 0;
        const uint32_t idx = valid ? c_idx : 0xFFFFFFFFu;
        const uint32_t key = valid ? float_key(c_score) : 0u;
        // ---- tally: votes and max score per distinct index (selection.hpp:359-375) ----
        uint32_t votes = 0, mk = 0;
        bool first = valid;
        for (int j = 0; j < 32; ++j) {
            const uint32_t oj = __shfl_sync(FULL, idx, j);
            const uint32_t ok = __shfl_sync(FULL, key, j);
            const bool ov = __shfl_sync(FULL, valid, j);
            if (valid && ov && oj == idx) {
                ++votes;
                mk = max(mk, ok);
                if (j < i) first = false;
            }
        }
        // ---- rank: votes desc, max score desc, index asc (selection.hpp:376-381) ----
        const bool rep = valid && first;
        uint32_t rank = 0;
        for (int j = 0; j < 32; ++j) {
            const bool rv = __shfl_sync(FULL, rep, j);
            const uint32_t vv = __shfl_sync(FULL, votes, j);
            const uint32_t kk = __shfl_sync(FULL, mk, j);
            const uint32_t ii = __shfl_sync(FULL, idx, j);
            if (rep && rv && (vv > votes || (vv == votes && (kk > mk || (kk == mk && ii < idx)))))
                ++rank;
        }
        const uint32_t U = __popc(__ballot_sync(FULL, rep));
        const uint32_t nw = min(io.k_prime, U);
        const bool win = rep && rank < nw;
        if (win && io.winners) io.winners[rank] = idx;
        // ---- spans (selection.hpp:425-456) ----
        uint32_t sb = 0, se = 0;
        bool bad = false;
        const bool do_spans = io.middle_len > 0;
        if (win && do_spans) {
            const uint32_t m = io.span_m;
            if (idx >= io.middle_len) bad = true;
            uint32_t st;
            if (io.span_mode == 0) {
                st = (idx / m) * m;
            } else {
                st = idx > m / 2 ? idx - m / 2 : 0u;
                if ((uint64_t)st + m > io.middle_len) st = io.middle_len > m ? io.middle_len - m : 0u;
            }
            sb = st;
            se = (uint32_t)min((uint64_t)st + m, (uint64_t)io.middle_len);
        }
        const bool any_bad = __any_sync(FULL, bad);
        const bool sw = win && do_spans && !any_bad;
        const unsigned long long skey = sw ? (((unsigned long long)sb << 32) | se) : ~0ull;
        // sorted position among winners by (begin, end), ties by vote rank
        uint32_t pos = 0;
        for (int j = 0; j < 32; ++j) {
            const bool ow = __shfl_sync(FULL, sw, j);
            const unsigned long long ok = __shfl_sync(FULL, skey, j);
            const uint32_t orank = __shfl_sync(FULL, rank, j);
            if (sw && ow && (ok < skey || (ok == skey && orank < rank))) ++pos;
        }
        // gather the sorted list into lane order: lane p holds the p-th smallest span
        const uint32_t nsw = __popc(__ballot_sync(FULL, sw));
        uint32_t pb = 0, pe = 0;
        for (int j = 0; j < 32; ++j) {
            const bool ow = __shfl_sync(FULL, sw, j);
            const uint32_t op = __shfl_sync(FULL, pos, j);
            const uint32_t ob = __shfl_sync(FULL, sb, j);
            const uint32_t oe = __shfl_sync(FULL, se, j);
            if (ow && op == (uint32_t)i) {
                pb = ob;
                pe = oe;
            }
        }
        const bool have = (uint32_t)i < nsw;
        // inclusive prefix max of ends (the running group end of the centered merge)
        uint32_t pm = have ? pe : 0u;
        for (int off = 1; off < 32; off <<= 1) {
            const uint32_t t = __shfl_up_sync(FULL, pm, off);
            if (i >= off) pm = max(pm, t);
        }
        const uint32_t prev_pm = __shfl_up_sync(FULL, pm, 1);
        const uint32_t prev_b = __shfl_up_sync(FULL, pb, 1);
        const uint32_t prev_e = __shfl_up_sync(FULL, pe, 1);
        bool keep;
        if (io.span_mode == 1)
            keep = have && (i == 0 || pb > prev_pm);  // merge overlapping/touching
        else
            keep = have && (i == 0 || pb != prev_b || pe != prev_e);  // drop duplicates
        const uint32_t kmask = __ballot_sync(FULL, keep);
        uint32_t gend = pe;
        if (io.span_mode == 1) {
            // group end = prefix max at the entry before the next kept entry
            const uint32_t later = kmask & ~((2u << i) - 1u);
            const int last_member = later ? (__ffs(later) - 2) : (int)nsw - 1;
            gend = __shfl_sync(FULL, pm, max(last_member, 0));
        }
        const uint32_t ns = __popc(kmask);
        const uint32_t outp = __popc(kmask & ((1u << i) - 1u));
        const uint32_t len = keep ? gend - pb : 0u;
        uint32_t ex = len;  // exclusive scan of kept lengths (in kept order == lane order)
        for (int off = 1; off < 32; off <<= 1) {
            const uint32_t t = __shfl_up_sync(FULL, ex, off);
            if (i >= off) ex += t;
        }
        const uint32_t cov = __shfl_sync(FULL, ex, 31);
        ex -= len;
        if (keep) {
            sm.b[outp] = pb;
            sm.off[outp] = ex;
            if (io.span_b) io.span_b[outp] = pb;
            if (io.span_e) io.span_e[outp] = gend;
        }
        if (i == 0) {
            uint32_t err = any_bad ? (uint32_t)kScopeErrWinnerRange : 0u;
            const uint64_t L = (uint64_t)io.g_end + cov + (io.total - io.l_start);
            if (err == 0 && L > io.window) err = kScopeErrWindow;
            if (err == 0 && io.n_q > L) err = kScopeErrQueryLong;
            sm.ns = any_bad ? 0u : ns;
            sm.cov = any_bad ? 0u : cov;
            sm.L = (uint32_t)L;
            sm.err = err;
            if (io.hdr) {
                ScopeHeader h;
                h.L = (uint32_t)L;
                h.n_spans = sm.ns;
                h.coverage = sm.cov;
                h.n_winners = nw;
                h.error = (int32_t)err;
                h.pad[0] = h.pad[1] = h.pad[2] = 0;
                *io.hdr = h;
            }
        }
    }
    __syncthreads();
    // ---- scope table: global ++ spans ++ local (scope.hpp:265-272) ----
    if (sm.err == 0 && io.scope_src) {
        const uint32_t g = io.g_end, cov = sm.cov, ns = sm.ns, L = sm.L;
        for (uint32_t r = tid; r < L; r += blockDim.x) {
            uint32_t src;
            if (r < g) {
                src = r;
            } else if (r < g + cov) {
                const uint32_t o = r - g;
                int lo = 0, hi = (int)ns - 1;
                while (lo < hi) {
                    const int mid = (lo + hi + 1) >> 1;
                    if (sm.off[mid] <= o) lo = mid;
                    else hi = mid - 1;
                }
                src = g + sm.b[lo] + (o - sm.off[lo]);
            } else {
                src = io.l_start + (r - g - cov);
            }
            io.scope_src[r] = src;
        }
    }
}

}  // namespace reattn_impl
