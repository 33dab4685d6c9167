// K2 — prefill score scan on the 5th-gen tensor cores (tcgen05 + TMEM), fused exact top-k.
//
// Same contract as fused_topk_scores (reference selection.hpp:168-248) for a prefill chunk
// (n_q up to l_chunk = 4096 queries): per (kv head, query) the top-k of mq · k over the
// middle, ties to the lower index -- with the reference's own fp32 scores, bit for bit.
//
//   1. S_hi[q, j] = hi(mq)[q, :] · K[j, :] on tcgen05.mma (kind::f16: bf16 operands, fp32
//      accumulators in TMEM; 128 queries x 128 keys per tile, d = 128), ONE pass.  mq is the
//      exact fp32 group mean (selection.hpp:143-151), hi(mq) its bf16 rounding.
//   2. Error bound per query row: |dot_f32(mq, k_j) - S_hi[j]| < delta :=
//      (||mq - hi(mq)||_1 + 2^-12 ||mq||_1) * max|k|.  The first term is the exact rounding
//      residual of the operand; 2^-12 covers both fp32 accumulations (the reference's 8-lane
//      dot: <= ~20 * 2^-24, the tensor core's 128-term sum: assumed <= 2^-13) with margin.
//   3. Epilogue (streaming): each (row, column half) keeps the top L = KT + 8 keys by S_hi
//      and admits a key only if S_hi > (its KT-th best S_hi) - 2 delta.  A key that is
//      admitted but falls off the list raises `dropped` (the largest S_hi ever dropped).
//   4. prefill_exact_merge_kernel (one warp per (kv head, query)): T = k-th best S_hi over all
//      key-range parts; every key of the exact top-k has S_hi > T - 2 delta (the k keys
//      with S_hi >= T score exactly >= T - delta).  Listed keys in that window are re-scored
//      with the reference's own dot_f32 (dense_matrix.hpp:41-56: 8 lanes over elements
//      j, j+8, ..., fixed tree; unfused or FMA lanes) -- about k + epsilon dots per query --
//      and a part whose `dropped` reaches the window (near-ties: more than L - KT keys
//      within 2 delta of the k-th best; ~1e-6 of rows at L = KT + 8, ~2% at KT + 4) is
//      re-scanned exactly.  Selected indices and scores are therefore identical to the
//      reference (tests/test_prefill_tc.py compares bitwise) while the tensor cores run the
//      score GEMM once and the streaming epilogue does no exact math.
//
// Warp roles (576 threads, 1 CTA/SM):
//   warp 0  TMA producer: the CTA's two hi(mq) tiles once, then K tiles (4-stage ring of 32 KB)
//   warp 1  TMEM allocator (512 columns = 2 pairs x 2 query tiles x 128) + single-thread MMA
//           issue: every K tile feeds BOTH query tiles (M = 256 per K tile), halving the K
//           feed per FLOP; the MMA commit releases the K stage and the accumulator pair
//   warps 2-17  epilogue, four per TMEM lane quarter (column half x query tile): two
//           tcgen05.ld 32x32b.x32, 8 group maxes against the admission limit, a warp vote,
//           rare per-column list inserts, release the accumulator pair.  The limit is kept
//           in a register and recomputed only when an input changes (an insert, the other
//           half's KT-th best, the board): round 2 cut the common path from ~244 to ~118
//           instructions per tile and warp (2.50 -> 2.33 ms per config-3 chunk).  Tried and
//           dropped: releasing the accumulator right after the loads with a one-group
//           shared-memory stash for the inserts (2.86 ms: the stash bookkeeping spilled).
//   Measured (config 3 chunk, incl. ~0.19 ms prep/kmax/merge): 2.50 ms (0.53 of the bf16
//   burst) in round 1, 2.33 ms (0.57) in round 2, vs 2.67 ms with one query tile per CTA.  Ablations (REATTN_K2_NULL_EPILOGUE /
//   REATTN_K2_NO_MMA): epilogue ablated 1.69 ms (was 1.96), feed alone 0.63 ms (was 0.85);
//   the MMA alone dispatches 128x128x16 in 64 cycles (tools/micro/mma_rate.cu).  The two
//   query tiles made the feed no longer the bound; the epilogue's admissions now are.
// Grid: (query-tile pair, kv head, key split): the key range of each pair is cut into
// `splits` contiguous parts chosen to fill whole waves; the exact merge reduces them.
#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"
#include "tcgen05.cuh"

using namespace reattn_dev;

namespace reattn_impl {

namespace {

constexpr int kPM = 128;  // queries per CTA = UMMA M
constexpr int kPN = 128;  // keys per tile = UMMA N
constexpr int kPD = 128;  // head dim
constexpr int kPQT = 2;     // query tiles per CTA: every K tile feeds M = 256 queries
constexpr int kPStages = 4;
constexpr int kPPairs = 2;  // TMEM: kPPairs x kPQT accumulators of kPN columns = 512
constexpr int kPQBytes = kPM * kPD * 2;  // hi(mq) tile: 32 KB
constexpr int kPKBytes = kPN * kPD * 2;  // one K stage: 32 KB
constexpr int kPEpi = 16;                // epilogue warps: (lane quarter, column half, query tile)
constexpr int kPThreads = (2 + kPEpi) * 32;  // producer, MMA, epilogue
constexpr int kPKMax = 8;                // largest k
constexpr int kPExtra = 8;               // list slots beyond KT (near-tie margin)
constexpr int kPL = 16;                  // part-list stride (>= kPKMax + kPExtra)
constexpr int kPMaxSplits = 8;
constexpr float kPAccumCoef = 0.000244140625f;  // 2^-12
constexpr size_t kPSmem = 1024 + kPQT * kPQBytes + kPStages * kPKBytes + 256 + kPQT * 2 * kPM * 4;
static_assert(kPStages * kPKBytes >= kPQT * kPM * (kPL * 8 + 4), "half-merge lists reuse the K ring");

struct PrefillArgs {
    int n_q, n_qpad, n_kv, k;
    uint32_t count;
    uint64_t head_stride, row0;
    int tiles;              // key tiles of the whole middle
    int splits;             // key-range parts per query tile (gridDim.z)
    const float* dl;        // [n_kv][n_qpad] delta / max|k|
    const unsigned* kmax;   // [n_kv] max |k| over the middle (float bits)
    unsigned* board;        // [n_kv][n_qpad] best published KT-th S_hi (ordered bits, 0 = none)
    const __nv_bfloat16* qhi;  // [n_kv][n_qpad][128] hi(mq), the MMA's A operand
    int null_epilogue;         // ablation (REATTN_K2_NULL_EPILOGUE): load + release only
    int no_mma;                // ablation (REATTN_K2_NO_MMA): the K-tile feed alone
    int no_insert;             // ablation (REATTN_K2_NO_INSERT): admission test, no list work
    uint32_t* part_idx;     // [splits][n_kv][n_qpad][kPL], sorted by better(), kNoIndex-padded
    float* part_score;      // S_hi of those keys
    float* part_dropped;    // [splits][n_kv][n_qpad]
};

constexpr uint32_t prefill_idesc() { return idesc_bf16_f32<kPM, kPN>(); }

// Insert (cs, ci) into the descending list ts/ti, given cs > ts[N-1].  One thread sees its
// candidates in increasing key order, so an equal score never displaces an entry and
// better() reduces to a strict >.  All compares use the original list: branch-free shift.
template <int N>
__device__ __forceinline__ void insert_in_order(float (&ts)[N], uint32_t (&ti)[N], float cs,
                                                uint32_t ci) {
#pragma unroll
    for (int j = N - 1; j >= 0; --j) {
        const bool here = cs > ts[j];
        const bool above = j > 0 && cs > ts[j > 0 ? j - 1 : 0];
        if (here) {
            ts[j] = above ? ts[j - (j > 0)] : cs;
            ti[j] = above ? ti[j - (j > 0)] : ci;
        }
    }
}

// nextafterf(x, -inf) for the admission limit's values (finite or -inf), without the
// library call's NaN / denormal branches
__device__ __forceinline__ float next_down(float x) {
    const uint32_t u = __float_as_uint(x);
    if (x == 0.0f) return __uint_as_float(0x80000001u);  // -denorm_min, from +0 and -0
    return __uint_as_float(x > 0.0f ? u - 1u : (x == -INFINITY ? u : u + 1u));
}

// float <-> unsigned with the same order (for atomicMax); 0 encodes "nothing published"
__device__ __forceinline__ unsigned ord_enc(float f) {
    const unsigned b = __float_as_uint(f);
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float ord_dec(unsigned u) {
    if (u == 0u) return -INFINITY;
    return __uint_as_float((u & 0x80000000u) ? (u & 0x7FFFFFFFu) : ~u);
}

// KT-th largest of 8 values (KT <= 8): a lower bound of the KT-th largest of the 64 columns
// they are the group maxima of
template <int KT>
__device__ __forceinline__ float kth_of_8(const float (&g)[8]) {
    float h[KT];
#pragma unroll
    for (int j = 0; j < KT; ++j) h[j] = -INFINITY;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
        float v = g[c];
#pragma unroll
        for (int j = 0; j < KT; ++j) {
            const float hi_ = fmaxf(h[j], v);
            v = fminf(h[j], v);
            h[j] = hi_;
        }
    }
    return h[KT - 1];
}

template <int KT>
__global__ void __launch_bounds__(kPThreads, 1)
    prefill_scan_tc_kernel(const __grid_constant__ CUtensorMap q_map,
                           const __grid_constant__ CUtensorMap k_map, const PrefillArgs a) {
    constexpr int L = KT + kPExtra;
    extern __shared__ uint8_t psm_raw[];
    uint8_t* sm = (uint8_t*)(((uintptr_t)psm_raw + 1023) & ~(uintptr_t)1023);
    uint8_t* s_q = sm;                                   // kPQT hi(mq) tiles, SW128
    uint8_t* s_k = sm + kPQT * kPQBytes;                 // K ring
    uint64_t* bars = (uint64_t*)(s_k + kPStages * kPKBytes);
    uint64_t* q_full = bars;
    uint64_t* full = bars + 1;
    uint64_t* empty = full + kPStages;
    // per (pair, query tile): the MMA and the two query tiles' epilogue warps run as two
    // independent pipelines over the shared K stages, so a slow warp of one query tile does
    // not hold back the other's next accumulator
    uint64_t* tfull = empty + kPStages;   // [kPPairs][kPQT]: accumulator ready
    uint64_t* tempty = tfull + kPPairs * kPQT;
    uint32_t* s_tmem = (uint32_t*)(tempty + kPPairs * kPQT);
    float* s_thr = (float*)((uint8_t*)bars + 256);  // [kPQT][2 halves][128] KT-th best S_hi
    uint8_t* aux = s_k;  // half-merge lists, after the tile loop (the K ring is idle then)

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int qtile = blockIdx.x, kv = blockIdx.y, split = blockIdx.z;  // qtile: pair index
    const int t_first = (int)((int64_t)split * a.tiles / a.splits);
    const int n_tiles = (int)((int64_t)(split + 1) * a.tiles / a.splits) - t_first;

    if (warp == 1) tmem_alloc(s_tmem, 512);
    for (int i = tid; i < kPQT * 2 * kPM; i += kPThreads) s_thr[i] = -INFINITY;
    if (tid == 0) {
        mbar_init(q_full, 1);
        for (int s = 0; s < kPStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);  // MMA commit: the stage has been read
        }
        for (int b = 0; b < kPPairs * kPQT; ++b) {
            mbar_init(&tfull[b], 1);
            mbar_init(&tempty[b], kPEpi * 32 / kPQT);
        }
        fence_barrier_init();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *s_tmem;

    if (warp == 0) {
        if (lane == 0) {  // ===== TMA producer =====
            prefetch_tensormap(&q_map);
            prefetch_tensormap(&k_map);
            const uint64_t pol = policy_evict_first();
            const uint64_t keep = policy_evict_last();  // K tiles: re-read by every query tile
            mbar_arrive_expect_tx(q_full, kPQT * kPQBytes);
#pragma unroll
            for (int qt = 0; qt < kPQT; ++qt) {
                const int32_t qrow = (int32_t)(kv * a.n_qpad + (qtile * kPQT + qt) * kPM);
                tma_load_2d(s_q + qt * kPQBytes, &q_map, 0, qrow, q_full, pol);
                tma_load_2d(s_q + qt * kPQBytes + kPQBytes / 2, &q_map, 64, qrow, q_full, pol);
            }
            for (int t = 0; t < n_tiles; ++t) {
                const int s = t % kPStages;
                const uint32_t ph = (t / kPStages) & 1u;
                if (t >= kPStages) mbar_wait(&empty[s], ph ^ 1u);
                const int32_t krow =
                    (int32_t)(kv * a.head_stride + a.row0 + (uint64_t)(t_first + t) * kPN);
                mbar_arrive_expect_tx(&full[s], kPKBytes);
                uint8_t* dst = s_k + (size_t)s * kPKBytes;
                tma_load_2d(dst, &k_map, 0, krow, &full[s], keep);
                tma_load_2d(dst + kPKBytes / 2, &k_map, 64, krow, &full[s], keep);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {  // ===== MMA issuer: S_hi = hi(mq) · K^T for both query tiles =====
            const uint32_t idesc = prefill_idesc();
            mbar_wait(q_full, 0);
            tc_fence_after();
            const uint32_t q0 = smem_u32(s_q);
            for (int t = 0; t < n_tiles; ++t) {
                const int s = t % kPStages;
                const uint32_t ph = (t / kPStages) & 1u;
                const int p = t % kPPairs;
                const uint32_t pph = (t / kPPairs) & 1u;
                mbar_wait(&full[s], ph);
                const uint32_t kbase = smem_u32(s_k + (size_t)s * kPKBytes);
#pragma unroll
                for (int qt = 0; qt < kPQT; ++qt) {
                    if (t >= kPPairs) mbar_wait(&tempty[p * kPQT + qt], pph ^ 1u);
                    tc_fence_after();
                    if (!a.no_mma) {
                        const uint32_t d_tmem = tmem + (uint32_t)((p * kPQT + qt) * kPN);
#pragma unroll
                        for (int kb = 0; kb < 2; ++kb)
#pragma unroll
                            for (int ks = 0; ks < 4; ++ks) {
                                const uint64_t ad = umma_desc_sw128(q0 + qt * kPQBytes + kb * (kPQBytes / 2) + ks * 32);
                                const uint64_t bd = umma_desc_sw128(kbase + kb * (kPKBytes / 2) + ks * 32);
                                mma_bf16_ss(d_tmem, ad, bd, idesc, (kb | ks) ? 1u : 0u);
                            }
                    }
                    mma_commit(&tfull[p * kPQT + qt]);  // this query tile's accumulator is ready
                }
                mma_commit(&empty[s]);  // K stage consumed (both query tiles' MMAs)
            }
        }
    } else {
        // ===== epilogue: 16 warps, four per TMEM lane quarter: warp (quarter, half, qt) owns
        // query row quarter*32 + lane of query tile qt, for one half (64 columns) of every
        // key tile =====
        const int ew = warp - 2;          // 0..15
        const int quarter = warp & 3;     // TMEM lane quarter this warp may access
        const int half = (ew >> 2) & 1;   // column half of the 128-key tile
        const int qt = ew >> 3;           // query tile of the CTA
        const int row = quarter * 32 + lane;
        const size_t qrow = (size_t)kv * a.n_qpad + (size_t)(qtile * kPQT + qt) * kPM + row;
        const float d2 = 2.0f * a.dl[qrow] * __uint_as_float(a.kmax[kv]);  // 2 delta
        float as[L];
        uint32_t ai[L];
#pragma unroll
        for (int j = 0; j < L; ++j) {
            as[j] = -INFINITY;
            ai[j] = kNoIndex;
        }
        float dropped = -INFINITY;
        // Threshold board: every part of this row publishes its KT-th best S_hi (KT keys score
        // at least that, so it bounds the row's k-th best from below) and admits nothing at or
        // below the best published value - 2 delta.  Parts of later waves start near the final
        // threshold instead of paying k ln(n/k) admissions from -inf.
        unsigned* board = a.board + qrow;
        float tb = ord_dec(*(volatile unsigned*)board);
        float* thr_mine = s_thr + (qt * 2 + half) * kPM;
        const uint32_t thr_other = smem_u32(s_thr + (qt * 2 + (half ^ 1)) * kPM + row);
        // the limit's inputs change rarely (an insert, the other half's list, the board every
        // 32 tiles): it is recomputed only then -- the common tile is 64 columns reduced to 8
        // group maxima, one compare against the limit and a warp vote
        float other_seen = -INFINITY;
        float lim = -INFINITY;
        bool dirty = true;
        for (int t = 0; t < n_tiles; ++t) {
            if ((t & 31) == 31) {
                if (as[KT - 1] > -INFINITY) atomicMax(board, ord_enc(as[KT - 1]));
                tb = ord_dec(*(volatile unsigned*)board);
                dirty = true;
            }
            const int p = t % kPPairs;
            const uint32_t pph = (t / kPPairs) & 1u;
            mbar_wait(&tfull[p * kPQT + qt], pph);
            tc_fence_after();
            const uint32_t taddr = tmem + ((uint32_t)(quarter * 32) << 16) +
                                   (uint32_t)((p * kPQT + qt) * kPN + half * 64);
            const uint32_t key0 = (uint32_t)(t_first + t) * kPN + half * 64;
            if (a.null_epilogue) {  // ablation: the TMA / MMA / TMEM-read floor
                uint32_t r[64];
                TMEM_LD_X64(taddr, r);
                tmem_wait_ld();
                if (r[0] == 0x7FFFFFFFu && r[63] == 0x7FFFFFFFu) dropped = 1.0f;
                tc_fence_before();
                mbar_arrive(&tempty[p * kPQT + qt]);
                continue;
            }
            // 8 group maxima, 32 columns at a time (register pressure)
            float gx[8];
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
                uint32_t r[32];
                TMEM_LD_X32(taddr + 32 * hh, r);
                tmem_wait_ld();
                if (key0 + 64 > a.count) {  // tail tile: keys past the middle never qualify
#pragma unroll
                    for (int c = 0; c < 32; ++c)
                        if (key0 + 32 * hh + c >= a.count) r[c] = __float_as_uint(-INFINITY);
                }
#pragma unroll
                for (int g = 0; g < 4; ++g) {
                    float m = __uint_as_float(r[8 * g]);
#pragma unroll
                    for (int u = 1; u < 8; ++u) m = fmaxf(m, __uint_as_float(r[8 * g + u]));
                    gx[4 * hh + g] = m;
                }
            }
            // admission limit: (KT-th best S_hi so far) - 2 delta.  The other column half's
            // KT-th best is a lower bound of the row's k-th best too (any subset's is): a key
            // at or below it - 2 delta is outside the merge's window
            // (prefill_exact_merge_kernel).  Its keys are not ordered before ours, so one ulp
            // lower.  Read racily: every value ever stored is a valid bound.
            float other;
            asm volatile("ld.volatile.shared.f32 %0, [%1];" : "=f"(other) : "r"(thr_other));
            if (other != other_seen) {
                other_seen = other;
                dirty = true;
            }
            if (dirty) {
                lim = fmaxf(as[KT - 1] - d2, next_down(fmaxf(other, tb) - d2));
                dirty = false;
            }
            const float tmax = fmaxf(fmaxf(fmaxf(gx[0], gx[1]), fmaxf(gx[2], gx[3])),
                                     fmaxf(fmaxf(gx[4], gx[5]), fmaxf(gx[6], gx[7])));
            uint32_t gm = 0;  // this row's groups holding an admissible column
            float lim_t = lim;
            if (tmax > lim) {
                // Before the list holds KT keys, the KT-th largest group max of this tile
                // bounds the KT-th best from below; those keys are not listed yet, so one ulp
                // lower keeps an exact tie (delta == 0) with them admissible.
                if (as[KT - 1] == -INFINITY) lim_t = fmaxf(lim_t, next_down(kth_of_8<KT>(gx) - d2));
#pragma unroll
                for (int g = 0; g < 8; ++g) gm |= (gx[g] > lim_t ? 1u : 0u) << g;
            }
            // rare path, rolled: the warp walks the union of its rows' groups and re-reads
            // each group's 8 columns from TMEM (warp-uniform address, one row per lane)
            uint32_t ug = __reduce_or_sync(0xFFFFFFFFu, gm);
            if (a.no_insert) ug = 0u;
            if (ug) {
                const float kth0 = as[KT - 1];
                while (ug) {
                    const int g = __ffs(ug) - 1;
                    ug &= ug - 1u;
                    uint32_t v8[8];
                    tmem_ld8(taddr + (uint32_t)(8 * g), v8);
                    if ((gm >> g) & 1u) {
#pragma unroll
                        for (int u = 0; u < 8; ++u) {
                            const float v = __uint_as_float(v8[u]);
                            if (v > lim_t && key0 + (uint32_t)(8 * g + u) < a.count) {
                                if (v > as[L - 1]) {
                                    dropped = fmaxf(dropped, as[L - 1]);
                                    insert_in_order<L>(as, ai, v, key0 + (uint32_t)(8 * g + u));
                                } else {
                                    dropped = fmaxf(dropped, v);
                                }
                            }
                        }
                    }
                }
                if (as[KT - 1] != kth0) {
                    thr_mine[row] = as[KT - 1];
                    dirty = true;
                }
            }
            tc_fence_before();
            mbar_arrive(&tempty[p * kPQT + qt]);  // accumulator no longer read: the MMA warp may reuse it
        }
        // merge the two column halves of each row (disjoint key sets): top L under better(),
        // anything pushed off the end raises `dropped`.  The K ring is idle now (every MMA
        // that read it has completed: its tfull commit was waited on above); query tile qt
        // uses its own part of it.
        // every MMA has completed once both query tiles' warps have seen their last tfull:
        // only then may the K ring be overwritten
        named_bar_sync(2, kPEpi * 32);
        uint8_t* aq = aux + (size_t)qt * kPM * (kPL * 8 + 4);
        float* m_s = (float*)aq;                               // [128][L] scores
        uint32_t* m_i = (uint32_t*)(aq + kPM * kPL * 4);       // [128][L] indices
        float* m_d = (float*)(aq + kPM * kPL * 8);             // [128] dropped
        if (half == 1) {
#pragma unroll
            for (int j = 0; j < L; ++j) {
                m_s[row * kPL + j] = as[j];
                m_i[row * kPL + j] = ai[j];
            }
            m_d[row] = dropped;
        }
        named_bar_sync(1, kPEpi * 32);
        if (half == 0) {
            dropped = fmaxf(dropped, m_d[row]);
#pragma unroll
            for (int jj = 0; jj < L; ++jj) {
                float cs = m_s[row * kPL + jj];
                uint32_t ci = m_i[row * kPL + jj];
                if (ci == kNoIndex) continue;
#pragma unroll
                for (int j = 0; j < L; ++j) {
                    if (better(cs, ci, as[j], ai[j])) {
                        const float tt = as[j];
                        const uint32_t uu = ai[j];
                        as[j] = cs;
                        ai[j] = ci;
                        cs = tt;
                        ci = uu;
                    }
                }
                if (ci != kNoIndex) dropped = fmaxf(dropped, cs);
            }
            const size_t prow = (size_t)split * a.n_kv * a.n_qpad + qrow;
            uint32_t* pi = a.part_idx + prow * kPL;
            float* ps = a.part_score + prow * kPL;
#pragma unroll
            for (int j = 0; j < kPL; ++j) {
                pi[j] = j < L ? ai[j] : kNoIndex;
                ps[j] = j < L ? as[j] : -INFINITY;
            }
            a.part_dropped[prow] = dropped;
            if (as[KT - 1] > -INFINITY) atomicMax(board, ord_enc(as[KT - 1]));
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

// group-mean query (selection.hpp:143-151, exact fp32): the fp32 row, its bf16 rounding (the
// MMA operand) and delta / max|k| = ||mq - hi||_1 + 2^-12 ||mq||_1 per row (one warp per row)
__global__ void prefill_prep_kernel(const float* q, int n_q, int n_heads, int n_kv, int n_qpad,
                                    __nv_bfloat16* hi, float* mq, float* dl) {
    const int group = n_heads / n_kv;
    const float inv = __fdiv_rn(1.0f, (float)group);
    const int lane = threadIdx.x & 31;
    const size_t rows = (size_t)n_kv * n_qpad;
    for (size_t rq = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) / 32; rq < rows;
         rq += (size_t)gridDim.x * blockDim.x / 32) {
        const int qi = (int)(rq % n_qpad), kv = (int)(rq / n_qpad);
        float s1 = 0.0f, se = 0.0f;
        for (int c = lane; c < kPD; c += 32) {
            float m = 0.0f;
            if (qi < n_q) {
                float acc = 0.0f;
                for (int g = 0; g < group; ++g)
                    acc = __fadd_rn(acc, q[(size_t)qi * n_heads * kPD + (size_t)(kv * group + g) * kPD + c]);
                m = __fmul_rn(acc, inv);
            }
            const __nv_bfloat16 h = __float2bfloat16_rn(m);
            mq[rq * kPD + c] = m;
            hi[rq * kPD + c] = h;
            s1 += fabsf(m);
            se += fabsf(m - __bfloat162float(h));  // exact: m and h share the exponent range
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            s1 += __shfl_xor_sync(0xFFFFFFFFu, s1, off);
            se += __shfl_xor_sync(0xFFFFFFFFu, se, off);
        }
        // 1.001: the rounding of these sums themselves
        if (lane == 0) dl[rq] = (se + kPAccumCoef * s1) * 1.001f;
    }
}

// max |k| over the middle rows of each kv head (float bits: non-negative floats order as
// unsigned integers); out must be zeroed before the launch
__global__ void prefill_kmax_kernel(const __nv_bfloat16* keys, uint64_t head_stride, uint64_t row0,
                                    uint32_t count, int n_kv, unsigned* out) {
    const int kv = blockIdx.y;
    const uint4* base = reinterpret_cast<const uint4*>(keys + ((size_t)kv * head_stride + row0) * kPD);
    const size_t n = (size_t)count * kPD / 8;
    uint32_t mx = 0;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
         i += (size_t)gridDim.x * blockDim.x) {
        const uint4 w = __ldg(base + i);
        const uint32_t u[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            mx = max(mx, (u[j] << 16) & 0x7FFFFFFFu);           // |low bf16| as float bits
            mx = max(mx, u[j] & 0x7FFF0000u);                    // |high bf16|
        }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) mx = max(mx, __shfl_xor_sync(0xFFFFFFFFu, mx, off));
    if ((threadIdx.x & 31) == 0) atomicMax(out + kv, mx);
}

struct PrefillMergeArgs {
    const uint32_t* part_idx;
    const float* part_score;
    const float* part_dropped;
    int splits, tiles, n_kv, n_q, n_qpad, k;
    uint32_t count;
    const __nv_bfloat16* keys;
    uint64_t head_stride, row0;
    const float* mq;
    const float* dl;
    const unsigned* kmax;
    uint32_t* idx_out;
    float* score_out;
    // rows whose part lists overflowed inside the window: re-scanned by prefill_rescan_kernel
    uint32_t* resc_count;  // zeroed before the merge
    uint32_t* resc_row;    // [rows] e = kv * n_q + query
    uint32_t* resc_mask;   // [rows] parts to re-scan
    float* resc_ts;        // [rows][kPKMax] the row's top-k of the other parts
    uint32_t* resc_ti;
};

// Insert (cs, ci) into the top-k list under better() (any arrival order).
template <int N>
__device__ __forceinline__ void insert_better(float (&ts)[N], uint32_t (&ti)[N], int k, float cs,
                                              uint32_t ci) {
#pragma unroll
    for (int j = 0; j < N; ++j) {
        if (j < k && better(cs, ci, ts[j], ti[j])) {
            const float tt = ts[j];
            const uint32_t uu = ti[j];
            ts[j] = cs;
            ti[j] = ci;
            cs = tt;
            ci = uu;
        }
    }
}

// Exact dot_f32 (dense_matrix.hpp:41-56) of this lane's query with key `key`, 8 lanes per
// key: lane t of the group accumulates the reference's lane t (elements t, t+8, ..., in
// order) and the fixed tree ((l0+l1)+(l2+l3))+((l4+l5)+(l6+l7)) is three xor-shuffle adds
// (IEEE addition commutes: every lane of the group ends with the same bits).
template <int LANES>
__device__ __forceinline__ float exact_dot8(const float (&qv)[16], const __nv_bfloat16* krow,
                                            bool live, int t) {
    float l = 0.0f;
    if (live) {
        float kf[16];
#pragma unroll
        for (int c = 0; c < 16; ++c) kf[c] = __bfloat162float(krow[t + 8 * c]);
#pragma unroll
        for (int c = 0; c < 16; ++c) {
            if (LANES == kLanesFma)
                l = __fmaf_rn(qv[c], kf[c], l);
            else
                l = __fadd_rn(l, __fmul_rn(qv[c], kf[c]));
        }
    }
    float s = __fadd_rn(l, __shfl_xor_sync(0xFFFFFFFFu, l, 1));
    s = __fadd_rn(s, __shfl_xor_sync(0xFFFFFFFFu, s, 2));
    s = __fadd_rn(s, __shfl_xor_sync(0xFFFFFFFFu, s, 4));
    return s;
}

// Exact dot_f32 of a whole key row by ONE thread (the re-scan path: lane = key): element
// block c (16 bytes of the row) holds the c-th element of each of the reference's 8 lanes,
// l_t += q[8c + t] * k[8c + t] in order, then the fixed tree -- the same bits as exact_dot8.
template <int LANES>
__device__ __forceinline__ float exact_dot_row(const float* __restrict__ sq, const __nv_bfloat16* krow) {
    float l[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    const uint4* k4 = reinterpret_cast<const uint4*>(krow);
#pragma unroll 4
    for (int c = 0; c < kPD / 8; ++c) {
        const uint4 w = __ldg(k4 + c);
        const float4 qa = reinterpret_cast<const float4*>(sq + 8 * c)[0];
        const float4 qb = reinterpret_cast<const float4*>(sq + 8 * c)[1];
        const float kf[8] = {__uint_as_float(w.x << 16), __uint_as_float(w.x & 0xFFFF0000u),
                             __uint_as_float(w.y << 16), __uint_as_float(w.y & 0xFFFF0000u),
                             __uint_as_float(w.z << 16), __uint_as_float(w.z & 0xFFFF0000u),
                             __uint_as_float(w.w << 16), __uint_as_float(w.w & 0xFFFF0000u)};
        const float qf[8] = {qa.x, qa.y, qa.z, qa.w, qb.x, qb.y, qb.z, qb.w};
#pragma unroll
        for (int t = 0; t < 8; ++t)
            l[t] = LANES == kLanesFma ? __fmaf_rn(qf[t], kf[t], l[t]) : __fadd_rn(l[t], __fmul_rn(qf[t], kf[t]));
    }
    return __fadd_rn(__fadd_rn(__fadd_rn(l[0], l[1]), __fadd_rn(l[2], l[3])),
                     __fadd_rn(__fadd_rn(l[4], l[5]), __fadd_rn(l[6], l[7])));
}

// One warp per (kv head, query): T = k-th best S_hi over the parts' lists, exact re-scoring
// of the listed keys with S_hi >= T - 2 delta, exact re-scan of any part whose dropped S_hi
// reaches that window, exact top-k of the union (every lane holds the same list).
template <int LANES, int KT>
__global__ void __launch_bounds__(256, 4) prefill_exact_merge_kernel(const PrefillMergeArgs m) {
    __shared__ float s_sc[8][kPMaxSplits * kPL];
    __shared__ uint32_t s_ix[8][kPMaxSplits * kPL];
    const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int e = blockIdx.x * 8 + wib;
    if (e >= m.n_kv * m.n_q) return;
    {
    const int kv = e / m.n_q, query = e % m.n_q;
    const size_t qrow = (size_t)kv * m.n_qpad + query;
    const int n = m.splits * kPL;
    float* sc = s_sc[wib];
    uint32_t* ix = s_ix[wib];
    const float dsp = lane < m.splits ? m.part_dropped[(((size_t)lane * m.n_kv + kv) * m.n_qpad + query)]
                                      : -INFINITY;
    {  // every list entry's index and score loaded before any is used (no dependent load)
        constexpr int kU = kPMaxSplits * kPL / 32;
        uint32_t id[kU];
        float sv[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const int i = lane + 32 * u;
            id[u] = kNoIndex;
            sv[u] = -INFINITY;
            if (i < n) {
                const size_t o = (((size_t)(i / kPL) * m.n_kv + kv) * m.n_qpad + query) * kPL + (i % kPL);
                id[u] = m.part_idx[o];
                sv[u] = m.part_score[o];
            }
        }
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const int i = lane + 32 * u;
            if (i < n) {
                ix[i] = id[u];
                sc[i] = id[u] == kNoIndex ? -INFINITY : sv[u];
            }
        }
    }
    __syncwarp();
    // T: k rounds of "best list head" across the (sorted) part lists, lane s owns part s
    int pos = 0;
    float T = -INFINITY;
    for (int r = 0; r < m.k; ++r) {
        float bs = -INFINITY;
        uint32_t bi = kNoIndex;
        if (lane < m.splits && pos < kPL) {
            bs = sc[lane * kPL + pos];
            bi = ix[lane * kPL + pos];
        }
        int bl = lane;
#pragma unroll
        for (int off = 1; off < kPMaxSplits; off <<= 1) {
            const float os = __shfl_xor_sync(0xFFFFFFFFu, bs, off);
            const uint32_t oi = __shfl_xor_sync(0xFFFFFFFFu, bi, off);
            const int ol = __shfl_xor_sync(0xFFFFFFFFu, bl, off);
            if (oi != kNoIndex && (bi == kNoIndex || better(os, oi, bs, bi))) {
                bs = os;
                bi = oi;
                bl = ol;
            }
        }
        bs = __shfl_sync(0xFFFFFFFFu, bs, 0);
        bi = __shfl_sync(0xFFFFFFFFu, bi, 0);
        bl = __shfl_sync(0xFFFFFFFFu, bl, 0);
        if (bi == kNoIndex) {  // fewer than k listed keys: every listed key is a candidate
            T = -INFINITY;
            break;
        }
        T = bs;
        if (lane == bl) ++pos;
    }
    const float w = T - 2.0f * m.dl[qrow] * __uint_as_float(m.kmax[kv]);
    // parts to re-scan exactly (bit s = lane s; the dropped values were loaded up front)
    const uint32_t rescan = __ballot_sync(0xFFFFFFFFu, lane < m.splits && dsp > -INFINITY && dsp >= w);
    // compact the candidates (listed, S_hi >= w, part not re-scanned) to the front of ix
    int nc = 0;
    for (int i0 = 0; i0 < n; i0 += 32) {
        const int i = i0 + lane;
        const bool c = i < n && ix[i] != kNoIndex && sc[i] >= w && !((rescan >> (i / kPL)) & 1u);
        const uint32_t id = i < n ? ix[i] : kNoIndex;
        const uint32_t bal = __ballot_sync(0xFFFFFFFFu, c);
        __syncwarp();
        if (c) ix[nc + __popc(bal & ((1u << lane) - 1u))] = id;
        nc += __popc(bal);
        __syncwarp();
    }
    const int t = lane & 7, j = lane >> 3;
    float qv[16];
#pragma unroll
    for (int c = 0; c < 16; ++c) qv[c] = m.mq[qrow * kPD + t + 8 * c];
    const __nv_bfloat16* kbase = m.keys + ((size_t)kv * m.head_stride + m.row0) * kPD;
    float ts[KT];
    uint32_t ti[KT];
#pragma unroll
    for (int q = 0; q < KT; ++q) {
        ts[q] = -INFINITY;
        ti[q] = kNoIndex;
    }
    auto consume = [&](uint32_t key, bool live) {
        const float v = exact_dot8<LANES>(qv, kbase + (size_t)key * kPD, live, t);
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
            const float vj = __shfl_sync(0xFFFFFFFFu, v, 8 * jj);
            const uint32_t kj = __shfl_sync(0xFFFFFFFFu, key, 8 * jj);
            const bool lj = __shfl_sync(0xFFFFFFFFu, live, 8 * jj);
            if (lj) insert_better(ts, ti, m.k, vj, kj);
        }
    };
    for (int p = 0; p < nc; p += 4) {
        const bool live = p + j < nc;
        consume(live ? ix[p + j] : 0u, live);
    }
    if (rescan) {  // finished by prefill_rescan_kernel
        uint32_t slot = 0;
        if (lane == 0) slot = atomicAdd(m.resc_count, 1u);
        slot = __shfl_sync(0xFFFFFFFFu, slot, 0);
        if (lane == 0) {
            m.resc_row[slot] = (uint32_t)e;
            m.resc_mask[slot] = rescan;
#pragma unroll
            for (int q = 0; q < kPKMax; ++q) {
                m.resc_ts[(size_t)slot * kPKMax + q] = q < KT ? ts[q < KT ? q : 0] : -INFINITY;
                m.resc_ti[(size_t)slot * kPKMax + q] = q < KT ? ti[q < KT ? q : 0] : kNoIndex;
            }
        }
    } else if (lane == 0) {
        const size_t o = ((size_t)kv * m.n_q + query) * m.k;
#pragma unroll
        for (int q = 0; q < KT; ++q)
            if (q < m.k) {
                m.idx_out[o + q] = ti[q];
                m.score_out[o + q] = ts[q];
            }
    }
    }
}

// A part whose list overflowed inside the window (near-ties, ~1e-6 of rows) is scanned again
// exactly by all 8 warps of a CTA: 32 keys per warp step, one key row per lane (16-byte
// loads), each warp keeping the top-k of its keys; warp 0 merges them with the row's top-k of
// the other parts.  (One warp with 8 lanes per key took ~20 ms for one 60K-key part.)  A
// separate launch keeps the re-scan's registers out of the merge's occupancy; with nothing
// queued its CTAs exit at once.
template <int LANES, int KT>
__global__ void __launch_bounds__(256) prefill_rescan_kernel(const PrefillMergeArgs m) {
    __shared__ __align__(16) float s_q[kPD];
    __shared__ float s_ws[8][KT];
    __shared__ uint32_t s_wi[8][KT];
    const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t n = *(volatile const uint32_t*)m.resc_count;
#pragma unroll 1
    for (uint32_t it = blockIdx.x; it < n; it += gridDim.x) {
        const uint32_t ep = m.resc_row[it], rescan = m.resc_mask[it];
        const int kvp = (int)(ep / m.n_q), qp = (int)(ep % m.n_q);
        const size_t qrow = (size_t)kvp * m.n_qpad + qp;
        __syncthreads();  // the previous row's shared state is consumed
        for (int c = threadIdx.x; c < kPD; c += blockDim.x) s_q[c] = m.mq[qrow * kPD + c];
        __syncthreads();
        const __nv_bfloat16* kb = m.keys + ((size_t)kvp * m.head_stride + m.row0) * kPD;
        float ts[KT];
        uint32_t ti[KT];
#pragma unroll
        for (int q = 0; q < KT; ++q) {
            ts[q] = -INFINITY;
            ti[q] = kNoIndex;
        }
        for (int s = 0; s < m.splits; ++s) {
            if (!((rescan >> s) & 1u)) continue;
            const uint32_t lo = (uint32_t)((int64_t)s * m.tiles / m.splits) * kPN;
            const uint32_t hi = min(m.count, (uint32_t)((int64_t)(s + 1) * m.tiles / m.splits) * kPN);
            for (uint32_t b0 = lo + 32u * (uint32_t)wib; b0 < hi; b0 += 32u * 8u) {
                const uint32_t key = b0 + (uint32_t)lane;
                const bool live = key < hi;
                const float v = live ? exact_dot_row<LANES>(s_q, kb + (size_t)key * kPD) : -INFINITY;
                float ws = ts[KT - 1];
                uint32_t wi = ti[KT - 1];
#pragma unroll
                for (int q = 0; q < KT; ++q)
                    if (q == m.k - 1) {
                        ws = ts[q];
                        wi = ti[q];
                    }
                uint32_t cand = __ballot_sync(0xFFFFFFFFu, live && better(v, key, ws, wi));
                while (cand) {
                    const int src = __ffs(cand) - 1;
                    cand &= cand - 1u;
                    insert_better(ts, ti, m.k, __shfl_sync(0xFFFFFFFFu, v, src), b0 + (uint32_t)src);
                }
            }
        }
        if (lane == 0) {
#pragma unroll
            for (int q = 0; q < KT; ++q) {
                s_ws[wib][q] = ts[q];
                s_wi[wib][q] = ti[q];
            }
        }
        __syncthreads();
        if (wib == 0) {
            float fs[KT];
            uint32_t fi[KT];
#pragma unroll
            for (int q = 0; q < KT; ++q) {
                fs[q] = m.resc_ts[(size_t)it * kPKMax + q];
                fi[q] = m.resc_ti[(size_t)it * kPKMax + q];
            }
            for (int w = 0; w < 8; ++w)
                for (int q = 0; q < m.k && q < KT; ++q)
                    if (s_wi[w][q] != kNoIndex) insert_better(fs, fi, m.k, s_ws[w][q], s_wi[w][q]);
            if (lane == 0) {
                const size_t o = ((size_t)kvp * m.n_q + qp) * m.k;
#pragma unroll
                for (int q = 0; q < KT; ++q)
                    if (q < m.k) {
                        m.idx_out[o + q] = fi[q];
                        m.score_out[o + q] = fs[q];
                    }
            }
        }
    }
}

int num_sms() {
    static int n = [] {
        int dev = 0, v = 148;
        if (cudaGetDevice(&dev) == cudaSuccess &&
            cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess)
            return v;
        return 148;
    }();
    return n;
}

// key-range parts per query tile: the fewest whose CTA count fills whole waves within 2%
// (1 CTA per SM), keeping >= 64 key tiles per part so the pipeline fill stays amortised
int choose_splits(int ctas, int tiles) {
    const int sms = num_sms();
    int best = 1;
    double best_eff = 0.0;
    for (int s = 1; s <= kPMaxSplits && (s == 1 || tiles / s >= 64); ++s) {
        const long units = (long)ctas * s;
        const double eff = (double)units / ((units + sms - 1) / sms * sms);
        if (eff > best_eff + 0.02) {
            best = s;
            best_eff = eff;
        }
    }
    return best;
}

struct PrefillGeom {
    int n_qpad, tiles, splits;
    size_t hi_bytes, mq_bytes, dl_bytes, kmax_bytes, board_bytes, list_bytes, dropped_bytes, resc_bytes;
};

size_t al256(size_t x) { return (x + 255) / 256 * 256; }

PrefillGeom prefill_geom(const ScanArgs& a) {
    PrefillGeom g;
    g.n_qpad = (a.n_q + kPM * kPQT - 1) / (kPM * kPQT) * (kPM * kPQT);
    g.tiles = (int)((a.count + kPN - 1) / kPN);
    g.splits = choose_splits(g.n_qpad / (kPM * kPQT) * a.n_kv, g.tiles);
    if (const char* e = std::getenv("REATTN_K2_SPLITS"))  // experiments only
        g.splits = std::max(1, std::min(kPMaxSplits, std::atoi(e)));
    const size_t rows = (size_t)a.n_kv * g.n_qpad;
    g.hi_bytes = al256(rows * kPD * sizeof(__nv_bfloat16));
    g.mq_bytes = al256(rows * kPD * sizeof(float));
    g.dl_bytes = al256(rows * sizeof(float));
    g.kmax_bytes = al256((size_t)a.n_kv * sizeof(unsigned));
    g.board_bytes = al256(rows * sizeof(unsigned));
    g.list_bytes = al256((size_t)g.splits * rows * kPL * 4);  // one of indices / scores
    g.dropped_bytes = al256((size_t)g.splits * rows * 4);
    // re-scan queue: count, row, mask, top-k scores and indices per queued row
    g.resc_bytes = al256(4) + 2 * al256(rows * 4) + 2 * al256(rows * kPKMax * 4);
    return g;
}

}  // namespace

bool prefill_tc_supported(const ScanArgs& a) {
    return a.d == kPD && a.dtype == kBF16 && a.k >= 1 && a.k <= kPKMax && a.count > 0 && a.n_q >= 1;
}

size_t prefill_tc_workspace(const ScanArgs& a) {
    const PrefillGeom g = prefill_geom(a);
    return g.hi_bytes + g.mq_bytes + g.dl_bytes + g.kmax_bytes + g.board_bytes + 2 * g.list_bytes + g.dropped_bytes +
           g.resc_bytes + 1024;
}

cudaError_t launch_prefill_tc(const ScanArgs& a, const CUtensorMap& kmap, void* ws,
                              cudaStream_t s) {
    const PrefillGeom g = prefill_geom(a);
    const int n_qpad = g.n_qpad;
    uint8_t* w = (uint8_t*)ws;
    __nv_bfloat16* hi = (__nv_bfloat16*)w;
    w += g.hi_bytes;
    float* mq = (float*)w;
    w += g.mq_bytes;
    float* dl = (float*)w;
    w += g.dl_bytes;
    unsigned* kmax = (unsigned*)w;
    w += g.kmax_bytes;
    unsigned* board = (unsigned*)w;
    w += g.board_bytes;
    uint32_t* part_idx = (uint32_t*)w;
    w += g.list_bytes;
    float* part_score = (float*)w;
    w += g.list_bytes;
    float* part_dropped = (float*)w;
    w += g.dropped_bytes;
    const size_t rows = (size_t)a.n_kv * n_qpad;
    uint32_t* resc_count = (uint32_t*)w;
    w += al256(4);
    uint32_t* resc_row = (uint32_t*)w;
    w += al256(rows * 4);
    uint32_t* resc_mask = (uint32_t*)w;
    w += al256(rows * 4);
    float* resc_ts = (float*)w;
    w += al256(rows * kPKMax * 4);
    uint32_t* resc_ti = (uint32_t*)w;
    prefill_prep_kernel<<<(int)std::min<size_t>(148 * 16, (rows * 32 + 255) / 256), 256, 0, s>>>(
        a.q, a.n_q, a.n_heads, a.n_kv, n_qpad, hi, mq, dl);
    cudaError_t e = cudaMemsetAsync(kmax, 0, (size_t)a.n_kv * sizeof(unsigned), s);
    if (e != cudaSuccess) return e;
    e = cudaMemsetAsync(board, 0, rows * sizeof(unsigned), s);
    if (e != cudaSuccess) return e;
    prefill_kmax_kernel<<<dim3(std::max(1, num_sms() * 4 / std::max(1, a.n_kv)), a.n_kv), 256, 0, s>>>(
        (const __nv_bfloat16*)a.keys, a.head_stride, a.row0, a.count, a.n_kv, kmax);
    PrefillArgs p;
    p.n_q = a.n_q;
    p.n_qpad = n_qpad;
    p.n_kv = a.n_kv;
    p.k = a.k;
    p.count = a.count;
    p.head_stride = a.head_stride;
    p.row0 = a.row0;
    p.tiles = g.tiles;
    p.splits = g.splits;
    p.dl = dl;
    p.kmax = kmax;
    p.board = board;
    p.part_idx = part_idx;
    p.part_score = part_score;
    p.part_dropped = part_dropped;
    p.qhi = hi;
    CUtensorMap qh;
    if (!make_key_tensor_map(&qh, hi, kBF16, kPD, (uint64_t)a.n_kv * n_qpad, kPM))
        return cudaErrorInvalidValue;
    p.null_epilogue = std::getenv("REATTN_K2_NULL_EPILOGUE") ? 1 : 0;
    p.no_mma = std::getenv("REATTN_K2_NO_MMA") ? 1 : 0;
    p.no_insert = std::getenv("REATTN_K2_NO_INSERT") ? 1 : 0;
    dim3 grid(n_qpad / (kPM * kPQT), a.n_kv, g.splits);
    auto launch = [&](auto kernel) {
        cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kPSmem);
        kernel<<<grid, kPThreads, kPSmem, s>>>(qh, kmap, p);
    };
    if (a.k <= 1)
        launch(prefill_scan_tc_kernel<1>);
    else if (a.k <= 2)
        launch(prefill_scan_tc_kernel<2>);
    else if (a.k <= 4)
        launch(prefill_scan_tc_kernel<4>);
    else
        launch(prefill_scan_tc_kernel<8>);
    PrefillMergeArgs mg;
    mg.part_idx = part_idx;
    mg.part_score = part_score;
    mg.part_dropped = part_dropped;
    mg.splits = g.splits;
    mg.tiles = g.tiles;
    mg.n_kv = a.n_kv;
    mg.n_q = a.n_q;
    mg.n_qpad = n_qpad;
    mg.k = a.k;
    mg.count = a.count;
    mg.keys = (const __nv_bfloat16*)a.keys;
    mg.head_stride = a.head_stride;
    mg.row0 = a.row0;
    mg.mq = mq;
    mg.dl = dl;
    mg.kmax = kmax;
    mg.idx_out = a.idx_out;
    mg.score_out = a.score_out;
    mg.resc_count = resc_count;
    mg.resc_row = resc_row;
    mg.resc_mask = resc_mask;
    mg.resc_ts = resc_ts;
    mg.resc_ti = resc_ti;
    if ((e = cudaMemsetAsync(resc_count, 0, 4, s)) != cudaSuccess) return e;
    const int nw = a.n_kv * a.n_q;
    auto merge = [&](auto mk, auto rk) {
        mk<<<(nw + 7) / 8, 256, 0, s>>>(mg);
        rk<<<num_sms(), 256, 0, s>>>(mg);
    };
    const bool fma = a.lanes == kLanesFma;
    if (a.k <= 1)
        fma ? merge(prefill_exact_merge_kernel<kLanesFma, 1>, prefill_rescan_kernel<kLanesFma, 1>)
            : merge(prefill_exact_merge_kernel<kLanesUnfused, 1>, prefill_rescan_kernel<kLanesUnfused, 1>);
    else if (a.k <= 2)
        fma ? merge(prefill_exact_merge_kernel<kLanesFma, 2>, prefill_rescan_kernel<kLanesFma, 2>)
            : merge(prefill_exact_merge_kernel<kLanesUnfused, 2>, prefill_rescan_kernel<kLanesUnfused, 2>);
    else if (a.k <= 4)
        fma ? merge(prefill_exact_merge_kernel<kLanesFma, 4>, prefill_rescan_kernel<kLanesFma, 4>)
            : merge(prefill_exact_merge_kernel<kLanesUnfused, 4>, prefill_rescan_kernel<kLanesUnfused, 4>);
    else
        fma ? merge(prefill_exact_merge_kernel<kLanesFma, 8>, prefill_rescan_kernel<kLanesFma, 8>)
            : merge(prefill_exact_merge_kernel<kLanesUnfused, 8>, prefill_rescan_kernel<kLanesUnfused, 8>);
    return cudaGetLastError();
}

int prefill_tc_key_box_rows() { return kPN; }

}  // namespace reattn_impl
