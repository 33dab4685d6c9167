// K1 — position-agnostic q·Kᵀ scan fused with an exact running top-k.
//
// Restates reattn::fused_topk_scores (reference selection.hpp:168-248) on sm_100a:
//   * group-mean query per KV head (selection.hpp:139-156): sequential fp32 adds, then
//     multiply by float(1/group);
//   * score = dot_f32 (dense_matrix.hpp:41-56): eight lanes over elements j, j+8, ...,
//     then ((l0+l1)+(l2+l3))+((l4+l5)+(l6+l7)).  The lane update is emulated exactly in
//     either of the two codegen variants the reference compiles to:
//     unfused (round(a*b) then round(l+p)) or FMA — so scores are bit-identical;
//   * exact top-k with ties to the lower index (selection.hpp:81-135), output sorted by
//     (score desc, index asc).
//
// Fast path (decode, d=128, n_q=1, k<=8): a persistent grid, one CTA per SM.  A producer
// warp streams 64 KB tiles of key rows with TMA (cp.async.bulk.tensor, SWIZZLE_128B) into
// a 3-stage shared-memory ring; each consumer thread owns one key row per tile, holds the
// group-mean query in registers as 64 packed fp32x2 pairs and evaluates the 8-lane dot
// with FMUL2/FADD2 (or FFMA2), then keeps a register top-k (the common reject is one
// compare against a register threshold, as selection.hpp:230-236).  Per-CTA top-k go to a
// slot array; CTA 0 (scanning fewer tiles, its merge code warmed by a dry pass) waits for the
// others' done count and merges them deterministically, then runs the fused vote/spans/scope.
//
// Generic path (any d / n_q / k): one CTA per (query, kv head) streaming the whole
// middle, appending candidates above the running k-th key into a shared buffer and
// compacting it with a bitonic sort — bounded scratch, exact, deterministic.
#include <algorithm>
#include <cstdlib>
#include <mutex>

#include "common.cuh"
#include "kernels.h"
#include "select_small.cuh"

using namespace reattn_dev;

namespace reattn_impl {

namespace {

template <typename KT>
struct FastCfg {
    static constexpr int D = 128;
    static constexpr int ESZ = (int)sizeof(KT);
    static constexpr int ROW_BYTES = D * ESZ;       // 256 (bf16) / 512 (fp32)
    // key rows per stage = consumer threads.  bf16: 8 consumer warps (2 per SM sub-partition,
    // evenly loaded); thread 0 also issues the TMA loads, so ptxas keeps 255 registers per
    // thread for the 128-float query held in registers (9 warps would cap it at 168).
    static constexpr int ROWS = ESZ == 2 ? 256 : 128;
    // fp32: two threads per key row, each summing four of the reference's eight lanes (half
    // the query in registers), so the CTA keeps 8 warps like bf16 -- the merger CTA's merge
    // and select run on 8 warps, and twice the loads are in flight per stage
    static constexpr int ROW_THREADS = ESZ == 2 ? 1 : 2;
    static constexpr int NBOX = ROW_BYTES / 128;    // 128-byte TMA boxes per row
    static constexpr int BOX_ELEMS = 128 / ESZ;
    static constexpr int STAGE_BYTES = ROWS * ROW_BYTES;
    static constexpr int STAGES = 3;
    static constexpr int CONSUMERS = ROWS * ROW_THREADS;
    static constexpr int CWARPS = CONSUMERS / 32;
    static constexpr int THREADS = CONSUMERS;  // thread 0 doubles as the TMA producer
    static constexpr int KMAX = 8;
    static constexpr size_t SMEM = 1024 /*align slack*/ + (size_t)STAGES * STAGE_BYTES +
                                   2 * STAGES * sizeof(uint64_t) + D * sizeof(float) +
                                   CWARPS * KMAX * (sizeof(float) + sizeof(uint32_t)) + 16;
};

struct FastArgs {
    const float* q;
    int n_heads, n_kv, group;
    uint64_t head_stride, row0;
    uint32_t count;
    int k;
    uint32_t tiles_per_head, total_tiles;
    uint32_t* slot_idx;
    float* slot_score;
    unsigned int* ticket;
    uint32_t* idx_out;
    float* score_out;
    int fuse_select;
    SmallSelectIO sel;
    uint64_t* trace;  // diagnostics (misc.cu layout) or null
    uint32_t tiles0;  // tiles of CTA 0 (the merger; see the tail below)
    uint32_t part_q, part_r;  // (T - T0) = part_q (G - 1) + part_r
    struct Balance* bal;      // adaptive partition state (plans), or null
    // device-resident cache length (plans that survive cache growth): when non-null, the middle
    // (kv_cache.hpp:65-67), the tile partition and the select's geometry are derived from it
    const uint32_t* dev_total;
    uint32_t l_global, l_local;
    int tail_tiles;
};

// The launch's geometry: from the host (a frozen plan) or from the device cache length.
struct FastGeo {
    uint32_t count, tph, T, T0, pq, pr, g_end, l_start, total;
};
__device__ __forceinline__ FastGeo fast_geo(const FastArgs& a, uint32_t G, int rows) {
    FastGeo g;
    if (!a.dev_total) {
        g.count = a.count;
        g.tph = a.tiles_per_head;
        g.T = a.total_tiles;
        g.T0 = G == 1 ? g.T : a.tiles0;
        g.pq = a.part_q;
        g.pr = a.part_r;
        g.g_end = a.sel.g_end;
        g.l_start = a.sel.l_start;
        g.total = a.sel.total;
        return g;
    }
    uint32_t total;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(total) : "l"(a.dev_total));
    g.total = total;
    g.g_end = min(total, a.l_global);
    g.l_start = total - min(total - g.g_end, a.l_local);
    g.count = g.l_start - g.g_end;
    g.tph = (g.count + rows - 1) / rows;
    g.T = g.tph * (uint32_t)a.n_kv;
    const uint32_t share = g.T / G;
    g.T0 = G == 1 ? g.T : (share > (uint32_t)a.tail_tiles ? share - (uint32_t)a.tail_tiles : 0u);
    const uint32_t rest = g.T - g.T0;
    g.pq = G > 1 ? rest / (G - 1) : 0u;
    g.pr = G > 1 ? rest % (G - 1) : 0u;
    return g;
}

// Adaptive tile partition.  The scan CTAs do not stream at equal rates (with the decode fork
// the slowest finish ~10 us after the median, on the same SMs every step), so for long scans
// the partition follows measured rates: every CTA records its loop time, and CTA 0, in the
// slack before it merges, turns launch e-1's rates (smoothed, clamped to +-30% of the mean)
// into the table launch e+1 uses.  Tables and durations are double-buffered by epoch parity;
// a header (T, G, T0) guards against a workspace reused for another geometry.  The top-k is
// exact under any partition, so results do not depend on it.
constexpr int kBalMaxG = 160;
struct Balance {
    uint32_t T, G, T0, epoch;        // epoch = launches completed with this header
    uint32_t tbv[2];                 // table p valid for launch tbv[p] - 1
    uint32_t durv[2];                // dur/cnt p hold launch durv[p] - 1
    uint32_t tb[2][kBalMaxG + 1];
    uint32_t dur[2][kBalMaxG];
    uint32_t cnt[2][kBalMaxG];
    float rate[kBalMaxG];
};

// Static tile partition: CTA 0 (the merger) takes T0 tiles, the other G-1 CTAs split the
// rest evenly: begin(b) = T0 + floor((b-1)(T-T0)/(G-1)) = T0 + (b-1)q + floor((b-1)r/(G-1))
// with (T-T0) = q(G-1) + r from the host -- 32-bit arithmetic only (a 64-bit integer or f64
// division is a long software sequence, and this runs in every CTA and in the merge).
__device__ __forceinline__ uint32_t tile_begin(uint32_t b, uint32_t G, uint32_t T, uint32_t T0,
                                               uint32_t q, uint32_t r) {
    if (b == 0) return 0u;
    if (b >= G) return T;
    return T0 + (b - 1) * q + ((b - 1) * r) / (G - 1);
}

constexpr uint32_t kDryFlush = 0xFFFFFFFEu;  // flush() without slot writes (code warm-up)

template <int KMAX>
__device__ __forceinline__ void topk_reset(float (&ts)[KMAX], uint32_t (&ti)[KMAX]) {
#pragma unroll
    for (int j = 0; j < KMAX; ++j) {
        ts[j] = -INFINITY;
        ti[j] = kNoIndex;
    }
}

// Bubble (s, i) into the sorted list; full (score desc, index asc) comparator.
template <int KMAX>
__device__ __forceinline__ void topk_insert(float (&ts)[KMAX], uint32_t (&ti)[KMAX], int k,
                                            float s, uint32_t i) {
#pragma unroll
    for (int j = 0; j < KMAX; ++j) {
        if (j < k && better(s, i, ts[j], ti[j])) {
            const float t = ts[j];
            const uint32_t u = ti[j];
            ts[j] = s;
            ti[j] = i;
            s = t;
            i = u;
        }
    }
}

template <int KMAX>
__device__ __forceinline__ float topk_threshold(const float (&ts)[KMAX], int k) {
    float thr = ts[0];
#pragma unroll
    for (int j = 1; j < KMAX; ++j)
        if (j == k - 1) thr = ts[j];
    return thr;
}

template <int KMAX>
__device__ __forceinline__ void topk_pop(float (&ts)[KMAX], uint32_t (&ti)[KMAX]) {
#pragma unroll
    for (int j = 0; j + 1 < KMAX; ++j) {
        ts[j] = ts[j + 1];
        ti[j] = ti[j + 1];
    }
    ts[KMAX - 1] = -INFINITY;
    ti[KMAX - 1] = kNoIndex;
}

template <int LANES>
__device__ __forceinline__ void lane_step(f2_t& acc, f2_t q, f2_t k) {
    if (LANES == kLanesFma)
        acc = f2_fma(q, k, acc);
    else
        // unfused lane: round(q*k), then round(acc + .).  The product comes from an FFMA2 with
        // a +0 addend -- ptxas cannot contract an FMA into the following add (it does contract
        // mul.rn.f32x2 + add.rn.f32x2, even with --fmad=false).  RN(q*k + 0) == RN(q*k) except
        // for an exact -0 product, which becomes +0; the accumulator starts at +0 and sums of
        // floats never round to -0, so acc + (+0) == acc + (-0) and the lanes stay bit-exact.
        acc = f2_add(acc, f2_fma(q, k, 0ull));
}

__device__ __forceinline__ float lane_tree(f2_t a0, f2_t a1, f2_t a2, f2_t a3) {
    const float s01 = __fadd_rn(f2_lo(a0), f2_hi(a0));
    const float s23 = __fadd_rn(f2_lo(a1), f2_hi(a1));
    const float s45 = __fadd_rn(f2_lo(a2), f2_hi(a2));
    const float s67 = __fadd_rn(f2_lo(a3), f2_hi(a3));
    return __fadd_rn(__fadd_rn(s01, s23), __fadd_rn(s45, s67));
}

template <typename KT, int LANES>
__global__ void __launch_bounds__(FastCfg<KT>::THREADS, 1)
    scan_fast_kernel(const __grid_constant__ CUtensorMap kmap, const FastArgs a) {
    // let a programmatic dependent (the decode attention) launch now: its CTAs become
    // resident as this grid's CTAs retire and wait in griddepcontrol.wait for our results
    asm volatile("griddepcontrol.launch_dependents;");
    using C = FastCfg<KT>;
    constexpr int KMAX = C::KMAX;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    uint8_t* stages = smem;
    uint64_t* full = (uint64_t*)(smem + (size_t)C::STAGES * C::STAGE_BYTES);
    uint64_t* empty = full + C::STAGES;
    float* s_mq = (float*)(empty + C::STAGES);
    float* s_ws = s_mq + C::D;
    uint32_t* s_wi = (uint32_t*)(s_ws + C::CWARPS * KMAX);
    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const uint32_t G = gridDim.x, b = blockIdx.x;
    const FastGeo fg = fast_geo(a, G, C::ROWS);
    const uint32_t T = fg.T, T0 = fg.T0;
    Balance* bal = (a.bal && G <= kBalMaxG && G > 2) ? a.bal : nullptr;
    uint32_t epoch = 0;
    const uint32_t* tab = nullptr;
    if (bal) {
        epoch = bal->epoch;
        if (bal->T != T || bal->G != G || bal->T0 != T0) epoch = 0;  // another geometry
        if (epoch > 0 && bal->tbv[epoch & 1] == epoch + 1) tab = bal->tb[epoch & 1];
    }
    auto tbeg = [&](uint32_t c) {
        return tab ? tab[c] : tile_begin(c, G, T, T0, fg.pq, fg.pr);
    };
    const uint32_t t_begin = tbeg(b), t_end = tbeg(b + 1);
    const uint64_t t_start = bal ? globaltimer() : 0ull;
    const int k = a.k;

    if (tid == 0) {
        for (int s = 0; s < C::STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], C::CWARPS);
        }
        fence_barrier_init();
    }
    __syncthreads();
    if (a.trace && tid == 0) a.trace[b] = globaltimer();

    // ===== TMA issue (thread 0): the first STAGES tiles now, then each stage is refilled
    // as soon as every warp has released it (end of the consumer iteration below) =====
    const uint64_t pol = policy_evict_first();
    auto issue = [&](uint32_t it) {
        const uint32_t t = t_begin + it;
        const int s = it % C::STAGES;
        const uint32_t kv = t / fg.tph, j = t % fg.tph;
        const int32_t row = (int32_t)(kv * a.head_stride + (a.dev_total ? fg.g_end : a.row0) +
                                      (uint64_t)j * C::ROWS);
        mbar_arrive_expect_tx(&full[s], C::STAGE_BYTES);
#pragma unroll
        for (int box = 0; box < C::NBOX; ++box)
            tma_load_2d(stages + (size_t)s * C::STAGE_BYTES + box * C::ROWS * 128, &kmap,
                        box * C::BOX_ELEMS, row, &full[s], pol);
    };
    if (tid == 0) {
        prefetch_tensormap(&kmap);
        for (uint32_t it = 0; it < (uint32_t)C::STAGES && t_begin + it < t_end; ++it) issue(it);
    }
    {
        // ===== consumers: one key row per thread (bf16) or per thread pair (fp32) per tile =====
        constexpr int RT = C::ROW_THREADS;
        const uint32_t rrow = (uint32_t)tid / RT, half = (uint32_t)tid % RT;
        f2_t qv[C::D / 2 / RT];
        float ts[KMAX];
        uint32_t ti[KMAX];
        float thr = -INFINITY;
        topk_reset<KMAX>(ts, ti);
        uint32_t cur_kv = kNoIndex;
        const uint32_t sw = rrow & 7u;

        auto flush = [&](uint32_t kv) {
            // warp-level top-k of the warp's 32 lists, then warp 0 merges the warps
            for (int r = 0; r < k; ++r) {
                float bs = ts[0];
                uint32_t bi = ti[0];
                warp_best(bs, bi);
                if (lane == 0) {
                    s_ws[warp * KMAX + r] = bs;
                    s_wi[warp * KMAX + r] = bi;
                }
                if (bi != kNoIndex && ti[0] == bi) topk_pop<KMAX>(ts, ti);
            }
            named_bar_sync(1, C::CONSUMERS);
            if (warp == 0) {
                float ls[2];
                uint32_t li[2];
                ls[0] = ls[1] = -INFINITY;
                li[0] = li[1] = kNoIndex;
                const int n = C::CWARPS * k;
                for (int e = lane; e < n; e += 32) {
                    const int w = e / k, r = e % k;
                    float s = s_ws[w * KMAX + r];
                    uint32_t i = s_wi[w * KMAX + r];
                    if (better(s, i, ls[0], li[0])) {
                        ls[1] = ls[0];
                        li[1] = li[0];
                        ls[0] = s;
                        li[0] = i;
                    } else if (better(s, i, ls[1], li[1])) {
                        ls[1] = s;
                        li[1] = i;
                    }
                }
                for (int r = 0; r < k; ++r) {
                    float bs = ls[0];
                    uint32_t bi = li[0];
                    warp_best(bs, bi);
                    if (lane == 0 && kv != kDryFlush) {
                        const size_t slot = ((size_t)kv * G + b) * KMAX + r;
                        a.slot_score[slot] = bs;
                        a.slot_idx[slot] = bi;
                    }
                    if (bi != kNoIndex && li[0] == bi) {
                        ls[0] = ls[1];
                        li[0] = li[1];
                        ls[1] = -INFINITY;
                        li[1] = kNoIndex;
                    }
                }
                __threadfence();
            }
            named_bar_sync(1, C::CONSUMERS);
            topk_reset<KMAX>(ts, ti);
            thr = -INFINITY;
        };

        // One flush call site: a dry flush at the first tile (warms its code while the first
        // TMA tiles land; it runs once per launch otherwise, so the slowest CTA's final flush
        // would run cold, ~2 us), the head switches, and the final flush at t == t_end.
        uint32_t it = 0;
        cur_kv = kDryFlush;
        for (uint32_t t = t_begin;; ++t, ++it) {
            const bool done = t >= t_end;
            const uint32_t kv = done ? kNoIndex : t / fg.tph, j = t % fg.tph;
            if (kv != cur_kv) {
                if (cur_kv != kNoIndex) flush(cur_kv);
                if (done) break;
                // group-mean query for this kv head (selection.hpp:143-151)
                if (tid < C::D) {
                    const float inv = __fdiv_rn(1.0f, (float)a.group);
                    float acc = 0.0f;
                    for (int g = 0; g < a.group; ++g)
                        acc = __fadd_rn(acc, a.q[(size_t)(kv * a.group + g) * C::D + tid]);
                    s_mq[tid] = __fmul_rn(acc, inv);
                }
                named_bar_sync(1, C::CONSUMERS);
                if (RT == 1) {
#pragma unroll
                    for (int p = 0; p < C::D / 2 / RT; ++p) qv[p] = f2_packf(s_mq[2 * p], s_mq[2 * p + 1]);
                } else {  // this thread's lanes 4h..4h+3: elements 8c + 4h + {0..3}
#pragma unroll
                    for (int c = 0; c < C::D / 8; ++c) {
                        qv[(2 * c) % (C::D / 2 / RT)] = f2_packf(s_mq[8 * c + 4 * half], s_mq[8 * c + 4 * half + 1]);
                        qv[(2 * c + 1) % (C::D / 2 / RT)] =
                            f2_packf(s_mq[8 * c + 4 * half + 2], s_mq[8 * c + 4 * half + 3]);
                    }
                }
                cur_kv = kv;
            }
            const int s = it % C::STAGES;
            const uint32_t ph = (it / C::STAGES) & 1u;
            mbar_wait(&full[s], ph);
            const uint32_t row = j * C::ROWS + rrow;
            const bool live = row < fg.count;  // the same for both threads of a row
            const uint32_t sbase = smem_u32(stages + (size_t)s * C::STAGE_BYTES) + rrow * 128u;
            f2_t a0 = f2_pack(0u, 0u), a1 = a0, a2 = a0, a3 = a0;
            if (live) {
#pragma unroll
                for (int c = 0; c < C::D / 8; ++c) {
                    if (C::ESZ == 2) {
                        const int box = c >> 3, cb = c & 7;
                        const uint4 w = lds128(sbase + box * C::ROWS * 128 + (((uint32_t)cb ^ sw) << 4));
                        lane_step<LANES>(a0, qv[(4 * c + 0) % (C::D / 2 / RT)], bf16x2_to_f2(w.x));
                        lane_step<LANES>(a1, qv[(4 * c + 1) % (C::D / 2 / RT)], bf16x2_to_f2(w.y));
                        lane_step<LANES>(a2, qv[(4 * c + 2) % (C::D / 2 / RT)], bf16x2_to_f2(w.z));
                        lane_step<LANES>(a3, qv[(4 * c + 3) % (C::D / 2 / RT)], bf16x2_to_f2(w.w));
                    } else {  // 16 bytes: the row's elements 8c + 4h .. 8c + 4h + 3 (lanes 4h..4h+3)
                        const int box = c >> 2, u = (c & 3) * 2 + (int)half;
                        const uint4 w = lds128(sbase + box * C::ROWS * 128 + (((uint32_t)u ^ sw) << 4));
                        lane_step<LANES>(a0, qv[(2 * c) % (C::D / 2 / RT)], f2_pack(w.x, w.y));
                        lane_step<LANES>(a1, qv[(2 * c + 1) % (C::D / 2 / RT)], f2_pack(w.z, w.w));
                    }
                }
            }
            float score;
            if (RT == 1) {
                score = lane_tree(a0, a1, a2, a3);
            } else {
                // ((l0+l1)+(l2+l3)) on the even thread, ((l4+l5)+(l6+l7)) on the odd one, and
                // their sum on both (IEEE addition commutes): the reference's tree, bit for bit
                const float part = __fadd_rn(__fadd_rn(f2_lo(a0), f2_hi(a0)), __fadd_rn(f2_lo(a1), f2_hi(a1)));
                score = __fadd_rn(part, __shfl_xor_sync(0xFFFFFFFFu, part, 1));
            }
            if (live && half == 0) {
                if (score > thr) {
                    topk_insert<KMAX>(ts, ti, k, score, row);
                    thr = topk_threshold<KMAX>(ts, k);
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
            if (tid == 0 && t + C::STAGES < t_end) {
                mbar_wait(&empty[s], ph);  // all warps are done with this stage
                issue(it + C::STAGES);
            }
        }
    }

    // ===== cross-CTA merge and select by CTA 0 =====
    // The merge + vote/spans/scope tail is ~1.5K instructions executed once per launch, so it
    // runs from a cold instruction cache (~0.3-0.5 us per fetch miss: 10+ us measured).  CTA 0
    // therefore scans fewer tiles, runs the tail once in dry mode (same code, global stores
    // predicated off) to warm its instruction cache while the others still scan, waits for
    // their done count, and runs it for real (~4 us).
    __syncthreads();
    if (bal && tid == 0) {
        bal->dur[epoch & 1][b] = (uint32_t)min(globaltimer() - t_start, (uint64_t)0xFFFFFFFFu);
        bal->cnt[epoch & 1][b] = t_end - t_begin;
    }
    if (a.trace && tid == 0) {
        a.trace[512 + b] = globaltimer();
        uint32_t smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        a.trace[1100 + b] = smid;
    }
    if (b != 0) {
        if (tid == 0) {
            __threadfence();
            atomicAdd(a.ticket, 1u);  // release: this CTA's slots are written
        }
        return;
    }
    // merged candidate i = kv * kk + r goes straight to the select's shared candidates
    __shared__ SmallSelectSmem ssel;
    constexpr int kMergeCache = 64;  // kv heads whose covering CTA range is cached
    __shared__ uint32_t s_b0[kMergeCache], s_b1[kMergeCache];
    const int kk = (int)min((uint32_t)k, fg.count);
    SmallSelectIO sel = a.sel;  // the select's geometry (device-derived for growing caches)
    if (a.dev_total) {
        sel.middle_len = fg.count;
        sel.g_end = fg.g_end;
        sel.l_start = fg.l_start;
        sel.total = fg.total;
    }
    const int nwarps = C::THREADS / 32;
#pragma unroll 1
    for (int pass = 0; pass < 2; ++pass) {
        const bool dry = pass == 0;
        if (!dry && bal && warp == 0 && epoch > 0 && bal->durv[(epoch + 1) & 1] == epoch) {
            // next launch's table from launch epoch-1's rates (same parity as the table written)
            const int p = (epoch + 1) & 1;
            const uint32_t n = G - 1;  // CTAs 1..G-1 share T - T0
            const uint32_t per = (n + 31) / 32, lo = 1 + lane * per, hi = min(G, lo + per);
            float r[6];
            float rs = 0.0f;
#pragma unroll
            for (int u = 0; u < 6; ++u) {
                const uint32_t c = lo + u;
                r[u] = 0.0f;
                if (c < hi) {
                    const uint32_t d = bal->dur[p][c];
                    r[u] = d ? (float)bal->cnt[p][c] / (float)d : 0.0f;
                    rs += r[u];
                }
            }
            float tot = rs;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(0xFFFFFFFFu, tot, o);
            const float mean = tot / (float)n;
            float ws = 0.0f;
#pragma unroll
            for (int u = 0; u < 6; ++u) {
                const uint32_t c = lo + u;
                if (c < hi) {
                    float x = mean > 0.0f ? fminf(fmaxf(r[u], 0.7f * mean), 1.3f * mean) : 1.0f;
                    const float old = bal->rate[c];
                    if (old > 0.0f) x = 0.5f * (old + x);
                    bal->rate[c] = x;
                    r[u] = x;
                    ws += x;
                } else {
                    r[u] = 0.0f;
                }
            }
            // exclusive prefix of the lanes' sums (lane order == CTA order)
            float incl = ws;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const float t = __shfl_up_sync(0xFFFFFFFFu, incl, o);
                if (lane >= o) incl += t;
            }
            const float total = __shfl_sync(0xFFFFFFFFu, incl, 31);
            double run = (double)(incl - ws);
            uint32_t* tb = bal->tb[(epoch + 1) & 1];
#pragma unroll
            for (int u = 0; u < 6; ++u) {
                const uint32_t c = lo + u;
                if (c < hi) tb[c] = T0 + (uint32_t)((double)(T - T0) * run / (double)total);
                run += (double)r[u];
            }
            if (lane == 0) {
                tb[0] = 0u;
                tb[G] = T;
            }
            __syncwarp();
            if (lane == 0) {
                __threadfence();
                bal->tbv[(epoch + 1) & 1] = epoch + 2;
            }
        }
        if (!dry) {
            if (tid == 0) {
                while (ld_acquire_u32(a.ticket) < G - 1) __nanosleep(32);
                *a.ticket = 0u;  // re-arm for the next launch (graph replay)
                if (a.trace) a.trace[1024] = globaltimer();
            }
            __syncthreads();
        }
        for (int kv = warp; kv < a.n_kv; kv += nwarps) {
            float ls[KMAX];
            uint32_t li[KMAX];
            topk_reset<KMAX>(ls, li);
            // CTAs whose (non-empty) tile range meets this head's tiles [h0, h1): contiguous
            const uint32_t h0 = (uint32_t)kv * fg.tph, h1 = h0 + fg.tph;
            // (computed in the dry pass and kept in shared memory: the partition is fixed for
            // the launch)
            uint32_t b0 = G, b1 = 0;
            if (!dry && kv < kMergeCache) {
                b0 = s_b0[kv];
                b1 = s_b1[kv];
            } else {
                for (uint32_t c = lane; c < G; c += 32) {
                    const uint32_t cb = tbeg(c), ce = tbeg(c + 1);
                    const bool meets = cb < ce && cb < h1 && ce > h0;
                    if (meets) {
                        b0 = min(b0, c);
                        b1 = max(b1, c);
                    }
                }
                b0 = __reduce_min_sync(0xFFFFFFFFu, b0);
                b1 = __reduce_max_sync(0xFFFFFFFFu, b1);
                if (dry && kv < kMergeCache && lane == 0) {
                    s_b0[kv] = b0;
                    s_b1[kv] = b1;
                }
            }
            const int n = b0 <= b1 ? (int)(b1 - b0 + 1) * k : 0;
            // all of a batch's loads are issued before any insert: one L2 round trip per batch
            for (int e0 = 0; e0 < n; e0 += 128) {
                float s4[4];
                uint32_t i4[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int e = e0 + 32 * u + lane;
                    s4[u] = -INFINITY;
                    i4[u] = kNoIndex;
                    if (e < n) {
                        const size_t slot = ((size_t)kv * G + b0 + e / k) * KMAX + e % k;
                        s4[u] = __ldcg(a.slot_score + slot);
                        i4[u] = __ldcg(a.slot_idx + slot);
                    }
                }
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    if (i4[u] != kNoIndex) topk_insert<KMAX>(ls, li, k, s4[u], i4[u]);
            }
            if (a.trace && !dry && lane == 0 && kv == 0) a.trace[1027] = globaltimer();
            for (int r = 0; r < k; ++r) {
                float bs = ls[0];
                uint32_t bi = li[0];
                warp_best(bs, bi);
                if (lane == 0) {
                    if (!dry) {
                        a.idx_out[(size_t)kv * k + r] = bi;
                        a.score_out[(size_t)kv * k + r] = bs;
                    }
                    const int c = kv * kk + r;
                    if (a.fuse_select && r < kk && c < 32) {
                        ssel.idx[c] = bi;
                        ssel.key[c] = float_key(bs);
                    }
                }
                if (bi != kNoIndex && li[0] == bi) topk_pop<KMAX>(ls, li);
            }
        }
        if (a.fuse_select) {
            // vote + spans + scope on the merged candidates [kv][0..kk) (selection.hpp:252-349)
            const int n = a.n_kv * kk;  // <= 32 (fuse_select condition)
            if (tid == 0) ssel.vmask = n >= 32 ? 0xFFFFFFFFu : ((1u << n) - 1u);
            __syncthreads();
            if (a.trace && !dry && tid == 0) {
                a.trace[1025] = a.trace[1028] = globaltimer();
                a.trace[1040] = clock64();
            }
            small_select_scope_smem(sel, ssel, dry ? nullptr : a.trace, dry);
            if (a.trace && !dry) {
                __syncthreads();
                if (tid == 0) a.trace[1026] = globaltimer();
            }
        }
        __syncthreads();
    }
    if (bal && tid == 0) {  // every CTA's duration is in: publish this launch's state
        bal->durv[epoch & 1] = epoch + 1;
        bal->T = T;
        bal->G = G;
        bal->T0 = T0;
        bal->epoch = epoch + 1;
    }
}

// ------------------------------------------------------------------------------------
// Generic exact path.
struct GenArgs {
    const float* q;
    int n_q, n_heads, n_kv, d, group;
    const void* keys;
    uint64_t head_stride, row0;
    uint32_t count;
    int k;
    int nbuf;  // power of two >= k + 512
    uint32_t* idx_out;
    float* score_out;
};

__device__ void bitonic_desc_u64(unsigned long long* buf, int n) {
    for (int k2 = 2; k2 <= n; k2 <<= 1) {
        for (int j = k2 >> 1; j > 0; j >>= 1) {
            for (int i = threadIdx.x; i < n; i += blockDim.x) {
                const int ixj = i ^ j;
                if (ixj > i) {
                    const unsigned long long x = buf[i], y = buf[ixj];
                    const bool desc = (i & k2) == 0;
                    if (desc ? (x < y) : (x > y)) {
                        buf[i] = y;
                        buf[ixj] = x;
                    }
                }
            }
            __syncthreads();
        }
    }
}

template <typename KT, int LANES>
__global__ void __launch_bounds__(256) scan_generic_kernel(const GenArgs a) {
    extern __shared__ unsigned long long gsm[];
    unsigned long long* buf = gsm;                  // [nbuf]
    float* mq = (float*)(gsm + a.nbuf);             // [d]
    __shared__ unsigned int s_nb;
    const int qi = blockIdx.x, kv = blockIdx.y, tid = threadIdx.x;
    const int d = a.d;
    // group-mean query (selection.hpp:143-151)
    const float inv = __fdiv_rn(1.0f, (float)a.group);
    for (int c = tid; c < d; c += blockDim.x) {
        float acc = 0.0f;
        for (int g = 0; g < a.group; ++g)
            acc = __fadd_rn(acc, a.q[(size_t)qi * a.n_heads * d + (size_t)(kv * a.group + g) * d + c]);
        mq[c] = __fmul_rn(acc, inv);
    }
    if (tid == 0) s_nb = 0;
    __syncthreads();

    const KT* keys = (const KT*)a.keys + ((size_t)kv * a.head_stride + a.row0) * d;
    uint32_t r = 0;                // valid sorted entries at buf[0, r)
    unsigned long long thr = 0;    // key of the k-th best once r == k
    const uint32_t kk = (uint32_t)a.k;
    for (uint32_t base = 0; base < a.count; base += blockDim.x) {
        const uint32_t row = base + tid;
        if (row < a.count) {
            const KT* kr = keys + (size_t)row * d;
            float l[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
            int j = 0;
            for (; j + 8 <= d; j += 8) {
#pragma unroll
                for (int t = 0; t < 8; ++t) {
                    const float kvv = load_as_float<KT>(kr + j + t);
                    l[t] = (LANES == kLanesFma) ? __fmaf_rn(mq[j + t], kvv, l[t])
                                                : __fadd_rn(l[t], __fmul_rn(mq[j + t], kvv));
                }
            }
            for (; j < d; ++j) {
                const float kvv = load_as_float<KT>(kr + j);
                l[0] = (LANES == kLanesFma) ? __fmaf_rn(mq[j], kvv, l[0])
                                            : __fadd_rn(l[0], __fmul_rn(mq[j], kvv));
            }
            const float s = __fadd_rn(__fadd_rn(__fadd_rn(l[0], l[1]), __fadd_rn(l[2], l[3])),
                                      __fadd_rn(__fadd_rn(l[4], l[5]), __fadd_rn(l[6], l[7])));
            const unsigned long long key = topk_key(s, row);
            if (r < kk || key > thr) {
                const unsigned int pos = atomicAdd(&s_nb, 1u);
                buf[r + pos] = key;
            }
        }
        __syncthreads();
        const uint32_t nb = s_nb;
        const bool last = base + blockDim.x >= a.count;
        if (r + nb + blockDim.x > (uint32_t)a.nbuf || last) {
            for (int i = r + nb + tid; i < a.nbuf; i += blockDim.x) buf[i] = 0ull;
            __syncthreads();
            bitonic_desc_u64(buf, a.nbuf);
            r = min(kk, r + nb);
            thr = (r == kk) ? buf[kk - 1] : 0ull;
            if (tid == 0) s_nb = 0;
        }
        __syncthreads();
    }
    const size_t o = ((size_t)kv * a.n_q + qi) * a.k;
    for (uint32_t j = tid; j < r; j += blockDim.x) {
        RA_ASSERT(key_index(buf[j]) < a.count);
        a.idx_out[o + j] = key_index(buf[j]);
        a.score_out[o + j] = key_score(buf[j]);
    }
}

template <typename F>
void set_smem_once(F* fn, size_t bytes) {
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

}  // namespace

// ------------------------------------------------------------------------------------
int scan_fast_box_rows(int dtype) {
    return dtype == kBF16 ? FastCfg<__nv_bfloat16>::ROWS : FastCfg<float>::ROWS;
}

bool scan_fast_supported(const ScanArgs& a) {
    return a.d == 128 && a.n_q == 1 && a.k >= 1 && a.k <= 8 && a.count > 0 &&
           (a.dtype == kBF16 || a.dtype == kF32) &&
           (uint64_t)a.n_kv * a.head_stride < (1ull << 31) && a.n_kv <= 65535;
}

static uint32_t fast_tiles_per_head(const ScanArgs& a) {
    const uint32_t rows = (uint32_t)scan_fast_box_rows(a.dtype);
    return (a.count + rows - 1) / rows;
}

static size_t slots_bytes(const ScanArgs& a, int num_sms) {
    return (size_t)a.n_kv * (size_t)std::max(1, num_sms) * 8 * (sizeof(uint32_t) + sizeof(float));
}

size_t scan_fast_workspace(const ScanArgs& a, int num_sms) {
    // ticket (256 B aligned) + slots + the adaptive partition state
    return 256 + ((slots_bytes(a, num_sms) + 255) & ~(size_t)255) + sizeof(Balance);
}

typedef CUresult (*PFN_encodeTiled_t)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                       const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                       const cuuint32_t*, CUtensorMapInterleave,
                                       CUtensorMapSwizzle, CUtensorMapL2promotion,
                                       CUtensorMapFloatOOBfill);

static PFN_encodeTiled_t encode_fn() {
    static PFN_encodeTiled_t fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = (PFN_encodeTiled_t)p;
    });
    return fn;
}

bool make_key_tensor_map(CUtensorMap* map, const void* base, int dtype, uint64_t d, uint64_t rows,
                         int box_rows) {
    PFN_encodeTiled_t enc = encode_fn();
    if (!enc) return false;
    const uint64_t esz = dtype == kBF16 ? 2 : 4;
    cuuint64_t dims[2] = {(cuuint64_t)d, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)(d * esz)};
    cuuint32_t box[2] = {(cuuint32_t)(128 / esz), (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    const CUresult r = enc(map, dtype == kBF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16
                                               : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                           2, const_cast<void*>(base), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

bool make_tensor_map_2d(CUtensorMap* map, const void* base, int dtype, uint64_t inner, uint64_t outer,
                        uint64_t row_bytes, uint32_t box_inner, uint32_t box_outer) {
    PFN_encodeTiled_t enc = encode_fn();
    if (!enc) return false;
    cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
    cuuint64_t strides[1] = {(cuuint64_t)row_bytes};
    cuuint32_t box[2] = {box_inner, box_outer};
    cuuint32_t estr[2] = {1, 1};
    const CUresult r = enc(map, dtype == kBF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                           2, const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

cudaError_t launch_scan_fast(const ScanArgs& a, const CUtensorMap& kmap, void* workspace,
                             int num_sms, cudaStream_t s) {
    FastArgs f;
    f.q = a.q;
    f.n_heads = a.n_heads;
    f.n_kv = a.n_kv;
    f.group = a.n_heads / a.n_kv;
    f.head_stride = a.head_stride;
    f.row0 = a.row0;
    f.count = a.count;
    f.k = a.k;
    f.tiles_per_head = fast_tiles_per_head(a);
    f.total_tiles = f.tiles_per_head * (uint32_t)a.n_kv;
    uint8_t* ws = (uint8_t*)workspace;
    f.ticket = (unsigned int*)ws;
    f.slot_idx = (uint32_t*)(ws + 256);
    f.slot_score = (float*)(ws + 256 + (size_t)a.n_kv * num_sms * 8 * sizeof(uint32_t));
    // a growing cache keeps the grid of the plan: CTAs without tiles are fine
    const int G = a.dev_total ? std::max(1, num_sms)
                              : (int)std::min<uint32_t>((uint32_t)std::max(1, num_sms), f.total_tiles);
    f.dev_total = a.dev_total;
    f.l_global = a.l_global;
    f.l_local = a.l_local;
    f.idx_out = a.idx_out;
    f.score_out = a.score_out;
    f.fuse_select = a.fuse_select;
    f.sel = a.sel;
    f.trace = trace_buffer();
    {
        // CTA 0 scans kTailTiles fewer tiles than an even share: the time its dry tail pass
        // takes (~15 us cold; one 64 KB tile per CTA ~1.5 us at the HBM rate).
        static const int tail_tiles = [] {
            const char* e = std::getenv("REATTN_TAIL_TILES");
            return e ? std::atoi(e) : 10;
        }();
        f.tail_tiles = tail_tiles;
        const uint32_t share = f.total_tiles / (uint32_t)std::max(1, std::min<int>(num_sms, (int)f.total_tiles));
        f.tiles0 = share > (uint32_t)tail_tiles ? share - (uint32_t)tail_tiles : 0u;
        const uint32_t rest = G > 1 ? f.total_tiles - f.tiles0 : 0u;
        f.part_q = G > 1 ? rest / (uint32_t)(G - 1) : 0u;
        f.part_r = G > 1 ? rest % (uint32_t)(G - 1) : 0u;
    }
    // very long scans only (>= 400 tiles per CTA): the table reads cost the start an L2
    // round trip and the merge a few loads.  Measured A/B: 4M context (885 tiles per CTA)
    // 1225 -> 1203 us; 1M (233) neutral; 32K-128K a loss
    const char* bmin = std::getenv("REATTN_BALANCE_MIN_TILES");  // tests force it small
    const bool long_scan = f.total_tiles / (uint32_t)G >= (bmin ? (uint32_t)std::atoi(bmin) : 400u);
    f.bal = a.balance && long_scan && !std::getenv("REATTN_NO_BALANCE")
                ? (Balance*)(ws + 256 + ((slots_bytes(a, num_sms) + 255) & ~(size_t)255))
                : nullptr;
    if (a.dtype == kBF16) {
        using C = FastCfg<__nv_bfloat16>;
        if (a.lanes == kLanesFma) {
            static bool once = (set_smem_once(scan_fast_kernel<__nv_bfloat16, kLanesFma>, C::SMEM), true);
            (void)once;
            scan_fast_kernel<__nv_bfloat16, kLanesFma><<<G, C::THREADS, C::SMEM, s>>>(kmap, f);
        } else {
            static bool once = (set_smem_once(scan_fast_kernel<__nv_bfloat16, kLanesUnfused>, C::SMEM), true);
            (void)once;
            scan_fast_kernel<__nv_bfloat16, kLanesUnfused><<<G, C::THREADS, C::SMEM, s>>>(kmap, f);
        }
    } else {
        using C = FastCfg<float>;
        if (a.lanes == kLanesFma) {
            static bool once = (set_smem_once(scan_fast_kernel<float, kLanesFma>, C::SMEM), true);
            (void)once;
            scan_fast_kernel<float, kLanesFma><<<G, C::THREADS, C::SMEM, s>>>(kmap, f);
        } else {
            static bool once = (set_smem_once(scan_fast_kernel<float, kLanesUnfused>, C::SMEM), true);
            (void)once;
            scan_fast_kernel<float, kLanesUnfused><<<G, C::THREADS, C::SMEM, s>>>(kmap, f);
        }
    }
    return cudaGetLastError();
}

cudaError_t launch_scan_generic(const ScanArgs& a, cudaStream_t s) {
    GenArgs g;
    g.q = a.q;
    g.n_q = a.n_q;
    g.n_heads = a.n_heads;
    g.n_kv = a.n_kv;
    g.d = a.d;
    g.group = a.n_heads / a.n_kv;
    g.keys = a.keys;
    g.head_stride = a.head_stride;
    g.row0 = a.row0;
    g.count = a.count;
    g.k = a.k;
    int nbuf = 512;
    while (nbuf < a.k + 512) nbuf <<= 1;
    g.nbuf = nbuf;
    g.idx_out = a.idx_out;
    g.score_out = a.score_out;
    const size_t smem = (size_t)nbuf * sizeof(unsigned long long) + (size_t)a.d * sizeof(float);
    dim3 grid(a.n_q, a.n_kv);
#define GEN_LAUNCH(KT, L)                                                              \
    do {                                                                               \
        set_smem_once(scan_generic_kernel<KT, L>, smem);                               \
        scan_generic_kernel<KT, L><<<grid, 256, smem, s>>>(g);                         \
    } while (0)
    if (a.dtype == kBF16) {
        if (a.lanes == kLanesFma) GEN_LAUNCH(__nv_bfloat16, kLanesFma);
        else GEN_LAUNCH(__nv_bfloat16, kLanesUnfused);
    } else {
        if (a.lanes == kLanesFma) GEN_LAUNCH(float, kLanesFma);
        else GEN_LAUNCH(float, kLanesUnfused);
    }
#undef GEN_LAUNCH
    return cudaGetLastError();
}

}  // namespace reattn_impl
