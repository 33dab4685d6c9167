// K2 — prefill score scan on the 5th-gen tensor cores (tcgen05 + TMEM), fused top-k.
//
// Same contract as fused_topk_scores (reference selection.hpp:275-355) for a prefill
// chunk (n_q up to l_chunk = 4096 queries): per (kv head, query) the top-k of
// mq · k over the middle, ties to the lower index.  The score GEMM
//     S[q, j] = mq[q, :] · K[j, :]      (128 queries x 256 keys per MMA tile, d = 128)
// runs on tcgen05.mma (kind::f16, bf16 operands, fp32 accumulators in TMEM).  mq is the
// exact fp32 group mean (selection.hpp:250-258) split into bf16 hi + lo (16 significant
// bits); S = hi·K + lo·K accumulates both in the same TMEM tile.  Scores therefore carry
// an error <= (2^-16 + 2·d·2^-24)·Σ|mq_i k_i| against the reference's fp32 dot: index
// parity is the north_star ε-tie rule, not bit equality (the exact CUDA-core path stays
// the default; this path is opt-in, reattn_ctx_set_prefill).
//
// Warp roles (320 threads, 1 CTA/SM):
//   warp 0  TMA producer: the CTA's Q hi/lo tile once, then K tiles (2-stage ring, 64 KB)
//   warp 1  TMEM allocator (512 columns = 2 accumulators of 256) + single-thread MMA issue
//   warps 2-9  epilogue, two warps per TMEM lane quarter (one per 128-column half):
//           2 x tcgen05.ld 32x32b.x64, release the accumulator, then 16 group maxes decide
//           which 8-column groups enter the register top-k of the thread's query row.
//
// Grid: (query tile, kv head, key split).  256 query tiles on 148 SMs is 1.73 waves, so the
// key range of each query tile is cut into `splits` contiguous parts chosen to fill whole
// waves; each part writes a partial top-k list and prefill_merge_kernel reduces them.
#include <algorithm>

#include "common.cuh"
#include "kernels.h"
#include "tcgen05.cuh"

using namespace reattn_dev;

namespace reattn_impl {

namespace {

constexpr int kPM = 128;  // queries per CTA = UMMA M
constexpr int kPN = 256;  // keys per tile = UMMA N
constexpr int kPD = 128;  // head dim
constexpr int kPStages = 2;
constexpr int kPQBytes = kPM * kPD * 2;  // one of hi / lo: 32 KB
constexpr int kPKBytes = kPN * kPD * 2;  // one K stage: 64 KB
constexpr int kPThreads = 320;  // producer, MMA, 8 epilogue warps
constexpr int kPKMax = 8;
constexpr size_t kPSmem = 1024 + 2 * kPQBytes + kPStages * kPKBytes + 128 + 2 * kPM * kPKMax * 4 + 256 * 32;

struct PrefillArgs {
    int n_q, n_qpad, n_kv, k;
    uint32_t count;
    uint64_t head_stride, row0;
    int tiles;             // key tiles of the whole middle
    int splits;            // key-range parts per query tile (gridDim.z)
    uint32_t* idx_out;     // splits == 1: final [n_kv][n_q][k]
    float* score_out;
    uint32_t* part_idx;    // splits > 1: [splits][n_kv][n_qpad][kPKMax]
    float* part_score;
};

constexpr uint32_t prefill_idesc() { return idesc_bf16_f32<kPM, kPN>(); }

// Insert (cs, ci) into the descending list ts/ti, given cs > ts[KT-1].  One thread sees its
// candidates in increasing key order, so an equal score never displaces an entry and
// better() reduces to a strict >.  All compares use the original list: branch-free shift.
template <int KT>
__device__ __forceinline__ void insert_in_order(float (&ts)[KT], uint32_t (&ti)[KT], float cs,
                                                uint32_t ci) {
#pragma unroll
    for (int j = KT - 1; j >= 0; --j) {
        const bool here = cs > ts[j];
        const bool above = j > 0 && cs > ts[j > 0 ? j - 1 : 0];
        if (here) {
            ts[j] = above ? ts[j - (j > 0)] : cs;
            ti[j] = above ? ti[j - (j > 0)] : ci;
        }
    }
}

template <int KT>
__global__ void __launch_bounds__(kPThreads, 1)
    prefill_scan_tc_kernel(const __grid_constant__ CUtensorMap qhi_map,
                           const __grid_constant__ CUtensorMap qlo_map,
                           const __grid_constant__ CUtensorMap k_map, const PrefillArgs a) {
    extern __shared__ uint8_t psm_raw[];
    uint8_t* sm = (uint8_t*)(((uintptr_t)psm_raw + 1023) & ~(uintptr_t)1023);
    uint8_t* s_qhi = sm;
    uint8_t* s_qlo = sm + kPQBytes;
    uint8_t* s_k = sm + 2 * kPQBytes;
    uint64_t* bars = (uint64_t*)(s_k + kPStages * kPKBytes);
    uint64_t* q_full = bars;
    uint64_t* full = bars + 1;
    uint64_t* empty = full + kPStages;
    uint64_t* tfull = empty + kPStages;
    uint64_t* tempty = tfull + 2;
    uint32_t* s_tmem = (uint32_t*)(tempty + 2);
    uint8_t* aux = (uint8_t*)bars + 128;  // half-merge lists, then the group staging area

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int qtile = blockIdx.x, kv = blockIdx.y, split = blockIdx.z;
    const int t_first = (int)((int64_t)split * a.tiles / a.splits);
    const int n_tiles = (int)((int64_t)(split + 1) * a.tiles / a.splits) - t_first;

    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(s_tmem)),
                     "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        mbar_init(q_full, 1);
        for (int s = 0; s < kPStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&tfull[b], 1);
            mbar_init(&tempty[b], 256);
        }
        fence_barrier_init();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *s_tmem;

    if (warp == 0) {
        if (lane == 0) {  // ===== TMA producer =====
            prefetch_tensormap(&qhi_map);
            prefetch_tensormap(&qlo_map);
            prefetch_tensormap(&k_map);
            const uint64_t pol = policy_evict_first();
            const uint64_t keep = policy_evict_last();  // K tiles: re-read by every query tile
            const int32_t qrow = (int32_t)(kv * a.n_qpad + qtile * kPM);
            mbar_arrive_expect_tx(q_full, 2 * kPQBytes);
            tma_load_2d(s_qhi, &qhi_map, 0, qrow, q_full, pol);
            tma_load_2d(s_qhi + kPQBytes / 2, &qhi_map, 64, qrow, q_full, pol);
            tma_load_2d(s_qlo, &qlo_map, 0, qrow, q_full, pol);
            tma_load_2d(s_qlo + kPQBytes / 2, &qlo_map, 64, qrow, q_full, pol);
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
        if (lane == 0) {  // ===== MMA issuer =====
            const uint32_t idesc = prefill_idesc();
            mbar_wait(q_full, 0);
            tc_fence_after();
            const uint32_t qhi = smem_u32(s_qhi), qlo = smem_u32(s_qlo);
            for (int t = 0; t < n_tiles; ++t) {
                const int s = t % kPStages;
                const uint32_t ph = (t / kPStages) & 1u;
                const int b = t & 1;
                const uint32_t bph = (t >> 1) & 1u;
                if (t >= 2) mbar_wait(&tempty[b], bph ^ 1u);
                mbar_wait(&full[s], ph);
                tc_fence_after();
                const uint32_t kbase = smem_u32(s_k + (size_t)s * kPKBytes);
                const uint32_t d_tmem = tmem + (uint32_t)(b * kPN);
                uint32_t acc = 0;
#pragma unroll
                for (int hl = 0; hl < 2; ++hl) {
                    const uint32_t qb = hl ? qlo : qhi;
#pragma unroll
                    for (int kb = 0; kb < 2; ++kb)
#pragma unroll
                        for (int ks = 0; ks < 4; ++ks) {
                            const uint64_t ad = umma_desc_sw128(qb + kb * (kPQBytes / 2) + ks * 32);
                            const uint64_t bd = umma_desc_sw128(kbase + kb * (kPKBytes / 2) + ks * 32);
                            mma_bf16_ss(d_tmem, ad, bd, idesc, acc);
                            acc = 1;
                        }
                }
                mma_commit(&empty[s]);  // smem stage free once these MMAs retire
                mma_commit(&tfull[b]);  // accumulator ready for the epilogue
            }
        }
    } else {
        // ===== epilogue: 8 warps, two per TMEM lane quarter; the thread owning lane r owns
        // query row r of the tile for one half (128 columns) of every key tile =====
        const int ew = warp - 2;          // 0..7
        const int quarter = warp & 3;     // TMEM lane quarter this warp may access
        const int half = ew >> 2;         // column half of the 256-key tile
        const int row = quarter * 32 + lane;
        const int query = qtile * kPM + row;
        const int e = ew * 32 + lane;
        float ts[KT];
        uint32_t ti[KT];
#pragma unroll
        for (int j = 0; j < KT; ++j) {
            ts[j] = -INFINITY;
            ti[j] = kNoIndex;
        }
        float4* stage = (float4*)(aux + 2 * kPM * kPKMax * 4);  // [2][256] float4: one group
        for (int t = 0; t < n_tiles; ++t) {
            const int b = t & 1;
            const uint32_t bph = (t >> 1) & 1u;
            mbar_wait(&tfull[b], bph);
            tc_fence_after();
            const uint32_t col = (uint32_t)(b * kPN + half * (kPN / 2));
            const uint32_t taddr = tmem + ((uint32_t)(quarter * 32) << 16) + col;
            uint32_t r[128];
            TMEM_LD_X64(taddr, r);  // both loads in flight before the single wait
            TMEM_LD_X64(taddr + 64, (r + 64));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            tc_fence_before();
            mbar_arrive(&tempty[b]);  // accumulator copied out: the MMA warp may reuse it
            const uint32_t key0 = (uint32_t)(t_first + t) * kPN + half * (kPN / 2);
            if (key0 + 128 > a.count) {  // tail tile: keys past the middle never qualify
#pragma unroll
                for (int c = 0; c < 128; ++c)
                    if (key0 + c >= a.count) r[c] = __float_as_uint(-INFINITY);
            }
            // common path: 16 group maxes (8 columns each), one 16-bit qualifying mask.  A warp
            // enters the insert path whenever ANY lane qualifies (~32k/t of tiles), so the
            // insert path touches only the qualifying groups: the group is staged through
            // shared memory by predicated stores (registers cannot be indexed dynamically).
            const float thr = ts[KT - 1];
            uint32_t gmask = 0;
#pragma unroll
            for (int g = 0; g < 16; ++g) {
                float m = __uint_as_float(r[8 * g]);
#pragma unroll
                for (int u = 1; u < 8; ++u) m = fmaxf(m, __uint_as_float(r[8 * g + u]));
                gmask |= (m > thr ? 1u : 0u) << g;
            }
            while (gmask) {
                const int g = __ffs(gmask) - 1;
                gmask &= gmask - 1;
#pragma unroll
                for (int gg = 0; gg < 16; ++gg)
                    if (gg == g) {
                        stage[e] = make_float4(__uint_as_float(r[8 * gg]), __uint_as_float(r[8 * gg + 1]),
                                               __uint_as_float(r[8 * gg + 2]), __uint_as_float(r[8 * gg + 3]));
                        stage[256 + e] =
                            make_float4(__uint_as_float(r[8 * gg + 4]), __uint_as_float(r[8 * gg + 5]),
                                        __uint_as_float(r[8 * gg + 6]), __uint_as_float(r[8 * gg + 7]));
                    }
                const float4 v0 = stage[e], v1 = stage[256 + e];
                const float v[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
#pragma unroll
                for (int u = 0; u < 8; ++u)
                    if (v[u] > ts[KT - 1]) insert_in_order<KT>(ts, ti, v[u], key0 + 8 * g + u);
            }
        }
        // merge the two column halves of each row (disjoint key sets; full order)
        float* m_s = (float*)aux;                           // [128][kPKMax] scores
        uint32_t* m_i = (uint32_t*)(aux + kPM * kPKMax * 4);  // [128][kPKMax] indices
        if (half == 1)
#pragma unroll
            for (int j = 0; j < KT; ++j) {
                m_s[row * kPKMax + j] = ts[j];
                m_i[row * kPKMax + j] = ti[j];
            }
        named_bar_sync(1, 256);
        if (half == 0) {
#pragma unroll
            for (int jj = 0; jj < KT; ++jj) {
                float cs = m_s[row * kPKMax + jj];
                uint32_t ci = m_i[row * kPKMax + jj];
#pragma unroll
                for (int j = 0; j < KT; ++j) {
                    if (better(cs, ci, ts[j], ti[j])) {
                        const float tt = ts[j];
                        const uint32_t uu = ti[j];
                        ts[j] = cs;
                        ti[j] = ci;
                        cs = tt;
                        ci = uu;
                    }
                }
            }
            const int k = a.k;
            if (a.splits > 1) {
                const size_t o = (((size_t)split * a.n_kv + kv) * a.n_qpad + query) * kPKMax;
#pragma unroll
                for (int j = 0; j < KT; ++j)
                    if (j < k) {
                        a.part_idx[o + j] = ti[j];
                        a.part_score[o + j] = ts[j];
                    }
            } else if (query < a.n_q) {
                const size_t o = ((size_t)kv * a.n_q + query) * k;
#pragma unroll
                for (int j = 0; j < KT; ++j)
                    if (j < k) {
                        a.idx_out[o + j] = ti[j];
                        a.score_out[o + j] = ts[j];
                    }
            }
        }
    }
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
    }
}

// group-mean query (selection.hpp:250-258, exact fp32) split into bf16 hi + lo
__global__ void prefill_prep_kernel(const float* q, int n_q, int n_heads, int n_kv, int n_qpad,
                                    __nv_bfloat16* hi, __nv_bfloat16* lo) {
    const int group = n_heads / n_kv;
    const float inv = __fdiv_rn(1.0f, (float)group);
    const size_t n = (size_t)n_kv * n_qpad * kPD;
    for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < n;
         e += (size_t)gridDim.x * blockDim.x) {
        const int c = (int)(e % kPD);
        const size_t rq = e / kPD;
        const int qi = (int)(rq % n_qpad), kv = (int)(rq / n_qpad);
        float m = 0.0f;
        if (qi < n_q) {
            float acc = 0.0f;
            for (int g = 0; g < group; ++g)
                acc = __fadd_rn(acc, q[(size_t)qi * n_heads * kPD + (size_t)(kv * group + g) * kPD + c]);
            m = __fmul_rn(acc, inv);
        }
        const __nv_bfloat16 h = __float2bfloat16_rn(m);
        hi[e] = h;
        lo[e] = __float2bfloat16_rn(__fsub_rn(m, __bfloat162float(h)));
    }
}

// reduce the per-split partial lists of each (kv head, query): disjoint key ranges, so the
// union's top-k under better() is the top-k of the whole middle
__global__ void prefill_merge_kernel(const uint32_t* part_idx, const float* part_score, int splits,
                                     int n_kv, int n_q, int n_qpad, int k, uint32_t* idx_out,
                                     float* score_out) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n_kv * n_q) return;
    const int kv = e / n_q, query = e % n_q;
    float ts[kPKMax];
    uint32_t ti[kPKMax];
#pragma unroll
    for (int j = 0; j < kPKMax; ++j) {
        ts[j] = -INFINITY;
        ti[j] = kNoIndex;
    }
    for (int s = 0; s < splits; ++s) {
        const size_t o = (((size_t)s * n_kv + kv) * n_qpad + query) * kPKMax;
        for (int jj = 0; jj < k; ++jj) {
            float cs = part_score[o + jj];
            uint32_t ci = part_idx[o + jj];
            if (ci == kNoIndex) break;
#pragma unroll
            for (int j = 0; j < kPKMax; ++j) {
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
    }
    const size_t o = ((size_t)kv * n_q + query) * k;
    for (int j = 0; j < k; ++j) {
        idx_out[o + j] = ti[j];
        score_out[o + j] = ts[j];
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
// (1 CTA per SM), keeping >= 32 key tiles per part so the pipeline fill stays amortised
int choose_splits(int ctas, int tiles) {
    const int sms = num_sms();
    int best = 1;
    double best_eff = 0.0;
    for (int s = 1; s <= 8 && (s == 1 || tiles / s >= 32); ++s) {
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
    size_t q_bytes, part_bytes;
};

PrefillGeom prefill_geom(const ScanArgs& a) {
    PrefillGeom g;
    g.n_qpad = (a.n_q + kPM - 1) / kPM * kPM;
    g.tiles = (int)((a.count + kPN - 1) / kPN);
    g.splits = choose_splits(g.n_qpad / kPM * a.n_kv, g.tiles);
    g.q_bytes = 2 * (size_t)a.n_kv * g.n_qpad * kPD * sizeof(__nv_bfloat16);
    g.part_bytes = g.splits > 1 ? (size_t)g.splits * a.n_kv * g.n_qpad * kPKMax * 8 : 0;
    return g;
}

}  // namespace

bool prefill_tc_supported(const ScanArgs& a) {
    return a.d == kPD && a.dtype == kBF16 && a.k >= 1 && a.k <= kPKMax && a.count > 0 && a.n_q >= 1;
}

size_t prefill_tc_workspace(const ScanArgs& a) {
    const PrefillGeom g = prefill_geom(a);
    return g.q_bytes + g.part_bytes + 1024;
}

cudaError_t launch_prefill_tc(const ScanArgs& a, const CUtensorMap& kmap, void* ws,
                              cudaStream_t s) {
    const PrefillGeom g = prefill_geom(a);
    const int n_qpad = g.n_qpad;
    __nv_bfloat16* hi = (__nv_bfloat16*)ws;
    __nv_bfloat16* lo = hi + (size_t)a.n_kv * n_qpad * kPD;
    const size_t n = (size_t)a.n_kv * n_qpad * kPD;
    prefill_prep_kernel<<<(int)std::min<size_t>(148 * 16, (n + 255) / 256), 256, 0, s>>>(
        a.q, a.n_q, a.n_heads, a.n_kv, n_qpad, hi, lo);
    CUtensorMap qh, ql;
    if (!make_key_tensor_map(&qh, hi, kBF16, kPD, (uint64_t)a.n_kv * n_qpad, kPM) ||
        !make_key_tensor_map(&ql, lo, kBF16, kPD, (uint64_t)a.n_kv * n_qpad, kPM))
        return cudaErrorInvalidValue;
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
    p.idx_out = a.idx_out;
    p.score_out = a.score_out;
    uint8_t* part = (uint8_t*)ws + (g.q_bytes + 255) / 256 * 256;
    p.part_idx = (uint32_t*)part;
    p.part_score = (float*)(part + g.part_bytes / 2);
    dim3 grid(n_qpad / kPM, a.n_kv, g.splits);
    auto launch = [&](auto kernel) {
        cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kPSmem);
        kernel<<<grid, kPThreads, kPSmem, s>>>(qh, ql, kmap, p);
    };
    if (a.k <= 1)
        launch(prefill_scan_tc_kernel<1>);
    else if (a.k <= 2)
        launch(prefill_scan_tc_kernel<2>);
    else if (a.k <= 4)
        launch(prefill_scan_tc_kernel<4>);
    else
        launch(prefill_scan_tc_kernel<8>);
    if (g.splits > 1) {
        const int n = a.n_kv * a.n_q;
        prefill_merge_kernel<<<(n + 127) / 128, 128, 0, s>>>(p.part_idx, p.part_score, g.splits,
                                                             a.n_kv, a.n_q, n_qpad, a.k,
                                                             a.idx_out, a.score_out);
    }
    return cudaGetLastError();
}

int prefill_tc_key_box_rows() { return kPN; }

}  // namespace reattn_impl
