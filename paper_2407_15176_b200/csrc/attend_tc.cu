// K6 — prefill finite-scope attention on the 5th-gen tensor cores (tcgen05 + TMEM).
//
// Same contract as the f64 CUDA-core kernel in attend.cu for a prefill block.  It restates
// the reference's attend (attend.hpp:25-77) over the assembled scope
// (scope.hpp:63-76, engine.hpp:78-93): keys rotated at compact position j, queries at
// L'-n_q+i, scale 1/sqrt(d), causal boundary L'-n_q, output acc/denom and row entropy
// ln A - B/A.  It is opt-in with the prefill scan (reattn_ctx_set_prefill(TENSOR)).
//
// Precision (bf16 K/V cache; north_star bf16 tolerance, measured far below it):
//   S = Qhi·Khi + Qlo·Khi + Qhi·Klo      fp32 rotated q and k, each split into bf16 hi + lo
//   O += Phi·V + Plo·V                   p = exp(s - m) in fp32, split hi + lo; V exact bf16
//   A, B (softmax denominator and entropy numerator) summed per tile in fp32, across tiles
//   in f64.  The running max is rescaled lazily: only when a tile max exceeds the reference
//   max by more than 2^8 in p (the final acc/A and ln A - B/A are invariant to the
//   reference, so this changes rounding only).
//
// Two kernels:
//   flash_prep_kernel  gathers the scope once per kv head (not once per query block):
//                      K rotated at compact positions -> Khi, Klo [n_kv][Lpad][128] bf16;
//                      V transposed -> Vt [n_kv][128][Lpad] bf16 (K-major B operand of P·V)
//   flash_tc_kernel    one CTA per (128-query block, q head), 320 threads, 1 CTA/SM:
//     warp 0    TMA producer: K hi/lo and Vt tiles of 128 scope rows (2-stage rings)
//     warp 1    TMEM owner (512 cols) + single-thread MMA issue:
//                 S_t (TMEM cols 0/128, double-buffered) then O += P_{t-1}·V_{t-1} (cols
//                 256..383), so the softmax of tile t overlaps the S MMAs of tile t+1
//     warps 2-9 softmax, two warps per TMEM lane quarter: thread = (query row, 64-column
//               half).  Q rotation, scale and split into TMEM (cols 384..511); per tile:
//               S -> mask -> max (exchanged with the other half) -> lazy O rescale -> p ->
//               P hi/lo written over S_t in TMEM (A operand of the P·V MMA); final acc/A.
#include <algorithm>

#include "common.cuh"
#include "kernels.h"
#include "tcgen05.cuh"

using namespace reattn_dev;

namespace reattn_impl {

namespace {

constexpr int kFM = 128;  // query rows per CTA = UMMA M
constexpr int kFN = 128;  // scope rows per tile = UMMA N of S = K of P·V
constexpr int kFD = 128;  // d = dv
constexpr int kFStages = 2;
constexpr int kFKBytes = kFN * kFD * 2;  // K hi or K lo tile: 32 KB
constexpr int kFVBytes = kFD * kFN * 2;  // V^T tile: 32 KB
constexpr int kFThreads = 320;  // producer, MMA, 8 softmax warps
constexpr size_t kFSmem = 1024 + (size_t)kFStages * (2 * kFKBytes + kFVBytes) + 256 + 4 * kFM * 4 +
                          2 * kFM * 2 * 8;
constexpr uint32_t kColO = 256, kColQhi = 384, kColQlo = 448;
constexpr float kRescaleLog2 = 8.0f;  // rescale once p could exceed 2^8

struct FlashArgs {
    const float* q;
    uint64_t q_row_stride;
    int n_q, n_head, group;
    uint32_t Lpad;
    const ScopeHeader* hdr;
    uint32_t L_host;
    const float* rope_cos;
    const float* rope_sin;
    int causal, boundary_is_tail;
    uint32_t boundary_host;
    float scale_log2;  // log2(e) / sqrt(d)
    float* out;        // [n_q][n_head * 128]
    double* entropy;   // [n_q][n_head]
};

__device__ __forceinline__ uint32_t pack_bf16x2(float lo_elem, float hi_elem) {
    uint32_t r;
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi_elem), "f"(lo_elem));
    return r;
}
__device__ __forceinline__ float ex2_approx(float x) {
    float r;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ float bf16_lo_half(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf16_hi_half(uint32_t w) { return __uint_as_float(w & 0xFFFF0000u); }

// rotate the interleaved pair (x, y) by (c, s) with the reference's unfused fp32 ops
// (rope.hpp:49-60)
__device__ __forceinline__ void rotate_pair(float x, float y, float c, float s, float& rx, float& ry) {
    rx = __fsub_rn(__fmul_rn(x, c), __fmul_rn(y, s));
    ry = __fadd_rn(__fmul_rn(x, s), __fmul_rn(y, c));
}

// ---- scope gather: K rotated + split, V transposed; rows >= L are zero ---------------------
template <typename KT>
__global__ void __launch_bounds__(256) flash_prep_kernel(const AttnArgs a, uint32_t Lpad,
                                                         __nv_bfloat16* khi, __nv_bfloat16* klo,
                                                         __nv_bfloat16* vt) {
    if (a.hdr && a.hdr->error != 0) return;
    const uint32_t L = a.hdr ? a.hdr->L : a.L_host;
    const int kv = blockIdx.y;
    const uint32_t r0 = blockIdx.x * 32u;
    const int tid = threadIdx.x;
    __shared__ uint16_t vs[32][kFD + 2];
    // K: one thread per (row, pair)
    for (int e = tid; e < 32 * (kFD / 2); e += 256) {
        const int r = e / (kFD / 2), j = e % (kFD / 2);
        const uint32_t sr = r0 + r;
        float rx = 0.0f, ry = 0.0f;
        if (sr < L) {
            const uint32_t cr = a.src ? a.src[sr] : sr;
            const KT* row = (const KT*)a.k_base + ((size_t)kv * a.head_stride + cr) * kFD;
            const float x = load_as_float<KT>(row + 2 * j), y = load_as_float<KT>(row + 2 * j + 1);
            if (a.rope_cos)
                rotate_pair(x, y, a.rope_cos[(size_t)sr * (kFD / 2) + j],
                            a.rope_sin[(size_t)sr * (kFD / 2) + j], rx, ry);
            else {
                rx = x;
                ry = y;
            }
        }
        const uint32_t h = pack_bf16x2(rx, ry);
        const uint32_t l = pack_bf16x2(__fsub_rn(rx, bf16_lo_half(h)), __fsub_rn(ry, bf16_hi_half(h)));
        const size_t o = ((size_t)kv * Lpad + sr) * kFD + 2 * j;
        *(uint32_t*)(khi + o) = h;
        *(uint32_t*)(klo + o) = l;
    }
    // V: gather 32 rows, write transposed
    for (int e = tid; e < 32 * kFD; e += 256) {
        const int r = e / kFD, c = e % kFD;
        const uint32_t sr = r0 + r;
        uint16_t v = 0;
        if (sr < L) {
            const uint32_t cr = a.src ? a.src[sr] : sr;
            const KT* row = (const KT*)a.v_base + ((size_t)kv * a.head_stride + cr) * kFD;
            v = __bfloat16_as_ushort(__float2bfloat16_rn(load_as_float<KT>(row + c)));
        }
        vs[r][c] = v;
    }
    __syncthreads();
    for (int e = tid; e < 32 * kFD; e += 256) {
        const int c = e / 32, r = e % 32;
        ((uint16_t*)vt)[((size_t)kv * kFD + c) * Lpad + r0 + r] = vs[r][c];
    }
}

__global__ void __launch_bounds__(kFThreads, 1)
    flash_tc_kernel(const __grid_constant__ CUtensorMap khi_map,
                    const __grid_constant__ CUtensorMap klo_map,
                    const __grid_constant__ CUtensorMap vt_map, const FlashArgs a) {
    if (a.hdr && a.hdr->error != 0) return;
    extern __shared__ uint8_t fsm_raw[];
    uint8_t* sm = (uint8_t*)(((uintptr_t)fsm_raw + 1023) & ~(uintptr_t)1023);
    uint8_t* s_k = sm;                                  // [stage][hi | lo] 64 KB
    uint8_t* s_v = sm + kFStages * 2 * kFKBytes;        // [stage] 32 KB
    uint64_t* bars = (uint64_t*)(s_v + kFStages * kFVBytes);
    uint64_t* q_ready = bars;
    uint64_t* k_full = bars + 1;
    uint64_t* k_empty = k_full + kFStages;
    uint64_t* v_full = k_empty + kFStages;
    uint64_t* v_empty = v_full + kFStages;
    uint64_t* s_full = v_empty + kFStages;
    uint64_t* p_full = s_full + 2;
    uint64_t* o_done = p_full + 2;
    uint64_t* o_final = o_done + 1;              // completes once: the last P·V landed
    uint32_t* s_tmem = (uint32_t*)(o_final + 1);  // then s_max / s_ab (softmax exchange)

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int qblk = blockIdx.x, h = blockIdx.y, kv = h / a.group;
    const uint32_t L = a.hdr ? a.hdr->L : a.L_host;
    const uint32_t boundary = a.boundary_is_tail ? L - (uint32_t)a.n_q : a.boundary_host;
    const int q0 = qblk * kFM;
    const int q_last = min(q0 + kFM, a.n_q) - 1;
    const uint32_t key_end =
        a.causal ? (uint32_t)min((unsigned long long)L, (unsigned long long)boundary + q_last + 1) : L;
    const int n_tiles = (int)((key_end + kFN - 1) / kFN);

    if (warp == 1) tmem_alloc(s_tmem, 512);
    if (tid == 0) {
        mbar_init(q_ready, 256);
        for (int s = 0; s < kFStages; ++s) {
            mbar_init(&k_full[s], 1);
            mbar_init(&k_empty[s], 1);
            mbar_init(&v_full[s], 1);
            mbar_init(&v_empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&s_full[b], 1);
            mbar_init(&p_full[b], 256);
        }
        mbar_init(o_done, 1);
        mbar_init(o_final, 1);
        fence_barrier_init();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *s_tmem;

    if (warp == 0) {
        if (lane == 0) {  // ===== TMA producer =====
            prefetch_tensormap(&khi_map);
            prefetch_tensormap(&klo_map);
            prefetch_tensormap(&vt_map);
            const uint64_t keep = policy_evict_last();  // the scope is re-read by every CTA
            for (int t = 0; t < n_tiles; ++t) {
                const int s = t % kFStages;
                const uint32_t ph = (t / kFStages) & 1u;
                const int32_t krow = (int32_t)((uint32_t)kv * a.Lpad + (uint32_t)t * kFN);
                if (t >= kFStages) mbar_wait(&k_empty[s], ph ^ 1u);
                mbar_arrive_expect_tx(&k_full[s], 2 * kFKBytes);
                uint8_t* dk = s_k + (size_t)s * 2 * kFKBytes;
                tma_load_2d(dk, &khi_map, 0, krow, &k_full[s], keep);
                tma_load_2d(dk + kFKBytes / 2, &khi_map, 64, krow, &k_full[s], keep);
                tma_load_2d(dk + kFKBytes, &klo_map, 0, krow, &k_full[s], keep);
                tma_load_2d(dk + kFKBytes + kFKBytes / 2, &klo_map, 64, krow, &k_full[s], keep);
                if (t >= kFStages) mbar_wait(&v_empty[s], ph ^ 1u);
                mbar_arrive_expect_tx(&v_full[s], kFVBytes);
                uint8_t* dv = s_v + (size_t)s * kFVBytes;
                const int32_t vrow = (int32_t)(kv * kFD);
                tma_load_2d(dv, &vt_map, t * kFN, vrow, &v_full[s], keep);
                tma_load_2d(dv + kFVBytes / 2, &vt_map, t * kFN + 64, vrow, &v_full[s], keep);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {  // ===== MMA issuer =====
            constexpr uint32_t idesc = idesc_bf16_f32<kFM, kFN>();
            mbar_wait(q_ready, 0);
            tc_fence_after();
            for (int t = 0; t <= n_tiles; ++t) {
                if (t < n_tiles) {  // S_t = Qhi·Khi + Qlo·Khi + Qhi·Klo
                    const int s = t % kFStages;
                    mbar_wait(&k_full[s], (t / kFStages) & 1u);
                    tc_fence_after();
                    const uint32_t kb = smem_u32(s_k + (size_t)s * 2 * kFKBytes);
                    const uint32_t d_s = tmem + (uint32_t)((t & 1) * kFN);
#pragma unroll
                    for (int term = 0; term < 3; ++term) {
                        const uint32_t qa = tmem + (term == 1 ? kColQlo : kColQhi);
                        const uint32_t kt = kb + (term == 2 ? kFKBytes : 0);
#pragma unroll
                        for (int ks = 0; ks < kFD / 16; ++ks) {
                            const uint64_t bd =
                                umma_desc_sw128(kt + (ks >> 2) * (kFKBytes / 2) + (ks & 3) * 32);
                            mma_bf16_ts(d_s, qa + ks * 8, bd, idesc, (term | ks) ? 1u : 0u);
                        }
                    }
                    mma_commit(&k_empty[s]);
                    mma_commit(&s_full[t & 1]);
                }
                if (t >= 1) {  // O += Phi_u·V_u + Plo_u·V_u, u = t - 1
                    const int u = t - 1, s = u % kFStages, b = u & 1;
                    mbar_wait(&p_full[b], (u >> 1) & 1u);
                    mbar_wait(&v_full[s], (u / kFStages) & 1u);
                    tc_fence_after();
                    const uint32_t vb = smem_u32(s_v + (size_t)s * kFVBytes);
#pragma unroll
                    for (int hl = 0; hl < 2; ++hl)
#pragma unroll
                        for (int ks = 0; ks < kFN / 16; ++ks) {
                            const uint64_t bd =
                                umma_desc_sw128(vb + (ks >> 2) * (kFVBytes / 2) + (ks & 3) * 32);
                            const uint32_t pa = tmem + (uint32_t)(b * kFN + hl * 64 + ks * 8);
                            mma_bf16_ts(tmem + kColO, pa, bd, idesc, (u | hl | ks) ? 1u : 0u);
                        }
                    mma_commit(&v_empty[s]);
                    mma_commit(o_done);
                }
            }
            mma_commit(o_final);
        }
    } else {
        // ===== softmax: two warps per TMEM lane quarter; thread = (query row, 64-column
        // half of every tile).  Both halves of a row keep the same reference max m2 (the
        // tile max is exchanged through shared memory), so A / B split additively. =====
        const int sw = warp - 2;          // 0..7
        const int quarter = warp & 3;     // TMEM lane quarter this warp may access
        const int half = sw >> 2;         // column half
        const int row = quarter * 32 + lane;
        const int i = q0 + row;
        const bool live = i < a.n_q;
        const uint32_t lane_base = tmem + ((uint32_t)(quarter * 32) << 16);
        float* s_max = (float*)(o_final + 2);       // [2 parity][2 half][128]
        double* s_ab = (double*)(s_max + 2 * 2 * kFM);  // [2 half][128][2]
        // query: rotated at L'-n_q+i (engine.hpp:88-93), times log2(e)/sqrt(d) (so S is
        // already in log2 units), split into bf16 hi + lo; this half writes pairs [32h, 32h+32)
        {
            const float* qrow = a.q + (size_t)(live ? i : 0) * a.q_row_stride + (size_t)h * kFD;
            const uint32_t pos = L - (uint32_t)a.n_q + (uint32_t)(live ? i : 0);
            uint32_t hw[32], lw[32];
#pragma unroll
            for (int j = 0; j < 32; ++j) {
                const int pj = half * 32 + j;
                const float2 xy = *(const float2*)(qrow + 2 * pj);
                float rx = xy.x, ry = xy.y;
                if (a.rope_cos)
                    rotate_pair(xy.x, xy.y, a.rope_cos[(size_t)pos * (kFD / 2) + pj],
                                a.rope_sin[(size_t)pos * (kFD / 2) + pj], rx, ry);
                rx = live ? __fmul_rn(rx, a.scale_log2) : 0.0f;
                ry = live ? __fmul_rn(ry, a.scale_log2) : 0.0f;
                hw[j] = pack_bf16x2(rx, ry);
                lw[j] = pack_bf16x2(__fsub_rn(rx, bf16_lo_half(hw[j])), __fsub_rn(ry, bf16_hi_half(hw[j])));
            }
            TMEM_ST_X32(lane_base + kColQhi + half * 32, hw);
            TMEM_ST_X32(lane_base + kColQlo + half * 32, lw);
            tmem_wait_st();
            tc_fence_before();
            mbar_arrive(q_ready);
        }
        // visible keys of this row: [0, lim)
        const uint32_t lim =
            !live ? 1u
                  : (a.causal ? (uint32_t)min((unsigned long long)L, (unsigned long long)boundary + i + 1)
                              : L);
        constexpr float kMasked = -1.0e30f;  // finite: 2^(masked - m2) == 0 and 0 * d == 0
        float m2 = -INFINITY;                // reference max, log2 units
        double A = 0.0, B2 = 0.0;
        for (int t = 0; t < n_tiles; ++t) {
            const int b = t & 1;
            mbar_wait(&s_full[b], (t >> 1) & 1u);
            tc_fence_after();
            float y[64];
            TMEM_LD_X64(lane_base + b * kFN + half * 64, ((uint32_t*)y));
            tmem_wait_ld();
            const uint32_t k0 = (uint32_t)t * kFN + half * 64;
            if (k0 + 64 > lim) {
#pragma unroll
                for (int c = 0; c < 64; ++c) y[c] = k0 + c < lim ? y[c] : kMasked;
            }
            float mx0 = y[0], mx1 = y[1];
#pragma unroll
            for (int c = 2; c < 64; c += 2) {
                mx0 = fmaxf(mx0, y[c]);
                mx1 = fmaxf(mx1, y[c + 1]);
            }
            float mx = fmaxf(mx0, mx1);
            s_max[(b * 2 + half) * kFM + row] = mx;
            named_bar_sync(1 + quarter, 64);
            mx = fmaxf(mx, s_max[(b * 2 + (half ^ 1)) * kFM + row]);
            // lazy rescale: move the reference max only when p could exceed 2^8
            float f = 1.0f;
            if (mx > m2 + kRescaleLog2) {
                if (m2 == -INFINITY) {
                    A = 0.0;
                    B2 = 0.0;
                } else {
                    f = exp2f(m2 - mx);
                    B2 = (double)f * (B2 + (double)(m2 - mx) * A);
                    A *= (double)f;
                }
                m2 = mx;
            }
            if (t > 0 && __any_sync(0xFFFFFFFFu, f != 1.0f)) {
                // O row (this half's 64 columns) *= f once the previous P·V has landed
                mbar_wait(o_done, (uint32_t)(t - 1) & 1u);
                tc_fence_after();
#pragma unroll 1
                for (int c0 = 0; c0 < 64; c0 += 32) {
                    uint32_t o[32];
                    TMEM_LD_X32(lane_base + kColO + half * 64 + c0, o);
                    tmem_wait_ld();
#pragma unroll
                    for (int c = 0; c < 32; ++c) o[c] = __float_as_uint(__uint_as_float(o[c]) * f);
                    TMEM_ST_X32(lane_base + kColO + half * 64 + c0, o);
                }
            }
            // p = 2^(y - m2) (packed pairs), tile sums, P hi / lo over the S columns
            const f2_t nm = f2_packf(-m2, -m2);
            f2_t at = 0ull, bt = 0ull;
            uint32_t hw[32], lw[32];
#pragma unroll
            for (int j = 0; j < 32; ++j) {
                const f2_t dd = f2_add(f2_packf(y[2 * j], y[2 * j + 1]), nm);
                const float p0 = ex2_approx(f2_lo(dd)), p1 = ex2_approx(f2_hi(dd));
                const f2_t pp = f2_packf(p0, p1);
                at = f2_add(at, pp);
                bt = f2_fma(pp, dd, bt);
                hw[j] = pack_bf16x2(p0, p1);
                const f2_t lo = f2_add(pp, bf16x2_to_f2(hw[j]) ^ 0x8000000080000000ull);
                lw[j] = pack_bf16x2(f2_lo(lo), f2_hi(lo));
            }
            TMEM_ST_X32(lane_base + b * kFN + half * 32, hw);
            TMEM_ST_X32(lane_base + b * kFN + 64 + half * 32, lw);
            tmem_wait_st();
            tc_fence_before();
            mbar_arrive(&p_full[b]);
            A += (double)__fadd_rn(f2_lo(at), f2_hi(at));
            B2 += (double)__fadd_rn(f2_lo(bt), f2_hi(bt));
        }
        // combine the halves' (A, B2) and wait for all P·V.  (o_done cannot tell: when this
        // thread gets here it may be 0, 1 or 2 completions short of n_tiles, and parity waits
        // for "n_tiles - 2" then "n_tiles - 1" hung whenever the last P·V had already landed
        // -- a rare race, seen as a hang after tens of replays.  o_final completes once.)
        s_ab[(half * kFM + row) * 2 + 0] = A;
        s_ab[(half * kFM + row) * 2 + 1] = B2;
        named_bar_sync(1 + quarter, 64);
        const double At = s_ab[row * 2 + 0] + s_ab[(kFM + row) * 2 + 0];
        const double Bt = s_ab[row * 2 + 1] + s_ab[(kFM + row) * 2 + 1];
        mbar_wait(o_final, 0u);
        tc_fence_after();
        const double inv = 1.0 / At;
#pragma unroll 1
        for (int c0 = 0; c0 < 64; c0 += 32) {
            uint32_t o[32];
            TMEM_LD_X32(lane_base + kColO + half * 64 + c0, o);
            tmem_wait_ld();
            if (live) {
                float4* dst = (float4*)(a.out + (size_t)i * a.n_head * kFD + (size_t)h * kFD +
                                        half * 64 + c0);
#pragma unroll
                for (int c = 0; c < 32; c += 4)
                    dst[c / 4] = make_float4((float)(__uint_as_float(o[c]) * inv),
                                             (float)(__uint_as_float(o[c + 1]) * inv),
                                             (float)(__uint_as_float(o[c + 2]) * inv),
                                             (float)(__uint_as_float(o[c + 3]) * inv));
            }
        }
        if (live && half == 0) {
            const double hh = log(At) - Bt * 0.69314718055994530942 / At;
            a.entropy[(size_t)i * a.n_head + h] = hh < 0.0 ? 0.0 : hh;
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

uint32_t flash_lpad(uint32_t L_max) { return (std::max<uint32_t>(1, L_max) + kFN - 1) / kFN * kFN; }

}  // namespace

bool attend_tc_supported(const AttnArgs& a) {
    return a.d == kFD && a.dv == kFD && a.dtype == kBF16 && a.n_q >= 1 && a.group >= 1 &&
           a.n_head == a.n_kv * a.group;
}

size_t attend_tc_workspace(const AttnArgs& a, uint32_t L_max) {
    return 3 * (size_t)a.n_kv * flash_lpad(L_max) * kFD * sizeof(__nv_bfloat16) + 1024;
}

cudaError_t launch_attend_tc(const AttnArgs& a, uint32_t L_max, void* ws, cudaStream_t s) {
    const uint32_t Lpad = flash_lpad(L_max);
    const size_t plane = (size_t)a.n_kv * Lpad * kFD;
    __nv_bfloat16* khi = (__nv_bfloat16*)ws;
    __nv_bfloat16* klo = khi + plane;
    __nv_bfloat16* vt = klo + plane;
    flash_prep_kernel<__nv_bfloat16><<<dim3(Lpad / 32, a.n_kv), 256, 0, s>>>(a, Lpad, khi, klo, vt);
    CUtensorMap mh, ml, mv;
    if (!make_key_tensor_map(&mh, khi, kBF16, kFD, (uint64_t)a.n_kv * Lpad, kFN) ||
        !make_key_tensor_map(&ml, klo, kBF16, kFD, (uint64_t)a.n_kv * Lpad, kFN) ||
        !make_key_tensor_map(&mv, vt, kBF16, Lpad, (uint64_t)a.n_kv * kFD, kFD))
        return cudaErrorInvalidValue;
    FlashArgs f;
    f.q = a.q;
    f.q_row_stride = a.q_row_stride;
    f.n_q = a.n_q;
    f.n_head = a.n_head;
    f.group = a.group;
    f.Lpad = Lpad;
    f.hdr = a.hdr;
    f.L_host = a.L_host;
    f.rope_cos = a.rope_cos;
    f.rope_sin = a.rope_sin;
    f.causal = a.causal;
    f.boundary_is_tail = a.boundary_is_tail;
    f.boundary_host = a.boundary_host;
    f.scale_log2 = (float)(1.4426950408889634 / std::sqrt((double)kFD));
    f.out = a.out;
    f.entropy = a.entropy;
    static bool once = (cudaFuncSetAttribute(flash_tc_kernel,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)kFSmem),
                        true);
    (void)once;
    dim3 grid((a.n_q + kFM - 1) / kFM, a.n_head);
    flash_tc_kernel<<<grid, kFThreads, kFSmem, s>>>(mh, ml, mv, f);
    return cudaGetLastError();
}

}  // namespace reattn_impl
