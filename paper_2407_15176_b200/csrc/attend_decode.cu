// K5 (decode) — finite-scope flash-decode with a deep bulk-copy ring and a fused combine.
//
// Restates, for n_q == 1 and a bf16 cache (d == dv == 128):
//   assemble_scope copies   scope.hpp:63-76   rows fetched straight from the cache through
//                                               the device scope table (no assembled copy)
//   RotaryTable::rotate_row rope.hpp:49-60    keys at compact i, the query at L'-1
//                                               (engine.hpp:78-93), unfused fp32 ops
//   attend                  attend.hpp:25-77  scale 1/sqrt(d), row entropy ln A - B/A
//
// The decode scope is small (L' ~ 5K rows, 21 MB of K+V at 1M context) and the step is
// latency-bound unless a large part of it is in flight at once, so the layout is:
//   grid (n_parts, n_kv), one CTA per SM (197 KB smem); part p of kv head h owns a
//   contiguous range of 32-row chunks of its rows (sized from the device L').
//   warp 16 (producer): per chunk, one cp.async.bulk per run of consecutive cache rows for K
//     and for V (gathered through the scope table) plus the chunk's RoPE cos / sin rows, into
//     a 6-stage ring of 32 KB stages.
//   warps 0-15 (compute): 4 groups of 4 warps take chunks round-robin; a group rotates the
//     chunk's keys once into fp32 over the stage's cos/sin area (XOR-swizzled), then one warp
//     per q head: lane j = key j logits (fp32, query pre-scaled by log2(e)/sqrt(d)), warp
//     max / sums by shuffle, online (m, A, B) state (A, B in f64), P·V with lane = 4 output
//     columns and p_j broadcast by shuffle.  The groups merge through shared memory.
//   The last CTA of each kv head (atomic ticket, re-armed for graph replay) merges the parts'
//   partial states in part order (deterministic) and writes the output and entropy, or one
//   merged partial row per head (sharded decode).
// Modes: the whole scope, the local window beside the scan (decode fork), the rows after it,
// or a rank's ShardRanges (see BulkArgs).
// Numerics: fp32 logits / accumulation within a CTA, f64 across parts: max-abs ~1e-8 on the
// reference's f64 attend at the decode geometry (north_star fp32 bar: 1e-5).
#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

using namespace reattn_dev;

namespace reattn_impl {

namespace {

constexpr int kBC = 32;                        // scope rows per chunk
constexpr int kBD = 128;                       // d = dv
constexpr int kBStages = 6;
constexpr int kBGroups = 4;                    // compute groups (4 warps each) per CTA
// chunks c and c - 2*kBStages must belong to the same group (see the consumer's stage wait)
static_assert((2 * kBStages) % kBGroups == 0, "stage ring / group interleave");
constexpr int kBKVBytes = kBC * kBD * 2;       // K or V of one chunk (bf16): 8 KB
constexpr int kBRopeBytes = kBC * (kBD / 2) * 4;  // cos or sin rows of one chunk: 8 KB
constexpr int kBStageBytes = 2 * kBKVBytes + 2 * kBRopeBytes;
constexpr int kBCompute = kBGroups * 128;
constexpr int kBThreads = kBCompute + 32;
constexpr int kBPartBytes = kDecodePartBytes;  // double m2, A, B2, pad; float acc[128]
constexpr int kBMaxParts = 160;          // partial slots per kv head (head + local)
constexpr int kBSxBytes = kBGroups * 4 * 4 * kBC * 4;  // G <= 4 logit partials [gi][warp][h][key]
constexpr size_t kBSmem = 1024 + (size_t)kBStages * kBStageBytes + 8ull * kBD * 4 + kBSxBytes +
                          (size_t)kBStages * kBC + 256;

enum { kModeScope = 0, kModeLocal = 1, kModeHead = 2, kModeRanges = 3 };

struct BulkArgs {
    AttnArgs a;
    int mode;               // kModeScope: scope rows [0, L') through the scope table
                            // kModeLocal: cache rows [local_row0, +n_local) at positions
                            //   0 .. n_local-1, query at n_local-1 (RoPE is relative: the
                            //   logits equal the scope frame's up to rounding); partials only
                            // kModeHead: scope rows [0, L'-n_local); merges the local partials
                            // kModeRanges: the scope rows of a ShardRanges (sharded decode);
                            //   the merged state goes to `merged` as partial rows
    uint32_t n_local, local_row0;
    const uint32_t* ranges;  // kModeRanges: device ShardRanges
    uint8_t* merged;         // non-null: write merged partial rows [n_head] instead of out
    int n_parts;            // CTAs per kv head in this launch
    int part_base;          // first partial slot of this launch
    int n_slots;            // partial slots per kv head (merged by the combine)
    float scale_log2;
    unsigned int* tickets;  // [n_kv]
    uint8_t* part;          // [n_slots][n_kv][G] partial rows
    uint64_t* trace;        // diagnostics (misc.cu layout) or null
    int warm;               // dry-run the merge before griddepcontrol.wait (see merge_parts)
    int local_post;         // kModeLocal launched after the scan (DecodeFork::post)
    int local_hpc;          // kModeLocal: kv heads per CTA, processed one after the other
    // growing caches: n_local / local_row0 derived from the device-resident cache length
    const uint32_t* dev_total;
    uint32_t l_global, l_local;
};

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ float bx_ex2(float x) {
    float r;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

// rotated fp32 key row r, float4 column i (XOR-swizzled: conflict-free row-per-lane reads)
__device__ __forceinline__ int rot_idx4(int r, int i) { return r * (kBD / 4) + (i ^ (r & 7)); }

// The last part of a kv head merges the parts' partial rows in part order and writes the
// output and entropy (attend.hpp:69-76 normalisation), or one merged partial row per head.
// `role` is the calling warp's compute-warp index.  This code runs once per launch and
// would run from a cold instruction cache (~0.5 us per fetch miss: ~9 us measured for the
// merge), so every CTA first runs it dry (global and shared stores predicated off) while it
// waits for the scan's merger CTA (griddepcontrol.wait): the lines are then resident in the
// SM's instruction cache when the last CTA runs it for real.  __noinline__ keeps both calls
// on the same code.
template <int G, int NW = 16>
__device__ __noinline__ void merge_parts(const BulkArgs& B, int kv, int role, uint8_t* stages, bool dry) {
    const AttnArgs& a = B.a;
    const int lane = threadIdx.x & 31;
    // WPH warps per q head, warp j summing slots j, j + WPH, ...: every load of the step (slot
    // headers by lane = slot, acc rows by lane = 4 columns) is issued before any is used, so
    // the merge costs one L2 round trip plus an in-order combine of the WPH partial sums
    // through shared memory (deterministic).  Few registers (no spills) and no f64 library
    // calls on the path: this code runs once per launch, cold.
    constexpr int WPH = NW == 16 ? (G == 1 ? 16 : G == 2 ? 8 : G <= 4 ? 4 : 2)
                                 : (G == 1 ? NW : G == 2 ? NW / 2 : G <= 4 ? NW / 4 : 1);
    static_assert(WPH >= 1 && G * WPH <= NW, "merge roles exceed the compute warps");
    constexpr int kPre = 8;  // acc rows in flight per lane
    double* xo = (double*)stages;  // [G][WPH][kBD] partial sums
    if (role < G * WPH) {
        const int g = role / WPH, j = role % WPH;
        __syncwarp();
        auto prow = [&](int p) {
            return B.part + (((size_t)p * a.n_kv + kv) * G + g) * kBPartBytes;
        };
        const int n_slots = B.n_slots;
        RA_ASSERT(n_slots <= kBMaxParts);
        double hm = -INFINITY, ha = 0.0, hb = 0.0;  // header of slot `lane` (first page)
        if (lane < n_slots) {
            const double* hd = (const double*)prow(lane);
            hm = __ldcg(hd);
            ha = __ldcg(hd + 1);
            hb = __ldcg(hd + 2);
        }
        float4 v[kPre];
#pragma unroll
        for (int u = 0; u < kPre; ++u) {
            const int p = j + WPH * u;
            v[u] = p < n_slots ? __ldcg(reinterpret_cast<const float4*>(prow(p) + 32) + lane)
                               : make_float4(0.f, 0.f, 0.f, 0.f);
        }
        double M = ha > 0.0 ? hm : -INFINITY;
        for (int p = lane + 32; p < n_slots; p += 32) {  // beyond one page (n_kv < 5)
            const double* hd = (const double*)prow(p);
            if (__ldcg(hd + 1) > 0.0) M = fmax(M, __ldcg(hd));
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) M = fmax(M, __shfl_xor_sync(0xFFFFFFFFu, M, off));
        // slot weight 2^(m_p - M): the m are fp32 values, so the f32 exp2 of their exact f64
        // difference is within 2^-22 relative
        auto wgt = [&](double pm, double pa) -> double {
            return pa > 0.0 ? (double)exp2f((float)(pm - M)) : 0.0;
        };
        const double w0 = wgt(hm, ha);
        double At = ha * w0, Bt = w0 * (hb + (hm - M) * ha);
        if (!(ha > 0.0)) At = Bt = 0.0;
        for (int p = lane + 32; p < n_slots; p += 32) {
            const double* hd = (const double*)prow(p);
            const double pm = __ldcg(hd), pa = __ldcg(hd + 1), pb = __ldcg(hd + 2);
            if (pa > 0.0) {
                const double w = wgt(pm, pa);
                At += pa * w;
                Bt += w * (pb + (pm - M) * pa);
            }
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            At += __shfl_xor_sync(0xFFFFFFFFu, At, off);
            Bt += __shfl_xor_sync(0xFFFFFFFFu, Bt, off);
        }
        if (!dry && B.trace && lane == 0 && role == 0 && kv < 64) B.trace[3664 + kv] = globaltimer();
        auto weight = [&](int p) -> double {  // page 0 by shuffle, later pages from the header
            if (p < 32) return __shfl_sync(0xFFFFFFFFu, w0, p);
            const double* hd = (const double*)prow(p);
            return wgt(__ldcg(hd), __ldcg(hd + 1));
        };
        double o0 = 0.0, o1 = 0.0, o2 = 0.0, o3 = 0.0;
        for (int u0 = 0; j + WPH * u0 < n_slots; u0 += kPre) {
            if (u0 > 0) {
#pragma unroll
                for (int u = 0; u < kPre; ++u) {
                    const int p = j + WPH * (u0 + u);
                    v[u] = p < n_slots ? __ldcg(reinterpret_cast<const float4*>(prow(p) + 32) + lane)
                                       : make_float4(0.f, 0.f, 0.f, 0.f);
                }
            }
#pragma unroll
            for (int u = 0; u < kPre; ++u) {
                const int p = j + WPH * (u0 + u);
                const double w = weight(min(p, n_slots - 1));  // shuffle: the whole warp
                if (p < n_slots) {
                    o0 = fma((double)v[u].x, w, o0);
                    o1 = fma((double)v[u].y, w, o1);
                    o2 = fma((double)v[u].z, w, o2);
                    o3 = fma((double)v[u].w, w, o3);
                }
            }
        }
        if (!dry) {  // dry: the stage ring is live, keep out of shared memory
            double* mine = xo + ((size_t)(g * WPH + j) * kBD + 4 * lane);
            mine[0] = o0;
            mine[1] = o1;
            mine[2] = o2;
            mine[3] = o3;
            named_bar_sync(6, G * WPH * 32);
        }
        if (j == 0) {
            double r[4] = {0.0, 0.0, 0.0, 0.0};
            for (int jj = 0; jj < WPH; ++jj) {
                const double* o = xo + ((size_t)(g * WPH + jj) * kBD + 4 * lane);
#pragma unroll
                for (int c = 0; c < 4; ++c) r[c] += o[c];
            }
            const double inv = 1.0 / At;
            const int h = kv * G + g;
            if (B.merged) {  // one partial row per q head (sharded decode: combined across ranks)
                uint8_t* row = B.merged + (size_t)h * kBPartBytes;
                if (!dry)
                    reinterpret_cast<float4*>(row + 32)[lane] =
                        make_float4((float)r[0], (float)r[1], (float)r[2], (float)r[3]);
                if (lane == 0 && !dry) {
                    double* hd = (double*)row;
                    hd[0] = M;
                    hd[1] = At;
                    hd[2] = Bt;
                }
            } else {
                const float4 o4 = make_float4((float)(r[0] * inv), (float)(r[1] * inv),
                                              (float)(r[2] * inv), (float)(r[3] * inv));
                // computed in the warm-up too (the f64 log is a long routine that would
                // otherwise run cold); the asm keeps it from sinking into the store branch
                const double hh = log(At) - Bt * 0.69314718055994530942 * inv;
                asm volatile("" ::"d"(hh), "f"(o4.x), "f"(o4.y), "f"(o4.z), "f"(o4.w));
                if (!dry) reinterpret_cast<float4*>(a.out + (size_t)h * kBD)[lane] = o4;
                if (lane == 0 && !dry) a.entropy[h] = hh < 0.0 ? 0.0 : hh;
            }
        }
    }
}

template <int G>
__global__ void __launch_bounds__(kBThreads, 1) attend_decode_bulk_kernel(const __grid_constant__ BulkArgs B) {
    const AttnArgs& a = B.a;
    // while the scan's merger CTA still runs its tail: warm the merge code (see merge_parts)
    extern __shared__ __align__(16) uint8_t bsm_raw[];
    if (B.trace && threadIdx.x == 0 && blockIdx.x == 0 && blockIdx.y == 0) B.trace[3904] = globaltimer();
    if (B.warm && threadIdx.x < 32) merge_parts<G>(B, blockIdx.y, 0, bsm_raw, true);
    const bool local = B.mode == kModeLocal;  // independent of the selection: never reads the header
    // launched as a programmatic dependent of the scan / select: wait for its results (a
    // post-scan local launch waits at its end instead: it does not read them)
    if (!local) asm volatile("griddepcontrol.wait;" ::: "memory");
    // a post-scan local launch lets the head launch become resident as its CTAs retire
    if (local && B.local_post) asm volatile("griddepcontrol.launch_dependents;");
    if (!local && a.hdr && a.hdr->error != 0) return;
    uint32_t n_local = B.n_local, local_row0 = B.local_row0;
    if (B.dev_total) {  // kv_cache.hpp:65-67 on the device cache length
        uint32_t total;
        asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(total) : "l"(B.dev_total));
        const uint32_t g_end = min(total, B.l_global);
        local_row0 = total - min(total - g_end, B.l_local);
        n_local = total - local_row0;
    }
    const uint32_t L = local ? n_local : (a.hdr ? a.hdr->L : a.L_host);
    const uint32_t rows = B.mode == kModeHead ? L - n_local : L;
    const int part = blockIdx.x;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int cta_id = blockIdx.y * gridDim.x + blockIdx.x + (local ? 512 : 0);  // trace slot
    if (B.trace && tid == 0 && cta_id < 1024) B.trace[1536 + cta_id] = globaltimer();
    // the local window may give a CTA several kv heads (fewer SMs lent by the scan)
    const int hpc = local ? max(1, B.local_hpc) : 1;
#pragma unroll 1
    for (int hh = 0; hh < hpc; ++hh) {
    const int kv = blockIdx.y * hpc + hh;
    if (hh > 0) __syncthreads();  // the previous head's stages and barriers are idle
    ShardRanges R;
    R.n = 0;
    int chunks;
    if (B.mode == kModeRanges) {
        R = *(const ShardRanges*)B.ranges;
        chunks = 0;
        for (uint32_t i = 0; i < R.n; ++i) chunks += (int)((R.end[i] - R.begin[i] + kBC - 1) / kBC);
    } else {
        chunks = (int)((rows + kBC - 1) / kBC);
    }
    // chunk -> first scope row and row count (kModeRanges: chunks never straddle ranges)
    auto geom = [&](int cg, uint32_t& k0, int& nk) {
        if (B.mode != kModeRanges) {
            k0 = (uint32_t)cg * kBC;
            nk = (int)min((uint32_t)kBC, rows - k0);
            return;
        }
        for (uint32_t i = 0; i < R.n; ++i) {
            const int cc = (int)((R.end[i] - R.begin[i] + kBC - 1) / kBC);
            if (cg < cc) {
                k0 = R.begin[i] + (uint32_t)cg * kBC;
                nk = (int)min((uint32_t)kBC, R.end[i] - k0);
                return;
            }
            cg -= cc;
        }
        k0 = 0;
        nk = 0;
    };
    const int cpp = (chunks + B.n_parts - 1) / B.n_parts;
    const int c_begin = part * cpp;
    const int n_ch = max(0, min(chunks, c_begin + cpp) - c_begin);
    constexpr int HPW = (G + 3) / 4;  // q heads per compute warp

    // addressed straight from the shared array (an integer round trip for alignment would
    // turn every access into a generic load); bulk copies only need 16-B alignment
    uint8_t* stages = bsm_raw;
    float* qs = (float*)(stages + kBStages * kBStageBytes);  // [8][kBD]
    float* sx = qs + 8 * kBD;                                 // kBSxBytes (G <= 4 path)
    uint8_t* rowok = (uint8_t*)sx + kBSxBytes;                // [kBStages][kBC]
    uint64_t* full = (uint64_t*)(rowok + kBStages * kBC);  // 8-B aligned: offsets are multiples of 64
    uint64_t* empty = full + kBStages;
    __shared__ unsigned int s_last;

    if (tid == 0) {
        for (int s = 0; s < kBStages; ++s) {
            if (hh > 0) {  // the previous kv head's barriers are idle (synced above): retire them
                mbar_inval(&full[s]);
                mbar_inval(&empty[s]);
            }
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 4);  // the 4 warps of the group that consumed the stage
        }
        fence_barrier_init();
    }
    __syncthreads();

    if (warp == kBCompute / 32) {
        // ===== producer: bulk copies of the chunk's rows into the ring =====
        for (int c = 0; c < n_ch; ++c) {
            const int s = c % kBStages;
            if (c >= kBStages) mbar_wait(&empty[s], ((c / kBStages) & 1u) ^ 1u);
            uint32_t k0;
            int nk;
            geom(c_begin + c, k0, nk);
            uint8_t* st = stages + (size_t)s * kBStageBytes;
            const bool valid = lane < nk;
            const uint32_t cr = !valid ? kNoIndex
                                : local ? local_row0 + k0 + lane
                                : (a.src ? __ldg(a.src + k0 + lane) : k0 + lane);
            const bool own = valid && cr != kNoIndex;  // sharded scopes mask rows owned elsewhere
            const int n_own = __popc(__ballot_sync(0xFFFFFFFFu, own));
            rowok[s * kBC + lane] = own ? 1 : 0;
            if (!own) {  // masked / tail row: zeros keep 0 * v finite in the (always 32-row) P·V
                uint4* kz = (uint4*)(st + lane * kBD * 2);
                uint4* vz = (uint4*)(st + kBKVBytes + lane * kBD * 2);
#pragma unroll
                for (int i = 0; i < kBD * 2 / 16; ++i) kz[i] = vz[i] = make_uint4(0, 0, 0, 0);
            }
            __syncwarp();
            const uint32_t bytes = (uint32_t)n_own * 2u * kBD * 2u + (a.rope_cos ? 2u * nk * (kBD / 2) * 4u : 0u);
            if (lane == 0) mbar_arrive_expect_tx(&full[s], bytes);
            __syncwarp();
            // one copy per run of consecutive cache rows (spans are 32-row runs, the global
            // and local segments are contiguous): bulk copies take uniform operands, so
            // per-lane copies would serialise across the warp
            const uint32_t cr_prev = __shfl_up_sync(0xFFFFFFFFu, cr, 1);
            const bool own_prev = __shfl_up_sync(0xFFFFFFFFu, own ? 1 : 0, 1) != 0;
            const bool head = own && !(lane > 0 && own_prev && cr == cr_prev + 1u);
            const uint32_t heads = __ballot_sync(0xFFFFFFFFu, head);
            const uint32_t breaks = heads | __ballot_sync(0xFFFFFFFFu, !own);
            if (head) {
                RA_ASSERT(cr < a.head_stride);
                const uint32_t later = lane == 31 ? 0u : breaks & ~((2u << lane) - 1u);
                const int end = later ? __ffs(later) - 1 : 32;
                const uint32_t bytes_run = (uint32_t)(end - lane) * kBD * 2u;
                RA_ASSERT(cr + (uint32_t)(end - lane) <= a.head_stride);
                const size_t row = ((size_t)kv * a.head_stride + cr) * kBD;
                bulk_g2s(st + lane * kBD * 2, (const __nv_bfloat16*)a.k_base + row, bytes_run, &full[s]);
                bulk_g2s(st + kBKVBytes + lane * kBD * 2, (const __nv_bfloat16*)a.v_base + row, bytes_run,
                         &full[s]);
            }
            if (B.trace && lane == 0 && blockIdx.x == 0 && blockIdx.y == 0 && c < 64)
                B.trace[3712 + c] = globaltimer();  // chunk c's copies issued (CTA (0, 0))
            if (a.rope_cos && lane < 2) {
                const float* tab = lane == 0 ? a.rope_cos : a.rope_sin;
                bulk_g2s(st + 2 * kBKVBytes + lane * kBRopeBytes, tab + (size_t)k0 * (kBD / 2),
                         (uint32_t)nk * (kBD / 2) * 4u, &full[s]);
            }
        }
        __syncthreads();  // matches the compute side's state exchange barrier
    } else {
        // ===== compute: group gi = warps 4gi .. 4gi+3 takes chunks gi, gi+4, ... =====
        const int gi = warp >> 2, gw = warp & 3, gt = tid & 127;
        // the group's queries, rotated at L'-1 (engine.hpp:88-93), times log2(e)/sqrt(d)
        const uint32_t qpos = L - 1u;  // kModeLocal: L == n_local (shifted frame)
        for (int e = tid; e < G * (kBD / 2); e += kBCompute) {
            const int g = e / (kBD / 2), j = e % (kBD / 2);
            const float* qrow = a.q + (size_t)(kv * G + g) * kBD;
            const float x = qrow[2 * j], y = qrow[2 * j + 1];
            float rx = x, ry = y;
            if (a.rope_cos) {
                const float cs = a.rope_cos[(size_t)qpos * (kBD / 2) + j];
                const float sn = a.rope_sin[(size_t)qpos * (kBD / 2) + j];
                rx = __fsub_rn(__fmul_rn(x, cs), __fmul_rn(y, sn));
                ry = __fadd_rn(__fmul_rn(x, sn), __fmul_rn(y, cs));
            }
            qs[g * kBD + 2 * j] = __fmul_rn(rx, B.scale_log2);
            qs[g * kBD + 2 * j + 1] = __fmul_rn(ry, B.scale_log2);
        }
        named_bar_sync(5, kBCompute);
        if constexpr (G <= 4) {
        // ---- G <= 4: lane = (key kl of the warp's 8, q head hd); each warp keeps its own
        // online-softmax state for its key slice (no per-chunk exchange), merged at the end.
        // Logits read the rotated keys once per warp for all heads (8 rows x 16 B + 4 query
        // float4 per step: 2 wavefronts), P.V reads each V row once for all heads (lane = 4
        // columns): ~2x fewer shared-memory wavefronts than one warp per head.
        const int kl = lane & 7, hd = lane >> 3;
        const int r = 8 * gw + kl;  // this lane's key row within the chunk
        // every lane tracks every head's running max (to rescale its acc columns); the f64
        // sums A (softmax denominator) and B2 (entropy numerator) only for its own head
        float m2[4];
        double A = 0.0, B2 = 0.0;
        f2_t o01[4], o23[4];
#pragma unroll
        for (int h = 0; h < 4; ++h) {
            m2[h] = -INFINITY;
            o01[h] = o23[h] = 0ull;
        }
        for (int c = gi; c < n_ch; c += kBGroups) {
            const int s = c % kBStages;
            // see the parity note in the G > 4 path
            if (c >= kBStages) mbar_wait(&empty[s], ((c / kBStages) - 1) & 1u);
            mbar_wait(&full[s], (c / kBStages) & 1u);
            __syncwarp();
            const bool tr = B.trace && gw == 0 && lane == 0 && blockIdx.x == 0 && blockIdx.y == 0 && c < 64;
            if (tr) B.trace[3776 + c] = globaltimer();  // chunk c landed (group gi)
            uint32_t k0;
            int nk;
            geom(c_begin + c, k0, nk);
            uint8_t* st = stages + (size_t)s * kBStageBytes;
            float4* kr4 = (float4*)(st + 2 * kBKVBytes);  // rotated keys over the cos/sin rows
            {
                const uint32_t* kw = (const uint32_t*)st;  // bf16 pairs
                const float* cs = (const float*)(st + 2 * kBKVBytes);
                const float* sn = (const float*)(st + 2 * kBKVBytes + kBRopeBytes);
                float2 rot[kBC * (kBD / 2) / 128];
#pragma unroll
                for (int i = 0; i < kBC * (kBD / 2) / 128; ++i) {
                    const int e = gt + 128 * i, rr = e >> 6, j = e & 63;
                    const uint32_t w = kw[rr * (kBD / 2) + j];
                    const float x = __uint_as_float(w << 16), y = __uint_as_float(w & 0xFFFF0000u);
                    float rx = x, ry = y;
                    if (a.rope_cos && rr < nk) {
                        const float cc = cs[rr * (kBD / 2) + j], ss = sn[rr * (kBD / 2) + j];
                        rx = __fsub_rn(__fmul_rn(x, cc), __fmul_rn(y, ss));
                        ry = __fadd_rn(__fmul_rn(x, ss), __fmul_rn(y, cc));
                    }
                    rot[i] = make_float2(rx, ry);
                }
                named_bar_sync(1 + gi, 128);  // every read of cos / sin done
#pragma unroll
                for (int i = 0; i < kBC * (kBD / 2) / 128; ++i) {
                    const int e = gt + 128 * i, rr = e >> 6, j = e & 63;
                    float* dst = (float*)&kr4[rot_idx4(rr, j >> 1)] + (j & 1) * 2;
                    *(float2*)dst = rot[i];
                }
                named_bar_sync(1 + gi, 128);  // rotated keys ready
                __syncwarp();
            }
            const bool key_ok = hd < G && r < nk && rowok[s * kBC + r];
            // logits, split over the group's warps by dimension: warp gw sums dims
            // [32 gw, 32 gw + 32) for all 32 keys (lane = key) and all heads, so one rotated-key
            // LDS.128 serves G heads and the query float4s are warp-uniform broadcasts; the four
            // partials meet in shared memory and are summed in warp order
            {
                const ulonglong2* kv4 = reinterpret_cast<const ulonglong2*>(kr4);
                f2_t d01[G], d23[G];
#pragma unroll
                for (int h = 0; h < G; ++h) d01[h] = d23[h] = 0ull;
#pragma unroll
                for (int i = 8 * gw; i < 8 * gw + 8; ++i) {
                    const ulonglong2 k4 = kv4[rot_idx4(lane, i)];
#pragma unroll
                    for (int h = 0; h < G; ++h) {
                        const ulonglong2 q4 = reinterpret_cast<const ulonglong2*>(qs + h * kBD)[i];
                        d01[h] = f2_fma(q4.x, k4.x, d01[h]);
                        d23[h] = f2_fma(q4.y, k4.y, d23[h]);
                    }
                }
                float* sxg = sx + gi * (4 * 4 * kBC);  // [warp][h][key]
#pragma unroll
                for (int h = 0; h < G; ++h)
                    sxg[(gw * 4 + h) * kBC + lane] =
                        (f2_lo(d01[h]) + f2_hi(d01[h])) + (f2_lo(d23[h]) + f2_hi(d23[h]));
                named_bar_sync(1 + gi, 128);  // partial logits ready
            }
            float sc = -INFINITY;
            if (key_ok) {
                const float* sxg = sx + gi * (4 * 4 * kBC);
                sc = ((sxg[(0 * 4 + hd) * kBC + r] + sxg[(1 * 4 + hd) * kBC + r]) +
                      sxg[(2 * 4 + hd) * kBC + r]) + sxg[(3 * 4 + hd) * kBC + r];
            }
            float mc = sc;
#pragma unroll
            for (int off = 1; off < 8; off <<= 1) mc = fmaxf(mc, __shfl_xor_sync(0xFFFFFFFFu, mc, off));
            float mn[4], f[4];
#pragma unroll
            for (int h = 0; h < 4; ++h) {
                mn[h] = fmaxf(m2[h], __shfl_sync(0xFFFFFFFFu, mc, 8 * h));
                // m2 == -inf (only masked rows so far): f == 0 and the state stays empty
                f[h] = m2[h] != -INFINITY ? bx_ex2(m2[h] - mn[h]) : 0.0f;
            }
            const float mine = hd == 0 ? mn[0] : hd == 1 ? mn[1] : hd == 2 ? mn[2] : mn[3];
            const float fo = hd == 0 ? f[0] : hd == 1 ? f[1] : hd == 2 ? f[2] : f[3];
            const float mo = hd == 0 ? m2[0] : hd == 1 ? m2[1] : hd == 2 ? m2[2] : m2[3];
            const float dd = sc - mine;
            const float p = key_ok ? bx_ex2(dd) : 0.0f;
            float sa = p, sb = key_ok ? dd * p : 0.0f;
#pragma unroll
            for (int off = 1; off < 8; off <<= 1) {
                sa += __shfl_xor_sync(0xFFFFFFFFu, sa, off);
                sb += __shfl_xor_sync(0xFFFFFFFFu, sb, off);
            }
            B2 = (A > 0.0 ? (double)fo * (B2 + (double)(mo - mine) * A) : 0.0) + (double)sb;
            A = A * (double)fo + (double)sa;
#pragma unroll
            for (int h = 0; h < 4; ++h) {
                m2[h] = mn[h];
                const f2_t ff = f2_packf(f[h], f[h]);
                o01[h] = f2_mul(o01[h], ff);
                o23[h] = f2_mul(o23[h], ff);
            }
            // P.V over the warp's 8 keys, all heads (rows >= nk are zero with p == 0)
            const uint2* vrow = reinterpret_cast<const uint2*>(st + kBKVBytes) + lane;  // 4 bf16
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const uint2 w = vrow[(8 * gw + j) * (kBD / 4)];
                const f2_t v01 = bf16x2_to_f2(w.x), v23 = bf16x2_to_f2(w.y);
#pragma unroll
                for (int h = 0; h < G; ++h) {
                    const float pj = __shfl_sync(0xFFFFFFFFu, p, j + 8 * h);
                    const f2_t pp = f2_packf(pj, pj);
                    o01[h] = f2_fma(pp, v01, o01[h]);
                    o23[h] = f2_fma(pp, v23, o23[h]);
                }
            }
            __syncwarp();
            if (tr) B.trace[3840 + c] = globaltimer();  // chunk c consumed
            if (lane == 0) mbar_arrive(&empty[s]);
        }
        // ---- merge the 16 warps' states per head through shared memory ----
        __syncthreads();  // every stage consumed: reuse the ring as exchange space
        constexpr int NW = kBCompute / 32;
        double* xs = (double*)stages;                                  // [warp][g][4]
        float* xa = (float*)(stages + NW * 4 * 4 * sizeof(double));    // [warp][g][kBD]
#pragma unroll
        for (int h = 0; h < G; ++h)
            reinterpret_cast<float4*>(xa + (warp * 4 + h) * kBD)[lane] =
                make_float4(f2_lo(o01[h]), f2_hi(o01[h]), f2_lo(o23[h]), f2_hi(o23[h]));
        if (kl == 0 && hd < G) {
            xs[(warp * 4 + hd) * 4 + 0] = (double)(hd == 0 ? m2[0] : hd == 1 ? m2[1] : hd == 2 ? m2[2] : m2[3]);
            xs[(warp * 4 + hd) * 4 + 1] = A;
            xs[(warp * 4 + hd) * 4 + 2] = B2;
        }
        named_bar_sync(5, kBCompute);
        if (warp < G) {  // warp g combines head g's 16 warp states in warp order
            const int g = warp;
            double M = -INFINITY;
#pragma unroll
            for (int k = 0; k < NW; ++k)
                if (xs[(k * 4 + g) * 4 + 1] > 0.0) M = fmax(M, xs[(k * 4 + g) * 4 + 0]);
            double At = 0.0, Bt = 0.0;
            float4 o = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 4
            for (int k = 0; k < NW; ++k) {
                const double km = xs[(k * 4 + g) * 4 + 0], ka = xs[(k * 4 + g) * 4 + 1];
                if (!(ka > 0.0)) continue;
                const double w = (double)exp2f((float)(km - M));
                At += ka * w;
                Bt += w * (xs[(k * 4 + g) * 4 + 2] + (km - M) * ka);
                const float4 x = reinterpret_cast<const float4*>(xa + (k * 4 + g) * kBD)[lane];
                const float wf = (float)w;
                o.x = __fmaf_rn(x.x, wf, o.x);
                o.y = __fmaf_rn(x.y, wf, o.y);
                o.z = __fmaf_rn(x.z, wf, o.z);
                o.w = __fmaf_rn(x.w, wf, o.w);
            }
            uint8_t* row = B.part + (((size_t)(B.part_base + part) * a.n_kv + kv) * G + g) * kBPartBytes;
            reinterpret_cast<float4*>(row + 32)[lane] = o;
            if (lane == 0) {
                double* hdp = (double*)row;
                hdp[0] = M;
                hdp[1] = At;
                hdp[2] = Bt;
            }
        }
        } else {
        float m2[HPW];
        double A[HPW], B2[HPW];
        float4 acc[HPW];
#pragma unroll
        for (int u = 0; u < HPW; ++u) {
            m2[u] = -INFINITY;
            A[u] = 0.0;
            B2[u] = 0.0;
            acc[u] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
        for (int c = gi; c < n_ch; c += kBGroups) {
            const int s = c % kBStages;
            // Stage s holds chunks c-6, c, c+6 ... consumed by DIFFERENT groups, so a parity
            // wait on full[s] alone could be satisfied by chunk c-6's completed phase while
            // chunk c is not loaded yet.  Wait for chunk c-6's release first (unambiguous:
            // chunk c-12 belongs to this group and is consumed); after it, full[s] is at most
            // one phase ahead of what we wait for.
            if (c >= kBStages) mbar_wait(&empty[s], ((c / kBStages) - 1) & 1u);
            mbar_wait(&full[s], (c / kBStages) & 1u);
            __syncwarp();  // reconverge after the wait loop: the shuffles below stay simple
            uint32_t k0;
            int nk;
            geom(c_begin + c, k0, nk);
            uint8_t* st = stages + (size_t)s * kBStageBytes;
            float4* kr4 = (float4*)(st + 2 * kBKVBytes);  // rotated keys over the cos/sin rows
            // ---- rotate the chunk's keys once (rope.hpp:49-60): read all, then write ----
            {
                const uint32_t* kw = (const uint32_t*)st;  // bf16 pairs
                const float* cs = (const float*)(st + 2 * kBKVBytes);
                const float* sn = (const float*)(st + 2 * kBKVBytes + kBRopeBytes);
                float2 rot[kBC * (kBD / 2) / 128];
#pragma unroll
                for (int i = 0; i < kBC * (kBD / 2) / 128; ++i) {
                    const int e = gt + 128 * i, r = e >> 6, j = e & 63;
                    const uint32_t w = kw[r * (kBD / 2) + j];
                    const float x = __uint_as_float(w << 16), y = __uint_as_float(w & 0xFFFF0000u);
                    float rx = x, ry = y;
                    if (a.rope_cos && r < nk) {
                        const float cc = cs[r * (kBD / 2) + j], ss = sn[r * (kBD / 2) + j];
                        rx = __fsub_rn(__fmul_rn(x, cc), __fmul_rn(y, ss));
                        ry = __fadd_rn(__fmul_rn(x, ss), __fmul_rn(y, cc));
                    }
                    rot[i] = make_float2(rx, ry);
                }
                named_bar_sync(1 + gi, 128);  // every read of cos / sin done
#pragma unroll
                for (int i = 0; i < kBC * (kBD / 2) / 128; ++i) {
                    const int e = gt + 128 * i, r = e >> 6, j = e & 63;
                    float* dst = (float*)&kr4[rot_idx4(r, j >> 1)] + (j & 1) * 2;
                    *(float2*)dst = rot[i];
                }
                named_bar_sync(1 + gi, 128);  // rotated keys ready
                __syncwarp();
            }
            const bool key_ok = lane < nk && rowok[s * kBC + lane];
            const uint2* vrow = reinterpret_cast<const uint2*>(st + kBKVBytes) + lane;  // 4 bf16
#pragma unroll
            for (int u = 0; u < HPW; ++u) {
                const int g = gw + 4 * u;
                if (g >= G) break;
                const ulonglong2* qv = reinterpret_cast<const ulonglong2*>(qs + g * kBD);
                const ulonglong2* kv4 = reinterpret_cast<const ulonglong2*>(kr4);
                f2_t d01 = 0ull, d23 = 0ull;
#pragma unroll 8
                for (int i = 0; i < kBD / 4; ++i) {
                    const ulonglong2 k4 = kv4[rot_idx4(lane, i)], q4 = qv[i];
                    d01 = f2_fma(q4.x, k4.x, d01);
                    d23 = f2_fma(q4.y, k4.y, d23);
                }
                const float d0 = f2_lo(d01), d1 = f2_hi(d01), d2 = f2_lo(d23), d3 = f2_hi(d23);
                const float sc = key_ok ? (d0 + d1) + (d2 + d3) : -INFINITY;
                float mc = sc;
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) mc = fmaxf(mc, __shfl_xor_sync(0xFFFFFFFFu, mc, off));
                // mn == -inf (only masked rows so far) leaves p == 0, f == 0, A == B2 == 0
                const float mn = fmaxf(m2[u], mc);
                const float dd = sc - mn;
                const float p = key_ok ? bx_ex2(dd) : 0.0f;
                float sa = p, sb = key_ok ? dd * p : 0.0f;
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) {
                    sa += __shfl_xor_sync(0xFFFFFFFFu, sa, off);
                    sb += __shfl_xor_sync(0xFFFFFFFFu, sb, off);
                }
                const float f = A[u] > 0.0 ? bx_ex2(m2[u] - mn) : 0.0f;
                B2[u] = (A[u] > 0.0 ? (double)f * (B2[u] + (double)(m2[u] - mn) * A[u]) : 0.0) + (double)sb;
                A[u] = A[u] * (double)f + (double)sa;
                m2[u] = mn;
                const f2_t ff = f2_packf(f, f);
                f2_t o01 = f2_mul(f2_packf(acc[u].x, acc[u].y), ff);
                f2_t o23 = f2_mul(f2_packf(acc[u].z, acc[u].w), ff);
                auto pv = [&](int j) {
                    const float pj = __shfl_sync(0xFFFFFFFFu, p, j);
                    const f2_t pp = f2_packf(pj, pj);
                    const uint2 w = vrow[j * (kBD / 4)];
                    o01 = f2_fma(pp, bf16x2_to_f2(w.x), o01);
                    o23 = f2_fma(pp, bf16x2_to_f2(w.y), o23);
                };
#pragma unroll
                for (int j = 0; j < kBC; ++j) pv(j);  // rows >= nk are zero with p == 0
                const float4 o = make_float4(f2_lo(o01), f2_hi(o01), f2_lo(o23), f2_hi(o23));
                acc[u] = o;
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
        }
        // ---- merge the 4 groups' states per head through shared memory ----
        __syncthreads();  // every stage consumed: reuse the ring as exchange space
        double* xs = (double*)stages;                                  // [gi][g][4]
        float* xa = (float*)(stages + kBGroups * 8 * 4 * sizeof(double));  // [gi][g][kBD]
#pragma unroll
        for (int u = 0; u < HPW; ++u) {
            const int g = gw + 4 * u;
            if (g >= G) break;
            reinterpret_cast<float4*>(xa + (gi * 8 + g) * kBD)[lane] = acc[u];
            if (lane == 0) {
                xs[(gi * 8 + g) * 4 + 0] = (double)m2[u];
                xs[(gi * 8 + g) * 4 + 1] = A[u];
                xs[(gi * 8 + g) * 4 + 2] = B2[u];
            }
        }
        named_bar_sync(5, kBCompute);
        if (gi == 0) {
#pragma unroll
            for (int u = 0; u < HPW; ++u) {
                const int g = gw + 4 * u;
                if (g >= G) break;
                double M = -INFINITY;
#pragma unroll
                for (int k = 0; k < kBGroups; ++k)
                    if (xs[(k * 8 + g) * 4 + 1] > 0.0) M = fmax(M, xs[(k * 8 + g) * 4 + 0]);
                double At = 0.0, Bt = 0.0;
                float4 o = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
                for (int k = 0; k < kBGroups; ++k) {
                    const double km = xs[(k * 8 + g) * 4 + 0], ka = xs[(k * 8 + g) * 4 + 1];
                    if (!(ka > 0.0)) continue;
                    const double w = exp2(km - M);
                    At += ka * w;
                    Bt += w * (xs[(k * 8 + g) * 4 + 2] + (km - M) * ka);
                    const float4 x = reinterpret_cast<const float4*>(xa + (k * 8 + g) * kBD)[lane];
                    const float wf = (float)w;
                    o.x = __fmaf_rn(x.x, wf, o.x);
                    o.y = __fmaf_rn(x.y, wf, o.y);
                    o.z = __fmaf_rn(x.z, wf, o.z);
                    o.w = __fmaf_rn(x.w, wf, o.w);
                }
                uint8_t* row = B.part + (((size_t)(B.part_base + part) * a.n_kv + kv) * G + g) * kBPartBytes;
                reinterpret_cast<float4*>(row + 32)[lane] = o;
                if (lane == 0) {
                    double* hd = (double*)row;
                    hd[0] = M;
                    hd[1] = At;
                    hd[2] = Bt;
                }
            }
        }
        }  // G > 4
    }
    // ---- the last part of this kv head merges (attend.hpp:69-76 normalisation) ----
    if (B.trace && tid == 0 && cta_id < 1024) B.trace[2560 + cta_id] = globaltimer();
    if (local) {
        if (hh + 1 < hpc) continue;
        // complete only after the scan (and its merger CTA): the head launch's
        // griddepcontrol.wait then covers the scope as well as these partials
        if (B.local_post) asm volatile("griddepcontrol.wait;" ::: "memory");
        return;
    }
    __threadfence();
    __syncthreads();
    if (tid == 0) s_last = atomicAdd(&B.tickets[kv], 1u) == (unsigned)B.n_parts - 1u;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    if (B.trace && tid == 0 && kv < 64) B.trace[3600 + kv] = globaltimer();
    merge_parts<G>(B, kv, warp, stages, false);
    if (tid == 0) B.tickets[kv] = 0u;  // re-arm for the next launch (graph replay)
    if (B.trace) {
        __syncthreads();
        if (tid == 0 && kv < 512) B.trace[3584 + kv] = globaltimer();
    }
    }  // kv heads of this CTA
}

int bulk_parts(const AttnArgs& a, int num_sms) {
    return std::max(1, std::min(kBMaxParts - kMaxLocalParts, num_sms / std::max(1, a.n_kv)));
}

cudaError_t launch_bulk(const BulkArgs& Bin, int G, int n_kv, cudaStream_t s, bool pdl) {
    BulkArgs B = Bin;
    B.warm = pdl && B.mode != kModeLocal && !std::getenv("REATTN_NO_WARM") ? 1 : 0;
    dim3 grid(B.n_parts, n_kv);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(kBThreads);
    cfg.dynamicSmemBytes = kBSmem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl ? 1 : 0;
#define BULK_LAUNCH(GG)                                                                  \
    do {                                                                                 \
        cudaFuncSetAttribute(attend_decode_bulk_kernel<GG>,                              \
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kBSmem);  \
        cudaLaunchKernelEx(&cfg, attend_decode_bulk_kernel<GG>, B);                      \
    } while (0)
    switch (G) {
        case 1: BULK_LAUNCH(1); break;
        case 2: BULK_LAUNCH(2); break;
        case 3: BULK_LAUNCH(3); break;
        case 4: BULK_LAUNCH(4); break;
        case 5: BULK_LAUNCH(5); break;
        case 6: BULK_LAUNCH(6); break;
        case 7: BULK_LAUNCH(7); break;
        default: BULK_LAUNCH(8); break;
    }
#undef BULK_LAUNCH
    return cudaGetLastError();
}

BulkArgs bulk_args(const AttnArgs& a, void* ws, int num_sms, const DecodeFork* f) {
    BulkArgs B;
    B.a = a;
    B.mode = f ? kModeHead : kModeScope;
    B.n_local = f ? f->n_local : 0;
    B.local_row0 = f ? f->local_row0 : 0;
    B.dev_total = f ? f->dev_total : nullptr;
    B.l_global = f ? f->l_global : 0;
    B.l_local = f ? f->l_local : 0;
    B.ranges = nullptr;
    B.merged = nullptr;
    B.n_parts = bulk_parts(a, num_sms);
    B.part_base = 0;
    B.n_slots = B.n_parts + (f ? f->local_parts : 0);
    B.scale_log2 = (float)(1.4426950408889634 / std::sqrt((double)kBD));
    B.tickets = (unsigned int*)ws;
    B.part = (uint8_t*)ws + decode_ticket_bytes(a.n_kv);
    B.trace = trace_buffer();
    B.warm = 0;
    B.local_post = 0;
    B.local_hpc = 1;
    return B;
}

}  // namespace

bool decode_bulk_eligible(const AttnArgs& a) {
    return a.n_q == 1 && a.d == kBD && a.dv == kBD && a.group >= 1 && a.group <= 8 && a.causal &&
           a.boundary_is_tail && a.dtype == kBF16 && a.n_head == a.n_kv * a.group;
}

size_t decode_ticket_bytes(int n_kv) { return ((size_t)4 * std::max(1, n_kv) + 255) & ~(size_t)255; }

size_t decode_bulk_workspace(const AttnArgs& a, int num_sms) {
    return decode_ticket_bytes(a.n_kv) + (size_t)(bulk_parts(a, num_sms) + kMaxLocalParts) * a.n_kv * a.group * kBPartBytes;
}

cudaError_t launch_attend_decode_bulk(const AttnArgs& a, void* ws, int num_sms, cudaStream_t s) {
    return launch_bulk(bulk_args(a, ws, num_sms, nullptr), a.group, a.n_kv, s, true);
}

cudaError_t launch_attend_decode_bulk_ex(const AttnArgs& a, void* ws, int num_sms, cudaStream_t s,
                                         bool pdl) {
    return launch_bulk(bulk_args(a, ws, num_sms, nullptr), a.group, a.n_kv, s, pdl);
}

cudaError_t launch_attend_decode_local(const AttnArgs& a, void* ws, int num_sms, const DecodeFork& f,
                                       cudaStream_t s) {
    if (f.local_parts < 1 || f.local_parts > kMaxLocalParts) return cudaErrorInvalidValue;
    BulkArgs B = bulk_args(a, ws, num_sms, &f);
    B.mode = kModeLocal;
    B.part_base = B.n_parts;  // after the head parts
    B.n_parts = f.local_parts;
    B.local_post = f.post;
    B.local_hpc = std::max(1, f.heads_per_cta);
    if (a.n_kv % B.local_hpc) return cudaErrorInvalidValue;
    return launch_bulk(B, a.group, a.n_kv / B.local_hpc, s, f.post != 0);
}

cudaError_t launch_attend_decode_head(const AttnArgs& a, void* ws, int num_sms, const DecodeFork& f,
                                      cudaStream_t s, bool pdl) {
    return launch_bulk(bulk_args(a, ws, num_sms, &f), a.group, a.n_kv, s, pdl);
}

cudaError_t launch_attend_decode_ranges(const AttnArgs& a, void* ws, int num_sms,
                                        const uint32_t* ranges, uint8_t* merged, cudaStream_t s) {
    BulkArgs B = bulk_args(a, ws, num_sms, nullptr);
    B.mode = kModeRanges;
    B.ranges = ranges;
    B.merged = merged;
    return launch_bulk(B, a.group, a.n_kv, s, false);
}

namespace {
// merge the ranks' partial rows of one q head (fixed source order): lane = 4 columns
__global__ void __launch_bounds__(32) combine_sources_kernel(const AttnArgs a, const uint8_t* parts,
                                                            int n_src, size_t stride) {
    // one launch per step after the partial-row all-gather, so cold: every header and acc
    // row is loaded before use (lane s < n_src: source s's header; all lanes: 4 columns of
    // up to 8 sources), f32 exp2 of the exact f64 differences, one f64 division
    if (a.hdr && a.hdr->error != 0) return;
    const int h = blockIdx.x, lane = threadIdx.x;
    auto row_of = [&](int src) { return parts + src * stride + (size_t)h * kBPartBytes; };
    double hm = -INFINITY, ha = 0.0, hb = 0.0;
    if (lane < n_src) {
        const double* hd = (const double*)row_of(lane);
        hm = hd[0];
        ha = hd[1];
        hb = hd[2];
    }
    constexpr int kPre = 8;
    float4 v[kPre];
#pragma unroll
    for (int s = 0; s < kPre; ++s)
        v[s] = s < n_src ? reinterpret_cast<const float4*>(row_of(s) + 32)[lane]
                         : make_float4(0.f, 0.f, 0.f, 0.f);
    double M = ha > 0.0 ? hm : -INFINITY;
    for (int s = lane + 32; s < n_src; s += 32) {  // more than 32 sources
        const double* hd = (const double*)row_of(s);
        if (hd[1] > 0.0) M = fmax(M, hd[0]);
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) M = fmax(M, __shfl_xor_sync(0xFFFFFFFFu, M, off));
    auto wgt = [&](double pm, double pa) -> double {
        return pa > 0.0 ? (double)exp2f((float)(pm - M)) : 0.0;
    };
    const double w0 = wgt(hm, ha);
    double At = ha > 0.0 ? ha * w0 : 0.0, Bt = ha > 0.0 ? w0 * (hb + (hm - M) * ha) : 0.0;
    for (int s = lane + 32; s < n_src; s += 32) {
        const double* hd = (const double*)row_of(s);
        if (hd[1] > 0.0) {
            const double w = wgt(hd[0], hd[1]);
            At += hd[1] * w;
            Bt += w * (hd[2] + (hd[0] - M) * hd[1]);
        }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        At += __shfl_xor_sync(0xFFFFFFFFu, At, off);
        Bt += __shfl_xor_sync(0xFFFFFFFFu, Bt, off);
    }
    double o[4] = {0.0, 0.0, 0.0, 0.0};
    for (int s0 = 0; s0 < n_src; s0 += kPre) {
        if (s0 > 0) {
#pragma unroll
            for (int s = 0; s < kPre; ++s)
                v[s] = s0 + s < n_src ? reinterpret_cast<const float4*>(row_of(s0 + s) + 32)[lane]
                                      : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int s = 0; s < kPre; ++s) {
            const int src = s0 + s;
            if (src >= n_src) break;
            double w;
            if (src < 32) {
                w = __shfl_sync(0xFFFFFFFFu, w0, src);
            } else {
                const double* hd = (const double*)row_of(src);
                w = wgt(hd[0], hd[1]);
            }
            o[0] = fma((double)v[s].x, w, o[0]);
            o[1] = fma((double)v[s].y, w, o[1]);
            o[2] = fma((double)v[s].z, w, o[2]);
            o[3] = fma((double)v[s].w, w, o[3]);
        }
    }
    const double inv = 1.0 / At;
    reinterpret_cast<float4*>(a.out + (size_t)h * kBD)[lane] =
        make_float4((float)(o[0] * inv), (float)(o[1] * inv), (float)(o[2] * inv), (float)(o[3] * inv));
    if (lane == 0) {
        const double hh = log(At) - Bt * 0.69314718055994530942 * inv;
        a.entropy[h] = hh < 0.0 ? 0.0 : hh;
    }
}
}  // namespace

cudaError_t launch_decode_combine_sources(const AttnArgs& a, const uint8_t* parts, int n_src,
                                          size_t src_stride, cudaStream_t s) {
    combine_sources_kernel<<<a.n_head, 32, 0, s>>>(a, parts, n_src, src_stride);
    return cudaGetLastError();
}

}  // namespace reattn_impl
