#include <algorithm>
// Elementwise / row kernels of the decoder block around attend_step (reference model.hpp):
// token embedding gather (model.hpp:181-190), RMS normalisation with the mean square carried
// in double (model.hpp:155-167), the gated-FFN activation silu(g) * u (model.hpp:170-178)
// and the greedy argmax with ties to the lowest token id (model.hpp:193-199).  The
// projections of a prefill block are plain fp32 GEMMs (cuBLAS, capi_engine.cpp); a decode
// token's projections are fp32 GEMVs (gemv_kernel below), a pure weight stream bound by HBM.
#include <cstdint>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

using namespace reattn_dev;

namespace reattn_impl {

namespace {

// REATTN_NO_PDL=1: the decode-token kernels launch without programmatic stream serialisation
bool gemv_pdl_env() {
    static const bool off = getenv("REATTN_NO_PDL") != nullptr;
    return !off;
}

// one row per CTA: out[r][c] = emb[tok[r]][c]
__global__ void embed_kernel(const uint32_t* __restrict__ tokens, const float* __restrict__ emb,
                             uint64_t d_model, float* __restrict__ out) {
    const uint64_t r = blockIdx.x;
    const float4* src = reinterpret_cast<const float4*>(emb + (uint64_t)tokens[r] * d_model);
    float4* dst = reinterpret_cast<float4*>(out + r * d_model);
    if ((d_model & 3) == 0) {
        for (uint64_t c = threadIdx.x; c < d_model / 4; c += blockDim.x) dst[c] = __ldg(src + c);
    } else {
        const float* s = emb + (uint64_t)tokens[r] * d_model;
        for (uint64_t c = threadIdx.x; c < d_model; c += blockDim.x) out[r * d_model + c] = s[c];
    }
}

// rmsnorm: ms = sum(double(x)^2) / cols; inv = float(1 / sqrt(ms + 1e-5)); out = x * inv * w
// (two fp32 multiplies in that order, as model.hpp:160-163).  One CTA per row, one float4 per
// thread per pass where the row allows (a decode row is one round trip, not a strided loop).
__global__ void rmsnorm_kernel(const float* __restrict__ x, uint64_t cols,
                               const float* __restrict__ w, float* __restrict__ out) {
    __shared__ double part[32];
    asm volatile("griddepcontrol.launch_dependents;");  // the projection after us may start
    asm volatile("griddepcontrol.wait;" ::: "memory");   // its weight stream under our tail
    const uint64_t r = blockIdx.x;
    const float* src = x + r * cols;
    float* dst = out + r * cols;
    const bool vec = (cols & 3) == 0 && ((uintptr_t)x & 15) == 0 && ((uintptr_t)w & 15) == 0 &&
                     ((uintptr_t)out & 15) == 0;
    double s = 0.0;
    if (vec) {
        for (uint64_t c = threadIdx.x; c < cols / 4; c += blockDim.x) {
            const float4 v = reinterpret_cast<const float4*>(src)[c];
            s += (double)v.x * v.x + (double)v.y * v.y + (double)v.z * v.z + (double)v.w * v.w;
        }
    } else {
        for (uint64_t c = threadIdx.x; c < cols; c += blockDim.x) {
            const double v = (double)src[c];
            s += v * v;
        }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xFFFFFFFFu, s, off);
    if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = s;
    __syncthreads();
    double ms = 0.0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) ms += part[i];
    const float inv = (float)(1.0 / sqrt(ms / (double)cols + 1e-5));
    if (vec) {
        for (uint64_t c = threadIdx.x; c < cols / 4; c += blockDim.x) {
            const float4 v = reinterpret_cast<const float4*>(src)[c];
            const float4 g = reinterpret_cast<const float4*>(w)[c];
            reinterpret_cast<float4*>(dst)[c] =
                make_float4(__fmul_rn(__fmul_rn(v.x, inv), g.x), __fmul_rn(__fmul_rn(v.y, inv), g.y),
                            __fmul_rn(__fmul_rn(v.z, inv), g.z), __fmul_rn(__fmul_rn(v.w, inv), g.w));
        }
    } else {
        for (uint64_t c = threadIdx.x; c < cols; c += blockDim.x)
            dst[c] = __fmul_rn(__fmul_rn(src[c], inv), w[c]);
    }
}

// gate[i] = gate[i] / (1 + exp(-gate[i])) * up[i]   (model.hpp:170-178, fp32 throughout)
__global__ void silu_mul_kernel(float* __restrict__ gate, const float* __restrict__ up, uint64_t n) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const float g = gate[i];
        gate[i] = __fmul_rn(__fdiv_rn(g, __fadd_rn(1.0f, expf(-g))), up[i]);
    }
}

// argmax over one row, ties to the lowest index (strict > in index order, model.hpp:193-199)
__global__ void argmax_kernel(const float* __restrict__ v, uint64_t n, uint32_t* __restrict__ out) {
    __shared__ float bs[32];
    __shared__ uint32_t bi[32];
    float best = -INFINITY;
    uint32_t idx = 0xFFFFFFFFu;
    auto take = [&](float x, uint64_t i) {  // per thread: ascending indices, strict >
        if (idx == 0xFFFFFFFFu || x > best) {
            best = x;
            idx = (uint32_t)i;
        }
    };
    if ((n & 3) == 0 && ((uintptr_t)v & 15) == 0) {  // 8 float4 loads in flight per thread
        const float4* v4 = reinterpret_cast<const float4*>(v);
        const uint64_t n4 = n / 4, bd = blockDim.x;
        uint64_t i = threadIdx.x;
        for (; i + 7 * bd < n4; i += 8 * bd) {
            float4 c[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) c[u] = v4[i + u * bd];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const uint64_t b = 4 * (i + u * bd);
                take(c[u].x, b);
                take(c[u].y, b + 1);
                take(c[u].z, b + 2);
                take(c[u].w, b + 3);
            }
        }
        for (; i < n4; i += bd) {
            const float4 c = v4[i];
            take(c.x, 4 * i);
            take(c.y, 4 * i + 1);
            take(c.z, 4 * i + 2);
            take(c.w, 4 * i + 3);
        }
    } else {
        for (uint64_t i = threadIdx.x; i < n; i += blockDim.x) take(v[i], i);
    }
    auto better = [](float a, uint32_t ia, float b, uint32_t ib) {
        if (ia == 0xFFFFFFFFu) return false;
        if (ib == 0xFFFFFFFFu) return true;
        return a > b || (a == b && ia < ib);
    };
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        const float ob = __shfl_xor_sync(0xFFFFFFFFu, best, off);
        const uint32_t oi = __shfl_xor_sync(0xFFFFFFFFu, idx, off);
        if (better(ob, oi, best, idx)) {
            best = ob;
            idx = oi;
        }
    }
    if ((threadIdx.x & 31) == 0) {
        bs[threadIdx.x >> 5] = best;
        bi[threadIdx.x >> 5] = idx;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        float b = bs[0];
        uint32_t i0 = bi[0];
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
            if (better(bs[w], bi[w], b, i0)) {
                b = bs[w];
                i0 = bi[w];
            }
        *out = i0;
    }
}

}  // namespace

cudaError_t launch_embed(const uint32_t* tokens, uint64_t rows, const float* emb, uint64_t d_model,
                         float* out, cudaStream_t s) {
    if (rows == 0) return cudaSuccess;
    embed_kernel<<<(unsigned)rows, 128, 0, s>>>(tokens, emb, d_model, out);
    return cudaGetLastError();
}

cudaError_t launch_rmsnorm(const float* x, uint64_t rows, uint64_t cols, const float* w, float* out,
                           cudaStream_t s) {
    if (rows == 0) return cudaSuccess;
    const unsigned threads = (unsigned)std::min<uint64_t>(1024, std::max<uint64_t>(32, ((cols + 3) / 4 + 31) & ~31ull));
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)rows);
    cfg.blockDim = dim3(threads);
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = gemv_pdl_env() ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, rmsnorm_kernel, x, cols, w, out);
}

cudaError_t launch_silu_mul(float* gate, const float* up, uint64_t n, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    const unsigned blocks = (unsigned)std::min<uint64_t>((n + 255) / 256, 148ull * 16);
    silu_mul_kernel<<<blocks, 256, 0, s>>>(gate, up, n);
    return cudaGetLastError();
}

cudaError_t launch_argmax(const float* v, uint64_t n, uint32_t* out, cudaStream_t s) {
    argmax_kernel<<<1, 1024, 0, s>>>(v, n, out);
    return cudaGetLastError();
}

namespace {
__global__ void scale_kernel(float* x, uint64_t n, float a) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        x[i] *= a;
}
}  // namespace

cudaError_t launch_scale(float* x, uint64_t n, float a, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    const int g = (int)std::min<uint64_t>((n + 255) / 256, 148 * 32);
    scale_kernel<<<g, 256, 0, s>>>(x, n, a);
    return cudaGetLastError();
}

// y[n] = sum_k x[k] W[k][n] (+ beta y[n]) for one row x, for up to three matrices sharing x
// (the q/k/v projections; gate/up) in one launch.  The weights are read exactly once, so the
// kernel is an HBM stream, and its work is split stream-K style so that every SM streams the
// same number of bytes whatever the shape: a tile is 128 columns of one matrix (a lane one
// float4), a unit is 64 rows of a tile (8 warps x 8 rows), and the tiles' units, laid end to
// end, are cut into one contiguous range per resident CTA.  A warp keeps the next unit's 8
// rows in flight (register double buffer) while it accumulates the current one, across tile
// boundaries too.  Where a CTA's range ends a tile segment it reduces its warps in order and,
// when the tile has several contributors, stores the partial at slot (cta + tile) -- unique,
// since contributors of consecutive tiles overlap in at most one CTA -- and the last
// contributor (a ticket counting units) sums the partials in CTA order: deterministic.  In
// the gated-FFN pair mode the gate and up tiles of the same columns share one ticket and the
// last contributor writes silu(g) * u (model.hpp:170-178) into the gate buffer.  Launched
// with programmatic stream serialisation: the first unit's weight rows are issued before
// griddepcontrol.wait, under the tail of the kernel before.  fp32, one FMA per row.
namespace {
constexpr int kGemvWarps = 8, kGemvCols = 128, kGemvRows = 8, kGemvUnitRows = kGemvWarps * kGemvRows;

__device__ __forceinline__ float4 ld_stream4(const float* p) {
    float4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "l"(p));
    return v;
}

__device__ __forceinline__ void add4(float4& a, const float4& b) {
    a.x += b.x;
    a.y += b.y;
    a.z += b.z;
    a.w += b.w;
}

struct GemvMat {
    const float* W;
    uint64_t ldw;
    float* y;           // kind 0: y[N]; kinds 1 / 2: the cache's K or V base ([n_kv][cap][d])
    uint32_t N, tile0;  // columns; first global tile of this matrix
    float beta;
    int kind;           // 0 dense fp32, 1 bf16 cache row, 2 fp32 cache row
    uint32_t d, row;    // cache row layout: column c -> head c / d, element c % d of row `row`
    uint64_t head_stride;
};

struct GemvBatch {
    GemvMat m[3];
    int count;
    int silu_pair;      // m[0] gate, m[1] up (same N): gate <- silu(g) * u
    uint32_t K, upt;    // rows; units per tile
    uint32_t tiles;     // tiles over all matrices
    uint64_t units;     // tiles * upt
    uint32_t* total_ptr;  // non-null: CTA 0 writes total_val (a cache's device length)
    uint32_t total_val;
    uint32_t prefetch;    // units prefetched into L2 ahead of the register double buffer
};

// y columns [col, col + 4) of M (the matrix's own column index), beta-accumulated for dense
// outputs; cache rows take the bf16 (round to nearest even, as the cache append) or fp32 value
__device__ __forceinline__ void gemv_store(const GemvMat& M, uint32_t col, float4 p) {
    if (M.kind == 0) {
        float4* yp = reinterpret_cast<float4*>(M.y + col);
        if (M.beta != 0.0f) {
            const float4 o = *yp;
            p.x = fmaf(M.beta, o.x, p.x);
            p.y = fmaf(M.beta, o.y, p.y);
            p.z = fmaf(M.beta, o.z, p.z);
            p.w = fmaf(M.beta, o.w, p.w);
        }
        *yp = p;
        return;
    }
    const uint32_t h = col / M.d, c = col % M.d;
    const size_t o = ((size_t)h * M.head_stride + M.row) * M.d + c;
    if (M.kind == 1) {
        const __nv_bfloat162 lo = __floats2bfloat162_rn(p.x, p.y), hi = __floats2bfloat162_rn(p.z, p.w);
        uint2 w;
        w.x = *reinterpret_cast<const uint32_t*>(&lo);
        w.y = *reinterpret_cast<const uint32_t*>(&hi);
        *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(M.y) + o) = w;
    } else {
        *reinterpret_cast<float4*>(M.y + o) = p;
    }
}

__device__ __forceinline__ uint32_t unit_begin(uint64_t c, uint64_t units, uint32_t G) {
    return (uint32_t)(c * units / G);
}
// the CTA whose range holds unit u: the largest c with unit_begin(c) <= u
__device__ __forceinline__ uint32_t unit_owner(uint64_t u, uint64_t units, uint32_t G) {
    return (uint32_t)(((u + 1) * G - 1) / units);
}

__device__ __forceinline__ int mat_of(const GemvBatch& B, uint32_t t) {
    return B.count > 2 && t >= B.m[2].tile0 ? 2 : B.count > 1 && t >= B.m[1].tile0 ? 1 : 0;
}

__global__ void __launch_bounds__(kGemvWarps * 32, 2) gemv_kernel(const float* __restrict__ x, GemvBatch B,
                                                                  float* ws, uint32_t* tickets) {
    __shared__ float4 red[2][kGemvWarps * 32];
    asm volatile("griddepcontrol.launch_dependents;");
    const uint32_t G = gridDim.x, c = blockIdx.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t u0 = unit_begin(c, B.units, G), u1 = unit_begin(c + 1, B.units, G);
    float4 w[2][kGemvRows];
    float xv[2][kGemvRows];
    auto load_w = [&](uint32_t u, int b) {
        const uint32_t t = u / B.upt;
        const GemvMat& M = B.m[mat_of(B, t)];
        const uint32_t col = (t - M.tile0) * kGemvCols + lane * 4;
        const uint32_t r0 = (u % B.upt) * kGemvUnitRows + warp;
        const float* wp = M.W + (uint64_t)r0 * M.ldw + col;
#pragma unroll
        for (int i = 0; i < kGemvRows; ++i)
            w[b][i] = col < M.N && r0 + i * kGemvWarps < B.K ? ld_stream4(wp + (uint64_t)i * kGemvWarps * M.ldw)
                                                            : make_float4(0.f, 0.f, 0.f, 0.f);
    };
    // L2 prefetch of a later unit's rows: DRAM requests in flight beyond the register buffers
    auto prefetch_w = [&](uint32_t u) {
        const uint32_t t = u / B.upt;
        const GemvMat& M = B.m[mat_of(B, t)];
        const uint32_t col = (t - M.tile0) * kGemvCols + lane * 4;
        const uint32_t r0 = (u % B.upt) * kGemvUnitRows + warp;
        const float* wp = M.W + (uint64_t)r0 * M.ldw + col;
        if ((lane & 7) == 0 && col < M.N) {  // one lane per 128-byte line
#pragma unroll
            for (int i = 0; i < kGemvRows; ++i)
                if (r0 + i * kGemvWarps < B.K)
                    asm volatile("prefetch.global.L2 [%0];" ::"l"(wp + (uint64_t)i * kGemvWarps * M.ldw));
        }
    };
    auto load_x = [&](uint32_t u, int b) {
        const uint32_t r0 = (u % B.upt) * kGemvUnitRows + warp;
#pragma unroll
        for (int i = 0; i < kGemvRows; ++i) xv[b][i] = r0 + i * kGemvWarps < B.K ? x[r0 + i * kGemvWarps] : 0.f;
    };
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    auto fma_rows = [&](int b) {
#pragma unroll
        for (int i = 0; i < kGemvRows; ++i) {
            acc.x = fmaf(xv[b][i], w[b][i].x, acc.x);
            acc.y = fmaf(xv[b][i], w[b][i].y, acc.y);
            acc.z = fmaf(xv[b][i], w[b][i].z, acc.z);
            acc.w = fmaf(xv[b][i], w[b][i].w, acc.w);
        }
    };
    auto silu = [](float gv, float uv) { return __fmul_rn(__fdiv_rn(gv, __fadd_rn(1.0f, expf(-gv))), uv); };
    int rb = 0;  // shared-memory reduction buffer of the next epilogue
    // the end of tile t's segment in this CTA: reduce the warps; a tile with one contributor
    // is written here, otherwise its partial goes to the workspace and the last contributor
    // of the tile (pair: of both tiles) finishes it (warp 0 only; the other warps stream on)
    auto epilogue = [&](uint32_t t) {
        red[rb][warp * 32 + lane] = acc;
        acc = make_float4(0.f, 0.f, 0.f, 0.f);
        __syncthreads();
        const int b = rb;
        rb ^= 1;
        if (warp != 0) return;
        float4 p = red[b][lane];
#pragma unroll
        for (int i = 1; i < kGemvWarps; ++i) add4(p, red[b][i * 32 + lane]);
        const bool pair = B.silu_pair != 0;
        const GemvMat& M = B.m[mat_of(B, t)];
        const uint32_t col = (t - M.tile0) * kGemvCols + lane * 4;
        const bool ok = col < M.N;
        const uint32_t cf = unit_owner((uint64_t)t * B.upt, B.units, G);
        const uint32_t cl = unit_owner((uint64_t)(t + 1) * B.upt - 1, B.units, G);
        if (!pair && cf == cl) {
            if (ok) gemv_store(M, col, p);
            return;
        }
        RA_ASSERT(c + t < G + B.tiles);
        if (ok) reinterpret_cast<float4*>(ws)[(uint64_t)(c + t) * 32 + lane] = p;
        // units of tile t in this CTA
        const uint64_t tb = (uint64_t)t * B.upt, te = tb + B.upt;
        const uint32_t mine = (uint32_t)((te < u1 ? te : (uint64_t)u1) - (tb > u0 ? tb : (uint64_t)u0));
        const uint32_t pt = pair ? B.m[1].tile0 : 0;  // pair: gate tiles [0, pt), up [pt, 2pt)
        const uint32_t ticket = pair ? t % pt : t;
        const uint32_t need = pair ? 2 * B.upt : B.upt;
        __threadfence();
        __syncwarp();
        uint32_t last = 0;
        if (lane == 0) {
            last = atomicAdd(&tickets[ticket], mine) + mine == need;
            if (last) tickets[ticket] = 0;  // the next launch on the stream starts from zero
        }
        if (!__shfl_sync(0xFFFFFFFFu, last, 0)) return;
        __threadfence();
        auto total_of = [&](uint32_t tt) {
            const uint32_t f = unit_owner((uint64_t)tt * B.upt, B.units, G);
            const uint32_t l = unit_owner((uint64_t)(tt + 1) * B.upt - 1, B.units, G);
            float4 q = make_float4(0.f, 0.f, 0.f, 0.f);
            if (!ok) return q;
            for (uint32_t j = f; j <= l; ++j)
                add4(q, __ldcg(reinterpret_cast<const float4*>(ws) + (uint64_t)(j + tt) * 32 + lane));
            return q;
        };
        if (!ok) return;
        if (pair) {
            const uint32_t tg = t % pt;
            const float4 g = total_of(tg), u = total_of(tg + pt);
            *reinterpret_cast<float4*>(B.m[0].y + col) =
                make_float4(silu(g.x, u.x), silu(g.y, u.y), silu(g.z, u.z), silu(g.w, u.w));
            return;
        }
        gemv_store(M, col, total_of(t));
    };
    if (u0 >= u1) {
        asm volatile("griddepcontrol.wait;" ::: "memory");
        if (B.total_ptr && c == 0 && threadIdx.x == 0) *B.total_ptr = B.total_val;
        return;
    }
    load_w(u0, 0);                                      // weights: constant
    asm volatile("griddepcontrol.wait;" ::: "memory");  // x, y, workspace: the kernel before
    // the cache's new device length: read only by kernels after this grid completes
    if (B.total_ptr && c == 0 && threadIdx.x == 0) *B.total_ptr = B.total_val;
    load_x(u0, 0);
    const uint32_t pd = B.prefetch;
    if (pd)
        for (uint32_t v = u0 + 1; v < min(u1, u0 + 1 + pd); ++v) prefetch_w(v);
    for (uint32_t u = u0;;) {
        if (u + 1 < u1) {
            load_w(u + 1, 1);
            load_x(u + 1, 1);
        }
        if (pd && u + 1 + pd < u1) prefetch_w(u + 1 + pd);
        fma_rows(0);
        if (u + 1 >= u1 || (u + 1) / B.upt != u / B.upt) epilogue(u / B.upt);
        if (++u >= u1) break;
        if (u + 1 < u1) {
            load_w(u + 1, 0);
            load_x(u + 1, 0);
        }
        if (pd && u + 1 + pd < u1) prefetch_w(u + 1 + pd);
        fma_rows(1);
        if (u + 1 >= u1 || (u + 1) / B.upt != u / B.upt) epilogue(u / B.upt);
        if (++u >= u1) break;
    }
}

// The TMA-fed variant (weights of every unit staged in shared memory by the tensor-memory
// accelerator): one CTA per SM, a producer thread keeps kTStages units (32 KB each) in flight
// -- 160 KB per SM, issued before griddepcontrol.wait since the weights do not depend on the
// kernel before -- and 8 consumer warps accumulate from shared memory with x staged once.
// Same stream-K split, epilogue and determinism as gemv_kernel.
constexpr int kTStages = 5, kTConsumers = 8, kTThreads = (kTConsumers + 1) * 32;
constexpr int kTStageBytes = kGemvUnitRows * kGemvCols * 4;  // 32 KB
constexpr int kTMaxK = 14336;                                 // x staged in shared memory
constexpr size_t kTSmem = 1024 + (size_t)kTStages * kTStageBytes + (size_t)kTMaxK * 4 + 256;

__global__ void __launch_bounds__(kTThreads, 1) gemv_tma_kernel(
    const __grid_constant__ CUtensorMap map0, const __grid_constant__ CUtensorMap map1,
    const __grid_constant__ CUtensorMap map2, const float* __restrict__ x, GemvBatch B, float* ws,
    uint32_t* tickets) {
    extern __shared__ uint8_t tsm_raw[];
    uint8_t* sm = (uint8_t*)(((uintptr_t)tsm_raw + 1023) & ~(uintptr_t)1023);
    float* ring = (float*)sm;                                            // [stages][64][128]
    float* sx = (float*)(sm + (size_t)kTStages * kTStageBytes);          // [K]
    uint64_t* full = (uint64_t*)(sx + kTMaxK);
    uint64_t* empty = full + kTStages;
    __shared__ float4 red[2][kTConsumers * 32];
    asm volatile("griddepcontrol.launch_dependents;");
    const uint32_t G = gridDim.x, c = blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t u0 = unit_begin(c, B.units, G), u1 = unit_begin(c + 1, B.units, G);
    if (tid == 0) {
        for (int i = 0; i < kTStages; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], kTConsumers);
        }
        fence_barrier_init();
    }
    __syncthreads();
    if (warp == kTConsumers) {  // ===== producer: one TMA load per unit =====
        if (lane == 0) {
            prefetch_tensormap(&map0);
            if (B.count > 1) prefetch_tensormap(&map1);
            if (B.count > 2) prefetch_tensormap(&map2);
            const uint64_t pol = policy_evict_first();
            for (uint32_t u = u0; u < u1; ++u) {
                const uint32_t i = u - u0, s = i % kTStages;
                if (i >= kTStages) mbar_wait(&empty[s], ((i / kTStages) - 1) & 1u);
                const uint32_t t = u / B.upt;
                const int mi = mat_of(B, t);
                const CUtensorMap* mp = mi == 0 ? &map0 : mi == 1 ? &map1 : &map2;
                mbar_arrive_expect_tx(&full[s], kTStageBytes);
                tma_load_2d(ring + (size_t)s * (kTStageBytes / 4), mp, (int32_t)((t - B.m[mi].tile0) * kGemvCols),
                            (int32_t)((u % B.upt) * kGemvUnitRows), &full[s], pol);
            }
        }
        asm volatile("griddepcontrol.wait;" ::: "memory");
        return;
    }
    // ===== consumers =====
    asm volatile("griddepcontrol.wait;" ::: "memory");  // x, y, workspace: the kernel before
    if (B.total_ptr && c == 0 && tid == 0) *B.total_ptr = B.total_val;
    for (uint32_t i = tid; i < B.K; i += kTConsumers * 32) sx[i] = x[i];
    named_bar_sync(1, kTConsumers * 32);
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    int rb = 0;
    auto silu = [](float gv, float uv) { return __fmul_rn(__fdiv_rn(gv, __fadd_rn(1.0f, expf(-gv))), uv); };
    auto epilogue = [&](uint32_t t) {
        red[rb][warp * 32 + lane] = acc;
        acc = make_float4(0.f, 0.f, 0.f, 0.f);
        named_bar_sync(1, kTConsumers * 32);
        const int b = rb;
        rb ^= 1;
        if (warp != 0) return;
        float4 p = red[b][lane];
#pragma unroll
        for (int i = 1; i < kTConsumers; ++i) add4(p, red[b][i * 32 + lane]);
        const bool pair = B.silu_pair != 0;
        const GemvMat& M = B.m[mat_of(B, t)];
        const uint32_t col = (t - M.tile0) * kGemvCols + lane * 4;
        const bool ok = col < M.N;
        const uint32_t cf = unit_owner((uint64_t)t * B.upt, B.units, G);
        const uint32_t cl = unit_owner((uint64_t)(t + 1) * B.upt - 1, B.units, G);
        if (!pair && cf == cl) {
            if (ok) gemv_store(M, col, p);
            return;
        }
        RA_ASSERT(c + t < G + B.tiles);
        if (ok) reinterpret_cast<float4*>(ws)[(uint64_t)(c + t) * 32 + lane] = p;
        const uint64_t tb = (uint64_t)t * B.upt, te = tb + B.upt;
        const uint32_t mine = (uint32_t)((te < u1 ? te : (uint64_t)u1) - (tb > u0 ? tb : (uint64_t)u0));
        const uint32_t pt = pair ? B.m[1].tile0 : 0;
        const uint32_t ticket = pair ? t % pt : t;
        const uint32_t need = pair ? 2 * B.upt : B.upt;
        __threadfence();
        __syncwarp();
        uint32_t last = 0;
        if (lane == 0) {
            last = atomicAdd(&tickets[ticket], mine) + mine == need;
            if (last) tickets[ticket] = 0;
        }
        if (!__shfl_sync(0xFFFFFFFFu, last, 0)) return;
        __threadfence();
        auto total_of = [&](uint32_t tt) {
            const uint32_t f = unit_owner((uint64_t)tt * B.upt, B.units, G);
            const uint32_t l = unit_owner((uint64_t)(tt + 1) * B.upt - 1, B.units, G);
            float4 q = make_float4(0.f, 0.f, 0.f, 0.f);
            if (!ok) return q;
            for (uint32_t j = f; j <= l; ++j)
                add4(q, __ldcg(reinterpret_cast<const float4*>(ws) + (uint64_t)(j + tt) * 32 + lane));
            return q;
        };
        if (!ok) return;
        if (pair) {
            const uint32_t tg = t % pt;
            const float4 g = total_of(tg), u = total_of(tg + pt);
            *reinterpret_cast<float4*>(B.m[0].y + col) =
                make_float4(silu(g.x, u.x), silu(g.y, u.y), silu(g.z, u.z), silu(g.w, u.w));
            return;
        }
        gemv_store(M, col, total_of(t));
    };
    for (uint32_t u = u0; u < u1; ++u) {
        const uint32_t i = u - u0, s = i % kTStages;
        mbar_wait(&full[s], (i / kTStages) & 1u);
        const float* st = ring + (size_t)s * (kTStageBytes / 4);
        const uint32_t r0 = (u % B.upt) * kGemvUnitRows;
#pragma unroll
        for (int j = 0; j < kGemvRows; ++j) {
            const uint32_t r = warp + j * kTConsumers, row = r0 + r;
            const float4 w = reinterpret_cast<const float4*>(st + r * kGemvCols)[lane];
            const float xv = row < B.K ? sx[row] : 0.f;  // rows past K: zero-filled by the TMA
            acc.x = fmaf(xv, w.x, acc.x);
            acc.y = fmaf(xv, w.y, acc.y);
            acc.z = fmaf(xv, w.z, acc.z);
            acc.w = fmaf(xv, w.w, acc.w);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
        if (u + 1 >= u1 || (u + 1) / B.upt != u / B.upt) epilogue(u / B.upt);
    }
}

int gemv_ctas() {
    static int g = [] {
        int dev = 0, sms = 148, occ = 2;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, gemv_kernel, kGemvWarps * 32, 0);
        const char* e = getenv("REATTN_GEMV_CTAS");
        return e ? std::max(1, atoi(e)) : sms * std::max(1, occ);
    }();
    return g;
}
}  // namespace

bool gemv_weight_map(CUtensorMap* map, const float* W, uint64_t ldw, uint64_t N, uint64_t K) {
    return make_tensor_map_2d(map, W, kF32, N, K, ldw * sizeof(float), kGemvCols, kGemvUnitRows);
}

size_t gemv_workspace_bytes(uint64_t n_max) {
    // partial slots cta + tile < ctas + tiles; one ticket per tile
    const uint64_t tiles = 3 * ((n_max + kGemvCols - 1) / kGemvCols);
    const uint64_t ctas = 148 * 8;
    return (size_t)(ctas + tiles) * kGemvCols * sizeof(float) + tiles * sizeof(uint32_t) + 256;
}

bool gemv_supported(uint64_t N, uint64_t K, uint64_t ldw, const void* x, const void* W, const void* y) {
    return N % 4 == 0 && ldw % 4 == 0 && N <= UINT32_MAX && K > 0 && K <= (1ull << 31) &&
           ((uintptr_t)W & 15) == 0 && ((uintptr_t)y & 15) == 0 && ((uintptr_t)x & 3) == 0;
}

cudaError_t launch_gemv_batch(const float* x, uint64_t K, const GemvDesc* mats, int count, bool silu_pair,
                              void* ws, uint64_t n_max, cudaStream_t s, uint32_t* total_ptr,
                              uint32_t total_val, const CUtensorMap* maps) {
    if (count < 1 || count > 3 || (silu_pair && (count != 2 || mats[0].N != mats[1].N)))
        return cudaErrorInvalidValue;
    GemvBatch B{};
    uint32_t tiles = 0;
    for (int i = 0; i < count; ++i) {
        if (mats[i].N > n_max) return cudaErrorInvalidValue;
        B.m[i] = GemvMat{mats[i].W, mats[i].ldw, mats[i].y, (uint32_t)mats[i].N, tiles, mats[i].beta,
                         mats[i].kind, (uint32_t)mats[i].d, (uint32_t)mats[i].row, mats[i].head_stride};
        if (mats[i].kind != 0 && (mats[i].d == 0 || mats[i].d % 4 != 0)) return cudaErrorInvalidValue;
        tiles += (uint32_t)((mats[i].N + kGemvCols - 1) / kGemvCols);
    }
    if (tiles == 0) return cudaSuccess;
    B.count = count;
    B.silu_pair = silu_pair ? 1 : 0;
    B.tiles = tiles;
    B.K = (uint32_t)K;
    B.upt = (uint32_t)((K + kGemvUnitRows - 1) / kGemvUnitRows);
    B.units = (uint64_t)tiles * B.upt;
    B.total_ptr = total_ptr;
    B.total_val = total_val;
    static const uint32_t pf = getenv("REATTN_GEMV_PREFETCH") ? (uint32_t)atoi(getenv("REATTN_GEMV_PREFETCH")) : 0u;
    B.prefetch = pf;
    if (B.units > UINT32_MAX) return cudaErrorInvalidValue;
    const uint32_t G = (uint32_t)std::min<uint64_t>(std::min(gemv_ctas(), 148 * 8), B.units);
    const uint64_t tiles_max = 3 * ((n_max + kGemvCols - 1) / kGemvCols);
    float* part = (float*)ws;
    uint32_t* tickets = (uint32_t*)(part + (148 * 8 + tiles_max) * kGemvCols);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(G);
    cfg.blockDim = dim3(kGemvWarps * 32);
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = gemv_pdl_env() ? 1 : 0;
    static const bool no_tma = getenv("REATTN_GEMV_NO_TMA") != nullptr;
    if (maps && K <= (uint64_t)kTMaxK && !no_tma) {
        static int sms = [] {
            int dev = 0, n = 148;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
            return n;
        }();
        static bool attr = [] {
            return cudaFuncSetAttribute(gemv_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)kTSmem) == cudaSuccess;
        }();
        if (!attr) return cudaErrorInvalidValue;
        const uint32_t GT = (uint32_t)std::min<uint64_t>((uint64_t)sms, B.units);
        cfg.gridDim = dim3(GT);
        cfg.blockDim = dim3(kTThreads);
        cfg.dynamicSmemBytes = kTSmem;
        const CUtensorMap& m0 = maps[0];
        const CUtensorMap& m1 = count > 1 ? maps[1] : maps[0];
        const CUtensorMap& m2 = count > 2 ? maps[2] : maps[0];
        return cudaLaunchKernelEx(&cfg, gemv_tma_kernel, m0, m1, m2, x, B, part, tickets);
    }
    return cudaLaunchKernelEx(&cfg, gemv_kernel, x, B, part, tickets);
}

cudaError_t launch_gemv(const float* x, const float* W, uint64_t ldw, uint64_t N, uint64_t K, float* y,
                        float beta, void* ws, uint64_t n_max, cudaStream_t s) {
    if (N == 0) return cudaSuccess;
    const GemvDesc m{W, ldw, N, y, beta, 0, 0, 0, 0};
    return launch_gemv_batch(x, K, &m, 1, false, ws, n_max, s);
}

}  // namespace reattn_impl
