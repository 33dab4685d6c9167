// Elementwise / row kernels of the decoder block around attend_step (reference model.hpp):
// token embedding gather (model.hpp:181-190), RMS normalisation with the mean square carried
// in double (model.hpp:155-167), the gated-FFN activation silu(g) * u (model.hpp:170-178)
// and the greedy argmax with ties to the lowest token id (model.hpp:193-199).  The
// projections themselves are plain fp32 GEMMs (cuBLAS, capi_engine.cpp).
#include <cstdint>

#include "common.cuh"
#include "kernels.h"

namespace reattn_impl {

namespace {

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
// (two fp32 multiplies in that order, as model.hpp:160-163).  One CTA of 256 threads per row.
__global__ void rmsnorm_kernel(const float* __restrict__ x, uint64_t cols,
                               const float* __restrict__ w, float* __restrict__ out) {
    __shared__ double part[8];
    const uint64_t r = blockIdx.x;
    const float* src = x + r * cols;
    double s = 0.0;
    for (uint64_t c = threadIdx.x; c < cols; c += blockDim.x) {
        const double v = (double)src[c];
        s += v * v;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xFFFFFFFFu, s, off);
    if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = s;
    __syncthreads();
    double ms = 0.0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) ms += part[i];
    const float inv = (float)(1.0 / sqrt(ms / (double)cols + 1e-5));
    float* dst = out + r * cols;
    for (uint64_t c = threadIdx.x; c < cols; c += blockDim.x)
        dst[c] = __fmul_rn(__fmul_rn(src[c], inv), w[c]);
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
    for (uint64_t i = threadIdx.x; i < n; i += blockDim.x) {
        const float x = v[i];
        if (idx == 0xFFFFFFFFu || x > best) {  // per thread: ascending indices, strict >
            best = x;
            idx = (uint32_t)i;
        }
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
    rmsnorm_kernel<<<(unsigned)rows, 256, 0, s>>>(x, cols, w, out);
    return cudaGetLastError();
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

}  // namespace reattn_impl
