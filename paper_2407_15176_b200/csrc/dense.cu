// Dense numerics of the drop-in API on the device, each the exact arithmetic of its reference
// function (host functions in the reference; batched here):
//   dot_f32             dense_matrix.hpp:41-56   8 fp32 lanes over j, j+8, ..., fixed tree; the
//                                                 lane update unfused or FMA (the context's lanes)
//   dot_f64             dense_matrix.hpp:59-74   the same lanes in f64 (unfused)
//   matmul              dense_matrix.hpp:77-90   c[i][j] accumulated in k order, unfused
//   group_mean_queries  selection.hpp:139-156    sequential fp32 adds, times float(1 / group)
//   naive_topk_scores   selection_reference.hpp:18-69: the full middle x n_q score matrix is
//                        materialised (the reference's point of comparison, scratch linear in
//                        the middle), then each row's top-k is selected by k block-wide argmax
//                        rounds under (score desc, index asc) -- an independent route to the
//                        same lists as K1 / K2 / the generic scan.
#include "common.cuh"
#include "kernels.h"

using namespace reattn_dev;

namespace reattn_impl {

namespace {

template <int LANES>
__device__ __forceinline__ float lane_upd(float l, float x, float y) {
    return LANES == kLanesFma ? __fmaf_rn(x, y, l) : __fadd_rn(l, __fmul_rn(x, y));
}

template <int LANES>
__device__ __forceinline__ float dot_f32_dev(const float* a, const float* b, uint32_t d) {
    float l[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    uint32_t j = 0;
    for (; j + 8 <= d; j += 8)
#pragma unroll
        for (int t = 0; t < 8; ++t) l[t] = lane_upd<LANES>(l[t], a[j + t], b[j + t]);
    for (; j < d; ++j) l[0] = lane_upd<LANES>(l[0], a[j], b[j]);
    return __fadd_rn(__fadd_rn(__fadd_rn(l[0], l[1]), __fadd_rn(l[2], l[3])),
                     __fadd_rn(__fadd_rn(l[4], l[5]), __fadd_rn(l[6], l[7])));
}

template <int LANES>
__global__ void dot_f32_kernel(const float* a, const float* b, uint64_t n, uint32_t d, float* out) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = dot_f32_dev<LANES>(a + i * d, b + i * d, d);
}

__global__ void dot_f64_kernel(const float* a, const float* b, uint64_t n, uint32_t d, double* out) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const float* x = a + i * d;
        const float* y = b + i * d;
        double l[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        uint32_t j = 0;
        for (; j + 8 <= d; j += 8)
#pragma unroll
            for (int t = 0; t < 8; ++t) l[t] = __dadd_rn(l[t], __dmul_rn((double)x[j + t], (double)y[j + t]));
        for (; j < d; ++j) l[0] = __dadd_rn(l[0], __dmul_rn((double)x[j], (double)y[j]));
        out[i] = __dadd_rn(__dadd_rn(__dadd_rn(l[0], l[1]), __dadd_rn(l[2], l[3])),
                           __dadd_rn(__dadd_rn(l[4], l[5]), __dadd_rn(l[6], l[7])));
    }
}

__global__ void matmul_kernel(const float* a, const float* b, uint64_t m, uint64_t k, uint64_t n,
                              float* c) {
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < m * n;
         e += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t i = e / n, j = e % n;
        float acc = 0.0f;
        for (uint64_t kk = 0; kk < k; ++kk) acc = __fadd_rn(acc, __fmul_rn(a[i * k + kk], b[kk * n + j]));
        c[e] = acc;
    }
}

__global__ void group_mean_kernel(const float* q, uint64_t n_q, uint32_t n_heads, uint32_t n_kv,
                                  uint32_t d, float* out) {
    const uint32_t group = n_heads / n_kv;
    const float inv = __fdiv_rn(1.0f, (float)group);
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < n_q * n_kv * d;
         e += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t r = e / ((uint64_t)n_kv * d);
        const uint32_t rem = (uint32_t)(e % ((uint64_t)n_kv * d)), kv = rem / d, c = rem % d;
        const float* src = q + r * (uint64_t)n_heads * d;
        float acc = 0.0f;
        for (uint32_t g = 0; g < group; ++g) acc = __fadd_rn(acc, src[(kv * group + g) * d + c]);
        out[e] = __fmul_rn(acc, inv);
    }
}

// scores[kv][q][i] = dot_f32(mq[q][kv], key_i)
template <typename KT, int LANES>
__global__ void naive_scores_kernel(const float* mq, uint32_t n_q, uint32_t n_kv, uint32_t d,
                                    const KT* keys, uint64_t head_stride, uint64_t row0,
                                    uint32_t count, float* scores) {
    extern __shared__ float s_row[];  // one key row, widened
    const uint32_t kv = blockIdx.y;
    for (uint32_t i = blockIdx.x; i < count; i += gridDim.x) {
        const KT* kr = keys + ((uint64_t)kv * head_stride + row0 + i) * d;
        __syncthreads();
        for (uint32_t c = threadIdx.x; c < d; c += blockDim.x) s_row[c] = load_as_float(kr + c);
        __syncthreads();
        for (uint32_t qq = threadIdx.x; qq < n_q; qq += blockDim.x)
            scores[((uint64_t)kv * n_q + qq) * count + i] =
                dot_f32_dev<LANES>(mq + ((uint64_t)qq * n_kv + kv) * d, s_row, d);
    }
}

// one CTA per (kv, q) row: k rounds of block argmax under (score desc, index asc), each round
// the best entry strictly behind the previous round's pick (the order is total: indices are
// distinct), so any k needs no record of the entries taken
__global__ void naive_select_kernel(const float* scores, uint32_t count, uint32_t kk, uint32_t k,
                                    uint32_t* idx_out, float* score_out) {
    const uint64_t row = blockIdx.x;
    const float* s = scores + row * count;
    __shared__ float ws[32];
    __shared__ uint32_t wi[32];
    __shared__ float s_ps;
    __shared__ uint32_t s_pi;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    float ps = INFINITY;  // previous pick (score, index); none yet
    uint32_t pi = kNoIndex;
    for (uint32_t r = 0; r < kk; ++r) {
        float bs = -INFINITY;
        uint32_t bi = kNoIndex;
        for (uint32_t i = threadIdx.x; i < count; i += blockDim.x) {
            const float v = s[i];
            const bool behind = pi == kNoIndex || better(ps, pi, v, i);
            if (behind && better(v, i, bs, bi)) {
                bs = v;
                bi = i;
            }
        }
        warp_best(bs, bi);
        if (lane == 0) {
            ws[warp] = bs;
            wi[warp] = bi;
        }
        __syncthreads();
        if (warp == 0) {
            bs = lane < nw ? ws[lane] : -INFINITY;
            bi = lane < nw ? wi[lane] : kNoIndex;
            warp_best(bs, bi);
            if (lane == 0) {
                idx_out[row * k + r] = bi;
                score_out[row * k + r] = bs;
                s_ps = bs;
                s_pi = bi;
            }
        }
        __syncthreads();
        ps = s_ps;
        pi = s_pi;
    }
}

int grid_of(uint64_t n) { return (int)std::min<uint64_t>((n + 255) / 256, 148 * 32); }

// softmax.hpp:13-27 stable_softmax of one vector, one CTA: the max, exp(l - max) in f64 for
// every element in parallel, then the f64 sum in element order by one thread (the reference's
// bits), then float(float(e) / sum)
__global__ void __launch_bounds__(1024) softmax_kernel(const float* __restrict__ l, uint32_t n, float* out,
                                                       double* scratch) {
    __shared__ float s_max[32];
    __shared__ double s_sum;
    float m = -INFINITY;
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) m = fmaxf(m, l[i]);
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xFFFFFFFFu, m, o));
    if ((threadIdx.x & 31) == 0) s_max[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x < 32) {
        m = threadIdx.x < (blockDim.x >> 5) ? s_max[threadIdx.x] : -INFINITY;
        for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xFFFFFFFFu, m, o));
        if (threadIdx.x == 0) s_max[0] = m;
    }
    __syncthreads();
    const double mx = (double)s_max[0];
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
        const double e = exp((double)l[i] - mx);
        scratch[i] = e;
        out[i] = (float)e;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double sum = 0.0;
        for (uint32_t i = 0; i < n; ++i) sum += scratch[i];
        s_sum = sum;
    }
    __syncthreads();
    const double sum = s_sum;
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) out[i] = (float)((double)out[i] / sum);
}

// softmax.hpp:29-36 attention_entropy: -sum w ln w over w > 0 in element order, clamped at 0
__global__ void __launch_bounds__(1024) entropy_kernel(const float* __restrict__ w, uint32_t n, double* out,
                                                       double* scratch) {
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
        const float v = w[i];
        scratch[i] = v > 0.0f ? (double)v * log((double)v) : 0.0;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double h = 0.0;
        for (uint32_t i = 0; i < n; ++i)
            if (w[i] > 0.0f) h -= scratch[i];
        *out = h < 0.0 ? 0.0 : h;
    }
}

}  // namespace

cudaError_t launch_dot_f32(const float* a, const float* b, uint64_t n, uint64_t d, int lanes,
                           float* out, cudaStream_t s) {
    if (lanes == kLanesFma)
        dot_f32_kernel<kLanesFma><<<grid_of(n), 256, 0, s>>>(a, b, n, (uint32_t)d, out);
    else
        dot_f32_kernel<kLanesUnfused><<<grid_of(n), 256, 0, s>>>(a, b, n, (uint32_t)d, out);
    return cudaGetLastError();
}

cudaError_t launch_dot_f64(const float* a, const float* b, uint64_t n, uint64_t d, double* out,
                           cudaStream_t s) {
    dot_f64_kernel<<<grid_of(n), 256, 0, s>>>(a, b, n, (uint32_t)d, out);
    return cudaGetLastError();
}

cudaError_t launch_matmul(const float* a, const float* b, uint64_t m, uint64_t k, uint64_t n,
                          float* c, cudaStream_t s) {
    matmul_kernel<<<grid_of(m * n), 256, 0, s>>>(a, b, m, k, n, c);
    return cudaGetLastError();
}

cudaError_t launch_group_mean(const float* q, uint64_t n_q, uint64_t n_heads, uint64_t n_kv,
                              uint64_t d, float* out, cudaStream_t s) {
    group_mean_kernel<<<grid_of(n_q * n_kv * d), 256, 0, s>>>(q, n_q, (uint32_t)n_heads,
                                                              (uint32_t)n_kv, (uint32_t)d, out);
    return cudaGetLastError();
}

cudaError_t launch_stable_softmax(const float* l, uint64_t n, float* out, double* scratch, cudaStream_t s) {
    softmax_kernel<<<1, 1024, 0, s>>>(l, (uint32_t)n, out, scratch);
    return cudaGetLastError();
}

cudaError_t launch_attention_entropy(const float* w, uint64_t n, double* out, double* scratch, cudaStream_t s) {
    entropy_kernel<<<1, 1024, 0, s>>>(w, (uint32_t)n, out, scratch);
    return cudaGetLastError();
}

size_t naive_topk_workspace(uint64_t n_q, uint64_t n_kv, uint64_t count, uint64_t d) {
    return (n_q * n_kv * d + n_q * n_kv * count) * sizeof(float) + 256;
}

cudaError_t launch_naive_topk(const ScanArgs& a, void* ws, cudaStream_t s) {
    float* mq = (float*)ws;
    float* scores = mq + (size_t)a.n_q * a.n_kv * a.d;
    cudaError_t e = launch_group_mean(a.q, a.n_q, a.n_heads, a.n_kv, a.d, mq, s);
    if (e != cudaSuccess) return e;
    const dim3 grid((unsigned)std::min<uint32_t>(a.count, 148u * 16u), (unsigned)a.n_kv);
    const size_t smem = (size_t)a.d * sizeof(float);
#define NAIVE(KT, L)                                                                        \
    naive_scores_kernel<KT, L><<<grid, 128, smem, s>>>(mq, (uint32_t)a.n_q, (uint32_t)a.n_kv, \
                                                       (uint32_t)a.d, (const KT*)a.keys,    \
                                                       a.head_stride, a.row0, a.count, scores)
    if (a.dtype == kBF16) {
        if (a.lanes == kLanesFma) NAIVE(__nv_bfloat16, kLanesFma);
        else NAIVE(__nv_bfloat16, kLanesUnfused);
    } else {
        if (a.lanes == kLanesFma) NAIVE(float, kLanesFma);
        else NAIVE(float, kLanesUnfused);
    }
#undef NAIVE
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    const uint32_t kk = std::min<uint32_t>((uint32_t)a.k, a.count);
    naive_select_kernel<<<(unsigned)(a.n_kv * a.n_q), 256, 0, s>>>(scores, a.count, kk, (uint32_t)a.k,
                                                                   a.idx_out, a.score_out);
    return cudaGetLastError();
}

}  // namespace reattn_impl
