// Small supporting kernels: cache append (kv_cache.hpp:54-68 layout change), scope gather
// for the assemble_scope API (scope.hpp:63-76), RoPE on device rows (rope.hpp:49-60),
// the deterministic synthetic-input generator used by tests and bench.py, and the RunStats
// entropy reduction in the reference's accumulation order (engine.hpp:100-106).
#include <cstdlib>

#include <algorithm>

#include "common.cuh"
#include "kernels.h"

using namespace reattn_dev;

namespace reattn_impl {

namespace {

template <typename T>
__device__ __forceinline__ void store_from_float(T* p, float v);
template <>
__device__ __forceinline__ void store_from_float<float>(float* p, float v) {
    *p = v;
}
template <>
__device__ __forceinline__ void store_from_float<__nv_bfloat16>(__nv_bfloat16* p, float v) {
    *p = __float2bfloat16_rn(v);
}

template <typename T>
__global__ void cache_append_kernel(const float* __restrict__ src, T* __restrict__ dst,
                                    uint64_t rows, uint64_t n_kv, uint64_t d,
                                    uint64_t head_stride, uint64_t row0) {
    const uint64_t n = rows * n_kv * d;
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < n;
         e += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t r = e / (n_kv * d), rem = e % (n_kv * d);
        const uint64_t h = rem / d, c = rem % d;
        store_from_float<T>(dst + (h * head_stride + row0 + r) * d + c, src[e]);
    }
}

template <typename T>
__global__ void gather_kernel(const T* __restrict__ base, uint64_t n_kv, uint64_t d,
                              uint64_t head_stride, const uint32_t* __restrict__ src, uint32_t L,
                              float* __restrict__ out) {
    const uint64_t n = n_kv * (uint64_t)L * d;
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < n;
         e += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t h = e / ((uint64_t)L * d), rem = e % ((uint64_t)L * d);
        const uint64_t r = rem / d, c = rem % d;
        out[e] = load_as_float<T>(base + (h * head_stride + src[r]) * d + c);
    }
}

__global__ void rope_rotate_kernel(float* rows, const uint32_t* pos, uint64_t n_rows, uint64_t d,
                                   const float* cos_t, const float* sin_t) {
    const uint64_t half = d / 2;
    const uint64_t n = n_rows * half;
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < n;
         e += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t r = e / half, i = e % half;
        float* v = rows + r * d;
        const float c = cos_t[(uint64_t)pos[r] * half + i];
        const float s = sin_t[(uint64_t)pos[r] * half + i];
        const float x = v[2 * i], y = v[2 * i + 1];
        v[2 * i] = __fsub_rn(__fmul_rn(x, c), __fmul_rn(y, s));
        v[2 * i + 1] = __fadd_rn(__fmul_rn(x, s), __fmul_rn(y, c));
    }
}

// splitmix64 of (seed, index) -> uniform [-1, 1) with 24 significant bits (exact in fp32).
__device__ __forceinline__ float synth_value(uint64_t seed, uint64_t i) {
    uint64_t z = seed * 0x9E3779B97F4A7C15ull + i + 0x632BE59BD9B4E019ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    return (float)(z >> 40) * (1.0f / 8388608.0f) - 1.0f;
}

template <typename T>
__global__ void synth_kernel(T* dst, uint64_t n, uint64_t seed, uint64_t offset) {
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < n;
         e += (uint64_t)gridDim.x * blockDim.x)
        store_from_float<T>(dst + e, synth_value(seed, offset + e));
}

__global__ void entropy_stats_kernel(const double* ent, int n_q, int n_head, double* out2) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        double mx = 0.0, sum = 0.0;
        for (int h = 0; h < n_head; ++h)
            for (int i = 0; i < n_q; ++i) {
                const double e = ent[(size_t)i * n_head + h];
                mx = fmax(mx, e);
                sum += e;
            }
        out2[0] = mx;
        out2[1] = sum;
    }
}

int grid_for(uint64_t n) {
    uint64_t g = (n + 255) / 256;
    if (g > 148ull * 16) g = 148ull * 16;
    return (int)(g ? g : 1);
}

}  // namespace

cudaError_t launch_cache_append(const float* src, void* dst, int dtype, uint64_t rows,
                                uint64_t n_kv, uint64_t d, uint64_t head_stride, uint64_t row0,
                                cudaStream_t s) {
    const int g = grid_for(rows * n_kv * d);
    if (dtype == kBF16)
        cache_append_kernel<__nv_bfloat16><<<g, 256, 0, s>>>(src, (__nv_bfloat16*)dst, rows, n_kv,
                                                              d, head_stride, row0);
    else
        cache_append_kernel<float><<<g, 256, 0, s>>>(src, (float*)dst, rows, n_kv, d, head_stride,
                                                     row0);
    return cudaGetLastError();
}

namespace {
// One decode step's K and V rows (DenseMatrix layout [1][n_kv * d] fp32, kv_cache.hpp:54-68)
// appended at the device-resident cache length, which is then advanced: the append node of a
// plan whose graph serves every decode step.  One CTA; thread 0 publishes the new length after
// the CTA's stores (the next kernel in the stream reads it).
template <typename T>
__global__ void __launch_bounds__(256) cache_append_step_kernel(const float* __restrict__ k_in,
                                                                const float* __restrict__ v_in,
                                                                T* keys, T* values, uint32_t n_kv,
                                                                uint32_t d, uint64_t head_stride,
                                                                uint32_t* dev_total) {
    const uint32_t row = *(volatile uint32_t*)dev_total;
    RA_ASSERT(row < head_stride);  // the plan checked capacity on the host mirror
    for (uint32_t e = threadIdx.x; e < n_kv * d; e += blockDim.x) {
        const uint32_t h = e / d, c = e % d;
        const size_t o = ((size_t)h * head_stride + row) * d + c;
        store_from_float<T>(keys + o, k_in[e]);
        store_from_float<T>(values + o, v_in[e]);
    }
    __syncthreads();
    if (threadIdx.x == 0) *(volatile uint32_t*)dev_total = row + 1u;
}

__global__ void set_u32_kernel(uint32_t* p, uint32_t v) { *p = v; }

// Zero-copy host I/O of a decode step (reattn_plan_step_host / run_host on pinned buffers):
// up to four host arrays read straight over the bus into device buffers, or written back, by a few CTAs -- no DMA set-up per array.  16-byte vectors when everything is
// aligned.
struct HostIo {
    const float* src[4];
    float* dst[4];
    uint32_t n[4];
    int count;
};

__global__ void __launch_bounds__(256) host_io_kernel(const HostIo io) {
    const uint32_t stride = gridDim.x * blockDim.x, t0 = blockIdx.x * blockDim.x + threadIdx.x;
#pragma unroll 1
    for (int a = 0; a < io.count; ++a) {
        const float* src = io.src[a];
        float* dst = io.dst[a];
        const uint32_t n = io.n[a];
        if ((((uintptr_t)src | (uintptr_t)dst) & 15) == 0) {
            const uint32_t n4 = n / 4;
            for (uint32_t i = t0; i < n4; i += stride)
                reinterpret_cast<float4*>(dst)[i] = reinterpret_cast<const float4*>(src)[i];
            for (uint32_t i = 4 * n4 + t0; i < n; i += stride) dst[i] = src[i];
        } else {
            for (uint32_t i = t0; i < n; i += stride) dst[i] = src[i];
        }
    }
}
}  // namespace

cudaError_t launch_host_io(const float* const* src, float* const* dst, const uint64_t* n, int count,
                           cudaStream_t s) {
    HostIo io{};
    uint64_t total = 0;
    for (int a = 0; a < count && a < 4; ++a) {
        io.src[a] = src[a];
        io.dst[a] = dst[a];
        io.n[a] = (uint32_t)n[a];
        total += n[a];
    }
    io.count = count < 4 ? count : 4;
    if (total == 0) return cudaSuccess;
    const int g = (int)std::min<uint64_t>(16, (total / 4 + 255) / 256 + 1);
    host_io_kernel<<<g, 256, 0, s>>>(io);
    return cudaGetLastError();
}

cudaError_t launch_cache_append_step(const float* k_in, const float* v_in, void* keys, void* values,
                                     int dtype, uint64_t n_kv, uint64_t d, uint64_t head_stride,
                                     uint32_t* dev_total, cudaStream_t s) {
    if (dtype == kBF16)
        cache_append_step_kernel<__nv_bfloat16><<<1, 256, 0, s>>>(
            k_in, v_in, (__nv_bfloat16*)keys, (__nv_bfloat16*)values, (uint32_t)n_kv, (uint32_t)d,
            head_stride, dev_total);
    else
        cache_append_step_kernel<float><<<1, 256, 0, s>>>(k_in, v_in, (float*)keys, (float*)values,
                                                          (uint32_t)n_kv, (uint32_t)d, head_stride,
                                                          dev_total);
    return cudaGetLastError();
}

cudaError_t launch_set_u32(uint32_t* p, uint32_t v, cudaStream_t s) {
    set_u32_kernel<<<1, 1, 0, s>>>(p, v);
    return cudaGetLastError();
}

cudaError_t launch_gather(const void* base, int dtype, uint64_t n_kv, uint64_t d,
                          uint64_t head_stride, const uint32_t* src, uint32_t L, float* out,
                          cudaStream_t s) {
    const int g = grid_for(n_kv * (uint64_t)L * d);
    if (dtype == kBF16)
        gather_kernel<__nv_bfloat16><<<g, 256, 0, s>>>((const __nv_bfloat16*)base, n_kv, d,
                                                        head_stride, src, L, out);
    else
        gather_kernel<float><<<g, 256, 0, s>>>((const float*)base, n_kv, d, head_stride, src, L,
                                               out);
    return cudaGetLastError();
}

cudaError_t launch_rope_rotate(float* rows, const uint32_t* pos, uint64_t n_rows, uint64_t d,
                               const float* cos_t, const float* sin_t, cudaStream_t s) {
    rope_rotate_kernel<<<grid_for(n_rows * (d / 2)), 256, 0, s>>>(rows, pos, n_rows, d, cos_t,
                                                                  sin_t);
    return cudaGetLastError();
}

cudaError_t launch_synth_uniform(void* dst, int dtype, uint64_t n, uint64_t seed, uint64_t offset,
                                 cudaStream_t s) {
    if (dtype == kBF16)
        synth_kernel<__nv_bfloat16><<<grid_for(n), 256, 0, s>>>((__nv_bfloat16*)dst, n, seed,
                                                                 offset);
    else
        synth_kernel<float><<<grid_for(n), 256, 0, s>>>((float*)dst, n, seed, offset);
    return cudaGetLastError();
}

cudaError_t launch_entropy_stats(const double* entropy, int n_q, int n_head, double* out2,
                                 cudaStream_t s) {
    entropy_stats_kernel<<<1, 32, 0, s>>>(entropy, n_q, n_head, out2);
    return cudaGetLastError();
}

}  // namespace reattn_impl

// ---- timeline trace ------------------------------------------------------------------
// Layout (uint64 words, %globaltimer ns):
//   K1 scan (G CTAs):   [b] CTA start, [512 + b] CTA main loop done,
//                       [1024] merger CTA 0 sees every CTA done, [1025] merge done, [1026] select done
//   K5 decode attention: [1536 + cta] CTA start (after griddepcontrol.wait),
//                       [2560 + cta] CTA compute done (cta = blockIdx.y * gridDim.x + blockIdx.x,
//                       + 512 for the local-window launch),
//                       [3584 + kv] kv head's final merge done
namespace reattn_impl {
namespace {
__device__ uint64_t g_trace[kTraceWords];
}
uint64_t* trace_buffer() {
    static int on = -1;
    if (on < 0) {
        const char* e = std::getenv("REATTN_TRACE");
        on = e && std::atoi(e) != 0;
    }
    if (!on) return nullptr;
    void* p = nullptr;
    return cudaGetSymbolAddress(&p, g_trace) == cudaSuccess ? (uint64_t*)p : nullptr;
}
}  // namespace reattn_impl
