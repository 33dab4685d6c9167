// TMEM read bandwidth microbenchmark: W warps per CTA, one CTA per SM, each warp loads
// tcgen05.ld 32x32b.x64 (8 KB per warp-load) from its lane quarter in a loop.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2407_15176_b200/csrc/common.cuh"
#include "../../paper_2407_15176_b200/csrc/tcgen05.cuh"
using namespace reattn_dev;

template <int W>
__global__ void __launch_bounds__(W * 32, 1) tmem_read(int iters, uint32_t* out, long long* cyc) {
    __shared__ uint32_t s_tmem;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) tmem_alloc(&s_tmem, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = s_tmem;
    const uint32_t base = tmem + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)((warp >> 2) * 64 % 512);
    uint32_t acc = 0;
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        uint32_t r[64];
        TMEM_LD_X64(base + (uint32_t)((i & 3) * 128 % 512), r);
        tmem_wait_ld();
#pragma unroll
        for (int c = 0; c < 64; ++c) acc ^= r[c];
    }
    __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

template <int W>
void run() {
    const int iters = 4096, sms = 148;
    uint32_t* out;
    long long* cyc;
    cudaMalloc(&out, sms * W * 32 * 4);
    cudaMalloc(&cyc, sms * 8);
    tmem_read<W><<<sms, W * 32>>>(16, out, cyc);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    tmem_read<W><<<sms, W * 32>>>(iters, out, cyc);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    long long c0;
    cudaMemcpy(&c0, cyc, 8, cudaMemcpyDeviceToHost);
    const double bytes_sm = (double)iters * W * 8192;
    printf("{\"warps\": %d, \"bytes_per_cycle_per_sm\": %.1f, \"ms\": %.3f, \"TB_s_chip\": %.1f, \"err\": \"%s\"}\n", W,
           bytes_sm / c0, ms, bytes_sm * sms / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
}

int main() {
    run<4>();
    run<8>();
    run<16>();
    return 0;
}
