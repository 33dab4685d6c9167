// tcgen05.mma dispatch rate on resident operands (no TMA, no epilogue): one CTA per SM, one
// thread issues `tiles` x 8 MMAs (K = 128 in steps of 16, bf16 -> f32) into a TMEM
// accumulator, then commits and waits.  Variants: SS (A and B in shared memory) with N = 128
// or 256, TS (A in TMEM) with N = 128.  Build: nvcc -gencode arch=compute_100a,code=sm_100a
//   -O3 -std=c++17 mma_rate.cu -o mma_rate
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#include "../../paper_2407_15176_b200/csrc/common.cuh"
#include "../../paper_2407_15176_b200/csrc/tcgen05.cuh"
using namespace reattn_dev;

template <int N, bool TS>
__global__ void __launch_bounds__(128, 1) mma_rate(int tiles, long long* cyc) {
    extern __shared__ uint8_t raw[];
    uint8_t* sm = (uint8_t*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
    uint8_t* sa = sm;               // 128 x 128 bf16, SW128 K-major: 32 KB
    uint8_t* sb = sm + 32768;       // N x 128 bf16: N * 256 B
    __shared__ uint64_t bar;
    __shared__ uint32_t s_tmem;
    for (int i = threadIdx.x; i < (32768 + N * 256) / 16; i += blockDim.x)
        reinterpret_cast<uint4*>(sm)[i] = make_uint4(0, 0, 0, 0);
    if (threadIdx.x < 32) tmem_alloc(&s_tmem, 512);
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        fence_barrier_init();
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = s_tmem;
    if (threadIdx.x == 0) {
        constexpr uint32_t idesc = idesc_bf16_f32<128, N>();
        const uint32_t a0 = smem_u32(sa), b0 = smem_u32(sb);
        const long long t0 = clock64();
        for (int t = 0; t < tiles; ++t) {
#pragma unroll
            for (int kb = 0; kb < 2; ++kb)
#pragma unroll
                for (int ks = 0; ks < 4; ++ks) {
                    const uint64_t bd = umma_desc_sw128(b0 + kb * (N * 128) + ks * 32);
                    if (TS)
                        mma_bf16_ts(tmem, tmem + 384 + kb * 32 + ks * 8, bd, idesc, 1u);
                    else
                        mma_bf16_ss(tmem, umma_desc_sw128(a0 + kb * 16384 + ks * 32), bd, idesc, 1u);
                }
        }
        mma_commit(&bar);
        mbar_wait(&bar, 0);
        cyc[blockIdx.x] = clock64() - t0;
    }
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x < 32) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

template <int N, bool TS>
void run(const char* name) {
    const int sms = 148, tiles = 4096;
    long long* cyc;
    cudaMalloc(&cyc, sms * 8);
    const int smem = 1024 + 32768 + N * 256;
    cudaFuncSetAttribute(mma_rate<N, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    mma_rate<N, TS><<<sms, 128, smem>>>(16, cyc);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    mma_rate<N, TS><<<sms, 128, smem>>>(tiles, cyc);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    long long c0;
    cudaMemcpy(&c0, cyc, 8, cudaMemcpyDeviceToHost);
    const double flop = 2.0 * 128 * N * 128 * (double)tiles * sms;
    printf("%-10s N=%3d: %.3f ms, %.0f TFLOP/s, %.1f cycles per 128xNx16 MMA\n", name, N, ms,
           flop / (ms * 1e-3) / 1e12, (double)c0 / (tiles * 8.0));
    printf("   err: %s\n", cudaGetErrorString(cudaGetLastError()));
}

int main() {
    run<128, false>("SS");
    run<128, true>("TS");
    run<256, false>("SS");
    return 0;
}
