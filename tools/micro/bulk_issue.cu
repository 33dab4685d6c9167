// Issue cost of cp.async.bulk (global -> shared, mbarrier complete_tx) as K5's producer uses
// it: one warp per SM, lane 0 issues `n` copies of `bytes` each from scattered rows of a large
// buffer, timed with clock64 around the issue loop only (and around the wait); LDGSTS
// (cp.async 16 B per lane) of the same bytes for comparison.  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 bulk_issue.cu -o bulk_issue
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#include "../../paper_2407_15176_b200/csrc/common.cuh"
using namespace reattn_dev;

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

__global__ void __launch_bounds__(32, 1) bulk_issue(const uint8_t* buf, size_t buf_bytes, int n,
                                                    int bytes, int mode, long long* out) {
    // span: sources scattered over buf_bytes (1 GB: a new 2 MB page per copy; 1 MB: one page)
    extern __shared__ __align__(128) uint8_t sm[];
    __shared__ uint64_t bar;
    const int lane = threadIdx.x;
    if (lane == 0) {
        mbar_init(&bar, 1);
        fence_barrier_init();
    }
    __syncwarp();
    // scattered sources: a hash of (block, i) over the buffer, 256-B aligned
    auto src_of = [&](int i) {
        const uint64_t h = (uint64_t)(blockIdx.x * 7919 + i * 104729) * 2654435761ull;
        return buf + ((h % (buf_bytes / 256 - 64)) * 256);
    };
    __shared__ const uint8_t* srcs[64];  // addresses computed outside the timed region
    for (int i = lane; i < n; i += 32) srcs[i] = src_of(i);
    __syncwarp();
    long long t0 = clock64();
    if (mode == 0) {  // bulk copies by lane 0
        if (lane == 0) {
            mbar_arrive_expect_tx(&bar, (uint32_t)n * bytes);
            for (int i = 0; i < n; ++i) bulk_g2s(sm + (size_t)i * bytes, srcs[i], bytes, &bar);
        }
    } else {  // LDGSTS: the warp copies the same bytes 16 B per lane
        for (int i = 0; i < n; ++i) {
            const uint8_t* s = srcs[i];
            for (int o = lane * 16; o < bytes; o += 512) {
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(sm + (size_t)i * bytes + o)),
                             "l"(s + o)
                             : "memory");
            }
        }
        asm volatile("cp.async.mbarrier.arrive.shared::cta.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
        if (lane == 0) mbar_arrive_expect_tx(&bar, 0);
    }
    __syncwarp();
    long long t1 = clock64();
    mbar_wait(&bar, 0);
    long long t2 = clock64();
    if (lane == 0) {
        out[blockIdx.x * 2] = t1 - t0;
        out[blockIdx.x * 2 + 1] = t2 - t0;
    }
}

int main() {
    const size_t buf_bytes = 1ull << 30;
    uint8_t* buf;
    cudaMalloc(&buf, buf_bytes);
    cudaMemset(buf, 1, buf_bytes);
    long long* out;
    const int blocks = 148;
    cudaMalloc(&out, blocks * 2 * sizeof(long long));
    long long h[blocks * 2];
    cudaFuncSetAttribute(bulk_issue, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    for (size_t span : {buf_bytes, (size_t)1 << 20})
    for (int mode = 0; mode < 2; ++mode)
        for (int bytes : {1024, 8192})
            for (int n : {1, 4, 16}) {
                if ((size_t)n * bytes > 190 * 1024) continue;
                for (int rep = 0; rep < 3; ++rep) {
                    bulk_issue<<<blocks, 32, n * bytes>>>(buf, span, n, bytes, mode, out);
                    cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
                }
                double iss = 0, tot = 0;
                for (int b = 0; b < blocks; ++b) {
                    iss += h[2 * b];
                    tot += h[2 * b + 1];
                }
                printf("span %10zu %s bytes %5d n %2d: issue %8.0f cyc (%6.0f per copy)  issue+land %8.0f cyc\n",
                       span, mode ? "ldgsts" : "bulk  ", bytes, n, iss / blocks, iss / blocks / n, tot / blocks);
            }
    cudaError_t e = cudaDeviceSynchronize();
    printf("status %s\n", cudaGetErrorString(e));
    return 0;
}
