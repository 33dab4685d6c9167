// Read-only HBM bandwidth ceiling on this GPU (what K1's scan could reach at best): every SM
// streams a contiguous slice of a 4 GiB buffer and only reduces it (a sum kept live), two ways:
//   ldg  : 1024 threads, LDG.128 (ld.global.nc.L1::no_allocate), U loads in flight per thread
//   bulk : one thread issues cp.async.bulk of `chunk` bytes into an S-stage shared ring, 512
//          threads consume each stage from shared memory (the scan's structure without TMA
//          tensor maps)
// Prints GB/s (bytes / CUDA-event time, best of 5).  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 hbm_read.cu -o hbm_read
#include <cstdint>
#include <cstdio>
#include <cuda.h>
#include <cuda_runtime.h>

#include "../../paper_2407_15176_b200/csrc/common.cuh"
using namespace reattn_dev;

template <int U>
__global__ void __launch_bounds__(1024, 1) ldg_read(const uint4* buf, size_t n16, uint32_t* sink) {
    const size_t per = n16 / gridDim.x;
    const uint4* p = buf + per * blockIdx.x;
    uint32_t acc = 0;
    for (size_t i = threadIdx.x; i + (U - 1) * 1024 < per; i += (size_t)U * 1024) {
        uint4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u)
            asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                         : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w)
                         : "l"(p + i + (size_t)u * 1024));
#pragma unroll
        for (int u = 0; u < U; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
    }
    if (acc == 0x12345678u) sink[0] = acc;
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

__global__ void __launch_bounds__(544, 1) bulk_read(const uint8_t* buf, size_t bytes, int chunk, int S,
                                                    uint32_t* sink) {
    extern __shared__ __align__(128) uint8_t sm[];
    __shared__ uint64_t full[16], empty[16];
    const size_t per = bytes / gridDim.x / chunk * chunk;
    const uint8_t* p = buf + per * blockIdx.x;
    const int n = (int)(per / chunk);
    const int tid = threadIdx.x, warp = tid >> 5;
    if (tid == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 16);
        }
        fence_barrier_init();
    }
    __syncthreads();
    if (warp == 16) {
        if ((tid & 31) == 0)
            for (int c = 0; c < n; ++c) {
                const int s = c % S;
                if (c >= S) mbar_wait(&empty[s], ((c / S) & 1u) ^ 1u);
                mbar_arrive_expect_tx(&full[s], chunk);
                bulk_g2s(sm + (size_t)s * chunk, p + (size_t)c * chunk, chunk, &full[s]);
            }
        return;
    }
    uint32_t acc = 0;
    for (int c = 0; c < n; ++c) {
        const int s = c % S;
        mbar_wait(&full[s], (c / S) & 1u);
        const uint4* st = reinterpret_cast<const uint4*>(sm + (size_t)s * chunk);
        for (int i = tid; i < chunk / 16; i += 512) {
            const uint4 v = st[i];
            acc ^= v.x ^ v.y ^ v.z ^ v.w;
        }
        __syncwarp();
        if ((tid & 31) == 0) mbar_arrive(&empty[s]);
    }
    if (acc == 0x12345678u) sink[0] = acc;
}

// the scan's own access: 2-D tensor map over [rows][128] bf16 with 128-byte boxes of `box_rows`
// rows (SWIZZLE_128B), two boxes per 256-byte row, S stages of box_rows * 256 bytes, optional
// L2 evict_first
__global__ void __launch_bounds__(288, 1) tma_read(const __grid_constant__ CUtensorMap map, uint32_t rows,
                                                   int box_rows, int S, int evict_first, uint32_t* sink) {
    extern __shared__ __align__(1024) uint8_t sm_raw[];
    uint8_t* sm = (uint8_t*)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
    __shared__ uint64_t full[16], empty[16];
    const uint32_t per = rows / gridDim.x / box_rows * box_rows;
    const uint32_t r0 = per * blockIdx.x;
    const int n = (int)(per / box_rows);
    const int stage = box_rows * 256;
    const int tid = threadIdx.x, warp = tid >> 5;
    if (tid == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 8);
        }
        fence_barrier_init();
    }
    __syncthreads();
    if (warp == 8) {
        if ((tid & 31) == 0) {
            uint64_t pol;
            if (evict_first)
                asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
            else
                asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
            for (int c = 0; c < n; ++c) {
                const int s = c % S;
                if (c >= S) mbar_wait(&empty[s], ((c / S) & 1u) ^ 1u);
                mbar_arrive_expect_tx(&full[s], stage);
                for (int b = 0; b < 2; ++b)
                    tma_load_2d(sm + (size_t)s * stage + b * box_rows * 128, &map, b * 64,
                                (int32_t)(r0 + (uint32_t)c * box_rows), &full[s], pol);
            }
        }
        return;
    }
    uint32_t acc = 0;
    for (int c = 0; c < n; ++c) {
        const int s = c % S;
        mbar_wait(&full[s], (c / S) & 1u);
        const uint4* st = reinterpret_cast<const uint4*>(sm + (size_t)s * stage);
        for (int i = tid; i < stage / 16; i += 256) {
            const uint4 v = st[i];
            acc ^= v.x ^ v.y ^ v.z ^ v.w;
        }
        __syncwarp();
        if ((tid & 31) == 0) mbar_arrive(&empty[s]);
    }
    if (acc == 0x12345678u) sink[0] = acc;
}

int main() {
    const size_t bytes = 4ull << 30;
    uint8_t* buf;
    uint32_t* sink;
    cudaMalloc(&buf, bytes);
    cudaMalloc(&sink, 4);
    cudaMemset(buf, 1, bytes);
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto timeit = [&](auto launch, const char* name) {
        float best = 1e30f;
        for (int r = 0; r < 6; ++r) {
            cudaEventRecord(e0);
            launch();
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (r > 0 && ms < best) best = ms;
        }
        printf("%-28s %8.1f GB/s  (%.3f ms, %s)\n", name, bytes / (best * 1e-3) / 1e9, best,
               cudaGetErrorString(cudaGetLastError()));
    };
    const size_t n16 = bytes / 16;
    timeit([&] { ldg_read<4><<<sms, 1024>>>((const uint4*)buf, n16, sink); }, "ldg U=4");
    timeit([&] { ldg_read<8><<<sms, 1024>>>((const uint4*)buf, n16, sink); }, "ldg U=8");
    timeit([&] { ldg_read<8><<<sms * 2, 1024>>>((const uint4*)buf, n16, sink); }, "ldg U=8, 2 CTAs/SM");
    for (int ctas : {sms, sms - 4}) {
        cudaFuncSetAttribute(bulk_read, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768 * 4);
        char name[64];
        snprintf(name, sizeof(name), "bulk 32K x 4, %d CTAs", ctas);
        timeit([&] { bulk_read<<<ctas, 544, 32768 * 4>>>(buf, bytes, 32768, 4, sink); }, name);
    }
    {
        CUtensorMap map;
        const uint32_t rows = (uint32_t)(bytes / 256);
        cuuint64_t dims[2] = {128, rows};
        cuuint64_t strides[1] = {256};
        for (int box_rows : {128, 256}) {
            cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
            cuuint32_t es[2] = {1, 1};
            CUresult r = cuTensorMapEncodeTiled(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, box, es,
                                                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            if (r != CUDA_SUCCESS) printf("tensor map failed %d\n", (int)r);
            for (int S : {2, 3, 4})
                for (int ef : {0, 1})
                    for (int ctas : {sms, sms - 4}) {
                        const int smem = box_rows * 256 * S + 1024;
                        if (smem > 220 * 1024) continue;
                        cudaFuncSetAttribute(tma_read, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
                        char name[64];
                        snprintf(name, sizeof(name), "tma %dr x %d ef%d %d CTAs", box_rows, S, ef, ctas);
                        timeit([&] { tma_read<<<ctas, 288, smem>>>(map, rows, box_rows, S, ef, sink); }, name);
                    }
        }
    }
    for (int chunk : {16384, 32768})
        for (int S : {4, 6}) {
            if ((size_t)chunk * S > 200 * 1024) continue;
            cudaFuncSetAttribute(bulk_read, cudaFuncAttributeMaxDynamicSharedMemorySize, chunk * S);
            char name[64];
            snprintf(name, sizeof(name), "bulk chunk %d x %d", chunk, S);
            timeit([&] { bulk_read<<<sms, 544, chunk * S>>>(buf, bytes, chunk, S, sink); }, name);
        }
    return 0;
}
