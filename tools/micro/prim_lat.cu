// Latency of block / warp primitives on one SM (256 threads), in SM cycles (clock64):
// bar.sync, bar.red.popc, redux.sync, dependent LDS, shared atomicOr, SHFL, a global store
// followed by __threadfence.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3
//   -std=c++17 prim_lat.cu -o prim_lat
#include <cstdio>
#include <cstdint>

__global__ void __launch_bounds__(256) prim_kernel(long long* out, unsigned* gbuf) {
    __shared__ unsigned sm[1024];
    __shared__ unsigned smask;
    const int tid = threadIdx.x;
    for (int i = tid; i < 1024; i += 256) sm[i] = (i * 7 + 1) & 1023;
    if (tid == 0) smask = 0;
    __syncthreads();
    constexpr int N = 200;
    unsigned v = tid;
    long long t0, t1;
    for (int rep = 0; rep < 2; ++rep) {  // rep 0 warms the i-cache
        int slot = 0;
        // 1. bar.sync
        t0 = clock64();
#pragma unroll 1
        for (int i = 0; i < N; ++i) __syncthreads();
        t1 = clock64();
        if (rep && tid == 0) out[slot] = (t1 - t0) / N;
        ++slot;
        // 2. bar.red.popc
        t0 = clock64();
#pragma unroll 1
        for (int i = 0; i < N; ++i) v += __syncthreads_count(v & 1);
        t1 = clock64();
        if (rep && tid == 0) out[slot] = (t1 - t0) / N;
        ++slot;
        // 3. redux.sync add (dependent)
        t0 = clock64();
#pragma unroll 1
        for (int i = 0; i < N; ++i) v = __reduce_add_sync(0xFFFFFFFFu, v) & 0xFF;
        t1 = clock64();
        if (rep && tid == 0) out[slot] = (t1 - t0) / N;
        ++slot;
        // 4. dependent LDS
        t0 = clock64();
#pragma unroll 1
        for (int i = 0; i < N; ++i) v = sm[v & 1023];
        t1 = clock64();
        if (rep && tid == 0) out[slot] = (t1 - t0) / N;
        ++slot;
        // 5. shared atomicOr (all threads, same word) then bar
        t0 = clock64();
#pragma unroll 1
        for (int i = 0; i < N; ++i) {
            atomicOr(&smask, 1u << (v & 31));
            __syncthreads();
        }
        t1 = clock64();
        if (rep && tid == 0) out[slot] = (t1 - t0) / N;
        ++slot;
        // 6. dependent SHFL
        t0 = clock64();
#pragma unroll 1
        for (int i = 0; i < N; ++i) v = __shfl_sync(0xFFFFFFFFu, v, (v + 1) & 31);
        t1 = clock64();
        if (rep && tid == 0) out[slot] = (t1 - t0) / N;
        ++slot;
        // 7. global store + threadfence (thread 0)
        t0 = clock64();
        if (tid == 0) {
#pragma unroll 1
            for (int i = 0; i < N; ++i) {
                gbuf[i] = v;
                __threadfence();
            }
        }
        t1 = clock64();
        if (rep && tid == 0) out[slot] = (t1 - t0) / N;
        ++slot;
        // 8. global atomicAdd returning (thread 0), dependent
        t0 = clock64();
        if (tid == 0) {
#pragma unroll 1
            for (int i = 0; i < N; ++i) v += atomicAdd(gbuf + 512 + (v & 7), 1u) & 1;
        }
        t1 = clock64();
        if (rep && tid == 0) out[slot] = (t1 - t0) / N;
        ++slot;
        // 9. bar.sync with one warp doing 4 dependent shuffles in between (warp-0 phase)
        t0 = clock64();
#pragma unroll 1
        for (int i = 0; i < N; ++i) {
            if (tid < 32) v = __shfl_up_sync(0xFFFFFFFFu, v, 1) + 1;
            __syncthreads();
        }
        t1 = clock64();
        if (rep && tid == 0) out[slot] = (t1 - t0) / N;
        ++slot;
    }
    gbuf[1000 + tid] = v;
}

int main() {
    long long* out;
    unsigned* gbuf;
    cudaMalloc(&out, 64 * sizeof(long long));
    cudaMalloc(&gbuf, 4096 * 4);
    cudaMemset(gbuf, 0, 4096 * 4);
    prim_kernel<<<1, 256>>>(out, gbuf);
    prim_kernel<<<1, 256>>>(out, gbuf);
    long long h[16];
    cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
    const char* names[] = {"bar.sync (256 thr)", "bar.red.popc", "redux.sync add (dep)",
                           "LDS (dep)", "smem atomicOr + bar", "SHFL (dep)",
                           "STG + membar.gl", "global atomicAdd (dep)", "bar + 1 warp shfl_up"};
    for (int i = 0; i < 9; ++i) printf("%-24s %6lld cycles\n", names[i], h[i]);
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
