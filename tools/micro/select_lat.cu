// Latency of the decode select (vote + spans + scope table, select_small.cuh) in one CTA,
// warm, stamped with %globaltimer per call; plus a probe of lone-warp SHFL / global-load
// round trips.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17
//   -I../../paper_2407_15176_b200/csrc select_lat.cu -o select_lat
#include <cstdio>
#include <vector>

#include "select_small.cuh"

using namespace reattn_impl;
using namespace reattn_dev;

__global__ void __launch_bounds__(256) sel_kernel(SmallSelectIO io, const uint32_t* cidx,
                                                  const float* cs, int n, uint64_t* stamps,
                                                  int reps) {
    __shared__ SmallSelectSmem ssel;
    for (int r = 0; r < reps; ++r) {
        __syncthreads();
        uint64_t* tr = stamps + 64 * r + 8 - 1024;  // select_small's trace slots 1028..
        const bool valid = threadIdx.x < n;
        const uint32_t ci = valid ? cidx[threadIdx.x] : 0;
        const float c = valid ? cs[threadIdx.x] : 0.f;
        __syncthreads();
        if (threadIdx.x == 0) tr[1028] = globaltimer();
        small_select_scope(io, ci, c, valid, ssel, tr);
        __syncthreads();
        if (threadIdx.x == 0) tr[1033] = globaltimer();
    }
}

__global__ void shfl_probe(uint64_t* stamps, const uint32_t* src, uint32_t* sink) {
    uint32_t v = threadIdx.x;
    const uint64_t c0 = clock64();
    const uint64_t t0 = globaltimer();
#pragma unroll 1
    for (int i = 0; i < 1000; ++i) v = __shfl_sync(0xFFFFFFFFu, v, (v + 1) & 31);
    const uint64_t t1 = globaltimer();
    uint32_t p = threadIdx.x;
#pragma unroll 1
    for (int i = 0; i < 100; ++i) p = __ldcg(src + p);
    const uint64_t t2 = globaltimer();
    if (threadIdx.x == 0) {
        stamps[0] = t1 - t0;
        stamps[1] = t2 - t1;
        stamps[2] = clock64() - c0;
        stamps[3] = globaltimer() - t0;
    }
    sink[threadIdx.x] = v + p;
}

int main() {
    const int n = 32, reps = 8;
    std::vector<uint32_t> hi(n);
    std::vector<float> hs(n);
    for (int i = 0; i < n; ++i) {
        hi[i] = (uint32_t)((i * 7919u * 131u) % 1000000u);
        hs[i] = 1.0f + 0.01f * i;
    }
    uint32_t *ci, *win, *sb, *se, *src;
    float* cs;
    uint64_t* st;
    ScopeHeader* hdr;
    cudaMalloc(&ci, n * 4);
    cudaMalloc(&cs, n * 4);
    cudaMalloc(&win, 512);
    cudaMalloc(&sb, 512);
    cudaMalloc(&se, 512);
    cudaMalloc(&src, 8192 * 4);
    cudaMalloc(&hdr, sizeof(ScopeHeader));
    cudaMalloc(&st, 4096 * 8);
    cudaMemcpy(ci, hi.data(), n * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(cs, hs.data(), n * 4, cudaMemcpyHostToDevice);
    SmallSelectIO io{};
    io.k_prime = 127;
    io.span_m = 32;
    io.middle_len = 1044448;
    io.span_mode = 0;
    io.g_end = 32;
    io.l_start = 1044480;
    io.total = 1048576;
    io.window = 8192;
    io.n_q = 1;
    io.winners = win;
    io.span_b = sb;
    io.span_e = se;
    io.scope_src = src;
    io.hdr = hdr;
    sel_kernel<<<1, 256>>>(io, ci, cs, n, st + 2048, reps);
    cudaDeviceSynchronize();
    std::vector<uint64_t> h(4096);
    cudaMemcpy(h.data(), st, 4096 * 8, cudaMemcpyDeviceToHost);
    for (int r = 0; r < reps; ++r) {
        const uint64_t* s = h.data() + 2048 + 64 * r + 8 - 1024;
        printf("select rep %d: tally %.2f rank/spans %.2f sort %.2f warp0 %.2f table %.2f us\n", r,
               (s[1030] - s[1028]) / 1e3, (s[1031] - s[1030]) / 1e3, (s[1032] - s[1031]) / 1e3,
               (s[1029] - s[1032]) / 1e3, (s[1033] - s[1029]) / 1e3);
    }
    uint32_t* sink;
    cudaMalloc(&sink, 128);
    std::vector<uint32_t> chain(8192);
    for (int i = 0; i < 8192; ++i) chain[i] = (i * 2654435761u + 977) % 8192;
    cudaMemcpy(src, chain.data(), 8192 * 4, cudaMemcpyHostToDevice);
    shfl_probe<<<1, 32>>>(st, src, sink);
    shfl_probe<<<1, 32>>>(st, src, sink);
    cudaDeviceSynchronize();
    cudaMemcpy(h.data(), st, 32, cudaMemcpyDeviceToHost);
    printf("probe: %llu cycles in %llu ns -> %.0f MHz\n", (unsigned long long)h[2],
           (unsigned long long)h[3], 1e3 * h[2] / (double)h[3]);
    printf("dependent SHFL: %.1f ns each; dependent ld.global.cg (L2 hit): %.1f ns each\n",
           h[0] / 1000.0, h[1] / 100.0);
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
