// Internal definitions shared by the C-ABI translation units (capi.cpp, capi_shard.cpp).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/reattn_cuda.h"
#include "kernels.h"

struct reattn_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    int lanes = REATTN_LANES_UNFUSED;
    int prefill = REATTN_PREFILL_TENSOR;  // reattn_prefill_mode bits (tcgen05 scan / attention)
    int num_sms = 148;
    std::string err;
    void* arena = nullptr;  // scratch for synchronous calls
    size_t arena_bytes = 0;
    // decode local-window fork: side stream + fork / join events (captured into plans)
    cudaStream_t side = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
};

struct reattn_cache {
    uint64_t n_kv, d, l_global, l_local_max, capacity, total = 0;
    int dtype;
    void* keys = nullptr;
    void* values = nullptr;
    // the length mirrored on the device (plans read it, so one graph serves every decode step
    // while the cache grows), and the storage generation (bumped when reserve reallocates)
    uint32_t* dev_total = nullptr;
    uint64_t generation = 0;
    uint64_t global_end() const { return std::min(total, l_global); }
    uint64_t local_start() const {
        const uint64_t g = global_end();
        return total - std::min(total - g, l_local_max);
    }
};

struct reattn_rope {
    uint64_t head_dim, max_position;
    double base;
    std::vector<float> cos_h, sin_h;
    float* cos_d = nullptr;
    float* sin_d = nullptr;
};

namespace reattn_capi {

using namespace reattn_impl;

inline int set_err(reattn_ctx* ctx, int code, const std::string& msg) {
    if (ctx) ctx->err = msg;
    return code;
}

#define CU(ctx, call)                                                                   \
    do {                                                                                \
        cudaError_t e_ = (call);                                                        \
        if (e_ != cudaSuccess)                                                          \
            return reattn_capi::set_err((ctx), REATTN_ECUDA,                            \
                                        std::string("CUDA error: ") +                   \
                                            cudaGetErrorString(e_) + " at " #call);     \
    } while (0)

inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// bump allocator over a device region (base == nullptr: sizing pass)
struct Carver {
    uint8_t* base;
    size_t off = 0;
    size_t cap;
    template <typename T>
    T* take(size_t n) {
        off = align_up(off, 256);
        T* p = (T*)(base ? base + off : nullptr);
        off += std::max<size_t>(n, 1) * sizeof(T);
        return p;
    }
};

inline int ensure_arena(reattn_ctx* ctx, size_t bytes) {
    if (bytes <= ctx->arena_bytes) return REATTN_OK;
    CU(ctx, cudaStreamSynchronize(ctx->stream));
    if (ctx->arena) CU(ctx, cudaFree(ctx->arena));
    ctx->arena = nullptr;
    ctx->arena_bytes = 0;
    const size_t nb = align_up(bytes + bytes / 4, 1 << 20);
    CU(ctx, cudaMalloc(&ctx->arena, nb));
    // zero in stream order: a legacy-stream cudaMemset is not ordered with this stream and
    // could land after the caller's first copy into the arena
    CU(ctx, cudaMemsetAsync(ctx->arena, 0, nb, ctx->stream));
    ctx->arena_bytes = nb;
    return REATTN_OK;
}

// enqueue the device mirror of cache->total (stream-ordered with the plans that read it)
// reattn_plan_stage_result on a given stream (the engine stages beside its main stream)
extern "C" int plan_stage_result_on(reattn_plan* p, cudaStream_t s);
// zero-copy host I/O around a captured graph (run_host / step_host on pinned buffers)
bool zero_copy_enabled();
bool host_pinned(const void* p);
int build_io_exec(reattn_ctx* ctx, cudaGraph_t body, const float* const* in_src, float* const* in_dst,
                  const uint64_t* in_n, int n_in, const float* out_src, float* out_dst, uint64_t out_n,
                  cudaGraphExec_t* exec);

inline int cache_sync_total(reattn_ctx* ctx, reattn_cache* c, cudaStream_t s) {
    if (c->dev_total) CU(ctx, launch_set_u32(c->dev_total, (uint32_t)c->total, s));
    return REATTN_OK;
}

inline int status_from_scope(reattn_ctx* ctx, int32_t e) {
    switch (e) {
        case kScopeOk: return REATTN_OK;
        case kScopeErrWindow: return set_err(ctx, REATTN_EINVAL, "scope exceeds pretrain window");
        case kScopeErrSpanRange:
            return set_err(ctx, REATTN_ERANGE, "assemble_scope: span outside middle");
        case kScopeErrQueryLong:
            return set_err(ctx, REATTN_ELOGIC, "attend_step: query block longer than scope");
        case kScopeErrWinnerRange:
            return set_err(ctx, REATTN_ERANGE, "expand_spans: winner outside middle");
        case kScopeErrTooMany:
            return set_err(ctx, REATTN_ERUNTIME, "vote: candidate count exceeds device capacity");
        default: return set_err(ctx, REATTN_ERUNTIME, "device scope error");
    }
}

// ---- scan dispatch -------------------------------------------------------------------
struct ScanPlan {
    ScanArgs a;
    bool fast = false;
    bool tc = false;  // prefill on tcgen05 (opt-in, ε-tie parity)
    CUtensorMap map;
    size_t ws_bytes = 0;
    int grid_sms = 0;  // fast scan CTAs (0: every SM); fewer when SMs are lent to the fork
};

inline int plan_scan(reattn_ctx* ctx, ScanPlan& sp) {
    sp.tc = false;
    if ((ctx->prefill & REATTN_PREFILL_TENSOR_SCAN) && sp.a.n_q > 1 && prefill_tc_supported(sp.a) &&
        make_key_tensor_map(&sp.map, sp.a.keys, sp.a.dtype, sp.a.d,
                            (uint64_t)sp.a.n_kv * sp.a.head_stride, prefill_tc_key_box_rows())) {
        sp.tc = true;
        sp.fast = false;
        sp.ws_bytes = prefill_tc_workspace(sp.a);
        return REATTN_OK;
    }
    sp.fast = scan_fast_supported(sp.a);
    sp.ws_bytes = 0;
    if (sp.fast) {
        sp.ws_bytes = scan_fast_workspace(sp.a, ctx->num_sms);
        if (!make_key_tensor_map(&sp.map, sp.a.keys, sp.a.dtype, sp.a.d,
                                 (uint64_t)sp.a.n_kv * sp.a.head_stride,
                                 scan_fast_box_rows(sp.a.dtype)))
            sp.fast = false;  // layout the TMA unit cannot describe: exact generic path
    }
    if (!sp.fast && sp.a.k > kGenericMaxK)
        return set_err(ctx, REATTN_EINVAL, "fused_topk_scores: k exceeds device capacity (7936)");
    return REATTN_OK;
}

// The fast scan's last-CTA ticket lives at offset 0 of its workspace and is re-armed by
// the kernel itself.  Plans own private, zero-initialised workspaces; the synchronous
// entry points share the context arena, so they clear the ticket first (zero_ticket).
inline int enqueue_scan(reattn_ctx* ctx, const ScanPlan& sp, void* ws, cudaStream_t s,
                        bool zero_ticket) {
    if (sp.tc) {
        CU(ctx, launch_prefill_tc(sp.a, sp.map, ws, s));
        return REATTN_OK;
    }
    if (sp.fast && zero_ticket) CU(ctx, cudaMemsetAsync(ws, 0, 256, s));
    if (sp.fast) {
        ScanArgs a = sp.a;
        a.balance = zero_ticket ? 0 : 1;
        CU(ctx, launch_scan_fast(a, sp.map, ws, sp.grid_sms ? sp.grid_sms : ctx->num_sms, s));
    }
    else
        CU(ctx, launch_scan_generic(sp.a, s));
    return REATTN_OK;
}

}  // namespace reattn_capi
