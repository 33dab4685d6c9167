// Decoder model + generation engine on the device: the reference's Engine (engine.hpp:119-216)
// around the attend_step pipeline, with ModelWeights (model.hpp:66-84), init_random
// (model.hpp:120-152) and the RATW weight file (model.hpp:204-339).
//
// forward_block per layer (engine.hpp:191-205), all on ctx->stream:
//   h = rmsnorm(x, norm_attn)                       rmsnorm_kernel (mean square in double)
//   q = h·wq                                        fp32 GEMM
//   cache.append(h·wk, h·wv)                        fp32 cache: one strided-batched GEMM per
//                                                   tensor writes each head's rows straight
//                                                   into [head][total..total+rows) -- the
//                                                   append IS the GEMM epilogue; bf16 cache:
//                                                   GEMM + the cache-append convert kernel
//   attn = attend_step(q, ...)                      reattn_attend_step (selection, scope,
//                                                   RoPE, attention; stats, spans)
//   x += attn·wo                                    GEMM with beta = 1 (residual fused)
//   h = rmsnorm(x, norm_ffn); x += (silu(h·wg) * (h·wu))·wd
// GEMMs are cuBLAS fp32 (default math mode: no TF32), i.e. library GEMMs; row-major
// C = A·B is issued as the column-major C^T = B^T·A^T.
#include <cublas_v2.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <memory>
#include <random>
#include <string>
#include <vector>

#include "capi_internal.h"

using namespace reattn_impl;
using namespace reattn_capi;

namespace {

constexpr int kNumKinds = 12;

bool is_layer_kind(int kind) { return kind >= REATTN_W_WQ && kind <= REATTN_W_NORM_FFN; }

}  // namespace

struct reattn_weights {
    reattn_model_config cfg{};
    int device = 0;
    // globals: embedding, norm_final, lm_head; per layer: wq..w_down, norm_attn, norm_ffn
    float* global[kNumKinds] = {};
    std::vector<std::vector<float*>> layer;  // [layer][kind]
    ~reattn_weights() {
        for (float* p : global)
            if (p) cudaFree(p);
        for (auto& l : layer)
            for (float* p : l)
                if (p) cudaFree(p);
    }
};

namespace {

void shape_of(const reattn_model_config& c, int kind, uint64_t* rows, uint64_t* cols) {
    uint64_t r = 0, k = 0;
    switch (kind) {
        case REATTN_W_EMBEDDING: r = c.vocab_size, k = c.d_model; break;
        case REATTN_W_WQ: r = c.d_model, k = c.n_head * c.d_head; break;
        case REATTN_W_WK:
        case REATTN_W_WV: r = c.d_model, k = c.n_kv_head * c.d_head; break;
        case REATTN_W_WO: r = c.d_model, k = c.d_model; break;
        case REATTN_W_GATE:
        case REATTN_W_UP: r = c.d_model, k = c.d_ff; break;
        case REATTN_W_DOWN: r = c.d_ff, k = c.d_model; break;
        case REATTN_W_NORM_ATTN:
        case REATTN_W_NORM_FFN:
        case REATTN_W_NORM_FINAL: r = 1, k = c.d_model; break;
        case REATTN_W_LM_HEAD: r = c.d_model, k = c.vocab_size; break;
        default: break;
    }
    *rows = r;
    *cols = k;
}

// ModelConfig::validate (model.hpp:51-61), same messages
int validate_model(reattn_ctx* ctx, const reattn_model_config& c) {
    if (c.n_layer == 0 || c.n_head == 0 || c.n_kv_head == 0 || c.d_model == 0 || c.d_head == 0 ||
        c.d_ff == 0 || c.vocab_size == 0 || c.pretrain_window == 0)
        return set_err(ctx, REATTN_EINVAL, "model config: all dimensions must be positive");
    if (c.n_head % c.n_kv_head != 0)
        return set_err(ctx, REATTN_EINVAL, "model config: n_head must be divisible by n_kv_head");
    if (c.d_model != c.n_head * c.d_head)
        return set_err(ctx, REATTN_EINVAL, "model config: d_model != n_head * d_head");
    if (c.d_head % 2 != 0)
        return set_err(ctx, REATTN_EINVAL, "model config: d_head must be even for rotation");
    return REATTN_OK;
}

// SelectionConfig::validate (selection.hpp:32-44), same messages
int validate_selection(reattn_ctx* ctx, const reattn_selection_config& s, uint64_t window) {
    if (s.k == 0) return set_err(ctx, REATTN_EINVAL, "selection: k must be >= 1");
    if (s.span_m == 0) return set_err(ctx, REATTN_EINVAL, "selection: span_m must be >= 1");
    if (s.tile_size == 0) return set_err(ctx, REATTN_EINVAL, "selection: tile_size must be >= 1");
    if (s.l_chunk == 0) return set_err(ctx, REATTN_EINVAL, "selection: l_chunk must be >= 1");
    if (s.l_chunk > s.l_local)
        return set_err(ctx, REATTN_EINVAL, "selection: l_chunk must not exceed l_local");
    const uint64_t budget = s.l_global + s.k_prime * s.span_m + s.l_local;
    if (budget > window)
        return set_err(ctx, REATTN_EINVAL,
                       "selection: budget l_global + k_prime*span_m + l_local = " +
                           std::to_string(budget) + " exceeds pretrain window " +
                           std::to_string(window));
    return REATTN_OK;
}

float** slot(reattn_weights* w, int kind, uint64_t layer) {
    if (is_layer_kind(kind)) return layer < w->layer.size() ? &w->layer[layer][kind] : nullptr;
    return &w->global[kind];
}
const float* cslot(const reattn_weights* w, int kind, uint64_t layer) {
    return *slot(const_cast<reattn_weights*>(w), kind, layer);
}

// the GEMV weight map of (kind, layer), or nullptr when it cannot be encoded
constexpr int kMapKinds = REATTN_W_DOWN + 1;
const CUtensorMap* wmap(reattn_engine* e, int kind, uint64_t layer);

int alloc_weights(reattn_ctx* ctx, const reattn_model_config& c, std::unique_ptr<reattn_weights>& w) {
    int rc = validate_model(ctx, c);
    if (rc) return rc;
    w.reset(new reattn_weights());
    w->cfg = c;
    w->device = ctx->device;
    w->layer.assign(c.n_layer, std::vector<float*>(kNumKinds, nullptr));
    auto alloc = [&](float** p, int kind) -> int {
        uint64_t r, k;
        shape_of(c, kind, &r, &k);
        CU(ctx, cudaMalloc(p, std::max<uint64_t>(r * k, 1) * sizeof(float)));
        if (kind >= REATTN_W_NORM_ATTN && kind <= REATTN_W_NORM_FINAL) {
            std::vector<float> ones(k, 1.0f);  // model.hpp:120-152: unit norm weights
            CU(ctx, cudaMemcpy(*p, ones.data(), k * sizeof(float), cudaMemcpyHostToDevice));
        } else {
            CU(ctx, cudaMemset(*p, 0, r * k * sizeof(float)));
        }
        return REATTN_OK;
    };
    for (int kind : {REATTN_W_EMBEDDING, REATTN_W_NORM_FINAL, REATTN_W_LM_HEAD})
        if ((rc = alloc(&w->global[kind], kind))) return rc;
    for (uint64_t l = 0; l < c.n_layer; ++l)
        for (int kind = REATTN_W_WQ; kind <= REATTN_W_NORM_FFN; ++kind)
            if ((rc = alloc(&w->layer[l][kind], kind))) return rc;
    return REATTN_OK;
}

// detail::GaussianSource (model.hpp:90-116): Box-Muller over mt19937_64, the spare sine draw
// returned on the next call.  Restated from the published recipe; the sequence is pinned.
struct Gaussian {
    std::mt19937_64 rng;
    double spare = 0.0;
    bool have = false;
    explicit Gaussian(uint64_t seed) : rng(seed) {}
    float next(float stddev) {
        if (have) {
            have = false;
            return (float)(spare * stddev);
        }
        const double top = (double)std::mt19937_64::max();
        const double u1 = ((double)rng() + 1.0) / (top + 2.0);
        const double u2 = (double)rng() / (top + 1.0);
        const double r = std::sqrt(-2.0 * std::log(u1));
        const double theta = 2.0 * 3.141592653589793238462643383279502884 * u2;
        spare = r * std::sin(theta);
        have = true;
        return (float)(r * std::cos(theta) * stddev);
    }
};

// ---- RATW file helpers (model.hpp:222-257) ----
constexpr char kMagic[4] = {'R', 'A', 'T', 'W'};
constexpr uint32_t kVersion = 1;

struct FileCloser {
    void operator()(FILE* f) const {
        if (f) std::fclose(f);
    }
};
using File = std::unique_ptr<FILE, FileCloser>;

template <typename T>
bool rd(FILE* f, T* v) {
    return std::fread(v, sizeof(T), 1, f) == 1;
}

}  // namespace

struct reattn_engine {
    reattn_ctx* ctx = nullptr;
    const reattn_weights* w = nullptr;
    reattn_selection_config sel{};
    int mode = REATTN_MODE_REATTENTION;
    int cache_dtype = REATTN_F32;
    reattn_rope* rope = nullptr;
    std::vector<reattn_cache*> caches;
    std::vector<std::vector<std::pair<uint64_t, uint64_t>>> spans;
    reattn_run_stats stats{};
    std::vector<double> latency_ms;
    std::vector<float> last_logits;
    cublasHandle_t blas = nullptr;
    // activations (rows_cap rows)
    uint64_t rows_cap = 0, last_rows = 0;
    uint32_t* tok = nullptr;
    uint32_t* next = nullptr;
    float *x = nullptr, *h = nullptr, *q = nullptr, *kb = nullptr, *vb = nullptr, *attn = nullptr,
          *gate = nullptr, *up = nullptr, *logits = nullptr;
    std::vector<uint64_t> sb, se;
    // decode: one CUDA-graph plan per layer that follows the growing cache (reattn_plan_*),
    // launched without a host synchronisation; their stats are read once per forward block
    std::vector<reattn_plan*> plans;
    std::vector<reattn_plan*> pending;  // plans whose staged results the next sync completes
    cudaStream_t side = nullptr;        // stats staging beside the main stream
    cudaEvent_t ev_stage = nullptr;
    // TMA tensor maps of the projection weights for the GEMV (built on first use; the weight
    // storage never moves): [layer * kMapKinds + kind], lm_head at the end
    std::vector<CUtensorMap> wmaps;
    std::vector<uint8_t> wmap_ok;
    // decode-token projections: GEMV workspace (split-k partials + self-resetting tickets)
    void* gemv_ws = nullptr;
    uint64_t gemv_n_max = 0;
    bool gemv_ok = false;  // every projection width a multiple of 4 (float4 columns)
    ~reattn_engine() {
        if (side) cudaStreamSynchronize(side);
        if (ev_stage) cudaEventDestroy(ev_stage);
        if (side) cudaStreamDestroy(side);
        if (gemv_ws) cudaFree(gemv_ws);
        for (auto* p : plans) reattn_plan_destroy(p);
        for (auto* c : caches) reattn_cache_destroy(c);
        if (rope) reattn_rope_destroy(rope);
        if (blas) cublasDestroy(blas);
        for (void* p : {(void*)tok, (void*)next, (void*)x, (void*)h, (void*)q, (void*)kb, (void*)vb,
                        (void*)attn, (void*)gate, (void*)up, (void*)logits})
            if (p) cudaFree(p);
    }
};

namespace {

#define BL(ctx, call)                                                                        \
    do {                                                                                     \
        cublasStatus_t s_ = (call);                                                          \
        if (s_ != CUBLAS_STATUS_SUCCESS)                                                     \
            return set_err((ctx), REATTN_ECUDA,                                              \
                           std::string("cuBLAS error ") + std::to_string((int)s_) + " at " #call); \
    } while (0)

// row-major C[M x N] = A[M x K] · B[K x N] + beta·C, leading dimensions in elements
const CUtensorMap* wmap(reattn_engine* e, int kind, uint64_t layer) {
    const reattn_model_config& c = e->w->cfg;
    const size_t n = c.n_layer * kMapKinds + 1;
    if (e->wmaps.size() != n) {
        e->wmaps.assign(n, CUtensorMap{});
        e->wmap_ok.assign(n, 0);
    }
    const size_t i = kind == REATTN_W_LM_HEAD ? n - 1 : layer * kMapKinds + kind;
    if (!e->wmap_ok[i]) {
        uint64_t rows, cols;
        shape_of(c, kind, &rows, &cols);
        e->wmap_ok[i] = gemv_weight_map(&e->wmaps[i], cslot(e->w, kind, layer), cols, cols, rows) ? 1 : 2;
    }
    return e->wmap_ok[i] == 1 ? &e->wmaps[i] : nullptr;
}

int gemm(reattn_engine* e, uint64_t M, uint64_t N, uint64_t K, const float* A, uint64_t lda,
         const float* B, uint64_t ldb, float* C, uint64_t ldc, float beta, const CUtensorMap* map = nullptr) {
    if (M == 0 || N == 0) return REATTN_OK;
    if (M == 1 && e->gemv_ok && N <= e->gemv_n_max && gemv_supported(N, K, ldb, A, B, C)) {
        const GemvDesc m{B, ldb, N, C, beta, 0, 0, 0, 0};
        CU(e->ctx, launch_gemv_batch(A, K, &m, 1, false, e->gemv_ws, e->gemv_n_max, e->ctx->stream, nullptr, 0,
                                     map));
        return REATTN_OK;
    }
    const float one = 1.0f;
    BL(e->ctx, cublasSgemm(e->blas, CUBLAS_OP_N, CUBLAS_OP_N, (int)N, (int)M, (int)K, &one, B,
                           (int)ldb, A, (int)lda, &beta, C, (int)ldc));
    return REATTN_OK;
}

int ensure_rows(reattn_engine* e, uint64_t rows) {
    if (rows <= e->rows_cap) return REATTN_OK;
    reattn_ctx* ctx = e->ctx;
    const reattn_model_config& c = e->w->cfg;
    CU(ctx, cudaStreamSynchronize(ctx->stream));
    for (void* p : {(void*)e->tok, (void*)e->x, (void*)e->h, (void*)e->q, (void*)e->kb, (void*)e->vb,
                    (void*)e->attn, (void*)e->gate, (void*)e->up, (void*)e->logits})
        if (p) CU(ctx, cudaFree(p));
    const uint64_t kvw = c.n_kv_head * c.d_head;
    CU(ctx, cudaMalloc(&e->tok, rows * sizeof(uint32_t)));
    CU(ctx, cudaMalloc(&e->x, rows * c.d_model * sizeof(float)));
    CU(ctx, cudaMalloc(&e->h, rows * c.d_model * sizeof(float)));
    CU(ctx, cudaMalloc(&e->q, rows * c.n_head * c.d_head * sizeof(float)));
    CU(ctx, cudaMalloc(&e->kb, rows * kvw * sizeof(float)));
    CU(ctx, cudaMalloc(&e->vb, rows * kvw * sizeof(float)));
    CU(ctx, cudaMalloc(&e->attn, rows * c.d_model * sizeof(float)));
    CU(ctx, cudaMalloc(&e->gate, rows * c.d_ff * sizeof(float)));
    CU(ctx, cudaMalloc(&e->up, rows * c.d_ff * sizeof(float)));
    CU(ctx, cudaMalloc(&e->logits, rows * c.vocab_size * sizeof(float)));
    e->rows_cap = rows;
    return REATTN_OK;
}

// K/V of `rows` tokens appended to the layer's cache (kv_cache.hpp:54-68): the fp32 cache
// takes the projection straight into its head-major rows, one strided-batched GEMM per tensor
int ensure_capacity(reattn_engine* e, reattn_cache* cache, uint64_t rows) {
    if (cache->total + rows <= cache->capacity) return REATTN_OK;
    return reattn_cache_reserve(e->ctx, cache, std::max(cache->capacity * 2, cache->total + rows));
}

int append_kv(reattn_engine* e, reattn_cache* cache, uint64_t layer, uint64_t rows) {
    reattn_ctx* ctx = e->ctx;
    const reattn_model_config& c = e->w->cfg;
    const uint64_t d = c.d_head, nkv = c.n_kv_head;
    if (int rc = ensure_capacity(e, cache, rows)) return rc;
    const float* wk = cslot(e->w, REATTN_W_WK, layer);
    const float* wv = cslot(e->w, REATTN_W_WV, layer);
    if (cache->dtype == REATTN_F32) {
        const float one = 1.0f, zero = 0.0f;
        for (int t = 0; t < 2; ++t) {
            float* dst = (float*)(t ? cache->values : cache->keys) + cache->total * d;
            // column-major: C_h^T (d x rows) = W_h^T (d x d_model, ld nkv*d) · H^T (d_model x rows)
            BL(ctx, cublasSgemmStridedBatched(e->blas, CUBLAS_OP_N, CUBLAS_OP_N, (int)d, (int)rows,
                                              (int)c.d_model, &one, t ? wv : wk, (int)(nkv * d),
                                              (long long)d, e->h, (int)c.d_model, 0LL, &zero, dst,
                                              (int)d, (long long)(cache->capacity * d), (int)nkv));
        }
        cache->total += rows;
        return cache_sync_total(ctx, cache, ctx->stream);
    }
    int rc = gemm(e, rows, nkv * d, c.d_model, e->h, c.d_model, wk, nkv * d, e->kb, nkv * d, 0.0f);
    if (rc) return rc;
    rc = gemm(e, rows, nkv * d, c.d_model, e->h, c.d_model, wv, nkv * d, e->vb, nkv * d, 0.0f);
    if (rc) return rc;
    return reattn_cache_append(ctx, cache, e->kb, e->vb, rows, 1);
}

// The layer's decode plan, when the layer's cache has a middle to select from (the plan then
// follows the cache as it grows, engine.hpp:163-198); rebuilt after a reserve reallocated the
// cache.  nullptr: this step runs the synchronous attend_step.
reattn_plan* layer_plan(reattn_engine* e, uint64_t l) {
    reattn_plan*& p = e->plans[l];
    const reattn_cache* cache = e->caches[l];
    if (p && reattn_plan_cache_generation(p) != cache->generation) {
        reattn_plan_destroy(p);
        p = nullptr;
    }
    if (p) return p;
    const uint64_t middle = cache->local_start() - cache->global_end();
    if (e->mode != REATTN_MODE_REATTENTION || e->sel.k_prime == 0 || middle < e->sel.k) return nullptr;
    reattn_plan* np = nullptr;
    if (reattn_plan_create(e->ctx, cache, e->rope, 1, e->w->cfg.n_head, &e->sel, e->mode, &np))
        return nullptr;  // (the synchronous step reports any error itself)
    if (!reattn_plan_follows_cache(np)) {
        reattn_plan_destroy(np);
        return nullptr;
    }
    return p = np;
}

void fold_stats(reattn_engine* e, uint64_t l, const reattn_step_stats& st) {
    auto& sp = e->spans[l];
    sp.clear();
    for (uint64_t i = 0; i < st.n_spans; ++i) sp.emplace_back(e->sb[i], e->se[i]);
    reattn_run_stats& S = e->stats;  // engine.hpp:64, :100-112 accumulation
    if (!st.coverage_total) S.coverage_total = 0;
    S.ood_positions += st.ood_positions;
    S.entropy_max = std::max(S.entropy_max, st.entropy_max);
    S.entropy_sum += st.entropy_sum;
    S.entropy_rows += st.entropy_rows;
    S.scope_len_max = std::max(S.scope_len_max, st.scope_len);
    S.max_position_used = std::max(S.max_position_used, st.max_position_used);
    S.peak_scratch_bytes = std::max(S.peak_scratch_bytes, st.peak_scratch_bytes);
}

// engine.hpp:191-205 over e->x (rows x d_model)
int forward_block(reattn_engine* e, uint64_t rows) {
    reattn_ctx* ctx = e->ctx;
    const reattn_model_config& c = e->w->cfg;
    const uint64_t D = c.d_model, QW = c.n_head * c.d_head, F = c.d_ff;
    const uint64_t cap = std::max<uint64_t>(1, e->sel.k_prime);
    e->sb.resize(cap);
    e->se.resize(cap);
    if (e->plans.size() != c.n_layer) e->plans.assign(c.n_layer, nullptr);
    std::vector<reattn_plan*> launched(c.n_layer, nullptr);
    // a decode token (one row, bf16 cache): the q/k/v projections are one GEMV launch and the
    // gate/up projections another, with the activation in its epilogue
    const bool token = rows == 1 && e->gemv_ok;
    const uint64_t KW = c.n_kv_head * c.d_head;
    for (uint64_t l = 0; l < c.n_layer; ++l) {
        CU(ctx, launch_rmsnorm(e->x, rows, D, cslot(e->w, REATTN_W_NORM_ATTN, l), e->h, ctx->stream));
        reattn_cache* cache = e->caches[l];
        int rc;
        reattn_plan* pl = nullptr;
        if (token) {
            // q -> the plan's query buffer; K / V rows written straight into the cache at its
            // length (the append of engine.hpp:196-198, kv_cache.hpp:54-68, fused into the
            // projection's epilogue), and the cache's device length advanced by the launch
            if ((rc = ensure_capacity(e, cache, 1))) return rc;
            pl = layer_plan(e, l);
            const int kind = cache->dtype == REATTN_BF16 ? 1 : 2;
            const GemvDesc m[3] = {
                {cslot(e->w, REATTN_W_WQ, l), QW, QW, pl ? reattn_plan_q(pl) : e->q, 0.0f, 0, 0, 0, 0},
                {cslot(e->w, REATTN_W_WK, l), KW, KW, (float*)cache->keys, 0.0f, kind, c.d_head, cache->total,
                 cache->capacity},
                {cslot(e->w, REATTN_W_WV, l), KW, KW, (float*)cache->values, 0.0f, kind, c.d_head, cache->total,
                 cache->capacity}};
            const CUtensorMap* mq = wmap(e, REATTN_W_WQ, l);
            const CUtensorMap* mk = wmap(e, REATTN_W_WK, l);
            const CUtensorMap* mv = wmap(e, REATTN_W_WV, l);
            CUtensorMap maps[3];
            const bool tma = mq && mk && mv;
            if (tma) {
                maps[0] = *mq;
                maps[1] = *mk;
                maps[2] = *mv;
            }
            CU(ctx, launch_gemv_batch(e->h, D, m, 3, false, e->gemv_ws, e->gemv_n_max, ctx->stream,
                                      cache->dev_total, (uint32_t)(cache->total + 1), tma ? maps : nullptr));
            cache->total += 1;
        } else {
            if ((rc = append_kv(e, cache, l, rows))) return rc;  // before attend_step (engine.hpp:196-198)
            pl = rows == 1 ? layer_plan(e, l) : nullptr;
            float* qd = pl ? reattn_plan_q(pl) : e->q;
            if ((rc = gemm(e, rows, QW, D, e->h, D, cslot(e->w, REATTN_W_WQ, l), QW, qd, QW, 0.0f)))
                return rc;
        }
        const float* attn = e->attn;
        if (pl) {  // the graph replay, no host synchronisation; stats after the block
            if ((rc = reattn_plan_launch(pl))) return rc;
            // the step's stats are copied to the host beside the main stream
            CU(ctx, cudaEventRecord(e->ev_stage, ctx->stream));
            CU(ctx, cudaStreamWaitEvent(e->side, e->ev_stage, 0));
            if ((rc = plan_stage_result_on(pl, e->side))) return rc;
            launched[l] = pl;
            attn = reattn_plan_out(pl);
        } else {
            reattn_step_stats st{};
            rc = reattn_attend_step(ctx, e->caches[l], e->rope, e->q, rows, c.n_head, &e->sel,
                                    e->mode, e->attn, &st, e->sb.data(), e->se.data(), nullptr);
            if (rc) return rc;
            fold_stats(e, l, st);
        }
        // x += attn · wo
        if ((rc = gemm(e, rows, D, D, attn, D, cslot(e->w, REATTN_W_WO, l), D, e->x, D, 1.0f,
                       token ? wmap(e, REATTN_W_WO, l) : nullptr)))
            return rc;
        CU(ctx, launch_rmsnorm(e->x, rows, D, cslot(e->w, REATTN_W_NORM_FFN, l), e->h, ctx->stream));
        if (token) {
            const GemvDesc m[2] = {{cslot(e->w, REATTN_W_GATE, l), F, F, e->gate, 0.0f, 0, 0, 0, 0},
                                   {cslot(e->w, REATTN_W_UP, l), F, F, e->up, 0.0f, 0, 0, 0, 0}};
            const CUtensorMap* mg = wmap(e, REATTN_W_GATE, l);
            const CUtensorMap* mu = wmap(e, REATTN_W_UP, l);
            CUtensorMap maps[2];
            if (mg && mu) {
                maps[0] = *mg;
                maps[1] = *mu;
            }
            CU(ctx, launch_gemv_batch(e->h, D, m, 2, true, e->gemv_ws, e->gemv_n_max, ctx->stream, nullptr, 0,
                                      mg && mu ? maps : nullptr));
        } else {
            if ((rc = gemm(e, rows, F, D, e->h, D, cslot(e->w, REATTN_W_GATE, l), F, e->gate, F, 0.0f)))
                return rc;
            if ((rc = gemm(e, rows, F, D, e->h, D, cslot(e->w, REATTN_W_UP, l), F, e->up, F, 0.0f)))
                return rc;
            CU(ctx, launch_silu_mul(e->gate, e->up, rows * F, ctx->stream));
        }
        if ((rc = gemm(e, rows, D, F, e->gate, F, cslot(e->w, REATTN_W_DOWN, l), D, e->x, D, 1.0f,
                       token ? wmap(e, REATTN_W_DOWN, l) : nullptr)))
            return rc;
    }
    // the plans' results are copied behind the block; folded in layer order after the next
    // synchronisation of the stream (fold_pending)
    e->pending = launched;
    e->last_rows = rows;
    return REATTN_OK;
}

// fold the staged results of the last block's plans (engine.hpp:100-112, layer order); the
// caller has synchronised the context stream
int fold_pending(reattn_engine* e) {
    if (!e->pending.empty()) CU(e->ctx, cudaStreamSynchronize(e->side));
    for (uint64_t l = 0; l < e->pending.size(); ++l) {
        if (!e->pending[l]) continue;
        reattn_step_stats st{};
        int rc = reattn_plan_staged_result(e->pending[l], &st, e->sb.data(), e->se.data(), nullptr);
        if (rc) return rc;
        fold_stats(e, l, st);
    }
    e->pending.clear();
    return REATTN_OK;
}

int check_tokens(reattn_ctx* ctx, const reattn_model_config& c, const uint32_t* t, uint64_t n) {
    for (uint64_t i = 0; i < n; ++i)
        if (t[i] >= c.vocab_size) return set_err(ctx, REATTN_ERANGE, "token id outside vocabulary");
    return REATTN_OK;
}

// rmsnorm(hidden, norm_final) · lm_head for `rows` rows in e->x -> e->logits
int logits_of_x(reattn_engine* e, uint64_t rows) {
    reattn_ctx* ctx = e->ctx;
    const reattn_model_config& c = e->w->cfg;
    CU(ctx, launch_rmsnorm(e->x, rows, c.d_model, cslot(e->w, REATTN_W_NORM_FINAL, 0), e->h,
                           ctx->stream));
    return gemm(e, rows, c.vocab_size, c.d_model, e->h, c.d_model, cslot(e->w, REATTN_W_LM_HEAD, 0),
                c.vocab_size, e->logits, c.vocab_size, 0.0f, rows == 1 ? wmap(e, REATTN_W_LM_HEAD, 0) : nullptr);
}

}  // namespace

extern "C" {

int reattn_model_config_validate(reattn_ctx* ctx, const reattn_model_config* cfg) {
    return validate_model(ctx, *cfg);
}

int reattn_weights_create(reattn_ctx* ctx, const reattn_model_config* cfg, reattn_weights** out) {
    *out = nullptr;
    std::unique_ptr<reattn_weights> w;
    int rc = alloc_weights(ctx, *cfg, w);
    if (rc) return rc;
    CU(ctx, cudaDeviceSynchronize());
    *out = w.release();
    return REATTN_OK;
}

int reattn_weights_init_random(reattn_ctx* ctx, const reattn_model_config* cfg, uint64_t seed,
                               reattn_weights** out) {
    *out = nullptr;
    std::unique_ptr<reattn_weights> w;
    int rc = alloc_weights(ctx, *cfg, w);
    if (rc) return rc;
    Gaussian g(seed);
    const float std_init = 0.02f;
    std::vector<float> buf;
    auto fill = [&](float* dst, int kind) -> int {
        uint64_t r, k;
        shape_of(*cfg, kind, &r, &k);
        buf.resize(r * k);
        for (float& v : buf) v = g.next(std_init);
        CU(ctx, cudaMemcpy(dst, buf.data(), buf.size() * sizeof(float), cudaMemcpyHostToDevice));
        return REATTN_OK;
    };
    // model.hpp:120-152 draw order: embedding, per layer wq wk wv wo w_gate w_up w_down, lm_head
    if ((rc = fill(w->global[REATTN_W_EMBEDDING], REATTN_W_EMBEDDING))) return rc;
    for (uint64_t l = 0; l < cfg->n_layer; ++l)
        for (int kind = REATTN_W_WQ; kind <= REATTN_W_DOWN; ++kind)
            if ((rc = fill(w->layer[l][kind], kind))) return rc;
    if ((rc = fill(w->global[REATTN_W_LM_HEAD], REATTN_W_LM_HEAD))) return rc;
    *out = w.release();
    return REATTN_OK;
}

int reattn_weights_synth(reattn_ctx* ctx, const reattn_model_config* cfg, uint64_t seed,
                         reattn_weights** out) {
    *out = nullptr;
    std::unique_ptr<reattn_weights> w;
    int rc = alloc_weights(ctx, *cfg, w);  // unit norms
    if (rc) return rc;
    auto fill = [&](float* dst, int kind, uint64_t salt) -> int {
        uint64_t r, k;
        shape_of(*cfg, kind, &r, &k);
        CU(ctx, launch_synth_uniform(dst, kF32, r * k, seed * 131 + salt, 0, ctx->stream));
        CU(ctx, launch_scale(dst, r * k, 0.02f, ctx->stream));
        return REATTN_OK;
    };
    if ((rc = fill(w->global[REATTN_W_EMBEDDING], REATTN_W_EMBEDDING, 1))) return rc;
    for (uint64_t l = 0; l < cfg->n_layer; ++l)
        for (int kind = REATTN_W_WQ; kind <= REATTN_W_DOWN; ++kind)
            if ((rc = fill(w->layer[l][kind], kind, 100 + l * 16 + kind))) return rc;
    if ((rc = fill(w->global[REATTN_W_LM_HEAD], REATTN_W_LM_HEAD, 2))) return rc;
    CU(ctx, cudaStreamSynchronize(ctx->stream));
    *out = w.release();
    return REATTN_OK;
}

int reattn_weights_config(const reattn_weights* w, reattn_model_config* cfg) {
    if (!w || !cfg) return REATTN_EINVAL;
    *cfg = w->cfg;
    return REATTN_OK;
}

int reattn_weights_shape(const reattn_weights* w, int kind, uint64_t* rows, uint64_t* cols) {
    if (!w || kind < 0 || kind >= kNumKinds) return REATTN_EINVAL;
    shape_of(w->cfg, kind, rows, cols);
    return REATTN_OK;
}

int reattn_weights_upload(reattn_ctx* ctx, reattn_weights* w, int kind, uint64_t layer,
                          const float* host, uint64_t n) {
    if (!w || kind < 0 || kind >= kNumKinds) return set_err(ctx, REATTN_EINVAL, "weights: bad tensor kind");
    float** p = slot(w, kind, layer);
    if (!p) return set_err(ctx, REATTN_ERANGE, "weights: layer out of range");
    uint64_t r, k;
    shape_of(w->cfg, kind, &r, &k);
    if (n != r * k) return set_err(ctx, REATTN_EINVAL, "weights: tensor size mismatch");
    CU(ctx, cudaMemcpy(*p, host, n * sizeof(float), cudaMemcpyHostToDevice));
    return REATTN_OK;
}

int reattn_weights_download(reattn_ctx* ctx, const reattn_weights* w, int kind, uint64_t layer,
                            float* host, uint64_t n) {
    if (!w || kind < 0 || kind >= kNumKinds) return set_err(ctx, REATTN_EINVAL, "weights: bad tensor kind");
    const float* p = is_layer_kind(kind) ? (layer < w->layer.size() ? w->layer[layer][kind] : nullptr)
                                         : w->global[kind];
    if (!p) return set_err(ctx, REATTN_ERANGE, "weights: layer out of range");
    uint64_t r, k;
    shape_of(w->cfg, kind, &r, &k);
    if (n != r * k) return set_err(ctx, REATTN_EINVAL, "weights: tensor size mismatch");
    CU(ctx, cudaMemcpy(host, p, n * sizeof(float), cudaMemcpyDeviceToHost));
    return REATTN_OK;
}

void reattn_weights_destroy(reattn_weights* w) { delete w; }

// save_weights (model.hpp:259-290)
int reattn_weights_save(reattn_ctx* ctx, const reattn_weights* w, const char* path) {
    const std::string p = path ? path : "";
    File f(std::fopen(p.c_str(), "wb"));
    if (!f) return set_err(ctx, REATTN_ERUNTIME, "cannot open for writing: " + p);
    const reattn_model_config& c = w->cfg;
    bool ok = std::fwrite(kMagic, 1, 4, f.get()) == 4;
    auto put = [&](const void* v, size_t n) { ok = ok && std::fwrite(v, 1, n, f.get()) == n; };
    const uint32_t hdr[8] = {kVersion, (uint32_t)c.n_layer, (uint32_t)c.n_head, (uint32_t)c.n_kv_head,
                             (uint32_t)c.d_model, (uint32_t)c.d_head, (uint32_t)c.d_ff,
                             (uint32_t)c.vocab_size};
    put(hdr, sizeof(hdr));
    const uint64_t pw = c.pretrain_window;
    put(&pw, 8);
    const double base = c.rope_base;
    put(&base, 8);
    const uint32_t mode = (uint32_t)c.attention_mode;
    put(&mode, 4);
    std::vector<float> buf;
    auto tensor = [&](int kind, uint64_t layer) -> int {
        uint64_t r, k;
        shape_of(c, kind, &r, &k);
        buf.resize(r * k);
        int rc = reattn_weights_download(ctx, w, kind, layer, buf.data(), buf.size());
        if (rc) return rc;
        put(&r, 8);
        put(&k, 8);
        put(buf.data(), buf.size() * sizeof(float));
        return REATTN_OK;
    };
    int rc;
    if ((rc = tensor(REATTN_W_EMBEDDING, 0))) return rc;
    for (uint64_t l = 0; l < c.n_layer; ++l)
        for (int kind = REATTN_W_WQ; kind <= REATTN_W_NORM_FFN; ++kind)
            if ((rc = tensor(kind, l))) return rc;
    if ((rc = tensor(REATTN_W_NORM_FINAL, 0))) return rc;
    if ((rc = tensor(REATTN_W_LM_HEAD, 0))) return rc;
    if (!ok || std::fflush(f.get()) != 0) return set_err(ctx, REATTN_ERUNTIME, "write failed: " + p);
    return REATTN_OK;
}

// load_weights (model.hpp:292-339): read order, checks and messages as the reference
int reattn_weights_load(reattn_ctx* ctx, const char* path, reattn_weights** out) {
    *out = nullptr;
    const std::string p = path ? path : "";
    File f(std::fopen(p.c_str(), "rb"));
    if (!f) return set_err(ctx, REATTN_ERUNTIME, "cannot open weights file: " + p);
    char magic[4];
    if (std::fread(magic, 1, 4, f.get()) != 4 || std::memcmp(magic, kMagic, 4) != 0)
        return set_err(ctx, REATTN_ERUNTIME, "weights file: bad magic");
    auto trunc = [&](const std::string& what) {
        return set_err(ctx, REATTN_ERUNTIME, "weights file truncated at " + what);
    };
    uint32_t version;
    if (!rd(f.get(), &version)) return trunc("version");
    if (version != kVersion)
        return set_err(ctx, REATTN_ERUNTIME, "weights file: unsupported version " + std::to_string(version));
    reattn_model_config c{};
    const char* names[7] = {"config.n_layer", "config.n_head",  "config.n_kv_head", "config.d_model",
                            "config.d_head",  "config.d_ff",    "config.vocab_size"};
    uint64_t* fields[7] = {&c.n_layer, &c.n_head, &c.n_kv_head, &c.d_model, &c.d_head, &c.d_ff, &c.vocab_size};
    for (int i = 0; i < 7; ++i) {
        uint32_t v;
        if (!rd(f.get(), &v)) return trunc(names[i]);
        *fields[i] = v;
    }
    if (!rd(f.get(), &c.pretrain_window)) return trunc("config.pretrain_window");
    if (!rd(f.get(), &c.rope_base)) return trunc("config.rope_base");
    uint32_t mode;
    if (!rd(f.get(), &mode)) return trunc("config.attention_mode");
    if (mode > 2) return set_err(ctx, REATTN_ERUNTIME, "weights file: bad attention mode");
    c.attention_mode = (int32_t)mode;
    std::unique_ptr<reattn_weights> w;
    int rc = alloc_weights(ctx, c, w);  // validate() first, as the reference
    if (rc) return rc;
    std::vector<float> buf;
    auto tensor = [&](int kind, uint64_t layer, const std::string& name) -> int {
        uint64_t want_r, want_k, r, k;
        shape_of(c, kind, &want_r, &want_k);
        if (!rd(f.get(), &r)) return trunc(name);
        if (!rd(f.get(), &k)) return trunc(name);
        if (r != want_r || k != want_k)
            return set_err(ctx, REATTN_ERUNTIME,
                           "weights file: tensor " + name + " has shape " + std::to_string(r) + "x" +
                               std::to_string(k) + ", expected " + std::to_string(want_r) + "x" +
                               std::to_string(want_k));
        buf.resize(r * k);
        if (std::fread(buf.data(), sizeof(float), buf.size(), f.get()) != buf.size()) return trunc(name);
        return reattn_weights_upload(ctx, w.get(), kind, layer, buf.data(), buf.size());
    };
    if ((rc = tensor(REATTN_W_EMBEDDING, 0, "embedding"))) return rc;
    const char* lnames[] = {nullptr, "wq", "wk", "wv", "wo", "w_gate", "w_up", "w_down", "norm_attn", "norm_ffn"};
    for (uint64_t l = 0; l < c.n_layer; ++l)
        for (int kind = REATTN_W_WQ; kind <= REATTN_W_NORM_FFN; ++kind)
            if ((rc = tensor(kind, l, "layer" + std::to_string(l) + "." + lnames[kind]))) return rc;
    if ((rc = tensor(REATTN_W_NORM_FINAL, 0, "norm_final"))) return rc;
    if ((rc = tensor(REATTN_W_LM_HEAD, 0, "lm_head"))) return rc;
    if (std::fgetc(f.get()) != EOF)
        return set_err(ctx, REATTN_ERUNTIME, "weights file: trailing bytes after lm_head");
    *out = w.release();
    return REATTN_OK;
}

int reattn_engine_create(reattn_ctx* ctx, const reattn_weights* w, const reattn_selection_config* sel,
                         int mode, int cache_dtype, reattn_engine** out) {
    *out = nullptr;
    if (!w || !sel) return set_err(ctx, REATTN_EINVAL, "engine: null weights or selection config");
    int rc = validate_model(ctx, w->cfg);
    if (rc) return rc;
    if (mode == REATTN_MODE_FULL)
        return set_err(ctx, REATTN_EINVAL,
                       "engine runs window or reattention modes; full attention is the reference path");
    if (mode != REATTN_MODE_WINDOW && mode != REATTN_MODE_REATTENTION)
        return set_err(ctx, REATTN_EINVAL, "unknown attention mode");
    if ((rc = validate_selection(ctx, *sel, w->cfg.pretrain_window))) return rc;
    if (cache_dtype != REATTN_F32 && cache_dtype != REATTN_BF16)
        return set_err(ctx, REATTN_EINVAL, "engine: cache dtype must be f32 or bf16");
    auto e = std::make_unique<reattn_engine>();
    e->ctx = ctx;
    e->w = w;
    e->sel = *sel;
    e->mode = mode;
    e->cache_dtype = cache_dtype;
    if (cublasCreate(&e->blas) != CUBLAS_STATUS_SUCCESS)
        return set_err(ctx, REATTN_ECUDA, "cuBLAS: cannot create handle");
    BL(ctx, cublasSetStream(e->blas, ctx->stream));
    BL(ctx, cublasSetMathMode(e->blas, CUBLAS_DEFAULT_MATH));  // fp32 GEMMs stay fp32 (no TF32)
    if ((rc = reattn_rope_create(ctx, w->cfg.d_head, w->cfg.rope_base, w->cfg.pretrain_window, &e->rope)))
        return rc;
    CU(ctx, cudaMalloc(&e->next, sizeof(uint32_t)));
    CU(ctx, cudaStreamCreateWithFlags(&e->side, cudaStreamNonBlocking));
    CU(ctx, cudaEventCreateWithFlags(&e->ev_stage, cudaEventDisableTiming));
    const reattn_model_config& mc = w->cfg;
    e->gemv_n_max = std::max({mc.vocab_size, mc.d_ff, mc.d_model, mc.n_head * mc.d_head,
                              mc.n_kv_head * mc.d_head});
    CU(ctx, cudaMalloc(&e->gemv_ws, gemv_workspace_bytes(e->gemv_n_max)));
    CU(ctx, cudaMemsetAsync(e->gemv_ws, 0, gemv_workspace_bytes(e->gemv_n_max), ctx->stream));
    e->gemv_ok = mc.d_model % 4 == 0 && mc.d_ff % 4 == 0 && mc.d_head % 4 == 0 && (mc.n_head * mc.d_head) % 4 == 0 &&
                 (mc.n_kv_head * mc.d_head) % 4 == 0 && getenv("REATTN_ENGINE_CUBLAS") == nullptr;
    if ((rc = reattn_engine_reset(e.get()))) return rc;
    *out = e.release();
    return REATTN_OK;
}

// reset (engine.hpp:134-143): fresh caches, spans and stats
int reattn_engine_reset(reattn_engine* e) {
    reattn_ctx* ctx = e->ctx;
    const reattn_model_config& c = e->w->cfg;
    e->pending.clear();
    for (auto* p : e->plans) reattn_plan_destroy(p);
    e->plans.assign(c.n_layer, nullptr);
    for (auto* cache : e->caches) reattn_cache_destroy(cache);
    e->caches.assign(c.n_layer, nullptr);
    const uint64_t cap0 = std::max<uint64_t>(e->sel.l_global + e->sel.l_local, 1024);
    for (uint64_t l = 0; l < c.n_layer; ++l) {
        int rc = reattn_cache_create(ctx, c.n_kv_head, c.d_head, e->sel.l_global, e->sel.l_local,
                                     cap0, e->cache_dtype, &e->caches[l]);
        if (rc) return rc;
    }
    e->spans.assign(c.n_layer, {});
    e->stats = reattn_run_stats{};
    e->stats.coverage_total = 1;
    e->latency_ms.clear();
    e->last_logits.clear();
    e->last_rows = 0;
    return REATTN_OK;
}

int reattn_engine_prefill(reattn_engine* e, const uint32_t* tokens, uint64_t n, uint64_t* rows_out) {
    reattn_ctx* ctx = e->ctx;
    const reattn_model_config& c = e->w->cfg;
    if (n == 0 || !tokens) return set_err(ctx, REATTN_EINVAL, "empty input");
    const uint64_t first = std::min<uint64_t>(n, e->sel.l_global + e->sel.l_local);
    int rc = ensure_rows(e, std::max<uint64_t>(first, std::min<uint64_t>(e->sel.l_chunk, n)));
    if (rc) return rc;
    uint64_t pos = 0;
    while (pos < n) {
        const uint64_t len = pos == 0 ? first : std::min<uint64_t>(e->sel.l_chunk, n - pos);
        if ((rc = check_tokens(ctx, c, tokens + pos, len))) return rc;  // embed (model.hpp:181-190)
        CU(ctx, cudaMemcpyAsync(e->tok, tokens + pos, len * sizeof(uint32_t), cudaMemcpyHostToDevice,
                                ctx->stream));
        CU(ctx, launch_embed(e->tok, len, cslot(e->w, REATTN_W_EMBEDDING, 0), c.d_model, e->x, ctx->stream));
        if ((rc = forward_block(e, len))) return rc;
        pos += len;
        ++e->stats.chunks_processed;
    }
    CU(ctx, cudaStreamSynchronize(ctx->stream));
    if ((rc = fold_pending(e))) return rc;
    if (rows_out) *rows_out = e->last_rows;
    return REATTN_OK;
}

int reattn_engine_hidden(reattn_engine* e, float* host, uint64_t n) {
    reattn_ctx* ctx = e->ctx;
    if (n != e->last_rows * e->w->cfg.d_model)
        return set_err(ctx, REATTN_EINVAL, "engine: hidden buffer size mismatch");
    CU(ctx, cudaMemcpyAsync(host, e->x, n * sizeof(float), cudaMemcpyDeviceToHost, ctx->stream));
    CU(ctx, cudaStreamSynchronize(ctx->stream));
    return REATTN_OK;
}

int reattn_engine_logits(reattn_engine* e, const float* hidden, uint64_t rows, float* logits) {
    reattn_ctx* ctx = e->ctx;
    const reattn_model_config& c = e->w->cfg;
    if (rows == 0) return REATTN_OK;
    int rc = ensure_rows(e, rows);
    if (rc) return rc;
    // logits() is a pure function of `hidden`: stage it in h's sibling buffer (attn)
    CU(ctx, cudaMemcpyAsync(e->attn, hidden, rows * c.d_model * sizeof(float), cudaMemcpyHostToDevice,
                            ctx->stream));
    CU(ctx, launch_rmsnorm(e->attn, rows, c.d_model, cslot(e->w, REATTN_W_NORM_FINAL, 0), e->h, ctx->stream));
    if ((rc = gemm(e, rows, c.vocab_size, c.d_model, e->h, c.d_model, cslot(e->w, REATTN_W_LM_HEAD, 0),
                   c.vocab_size, e->logits, c.vocab_size, 0.0f)))
        return rc;
    CU(ctx, cudaMemcpyAsync(logits, e->logits, rows * c.vocab_size * sizeof(float),
                            cudaMemcpyDeviceToHost, ctx->stream));
    CU(ctx, cudaStreamSynchronize(ctx->stream));
    return REATTN_OK;
}

int reattn_engine_decode_step(reattn_engine* e, uint32_t last_token, uint32_t* next_token) {
    reattn_ctx* ctx = e->ctx;
    const reattn_model_config& c = e->w->cfg;
    const auto t0 = std::chrono::steady_clock::now();
    int rc = check_tokens(ctx, c, &last_token, 1);
    if (rc) return rc;
    if ((rc = ensure_rows(e, 1))) return rc;
    CU(ctx, cudaMemcpyAsync(e->tok, &last_token, sizeof(uint32_t), cudaMemcpyHostToDevice, ctx->stream));
    CU(ctx, launch_embed(e->tok, 1, cslot(e->w, REATTN_W_EMBEDDING, 0), c.d_model, e->x, ctx->stream));
    if ((rc = forward_block(e, 1))) return rc;
    if ((rc = logits_of_x(e, 1))) return rc;
    CU(ctx, launch_argmax(e->logits, c.vocab_size, e->next, ctx->stream));
    e->last_logits.resize(c.vocab_size);
    uint32_t nt = 0;
    CU(ctx, cudaMemcpyAsync(e->last_logits.data(), e->logits, c.vocab_size * sizeof(float),
                            cudaMemcpyDeviceToHost, ctx->stream));
    CU(ctx, cudaMemcpyAsync(&nt, e->next, sizeof(uint32_t), cudaMemcpyDeviceToHost, ctx->stream));
    CU(ctx, cudaStreamSynchronize(ctx->stream));
    if ((rc = fold_pending(e))) return rc;
    const auto t1 = std::chrono::steady_clock::now();
    e->latency_ms.push_back(std::chrono::duration<double, std::milli>(t1 - t0).count());
    ++e->stats.decode_steps;
    if (next_token) *next_token = nt;
    return REATTN_OK;
}

int reattn_engine_last_logits(reattn_engine* e, float* host, uint64_t n) {
    if (n != e->last_logits.size()) return set_err(e->ctx, REATTN_EINVAL, "engine: logits size mismatch");
    std::copy(e->last_logits.begin(), e->last_logits.end(), host);
    return REATTN_OK;
}

int reattn_engine_stats(const reattn_engine* e, reattn_run_stats* st) {
    if (!e || !st) return REATTN_EINVAL;
    *st = e->stats;
    return REATTN_OK;
}

int reattn_engine_decode_latencies(const reattn_engine* e, double* out, uint64_t cap, uint64_t* n) {
    if (!e) return REATTN_EINVAL;
    if (n) *n = e->latency_ms.size();
    for (uint64_t i = 0; i < std::min<uint64_t>(cap, e->latency_ms.size()); ++i) out[i] = e->latency_ms[i];
    return REATTN_OK;
}

int reattn_engine_last_spans(const reattn_engine* e, uint64_t layer, uint64_t* begin, uint64_t* end,
                             uint64_t cap, uint64_t* n) {
    if (!e || layer >= e->spans.size()) return REATTN_ERANGE;
    const auto& sp = e->spans[layer];
    if (n) *n = sp.size();
    for (uint64_t i = 0; i < std::min<uint64_t>(cap, sp.size()); ++i) {
        begin[i] = sp[i].first;
        end[i] = sp[i].second;
    }
    return REATTN_OK;
}

int reattn_engine_synth_context(reattn_engine* e, uint64_t total, uint64_t seed) {
    reattn_ctx* ctx = e->ctx;
    const reattn_model_config& c = e->w->cfg;
    for (uint64_t l = 0; l < c.n_layer; ++l) {
        reattn_cache* cache = e->caches[l];
        int rc = reattn_cache_reserve(ctx, cache, total + 4096);
        if (rc) return rc;
        const int dt = cache->dtype == REATTN_BF16 ? kBF16 : kF32;
        const uint64_t n = cache->n_kv * cache->capacity * cache->d;
        CU(ctx, launch_synth_uniform(cache->keys, dt, n, seed * 977 + 2 * l, 0, ctx->stream));
        CU(ctx, launch_synth_uniform(cache->values, dt, n, seed * 977 + 2 * l + 1, 0, ctx->stream));
        if ((rc = reattn_cache_set_total(ctx, cache, total))) return rc;
    }
    CU(ctx, cudaStreamSynchronize(ctx->stream));
    return REATTN_OK;
}

size_t reattn_debug_gemv_workspace(uint64_t n) { return gemv_workspace_bytes(n); }

int reattn_debug_gemv(reattn_ctx* ctx, const float* x, const float* w, uint64_t ldw, uint64_t n,
                      uint64_t k, float* y, float beta, void* ws) {
    if (!gemv_supported(n, k, ldw, x, w, y)) return set_err(ctx, REATTN_EINVAL, "gemv: unsupported shape");
    CUtensorMap map;
    const bool tma = gemv_weight_map(&map, w, ldw, n, k);
    const GemvDesc m{w, ldw, n, y, beta, 0, 0, 0, 0};
    CU(ctx, launch_gemv_batch(x, k, &m, 1, false, ws, n, ctx->stream, nullptr, 0, tma ? &map : nullptr));
    return REATTN_OK;
}

const reattn_cache* reattn_engine_cache(const reattn_engine* e, uint64_t layer) {
    return e && layer < e->caches.size() ? e->caches[layer] : nullptr;
}

void reattn_engine_destroy(reattn_engine* e) { delete e; }

}  // extern "C"
