// C-ABI implementation (include/reattn_cuda.h): contexts, device KV cache, rotary tables,
// the synchronous reference-shaped entry points and CUDA-graph step plans.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "capi_internal.h"

using namespace reattn_impl;
using namespace reattn_capi;

namespace {

// ---- attend_step pipeline --------------------------------------------------------------
struct StepPlan {
    // shape
    uint64_t n_q, n_head, n_kv, d, group, g_end, l_start, total, middle, window;
    uint64_t kk;  // min(k, middle) when selecting
    bool select = false;
    uint32_t L_upper = 0;
    reattn_selection_config cfg;
    ScanPlan scan;
    // device buffers
    uint32_t* cand_idx = nullptr;
    float* cand_score = nullptr;
    void* scan_ws = nullptr;
    uint32_t* winners = nullptr;
    uint32_t* span_b = nullptr;
    uint32_t* span_e = nullptr;
    uint32_t* scope_src = nullptr;
    ScopeHeader* hdr = nullptr;
    double* part = nullptr;
    double* entropy = nullptr;
    bool large_vote = false;  // > kVoteMaxSmem candidates: device radix-sort vote
    size_t vote_ws_bytes = 0;
    void* vote_ws = nullptr;
    size_t part_bytes = 0;
    bool fork = false;        // decode: local-window attention beside the scan
    DecodeFork fk{};
    bool attn_tc = false;     // prefill attention on tcgen05 (ctx prefill mode TENSOR)
    size_t attn_tc_bytes = 0;
    void* attn_tc_ws = nullptr;
    size_t scratch_bytes = 0;
    uint64_t kernels = 0;
    // decode plans read the cache length from the device (reattn_cache::dev_total): one graph
    // serves every decode step while the cache grows (engine.hpp:163-198 appends every step)
    bool dynamic = false;
};

void plan_fork(reattn_ctx* ctx, StepPlan& P);

int plan_step(reattn_ctx* ctx, const reattn_cache* cache, const reattn_rope* rope, uint64_t n_q,
              uint64_t n_head, const reattn_selection_config* cfg, int mode, StepPlan& P,
              const float* q_dev, float* out_dev, bool allow_dynamic = false) {
    if (n_head % cache->n_kv != 0)
        return set_err(ctx, REATTN_EINVAL, "attend_step: n_head must be a multiple of kv heads");
    if (rope->head_dim != cache->d)
        return set_err(ctx, REATTN_EINVAL, "attend_step: rotary head_dim != cache d_head");
    if (cfg->k == 0) return set_err(ctx, REATTN_EINVAL, "selection: k must be >= 1");
    if (cfg->span_m == 0) return set_err(ctx, REATTN_EINVAL, "selection: span_m must be >= 1");
    P.cfg = *cfg;
    P.n_q = n_q;
    P.n_head = n_head;
    P.n_kv = cache->n_kv;
    P.d = cache->d;
    P.group = n_head / cache->n_kv;
    P.total = cache->total;
    P.g_end = cache->global_end();
    P.l_start = cache->local_start();
    P.middle = P.l_start - P.g_end;
    P.window = rope->max_position;
    P.select = mode == REATTN_MODE_REATTENTION && cfg->k_prime > 0 && P.middle > 0;
    P.kk = std::min<uint64_t>(cfg->k, P.middle);
    const uint64_t local = P.total - P.l_start;
    // at most min(k', #candidates) winners, each expanding to <= span_m rows
    const uint64_t max_winners = std::min<uint64_t>(cfg->k_prime, P.n_kv * n_q * P.kk);
    uint64_t sel_rows = P.select ? std::min<uint64_t>(P.middle, max_winners * cfg->span_m) : 0;
    P.L_upper = (uint32_t)std::min<uint64_t>(P.window, P.g_end + sel_rows + local);
    if (P.total >= (1ull << 32) || P.window >= (1ull << 31))
        return set_err(ctx, REATTN_EINVAL, "attend_step: cache too long for 32-bit indices");
    if (P.select) {
        const uint64_t n_cand = P.n_kv * n_q * P.kk;
        if (n_cand >= (1ull << 31))
            return set_err(ctx, REATTN_ERUNTIME, "vote: candidate count exceeds 2^31");
        P.large_vote = n_cand > kVoteMaxSmem;
        P.vote_ws_bytes = P.large_vote ? vote_large_workspace((uint32_t)n_cand, (uint32_t)P.middle,
                                                              (uint32_t)cfg->k_prime) : 0;
        ScanArgs& a = P.scan.a;
        a.q = q_dev;
        a.n_q = (int)n_q;
        a.n_heads = (int)n_head;
        a.n_kv = (int)P.n_kv;
        a.d = (int)P.d;
        a.keys = cache->keys;
        a.dtype = cache->dtype;
        a.head_stride = cache->capacity;
        a.row0 = P.g_end;
        a.count = (uint32_t)P.middle;
        a.k = (int)cfg->k;
        a.lanes = ctx->lanes;
        int rc = plan_scan(ctx, P.scan);
        if (rc) return rc;
    }
    P.attn_tc = (ctx->prefill & REATTN_PREFILL_TENSOR_ATTN) && n_q > 1 && cache->d == 128 &&
                cache->dtype == kBF16;
    plan_fork(ctx, P);
    // a decode plan whose selection runs in K1's merger CTA can follow a growing cache: the
    // scan, the select and the decode attention derive the segments from the device length
    if (allow_dynamic && P.select && n_q == 1 && P.scan.fast && P.kk == cfg->k &&
        P.n_kv * cfg->k <= kSmallSelectMax && cache->dev_total) {
        P.dynamic = true;
        P.scan.a.dev_total = cache->dev_total;
        P.scan.a.l_global = (uint32_t)cfg->l_global;
        P.scan.a.l_local = (uint32_t)cfg->l_local;
        P.fk.dev_total = cache->dev_total;
        P.fk.l_global = (uint32_t)cfg->l_global;
        P.fk.l_local = (uint32_t)cfg->l_local;
        // buffers sized for the largest scope any later step can have
        const uint64_t wmax = std::min<uint64_t>(cfg->k_prime, P.n_kv * cfg->k);
        P.L_upper = (uint32_t)std::min<uint64_t>(P.window, cfg->l_global + wmax * cfg->span_m + cfg->l_local);
    }
    (void)out_dev;
    return REATTN_OK;
}

// host copy of the step geometry at the cache's current length (dynamic plans)
void refresh_geometry(StepPlan& P, const reattn_cache* cache) {
    if (!P.dynamic) return;
    P.total = cache->total;
    P.g_end = cache->global_end();
    P.l_start = cache->local_start();
    P.middle = P.l_start - P.g_end;
}

// Decode local-window fork (DecodeFork in kernels.h): lend R = m * n_kv SMs to the local
// window's attention while the scan runs on the rest, when the local work fits well inside
// the scan (estimates: scan ~5.8 TB/s over the middle's keys; local ~0.8 us per 32-row chunk
// per SM, measured).  At 1M context on B200 it costs the scan ~3 us and saves ~7 us of
// post-select attention.  REATTN_FORK=0 disables it, REATTN_FORK=1 forces m = 1.
void plan_fork(reattn_ctx* ctx, StepPlan& P) {
    P.fork = false;
    P.scan.grid_sms = 0;
    const uint64_t n_local = P.total - P.l_start;
    if (!(P.n_q == 1 && P.d == 128 && P.select && P.scan.fast && P.scan.a.dtype == kBF16 &&
          P.group <= 8 && n_local > 0))
        return;
    const char* env_s = std::getenv("REATTN_FORK");
    const int env = env_s ? std::atoi(env_s) : -1;
    if (env == 0) return;
    if (env == 2) {
        // post-scan local launch on every SM (see DecodeFork::post)
        P.fork = true;
        P.fk.n_local = (uint32_t)n_local;
        P.fk.local_row0 = (uint32_t)P.l_start;
        P.fk.local_parts = std::max(1, std::min(kMaxLocalParts, ctx->num_sms / (int)P.n_kv));
        P.fk.heads_per_cta = 1;
        P.fk.post = 1;
        return;
    }
    // m CTAs per kv head, each CTA taking hpc kv heads in turn: the fewest lent SMs
    // (m * n_kv / hpc) whose local work (~0.8 us per 32-row chunk per CTA, measured) fits in
    // 70% of the scan (estimated at 5.8 TB/s over the middle's keys)
    int m = env == 1 ? 1 : 0, hpc = 1;
    if (env == 1) {  // forced fork (tests): REATTN_FORK_HPC kv heads per local CTA
        const char* h = std::getenv("REATTN_FORK_HPC");
        const int hh = h ? std::atoi(h) : 1;
        if (hh >= 1 && P.n_kv % (uint64_t)hh == 0) hpc = hh;
    }
    if (!m) {
        const double t_scan = (double)P.middle * P.n_kv * P.d * 2 / 5.8e6;  // us
        const double chunks_per_head = (double)((n_local + 31) / 32);
        int best_sms = 1 << 30;
        for (int mm = 1; mm <= 2; ++mm)
            for (int hh = 1; hh <= (int)P.n_kv; hh *= 2) {
                if (P.n_kv % hh) continue;
                const int sms = mm * (int)P.n_kv / hh;
                if (sms * 8 > ctx->num_sms) continue;
                if (chunks_per_head * hh / mm * 0.8 <= 0.7 * t_scan && sms < best_sms) {
                    best_sms = sms;
                    m = mm;
                    hpc = hh;
                }
            }
    }
    if (!m) return;
    P.fork = true;
    P.fk.n_local = (uint32_t)n_local;
    P.fk.local_row0 = (uint32_t)P.l_start;
    P.fk.local_parts = m;
    P.fk.heads_per_cta = hpc;
    P.fk.post = 0;
    P.scan.grid_sms = ctx->num_sms - m * (int)P.n_kv / hpc;
}

AttnArgs step_attn_args(const StepPlan& P, const reattn_cache* cache, const reattn_rope* rope,
                        const float* q_dev, float* out_dev) {
    AttnArgs a;
    a.q = q_dev;
    a.q_row_stride = P.n_head * P.d;
    a.n_q = (int)P.n_q;
    a.n_head = (int)P.n_head;
    a.n_kv = (int)P.n_kv;
    a.group = (int)P.group;
    a.d = (int)P.d;
    a.dv = (int)P.d;
    a.k_base = cache->keys;
    a.v_base = cache->values;
    a.dtype = cache->dtype;
    a.head_stride = cache->capacity;
    a.src = P.scope_src;
    a.hdr = P.hdr;
    a.L_host = 0;
    a.rope_cos = rope->cos_d;
    a.rope_sin = rope->sin_d;
    a.causal = 1;
    a.boundary_is_tail = 1;
    a.boundary_host = 0;
    a.part = P.part;
    a.out = out_dev;
    a.entropy = P.entropy;
    return a;
}

// carve (or size, when base == nullptr) the step buffers
void carve_step(StepPlan& P, const reattn_cache* cache, const reattn_rope* rope, Carver& c) {
    const uint64_t ncand = P.select ? P.n_kv * P.n_q * P.cfg.k : 1;
    P.cand_idx = c.take<uint32_t>(ncand);
    P.cand_score = c.take<float>(ncand);
    P.scan_ws = c.take<uint8_t>(P.scan.ws_bytes);
    const uint64_t kp = std::max<uint64_t>(1, P.cfg.k_prime);
    P.winners = c.take<uint32_t>(kp);
    P.span_b = c.take<uint32_t>(kp);
    P.span_e = c.take<uint32_t>(kp);
    P.scope_src = c.take<uint32_t>(std::max<uint64_t>(1, P.L_upper));
    P.hdr = c.take<ScopeHeader>(1);
    AttnArgs a = step_attn_args(P, cache, rope, nullptr, nullptr);
    P.part_bytes = attend_workspace(a, std::max<uint32_t>(1, P.L_upper));
    P.part = c.take<double>(P.part_bytes / sizeof(double) + 1);
    P.attn_tc = P.attn_tc && attend_tc_supported(a);
    P.attn_tc_bytes = P.attn_tc ? attend_tc_workspace(a, std::max<uint32_t>(1, P.L_upper)) : 0;
    P.attn_tc_ws = c.take<uint8_t>(P.attn_tc_bytes);
    P.entropy = c.take<double>(std::max<uint64_t>(1, P.n_q * P.n_head));
    P.vote_ws = c.take<uint8_t>(P.vote_ws_bytes);
    // the scan's scratch, what the reference's ScratchMeter meters (inside fused_topk_scores
    // only, selection.hpp:168-248, via engine.hpp:60-66): the candidate lists and the scan's
    // workspace -- not the vote, the scope table or the attention's partial rows
    P.scratch_bytes = ncand * (sizeof(uint32_t) + sizeof(float)) + P.scan.ws_bytes;
}

// The selection half of a step: the local-window fork (when planned), K1 (+ fused K3) or the
// standalone select / large vote.  Leaves the scope header and table on the device.
int enqueue_select_part(reattn_ctx* ctx, StepPlan& P, const reattn_cache* cache,
                        const reattn_rope* rope, const float* q_dev, float* out_dev, cudaStream_t s,
                        bool zero_ticket) {
    P.kernels = 0;
    SelectArgs sa;
    std::memset(&sa, 0, sizeof(sa));
    if (P.select) {
        sa.cand_idx = P.cand_idx;
        sa.cand_score = P.cand_score;
        sa.n_lists = (uint32_t)(P.n_kv * P.n_q);
        sa.list_len = (uint32_t)P.kk;
        sa.list_stride = (uint32_t)P.cfg.k;
        sa.k_prime = (uint32_t)P.cfg.k_prime;
    }
    sa.span_m = (uint32_t)P.cfg.span_m;
    sa.middle_len = (uint32_t)P.middle;
    sa.span_mode = P.cfg.span_mode;
    sa.build_scope = 1;
    sa.g_end = (uint32_t)P.g_end;
    sa.l_start = (uint32_t)P.l_start;
    sa.total = (uint32_t)P.total;
    sa.window = (uint32_t)P.window;
    sa.n_q = (uint32_t)P.n_q;
    sa.winners = P.winners;
    sa.span_b = P.span_b;
    sa.span_e = P.span_e;
    sa.scope_src = P.scope_src;
    sa.hdr = P.hdr;
    // Decode: <= 32 candidates -> vote/spans/scope run in the fast scan's merger CTA (one
    // launch fewer, no host round trip); otherwise the standalone select kernel.
    if (P.fork && !P.fk.post) {  // local window beside the scan (independent of the selection)
        AttnArgs la = step_attn_args(P, cache, rope, q_dev, out_dev);
        CU(ctx, cudaEventRecord(ctx->ev_fork, s));
        CU(ctx, cudaStreamWaitEvent(ctx->side, ctx->ev_fork, 0));
        CU(ctx, launch_attend_decode_local(la, P.part, ctx->num_sms, P.fk, ctx->side));
        CU(ctx, cudaEventRecord(ctx->ev_join, ctx->side));
        ++P.kernels;
    }
    bool fused = false;
    if (P.select) {
        P.scan.a.q = q_dev;
        P.scan.a.idx_out = P.cand_idx;
        P.scan.a.score_out = P.cand_score;
        fused = P.scan.fast && P.n_kv * P.n_q * P.kk <= kSmallSelectMax;
        P.scan.a.fuse_select = fused ? 1 : 0;
        if (fused) {
            SmallSelectIO& io = P.scan.a.sel;
            io.k_prime = sa.k_prime;
            io.span_m = sa.span_m;
            io.middle_len = sa.middle_len;
            io.span_mode = sa.span_mode;
            io.g_end = sa.g_end;
            io.l_start = sa.l_start;
            io.total = sa.total;
            io.window = sa.window;
            io.n_q = sa.n_q;
            io.winners = sa.winners;
            io.span_b = sa.span_b;
            io.span_e = sa.span_e;
            io.scope_src = sa.scope_src;
            io.hdr = sa.hdr;
            io.table_local = P.fork ? 0 : 1;
        }
        int rc = enqueue_scan(ctx, P.scan, P.scan_ws, s, zero_ticket);
        if (rc) return rc;
        ++P.kernels;
    }
    if (P.fork && P.fk.post) {  // local window after the scan, on the SMs its CTAs release
        AttnArgs la = step_attn_args(P, cache, rope, q_dev, out_dev);
        CU(ctx, launch_attend_decode_local(la, P.part, ctx->num_sms, P.fk, s));
        ++P.kernels;
    }
    if (!fused && P.large_vote) {
        // the bounded vote's tallies stay clean across replays; a fresh (arena) workspace
        // is zeroed first -- plans zero theirs at creation
        if (zero_ticket) CU(ctx, cudaMemsetAsync(P.vote_ws, 0, P.vote_ws_bytes, s));
        CU(ctx, launch_vote_large(sa, P.vote_ws, s));
        P.kernels += vote_large_kernels(sa.n_lists * sa.list_len, sa.middle_len, sa.k_prime);
    } else if (!fused) {
        CU(ctx, launch_select(sa, s));
        ++P.kernels;
    }
    return REATTN_OK;
}

// The attention half on stream `s`.  attn_sms < num_sms (batch pipelines): the decode
// attention runs on that many SMs beside another sequence's scan, without PDL.
int enqueue_attn_part(reattn_ctx* ctx, StepPlan& P, const reattn_cache* cache,
                      const reattn_rope* rope, const float* q_dev, float* out_dev, cudaStream_t s,
                      bool zero_ticket, int attn_sms) {
    if (P.n_q > 0) {
        AttnArgs a = step_attn_args(P, cache, rope, q_dev, out_dev);
        if (attn_sms > 0 && attn_sms < ctx->num_sms && decode_bulk_eligible(a) && !P.fork) {
            if (zero_ticket) CU(ctx, cudaMemsetAsync(P.part, 0, decode_ticket_bytes(a.n_kv), s));
            CU(ctx, launch_attend_decode_bulk_ex(a, P.part, attn_sms, s, false));
            ++P.kernels;
            return REATTN_OK;
        }
        // the bulk decode attention's tickets sit at the start of P.part (plans: zeroed once)
        if (zero_ticket && decode_bulk_eligible(a))
            CU(ctx, cudaMemsetAsync(P.part, 0, decode_ticket_bytes(a.n_kv), s));
        if (P.fork) {
            if (!P.fk.post) CU(ctx, cudaStreamWaitEvent(s, ctx->ev_join, 0));
            CU(ctx, launch_attend_decode_head(a, P.part, ctx->num_sms, P.fk, s, P.fk.post != 0));
            ++P.kernels;
        } else if (P.attn_tc) {
            CU(ctx, launch_attend_tc(a, std::max<uint32_t>(1, P.L_upper), P.attn_tc_ws, s));
            P.kernels += 2;
        } else {
            CU(ctx, launch_attend(a, std::max<uint32_t>(1, P.L_upper), s));
            P.kernels += attend_kernel_count(a, std::max<uint32_t>(1, P.L_upper));
        }
    }
    return REATTN_OK;
}

int enqueue_step(reattn_ctx* ctx, StepPlan& P, const reattn_cache* cache, const reattn_rope* rope,
                 const float* q_dev, float* out_dev, cudaStream_t s, bool zero_ticket) {
    int rc = enqueue_select_part(ctx, P, cache, rope, q_dev, out_dev, s, zero_ticket);
    if (rc) return rc;
    return enqueue_attn_part(ctx, P, cache, rope, q_dev, out_dev, s, zero_ticket, 0);
}

int stats_from_host(reattn_ctx* ctx, const StepPlan& P, const ScopeHeader& h, const double* ent,
                    reattn_step_stats* st, double* entropy_host);

int finish_step_stats(reattn_ctx* ctx, const StepPlan& P, const ScopeHeader& h,
                      reattn_step_stats* st, double* entropy_host) {
    int rc = status_from_scope(ctx, h.error);
    if (rc) return rc;
    if (P.n_q == 0 && h.L == 0) return set_err(ctx, REATTN_EINVAL, "empty key set");
    std::vector<double> ent(P.n_q * P.n_head);
    if (!ent.empty())
        CU(ctx, cudaMemcpy(ent.data(), P.entropy, ent.size() * sizeof(double),
                           cudaMemcpyDeviceToHost));
    return stats_from_host(ctx, P, h, ent.data(), st, entropy_host);
}

// the step's stats from its header and entropies already on the host
int stats_from_host(reattn_ctx* ctx, const StepPlan& P, const ScopeHeader& h, const double* ent_p,
                    reattn_step_stats* st, double* entropy_host) {
    int rc = status_from_scope(ctx, h.error);
    if (rc) return rc;
    if (P.n_q == 0 && h.L == 0) return set_err(ctx, REATTN_EINVAL, "empty key set");
    const uint64_t n_ent = P.n_q * P.n_head;
    if (entropy_host) std::copy(ent_p, ent_p + n_ent, entropy_host);
    if (st) {
        std::memset(st, 0, sizeof(*st));
        double mx = 0.0, sum = 0.0;
        for (uint64_t hh = 0; hh < P.n_head; ++hh)
            for (uint64_t i = 0; i < P.n_q; ++i) {
                const double e = ent_p[i * P.n_head + hh];
                mx = std::max(mx, e);
                sum += e;
            }
        st->entropy_max = mx;
        st->entropy_sum = sum;
        st->entropy_rows = P.n_q * P.n_head;
        st->scope_len = h.L;
        st->max_position_used = h.L ? h.L - 1 : 0;
        st->ood_positions = 0;  // every position < L' <= window (checked on device)
        st->n_spans = h.n_spans;
        st->coverage = h.coverage;
        st->coverage_total = h.coverage == P.middle ? 1 : 0;
        st->peak_scratch_bytes = P.scratch_bytes;
    }
    return REATTN_OK;
}

}  // namespace

struct reattn_plan {
    reattn_ctx* ctx;
    reattn_cache* cache;
    const reattn_rope* rope;
    StepPlan P;
    void* mem = nullptr;
    float* q = nullptr;
    float* out = nullptr;
    float* k_in = nullptr;  // append mode: this step's K / V rows [n_kv * d] fp32
    float* v_in = nullptr;
    bool append = false;
    uint64_t generation = 0;  // the cache storage the graph was captured over
    uint64_t total0 = 0;      // the cache length a frozen (non-dynamic) plan was built for
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    // staged results (reattn_plan_stage_result): pinned host copies of the step's header,
    // entropies and spans, filled by copies enqueued behind the replay
    void* staged = nullptr;
    bool staged_pending = false;
    // zero-copy host I/O (step_host / run_host on pinned buffers): the plan's graph with the
    // host reads before it and the output write after it, for the last host pointers seen
    cudaGraphExec_t io_exec = nullptr;
    const void* io_key[4] = {nullptr, nullptr, nullptr, nullptr};
    bool io_append = false;
};

namespace {
// The plan's graph: [append the step's K/V rows] + the attend_step pipeline.
int capture_plan(reattn_plan* p) {
    reattn_ctx* ctx = p->ctx;
    if (p->io_exec) cudaGraphExecDestroy(p->io_exec);  // holds a copy of the old graph
    p->io_exec = nullptr;
    if (p->exec) cudaGraphExecDestroy(p->exec);
    if (p->graph) cudaGraphDestroy(p->graph);
    p->exec = nullptr;
    p->graph = nullptr;
    cudaStream_t cs;
    CU(ctx, cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    CU(ctx, cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
    int rc = REATTN_OK;
    if (p->append) {
        const cudaError_t e = launch_cache_append_step(p->k_in, p->v_in, p->cache->keys,
                                                       p->cache->values, p->cache->dtype,
                                                       p->cache->n_kv, p->cache->d,
                                                       p->cache->capacity, p->cache->dev_total, cs);
        if (e != cudaSuccess) rc = set_err(ctx, REATTN_ECUDA, std::string("append capture: ") + cudaGetErrorString(e));
    }
    if (!rc) rc = enqueue_step(ctx, p->P, p->cache, p->rope, p->q, p->out, cs, false);
    cudaGraph_t g = nullptr;
    const cudaError_t ce = cudaStreamEndCapture(cs, &g);
    cudaStreamDestroy(cs);
    if (rc || ce != cudaSuccess) {
        if (g) cudaGraphDestroy(g);
        return rc ? rc : set_err(ctx, REATTN_ECUDA, std::string("graph capture: ") + cudaGetErrorString(ce));
    }
    p->graph = g;
    const cudaError_t e = cudaGraphInstantiate(&p->exec, g, 0);
    if (e != cudaSuccess)
        return set_err(ctx, REATTN_ECUDA, std::string("graph instantiate: ") + cudaGetErrorString(e));
    return REATTN_OK;
}

}  // namespace

namespace reattn_capi {

bool zero_copy_enabled() {
    static const bool off = std::getenv("REATTN_NO_ZERO_COPY") != nullptr;
    return !off;
}

bool host_pinned(const void* p) {
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeHost;
}

// An I/O graph: host arrays -> device (zero-copy reads), `body` as a child graph, device
// output -> host.  Used by the plans' run_host / step_host on pinned buffers.
int build_io_exec(reattn_ctx* ctx, cudaGraph_t body, const float* const* in_src, float* const* in_dst,
                  const uint64_t* in_n, int n_in, const float* out_src, float* out_dst, uint64_t out_n,
                  cudaGraphExec_t* exec) {
    *exec = nullptr;
    cudaStream_t cs;
    CU(ctx, cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    CU(ctx, cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
    cudaError_t e = launch_host_io(in_src, in_dst, in_n, n_in, cs);
    if (e == cudaSuccess) {
        cudaGraph_t cap = nullptr;
        const cudaGraphNode_t* deps = nullptr;
        size_t nd = 0;
        cudaStreamCaptureStatus st;
        cudaGraphNode_t child = nullptr;
        e = cudaStreamGetCaptureInfo(cs, &st, nullptr, &cap, &deps, &nd);
        if (e == cudaSuccess) e = cudaGraphAddChildGraphNode(&child, cap, deps, nd, body);
        if (e == cudaSuccess) e = cudaStreamUpdateCaptureDependencies(cs, &child, 1, cudaStreamSetCaptureDependencies);
    }
    if (e == cudaSuccess) {
        const float* osrc[1] = {out_src};
        float* odst[1] = {out_dst};
        const uint64_t on[1] = {out_n};
        e = launch_host_io(osrc, odst, on, 1, cs);
    }
    cudaGraph_t g = nullptr;
    const cudaError_t ce = cudaStreamEndCapture(cs, &g);
    cudaStreamDestroy(cs);
    if (e != cudaSuccess || ce != cudaSuccess) {
        if (g) cudaGraphDestroy(g);
        return set_err(ctx, REATTN_ECUDA, std::string("host I/O graph: ") +
                                              cudaGetErrorString(e != cudaSuccess ? e : ce));
    }
    e = cudaGraphInstantiate(exec, g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) {
        *exec = nullptr;
        return set_err(ctx, REATTN_ECUDA, std::string("host I/O graph instantiate: ") + cudaGetErrorString(e));
    }
    return REATTN_OK;
}

}  // namespace reattn_capi

namespace {

// the plan's I/O graph for these host pointers (rebuilt when they, the append mode or the
// plan graph change)
int ensure_io_graph(reattn_plan* p, const float* q_host, const float* k_host, const float* v_host,
                    float* out_host) {
    const void* key[4] = {q_host, k_host, v_host, out_host};
    if (p->io_exec && p->io_append == p->append && std::equal(key, key + 4, p->io_key)) return REATTN_OK;
    if (p->io_exec) cudaGraphExecDestroy(p->io_exec);
    p->io_exec = nullptr;
    const uint64_t qn = p->P.n_q * p->P.n_head * p->cache->d, kn = p->cache->n_kv * p->cache->d;
    const float* src[3] = {q_host, k_host, v_host};
    float* dst[3] = {p->q, p->k_in, p->v_in};
    const uint64_t n[3] = {qn, kn, kn};
    int rc = build_io_exec(p->ctx, p->graph, src, dst, n, p->append ? 3 : 1, p->out, out_host, qn, &p->io_exec);
    if (rc) return rc;
    std::copy(key, key + 4, p->io_key);
    p->io_append = p->append;
    return REATTN_OK;
}


// A plan replays the graph it captured: the cache storage must be the one it was built over
// (reserve reallocates), and a frozen plan also its length (replays used to attend
// a stale scope silently).  Append mode: one more row must fit.
int check_plan(reattn_plan* p) {
    if (p->cache->generation != p->generation)
        return set_err(p->ctx, REATTN_ERUNTIME,
                       "plan: the cache storage was reallocated (reserve) since the plan was built; rebuild the plan");
    if (!p->P.dynamic && p->cache->total != p->total0)
        return set_err(p->ctx, REATTN_ERUNTIME,
                       "plan: the cache length changed since the plan was built (this plan shape is frozen); rebuild the plan");
    if (p->append && p->cache->total + 1 > p->cache->capacity)
        return set_err(p->ctx, REATTN_ERUNTIME, "cache append: capacity exceeded");
    return REATTN_OK;
}
}  // namespace

extern "C" {

const char* reattn_version(void) {
#ifdef REATTN_DEBUG
    return "reattn-b200 0.1 (sm_100a, debug: device asserts, trapping mbarrier timeouts)";
#else
    return "reattn-b200 0.1 (sm_100a)";
#endif
}

int reattn_ctx_create(int device, reattn_ctx** out) {
    auto* ctx = new reattn_ctx();
    ctx->device = device;
    cudaError_t e = cudaSetDevice(device);
    // a BLOCKING stream: work the caller issues on the legacy default stream (e.g. torch's
    // default-stream uploads, cudaMemcpy) is ordered with this context's kernels
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ctx->stream, cudaStreamDefault);
    if (e != cudaSuccess) {
        delete ctx;
        *out = nullptr;
        return REATTN_ECUDA;
    }
    ctx->own_stream = true;
    cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, device);
    e = cudaStreamCreateWithFlags(&ctx->side, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ctx->ev_fork, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ctx->ev_join, cudaEventDisableTiming);
    if (e != cudaSuccess) {
        reattn_ctx_destroy(ctx);
        *out = nullptr;
        return REATTN_ECUDA;
    }
    *out = ctx;
    return REATTN_OK;
}

void reattn_ctx_destroy(reattn_ctx* ctx) {
    if (!ctx) return;
    cudaStreamSynchronize(ctx->stream);
    if (ctx->side) cudaStreamSynchronize(ctx->side);
    if (ctx->arena) cudaFree(ctx->arena);
    if (ctx->ev_fork) cudaEventDestroy(ctx->ev_fork);
    if (ctx->ev_join) cudaEventDestroy(ctx->ev_join);
    if (ctx->side) cudaStreamDestroy(ctx->side);
    if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
    delete ctx;
}

const char* reattn_last_error(const reattn_ctx* ctx) { return ctx ? ctx->err.c_str() : ""; }

int reattn_ctx_set_stream(reattn_ctx* ctx, void* s) {
    if (ctx->own_stream) {
        cudaStreamSynchronize(ctx->stream);
        cudaStreamDestroy(ctx->stream);
        ctx->own_stream = false;
    }
    ctx->stream = (cudaStream_t)s;
    return REATTN_OK;
}
void* reattn_ctx_stream(const reattn_ctx* ctx) { return (void*)ctx->stream; }

int reattn_ctx_set_lanes(reattn_ctx* ctx, int lanes) {
    if (lanes != REATTN_LANES_UNFUSED && lanes != REATTN_LANES_FMA)
        return set_err(ctx, REATTN_EINVAL, "unknown lane arithmetic");
    ctx->lanes = lanes;
    return REATTN_OK;
}
int reattn_ctx_set_prefill(reattn_ctx* ctx, int mode) {
    if (mode < REATTN_PREFILL_EXACT || mode > REATTN_PREFILL_TENSOR)
        return set_err(ctx, REATTN_EINVAL, "unknown prefill mode");
    ctx->prefill = mode;
    return REATTN_OK;
}
int reattn_ctx_synchronize(reattn_ctx* ctx) {
    CU(ctx, cudaStreamSynchronize(ctx->stream));
    return REATTN_OK;
}
int reattn_ctx_num_sms(const reattn_ctx* ctx) { return ctx->num_sms; }

int reattn_malloc(reattn_ctx* ctx, uint64_t bytes, void** out) {
    *out = nullptr;
    CU(ctx, cudaMalloc(out, std::max<uint64_t>(bytes, 1)));
    return REATTN_OK;
}
int reattn_free(reattn_ctx* ctx, void* p) {
    if (p) CU(ctx, cudaFree(p));
    return REATTN_OK;
}
int reattn_memcpy_h2d(reattn_ctx* ctx, void* dst, const void* src, uint64_t bytes) {
    if (!bytes) return REATTN_OK;
    CU(ctx, cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, ctx->stream));
    CU(ctx, cudaStreamSynchronize(ctx->stream));
    return REATTN_OK;
}
int reattn_memcpy_d2h(reattn_ctx* ctx, void* dst, const void* src, uint64_t bytes) {
    if (!bytes) return REATTN_OK;
    CU(ctx, cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, ctx->stream));
    CU(ctx, cudaStreamSynchronize(ctx->stream));
    return REATTN_OK;
}

// ---- cache ---------------------------------------------------------------------------
int reattn_cache_create(reattn_ctx* ctx, uint64_t n_kv, uint64_t d, uint64_t l_global,
                        uint64_t l_local_max, uint64_t capacity, int dtype, reattn_cache** out) {
    *out = nullptr;
    if (n_kv == 0 || d == 0)
        return set_err(ctx, REATTN_EINVAL, "cache needs at least one head and a positive head dim");
    if (l_local_max == 0) return set_err(ctx, REATTN_EINVAL, "l_local_max must be positive");
    if (dtype != REATTN_F32 && dtype != REATTN_BF16)
        return set_err(ctx, REATTN_EINVAL, "cache: unknown dtype");
    auto* c = new reattn_cache();
    c->n_kv = n_kv;
    c->d = d;
    c->l_global = l_global;
    c->l_local_max = l_local_max;
    c->capacity = std::max<uint64_t>(capacity, 1);
    c->dtype = dtype;
    const size_t bytes = n_kv * c->capacity * d * (dtype == REATTN_BF16 ? 2 : 4);
    cudaError_t e = cudaMalloc(&c->keys, bytes);
    if (e == cudaSuccess) e = cudaMalloc(&c->values, bytes);
    if (e == cudaSuccess) e = cudaMalloc(&c->dev_total, sizeof(uint32_t));
    if (e == cudaSuccess) e = cudaMemsetAsync(c->dev_total, 0, sizeof(uint32_t), ctx->stream);
    if (e != cudaSuccess) {
        if (c->keys) cudaFree(c->keys);
        if (c->values) cudaFree(c->values);
        delete c;
        return set_err(ctx, REATTN_ECUDA, std::string("cache allocation: ") + cudaGetErrorString(e));
    }
    *out = c;
    return REATTN_OK;
}

void reattn_cache_destroy(reattn_cache* c) {
    if (!c) return;
    cudaFree(c->keys);
    cudaFree(c->values);
    if (c->dev_total) cudaFree(c->dev_total);
    delete c;
}

int reattn_cache_append(reattn_ctx* ctx, reattn_cache* c, const float* keys, const float* values,
                        uint64_t rows, int src_on_device) {
    if (rows == 0) return REATTN_OK;
    if (c->total + rows > c->capacity)
        return set_err(ctx, REATTN_ERUNTIME, "cache append: capacity exceeded");
    const size_t bytes = rows * c->n_kv * c->d * sizeof(float);
    const float* ks = keys;
    const float* vs = values;
    if (!src_on_device) {
        int rc = ensure_arena(ctx, 2 * bytes + 512);
        if (rc) return rc;
        float* kd = (float*)ctx->arena;
        float* vd = (float*)((uint8_t*)ctx->arena + align_up(bytes, 256));
        CU(ctx, cudaMemcpyAsync(kd, keys, bytes, cudaMemcpyHostToDevice, ctx->stream));
        CU(ctx, cudaMemcpyAsync(vd, values, bytes, cudaMemcpyHostToDevice, ctx->stream));
        ks = kd;
        vs = vd;
    }
    CU(ctx, launch_cache_append(ks, c->keys, c->dtype, rows, c->n_kv, c->d, c->capacity, c->total,
                                ctx->stream));
    CU(ctx, launch_cache_append(vs, c->values, c->dtype, rows, c->n_kv, c->d, c->capacity,
                                c->total, ctx->stream));
    c->total += rows;  // boundaries follow kv_cache.hpp:65-67 (computed on demand)
    int rc = cache_sync_total(ctx, c, ctx->stream);
    if (rc) return rc;
    // host rows were staged in the context arena: drain before it can be reused (device
    // sources stay asynchronous, stream-ordered with the steps that read them)
    if (!src_on_device) CU(ctx, cudaStreamSynchronize(ctx->stream));
    return REATTN_OK;
}

int reattn_cache_reserve(reattn_ctx* ctx, reattn_cache* c, uint64_t cap) {
    if (cap <= c->capacity) return REATTN_OK;
    const uint64_t esz = c->dtype == REATTN_BF16 ? 2 : 4;
    void* nk = nullptr;
    void* nv = nullptr;
    CU(ctx, cudaMalloc(&nk, c->n_kv * cap * c->d * esz));
    CU(ctx, cudaMalloc(&nv, c->n_kv * cap * c->d * esz));
    if (c->total) {
        const size_t w = c->total * c->d * esz;
        CU(ctx, cudaMemcpy2DAsync(nk, cap * c->d * esz, c->keys, c->capacity * c->d * esz, w,
                                  c->n_kv, cudaMemcpyDeviceToDevice, ctx->stream));
        CU(ctx, cudaMemcpy2DAsync(nv, cap * c->d * esz, c->values, c->capacity * c->d * esz, w,
                                  c->n_kv, cudaMemcpyDeviceToDevice, ctx->stream));
    }
    CU(ctx, cudaStreamSynchronize(ctx->stream));
    cudaFree(c->keys);
    cudaFree(c->values);
    c->keys = nk;
    c->values = nv;
    c->capacity = cap;
    ++c->generation;  // plans over the old storage are invalid (checked at launch)
    return REATTN_OK;
}

int reattn_cache_set_total(reattn_ctx* ctx, reattn_cache* c, uint64_t total) {
    if (total > c->capacity) return set_err(ctx, REATTN_EINVAL, "cache: total exceeds capacity");
    c->total = total;
    return cache_sync_total(ctx, c, ctx->stream);
}

int reattn_cache_info(const reattn_cache* c, uint64_t* n_kv, uint64_t* d, uint64_t* l_global,
                      uint64_t* l_local_max, uint64_t* capacity, uint64_t* total,
                      uint64_t* global_end, uint64_t* local_start, int* dtype) {
    if (n_kv) *n_kv = c->n_kv;
    if (d) *d = c->d;
    if (l_global) *l_global = c->l_global;
    if (l_local_max) *l_local_max = c->l_local_max;
    if (capacity) *capacity = c->capacity;
    if (total) *total = c->total;
    if (global_end) *global_end = c->global_end();
    if (local_start) *local_start = c->local_start();
    if (dtype) *dtype = c->dtype;
    return REATTN_OK;
}
void* reattn_cache_keys(const reattn_cache* c) { return c->keys; }
void* reattn_cache_values(const reattn_cache* c) { return c->values; }

// ---- rope ----------------------------------------------------------------------------
int reattn_rope_create(reattn_ctx* ctx, uint64_t head_dim, double base, uint64_t max_position,
                       reattn_rope** out) {
    *out = nullptr;
    if (head_dim == 0 || head_dim % 2 != 0)
        return set_err(ctx, REATTN_EINVAL, "rotary head_dim must be even and positive");
    if (!(base > 0.0)) return set_err(ctx, REATTN_EINVAL, "rotary base must be positive");
    if (max_position == 0)
        return set_err(ctx, REATTN_EINVAL, "rotary max_position must be positive");
    auto* r = new reattn_rope();
    r->head_dim = head_dim;
    r->max_position = max_position;
    r->base = base;
    const uint64_t half = head_dim / 2;
    // table constant: float(cos/sin(p * base^(-2i/d))) computed in double (rope.hpp:27-39)
    std::vector<double> inv(half);
    for (uint64_t i = 0; i < half; ++i) inv[i] = std::pow(base, -2.0 * double(i) / double(head_dim));
    r->cos_h.resize(max_position * half);
    r->sin_h.resize(max_position * half);
    for (uint64_t p = 0; p < max_position; ++p)
        for (uint64_t i = 0; i < half; ++i) {
            const double ang = double(p) * inv[i];
            r->cos_h[p * half + i] = float(std::cos(ang));
            r->sin_h[p * half + i] = float(std::sin(ang));
        }
    const size_t bytes = r->cos_h.size() * sizeof(float);
    cudaError_t e = cudaMalloc(&r->cos_d, bytes);
    if (e == cudaSuccess) e = cudaMalloc(&r->sin_d, bytes);
    if (e == cudaSuccess) e = cudaMemcpy(r->cos_d, r->cos_h.data(), bytes, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(r->sin_d, r->sin_h.data(), bytes, cudaMemcpyHostToDevice);
    // a pageable-source cudaMemcpy may return before its DMA lands: complete it before any
    // stream (ordered with the legacy stream or not) can read the tables
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        cudaFree(r->cos_d);
        cudaFree(r->sin_d);
        delete r;
        return set_err(ctx, REATTN_ECUDA, std::string("rope upload: ") + cudaGetErrorString(e));
    }
    *out = r;
    return REATTN_OK;
}

void reattn_rope_destroy(reattn_rope* r) {
    if (!r) return;
    cudaFree(r->cos_d);
    cudaFree(r->sin_d);
    delete r;
}

int reattn_rope_tables_host(const reattn_rope* r, float* c, float* s) {
    if (c) std::copy(r->cos_h.begin(), r->cos_h.end(), c);
    if (s) std::copy(r->sin_h.begin(), r->sin_h.end(), s);
    return REATTN_OK;
}

int reattn_rope_rotate(reattn_ctx* ctx, const reattn_rope* r, float* rows, const uint64_t* pos,
                       uint64_t n_rows) {
    if (n_rows == 0) return REATTN_OK;
    std::vector<uint32_t> p32(n_rows);
    for (uint64_t i = 0; i < n_rows; ++i) {
        if (pos[i] >= r->max_position)
            return set_err(ctx, REATTN_ERANGE, "position out of pretrained range");
        p32[i] = (uint32_t)pos[i];
    }
    int rc = ensure_arena(ctx, n_rows * 4 + 256);
    if (rc) return rc;
    CU(ctx, cudaMemcpyAsync(ctx->arena, p32.data(), n_rows * 4, cudaMemcpyHostToDevice, ctx->stream));
    CU(ctx, launch_rope_rotate(rows, (const uint32_t*)ctx->arena, n_rows, r->head_dim, r->cos_d,
                               r->sin_d, ctx->stream));
    CU(ctx, cudaStreamSynchronize(ctx->stream));
    return REATTN_OK;
}

// ---- selection ---------------------------------------------------------------------------
int reattn_fused_topk(reattn_ctx* ctx, const float* q_dev, uint64_t n_q, uint64_t n_heads,
                      const void* keys_dev, int key_dtype, uint64_t n_kv, uint64_t head_stride,
                      uint64_t row0, uint64_t count, uint64_t d, uint64_t k, uint32_t* idx_out,
                      float* score_out, uint64_t* n_out, uint64_t* scratch_bytes) {
    if (n_kv == 0 || n_heads % n_kv != 0)
        return set_err(ctx, REATTN_EINVAL, "fused_topk_scores: n_heads must be a multiple of kv heads");
    if (k == 0) return set_err(ctx, REATTN_EINVAL, "selection: k must be >= 1");
    if (count >= (1ull << 32)) return set_err(ctx, REATTN_EINVAL, "fused_topk_scores: middle too long");
    if (n_out) *n_out = std::min(k, count);
    ScanPlan sp;
    ScanArgs& a = sp.a;
    a.q = q_dev;
    a.n_q = (int)n_q;
    a.n_heads = (int)n_heads;
    a.n_kv = (int)n_kv;
    a.d = (int)d;
    a.keys = keys_dev;
    a.dtype = key_dtype;
    a.head_stride = head_stride;
    a.row0 = row0;
    a.count = (uint32_t)count;
    a.k = (int)k;
    a.lanes = ctx->lanes;
    a.idx_out = idx_out;
    a.score_out = score_out;
    int rc = plan_scan(ctx, sp);
    if (rc) return rc;
    // fixed workspace: independent of `count` (the scratch contract, test_selection.cpp:228)
    // fixed workspace: independent of `count` (the scratch contract, test_selection.cpp:228)
    const size_t ws_fixed = std::max(scan_fast_workspace(a, ctx->num_sms), sp.ws_bytes);
    if (scratch_bytes) *scratch_bytes = ws_fixed + n_q * n_kv * k * 8;
    if (count == 0 || n_q == 0) return REATTN_OK;
    rc = ensure_arena(ctx, ws_fixed + 256);
    if (rc) return rc;
    rc = enqueue_scan(ctx, sp, ctx->arena, ctx->stream, true);
    if (rc) return rc;
    CU(ctx, cudaStreamSynchronize(ctx->stream));
    return REATTN_OK;
}

int reattn_naive_topk(reattn_ctx* ctx, const float* q_dev, uint64_t n_q, uint64_t n_heads,
                      const void* keys_dev, int key_dtype, uint64_t n_kv, uint64_t head_stride,
                      uint64_t row0, uint64_t count, uint64_t d, uint64_t k, uint32_t* idx_out,
                      float* score_out, uint64_t* n_out, uint64_t* scratch_bytes) {
    if (n_kv == 0 || n_heads % n_kv != 0)
        return set_err(ctx, REATTN_EINVAL, "naive_topk_scores: n_heads must be a multiple of kv heads");
    if (k == 0) return set_err(ctx, REATTN_EINVAL, "selection: k must be >= 1");
    if (count >= (1ull << 32)) return set_err(ctx, REATTN_EINVAL, "naive_topk_scores: middle too long");
    if (n_out) *n_out = std::min(k, count);
    // the reference's meter (selection_reference.hpp:37-41): mq + the score matrix (+ its
    // order buffer, which the device selection does not need)
    const size_t ws = naive_topk_workspace(n_q, n_kv, count, d);
    if (scratch_bytes) *scratch_bytes = ws;
    if (count == 0 || n_q == 0) return REATTN_OK;
    int rc = ensure_arena(ctx, ws + 256);
    if (rc) return rc;
    ScanArgs a{};
    a.q = q_dev;
    a.n_q = (int)n_q;
    a.n_heads = (int)n_heads;
    a.n_kv = (int)n_kv;
    a.d = (int)d;
    a.keys = keys_dev;
    a.dtype = key_dtype;
    a.head_stride = head_stride;
    a.row0 = row0;
    a.count = (uint32_t)count;
    a.k = (int)k;
    a.lanes = ctx->lanes;
    a.idx_out = idx_out;
    a.score_out = score_out;
    CU(ctx, launch_naive_topk(a, ctx->arena, ctx->stream));
    CU(ctx, cudaStreamSynchronize(ctx->stream));
    return REATTN_OK;
}

int reattn_dot_f32(reattn_ctx* ctx, const float* a, const float* b, uint64_t n, uint64_t d,
                   float* out) {
    if (n == 0) return REATTN_OK;
    CU(ctx, launch_dot_f32(a, b, n, d, ctx->lanes, out, ctx->stream));
    CU(ctx, cudaStreamSynchronize(ctx->stream));
    return REATTN_OK;
}

int reattn_dot_f64(reattn_ctx* ctx, const float* a, const float* b, uint64_t n, uint64_t d,
                   double* out) {
    if (n == 0) return REATTN_OK;
    CU(ctx, launch_dot_f64(a, b, n, d, out, ctx->stream));
    CU(ctx, cudaStreamSynchronize(ctx->stream));
    return REATTN_OK;
}

int reattn_matmul(reattn_ctx* ctx, const float* a, const float* b, uint64_t m, uint64_t k,
                  uint64_t n, float* c) {
    if (m * n == 0) return REATTN_OK;
    CU(ctx, launch_matmul(a, b, m, k, n, c, ctx->stream));
    CU(ctx, cudaStreamSynchronize(ctx->stream));
    return REATTN_OK;
}

int reattn_rmsnorm(reattn_ctx* ctx, const float* x_dev, uint64_t rows, uint64_t cols, const float* w_dev,
                   float* out_dev) {
    if (rows == 0 || cols == 0) return REATTN_OK;
    CU(ctx, launch_rmsnorm(x_dev, rows, cols, w_dev, out_dev, ctx->stream));
    CU(ctx, cudaStreamSynchronize(ctx->stream));
    return REATTN_OK;
}

int reattn_silu_mul(reattn_ctx* ctx, float* gate_dev, const float* up_dev, uint64_t n) {
    if (n == 0) return REATTN_OK;
    CU(ctx, launch_silu_mul(gate_dev, up_dev, n, ctx->stream));
    CU(ctx, cudaStreamSynchronize(ctx->stream));
    return REATTN_OK;
}

int reattn_stable_softmax(reattn_ctx* ctx, const float* logits_dev, uint64_t n, float* out_dev) {
    if (n == 0) return set_err(ctx, REATTN_EINVAL, "empty logits");
    if (n >= (1ull << 31)) return set_err(ctx, REATTN_EINVAL, "stable_softmax: too many logits");
    int rc = ensure_arena(ctx, n * sizeof(double) + 256);
    if (rc) return rc;
    CU(ctx, launch_stable_softmax(logits_dev, n, out_dev, (double*)ctx->arena, ctx->stream));
    CU(ctx, cudaStreamSynchronize(ctx->stream));
    return REATTN_OK;
}

int reattn_attention_entropy(reattn_ctx* ctx, const float* weights_dev, uint64_t n, double* entropy_out_dev) {
    if (n >= (1ull << 31)) return set_err(ctx, REATTN_EINVAL, "attention_entropy: too many weights");
    if (n == 0) {
        CU(ctx, cudaMemsetAsync(entropy_out_dev, 0, sizeof(double), ctx->stream));
        CU(ctx, cudaStreamSynchronize(ctx->stream));
        return REATTN_OK;
    }
    int rc = ensure_arena(ctx, n * sizeof(double) + 256);
    if (rc) return rc;
    CU(ctx, launch_attention_entropy(weights_dev, n, entropy_out_dev, (double*)ctx->arena, ctx->stream));
    CU(ctx, cudaStreamSynchronize(ctx->stream));
    return REATTN_OK;
}

int reattn_group_mean(reattn_ctx* ctx, const float* q, uint64_t n_q, uint64_t n_heads,
                      uint64_t n_kv, uint64_t d, float* out) {
    if (n_kv == 0 || n_heads % n_kv != 0)
        return set_err(ctx, REATTN_EINVAL, "fused_topk_scores: n_heads must be a multiple of kv heads");
    if (n_q * n_kv * d == 0) return REATTN_OK;
    CU(ctx, launch_group_mean(q, n_q, n_heads, n_kv, d, out, ctx->stream));
    CU(ctx, cudaStreamSynchronize(ctx->stream));
    return REATTN_OK;
}

int reattn_vote(reattn_ctx* ctx, const uint32_t* idx_dev, const float* score_dev, uint64_t n,
                uint64_t k_prime, uint32_t* winners_dev, uint64_t* n_winners) {
    *n_winners = 0;
    if (k_prime == 0 || n == 0) return REATTN_OK;
    if (n >= (1ull << 31)) return set_err(ctx, REATTN_ERUNTIME, "vote: candidate count exceeds 2^31");
    const bool large = n > kVoteMaxSmem;
    int rc = ensure_arena(ctx, 4096 + (large ? vote_large_workspace((uint32_t)n, 0, 0) : 0));
    if (rc) return rc;
    SelectArgs sa;
    std::memset(&sa, 0, sizeof(sa));
    sa.cand_idx = idx_dev;
    sa.cand_score = score_dev;
    sa.n_lists = 1;
    sa.list_len = (uint32_t)n;
    sa.list_stride = (uint32_t)n;
    sa.k_prime = (uint32_t)std::min<uint64_t>(k_prime, n);
    sa.winners = winners_dev;
    sa.hdr = (ScopeHeader*)ctx->arena;
    if (large)
        CU(ctx, launch_vote_large(sa, (uint8_t*)ctx->arena + 4096, ctx->stream));
    else
        CU(ctx, launch_select(sa, ctx->stream));
    ScopeHeader h;
    CU(ctx, cudaMemcpyAsync(&h, sa.hdr, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
    CU(ctx, cudaStreamSynchronize(ctx->stream));
    rc = status_from_scope(ctx, h.error);
    if (rc) return rc;
    *n_winners = h.n_winners;
    return REATTN_OK;
}

int reattn_tally(reattn_ctx* ctx, const uint32_t* idx_dev, const float* score_dev, uint64_t n,
                 uint32_t* idx_out, uint32_t* votes_out, float* score_out, uint64_t* n_unique) {
    *n_unique = 0;
    if (n == 0) return REATTN_OK;
    if (n >= (1ull << 31)) return set_err(ctx, REATTN_ERUNTIME, "vote: candidate count exceeds 2^31");
    const bool large = n > kVoteMaxSmem;
    int rc = ensure_arena(ctx, 4096 + (large ? vote_large_workspace((uint32_t)n, 0, 0) : 0));
    if (rc) return rc;
    SelectArgs sa;
    std::memset(&sa, 0, sizeof(sa));
    sa.cand_idx = idx_dev;
    sa.cand_score = score_dev;
    sa.n_lists = 1;
    sa.list_len = (uint32_t)n;
    sa.list_stride = (uint32_t)n;
    sa.k_prime = (uint32_t)n;
    sa.winners = idx_out;
    sa.rank_votes = votes_out;
    sa.rank_score = score_out;
    sa.hdr = (ScopeHeader*)ctx->arena;
    if (large)
        CU(ctx, launch_vote_large(sa, (uint8_t*)ctx->arena + 4096, ctx->stream));
    else
        CU(ctx, launch_select(sa, ctx->stream));
    ScopeHeader h;
    CU(ctx, cudaMemcpyAsync(&h, sa.hdr, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
    CU(ctx, cudaStreamSynchronize(ctx->stream));
    rc = status_from_scope(ctx, h.error);
    if (rc) return rc;
    *n_unique = h.n_winners;
    return REATTN_OK;
}

int reattn_expand_spans(reattn_ctx* ctx, const uint32_t* winners_dev, uint64_t n, uint64_t span_m,
                        uint64_t middle_len, int span_mode, uint32_t* begin_dev,
                        uint32_t* end_dev, uint64_t* n_spans) {
    *n_spans = 0;
    if (span_m == 0) return set_err(ctx, REATTN_EINVAL, "selection: span_m must be >= 1");
    if (n == 0 || middle_len == 0) return REATTN_OK;
    int rc = ensure_arena(ctx, 4096);
    if (rc) return rc;
    SelectArgs sa;
    std::memset(&sa, 0, sizeof(sa));
    sa.winners_in = winners_dev;
    sa.n_winners_in = (uint32_t)n;
    sa.k_prime = (uint32_t)n;
    sa.span_m = (uint32_t)span_m;
    sa.middle_len = (uint32_t)middle_len;
    sa.span_mode = span_mode;
    sa.winners = const_cast<uint32_t*>(winners_dev);
    sa.span_b = begin_dev;
    sa.span_e = end_dev;
    sa.hdr = (ScopeHeader*)ctx->arena;
    CU(ctx, launch_select(sa, ctx->stream));
    ScopeHeader h;
    CU(ctx, cudaMemcpyAsync(&h, sa.hdr, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
    CU(ctx, cudaStreamSynchronize(ctx->stream));
    rc = status_from_scope(ctx, h.error);
    if (rc) return rc;
    *n_spans = h.n_spans;
    return REATTN_OK;
}

int reattn_assemble_scope(reattn_ctx* ctx, const reattn_cache* c, const uint32_t* span_b_dev,
                          const uint32_t* span_e_dev, uint64_t n_spans, uint64_t window,
                          uint32_t* src_dev, float* keys_out, float* values_out,
                          uint64_t* length) {
    int rc = ensure_arena(ctx, 4096);
    if (rc) return rc;
    SelectArgs sa;
    std::memset(&sa, 0, sizeof(sa));
    sa.span_b_in = span_b_dev;
    sa.span_e_in = span_e_dev;
    sa.n_spans_in = (uint32_t)n_spans;
    if (n_spans == 0) {  // an empty SpanSet: still "given", never voted
        sa.span_b_in = span_b_dev ? span_b_dev : (const uint32_t*)ctx->arena;
        sa.span_e_in = sa.span_b_in;
    }
    sa.middle_len = (uint32_t)(c->local_start() - c->global_end());
    sa.build_scope = 1;
    sa.g_end = (uint32_t)c->global_end();
    sa.l_start = (uint32_t)c->local_start();
    sa.total = (uint32_t)c->total;
    sa.window = (uint32_t)std::min<uint64_t>(window, 0xFFFFFFFFull);
    sa.n_q = 0;
    sa.scope_src = src_dev;
    sa.hdr = (ScopeHeader*)((uint8_t*)ctx->arena + 256);
    CU(ctx, launch_select(sa, ctx->stream));
    ScopeHeader h;
    CU(ctx, cudaMemcpyAsync(&h, sa.hdr, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
    CU(ctx, cudaStreamSynchronize(ctx->stream));
    rc = status_from_scope(ctx, h.error);
    if (rc) return rc;
    *length = h.L;
    if (h.L && keys_out)
        CU(ctx, launch_gather(c->keys, c->dtype, c->n_kv, c->d, c->capacity, src_dev, h.L,
                              keys_out, ctx->stream));
    if (h.L && values_out)
        CU(ctx, launch_gather(c->values, c->dtype, c->n_kv, c->d, c->capacity, src_dev, h.L,
                              values_out, ctx->stream));
    CU(ctx, cudaStreamSynchronize(ctx->stream));
    return REATTN_OK;
}

int reattn_attend(reattn_ctx* ctx, const float* q_dev, uint64_t n_q, const float* k_dev,
                  const float* v_dev, uint64_t L, uint64_t d, uint64_t dv, int has_boundary,
                  uint64_t boundary, float* out_dev, double* entropy_dev) {
    if (L == 0) return set_err(ctx, REATTN_EINVAL, "empty key set");
    if (d > 4096 || dv > 4096) return set_err(ctx, REATTN_EINVAL, "attend: head dim too large");
    if (n_q == 0) return REATTN_OK;
    AttnArgs a;
    std::memset(&a, 0, sizeof(a));
    a.q = q_dev;
    a.q_row_stride = d;
    a.n_q = (int)n_q;
    a.n_head = 1;
    a.n_kv = 1;
    a.group = 1;
    a.d = (int)d;
    a.dv = (int)dv;
    a.dtype = kF32;
    a.head_stride = 0;
    a.src = nullptr;
    a.hdr = nullptr;
    a.L_host = (uint32_t)L;
    a.causal = has_boundary ? 1 : 0;
    a.boundary_is_tail = 0;
    a.boundary_host = (uint32_t)std::min<uint64_t>(boundary, 0xFFFFFFF0ull);
    a.out = out_dev;
    a.entropy = entropy_dev;
    // k and v have different row widths: run them as separate bases (head_stride unused)
    a.k_base = k_dev;
    a.v_base = v_dev;
    const size_t ws = attend_workspace(a, (uint32_t)L);
    int rc = ensure_arena(ctx, ws + 256);
    if (rc) return rc;
    a.part = (double*)ctx->arena;
    CU(ctx, launch_attend(a, (uint32_t)L, ctx->stream));
    CU(ctx, cudaStreamSynchronize(ctx->stream));
    return REATTN_OK;
}

int reattn_attend_step(reattn_ctx* ctx, const reattn_cache* cache, const reattn_rope* rope,
                       const float* q_dev, uint64_t n_q, uint64_t n_head,
                       const reattn_selection_config* cfg, int mode, float* out_dev,
                       reattn_step_stats* stats, uint64_t* span_b_host, uint64_t* span_e_host,
                       double* entropy_host) {
    StepPlan P;
    int rc = plan_step(ctx, cache, rope, n_q, n_head, cfg, mode, P, q_dev, out_dev);
    if (rc) return rc;
    Carver sizer{nullptr, 0, 0};
    carve_step(P, cache, rope, sizer);
    rc = ensure_arena(ctx, sizer.off + 256);
    if (rc) return rc;
    Carver c{(uint8_t*)ctx->arena, 0, ctx->arena_bytes};
    carve_step(P, cache, rope, c);
    rc = enqueue_step(ctx, P, cache, rope, q_dev, out_dev, ctx->stream, true);
    if (rc) return rc;
    ScopeHeader h;
    CU(ctx, cudaMemcpyAsync(&h, P.hdr, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
    CU(ctx, cudaStreamSynchronize(ctx->stream));
    rc = finish_step_stats(ctx, P, h, stats, entropy_host);
    if (rc) return rc;
    if (span_b_host && h.n_spans) {
        std::vector<uint32_t> b(h.n_spans), e(h.n_spans);
        CU(ctx, cudaMemcpy(b.data(), P.span_b, h.n_spans * 4, cudaMemcpyDeviceToHost));
        CU(ctx, cudaMemcpy(e.data(), P.span_e, h.n_spans * 4, cudaMemcpyDeviceToHost));
        for (uint32_t i = 0; i < h.n_spans; ++i) {
            span_b_host[i] = b[i];
            span_e_host[i] = e[i];
        }
    }
    return REATTN_OK;
}

// ---- plans ---------------------------------------------------------------------------
int reattn_plan_create(reattn_ctx* ctx, const reattn_cache* cache, const reattn_rope* rope,
                       uint64_t n_q, uint64_t n_head, const reattn_selection_config* cfg,
                       int mode, reattn_plan** out) {
    *out = nullptr;
    auto* p = new reattn_plan();
    p->ctx = ctx;
    p->cache = const_cast<reattn_cache*>(cache);  // append mode writes rows (through the graph)
    p->rope = rope;
    p->generation = cache->generation;
    p->total0 = cache->total;
    int rc = plan_step(ctx, cache, rope, n_q, n_head, cfg, mode, p->P, nullptr, nullptr, true);
    if (rc) {
        delete p;
        return rc;
    }
    Carver sizer{nullptr, 0, 0};
    sizer.take<float>(n_q * n_head * cache->d);
    sizer.take<float>(n_q * n_head * cache->d);
    sizer.take<float>(cache->n_kv * cache->d);
    sizer.take<float>(cache->n_kv * cache->d);
    carve_step(p->P, cache, rope, sizer);
    cudaError_t e = cudaMalloc(&p->mem, sizer.off + 256);
    if (e == cudaSuccess) e = cudaMemset(p->mem, 0, sizer.off + 256);
    if (e == cudaSuccess) e = cudaDeviceSynchronize();  // zeroed before any stream replays
    if (e != cudaSuccess) {
        delete p;
        return set_err(ctx, REATTN_ECUDA, std::string("plan allocation: ") + cudaGetErrorString(e));
    }
    Carver c{(uint8_t*)p->mem, 0, sizer.off + 256};
    p->q = c.take<float>(n_q * n_head * cache->d);
    p->out = c.take<float>(n_q * n_head * cache->d);
    p->k_in = c.take<float>(cache->n_kv * cache->d);
    p->v_in = c.take<float>(cache->n_kv * cache->d);
    carve_step(p->P, cache, rope, c);
    rc = capture_plan(p);
    if (rc) {
        reattn_plan_destroy(p);
        return rc;
    }
    *out = p;
    return REATTN_OK;
}

void reattn_plan_destroy(reattn_plan* p) {
    if (!p) return;
    cudaDeviceSynchronize();  // never touches the (possibly destroyed) context stream
    if (p->exec) cudaGraphExecDestroy(p->exec);
    if (p->graph) cudaGraphDestroy(p->graph);
    cudaFree(p->mem);
    if (p->staged) cudaFreeHost(p->staged);
    if (p->io_exec) cudaGraphExecDestroy(p->io_exec);
    delete p;
}
float* reattn_plan_q(const reattn_plan* p) { return p->q; }
float* reattn_plan_out(const reattn_plan* p) { return p->out; }

int reattn_plan_launch(reattn_plan* p) {
    int rc = check_plan(p);
    if (rc) return rc;
    CU(p->ctx, cudaGraphLaunch(p->exec, p->ctx->stream));
    if (p->append) ++p->cache->total;  // the host mirror of the row the graph appends
    return REATTN_OK;
}

int reattn_plan_set_append(reattn_plan* p, int enable) {
    if (enable && !p->P.dynamic)
        return set_err(p->ctx, REATTN_EINVAL,
                       "plan append: needs a decode plan that follows the cache length "
                       "(n_q == 1, selection on the K1 fast scan with the fused select)");
    if ((enable != 0) == p->append) return REATTN_OK;
    CU(p->ctx, cudaStreamSynchronize(p->ctx->stream));
    p->append = enable != 0;
    return capture_plan(p);
}
int reattn_plan_follows_cache(const reattn_plan* p) { return p->P.dynamic ? 1 : 0; }
uint64_t reattn_plan_cache_generation(const reattn_plan* p) { return p->generation; }
float* reattn_plan_k_in(const reattn_plan* p) { return p->k_in; }
float* reattn_plan_v_in(const reattn_plan* p) { return p->v_in; }

int reattn_plan_step_host(reattn_plan* p, const float* q_host, const float* k_host,
                          const float* v_host, float* out_host) {
    reattn_ctx* ctx = p->ctx;
    int rc = check_plan(p);
    if (rc) return rc;
    const size_t qb = p->P.n_q * p->P.n_head * p->cache->d * sizeof(float);
    const size_t kb = p->cache->n_kv * p->cache->d * sizeof(float);
    const void* key[4] = {q_host, p->append ? k_host : nullptr, p->append ? v_host : nullptr, out_host};
    const bool io_ready = p->io_exec && p->io_append == p->append && std::equal(key, key + 4, p->io_key);
    if (io_ready || (zero_copy_enabled() && host_pinned(q_host) && host_pinned(out_host) &&
                     (!p->append || (host_pinned(k_host) && host_pinned(v_host))))) {
        if ((rc = ensure_io_graph(p, q_host, p->append ? k_host : nullptr, p->append ? v_host : nullptr,
                                  out_host)))
            return rc;
        CU(ctx, cudaGraphLaunch(p->io_exec, ctx->stream));
        if (p->append) ++p->cache->total;
        CU(ctx, cudaStreamSynchronize(ctx->stream));
        return REATTN_OK;
    }
    CU(ctx, cudaMemcpyAsync(p->q, q_host, qb, cudaMemcpyHostToDevice, ctx->stream));
    if (p->append) {
        CU(ctx, cudaMemcpyAsync(p->k_in, k_host, kb, cudaMemcpyHostToDevice, ctx->stream));
        CU(ctx, cudaMemcpyAsync(p->v_in, v_host, kb, cudaMemcpyHostToDevice, ctx->stream));
    }
    CU(ctx, cudaGraphLaunch(p->exec, ctx->stream));
    if (p->append) ++p->cache->total;
    CU(ctx, cudaMemcpyAsync(out_host, p->out, qb, cudaMemcpyDeviceToHost, ctx->stream));
    CU(ctx, cudaStreamSynchronize(ctx->stream));
    return REATTN_OK;
}

int reattn_plan_launch_scan(reattn_plan* p) {
    if (!p->P.select) return REATTN_OK;
    int rc = check_plan(p);
    if (rc) return rc;
    return enqueue_scan(p->ctx, p->P.scan, p->P.scan_ws, p->ctx->stream, false);
}

int reattn_debug_trace(uint64_t* host_out, uint64_t n) {
    uint64_t* t = reattn_impl::trace_buffer();
    if (!t || n > (uint64_t)reattn_impl::kTraceWords) return REATTN_EINVAL;
    if (cudaDeviceSynchronize() != cudaSuccess ||
        cudaMemcpy(host_out, t, n * sizeof(uint64_t), cudaMemcpyDeviceToHost) != cudaSuccess)
        return REATTN_ECUDA;
    return REATTN_OK;
}

int reattn_plan_run_host(reattn_plan* p, const float* q_host, float* out_host) {
    const size_t bytes = p->P.n_q * p->P.n_head * p->cache->d * sizeof(float);
    reattn_ctx* ctx = p->ctx;
    if (p->append)
        return set_err(ctx, REATTN_EINVAL, "plan: append mode takes the step's K/V too (reattn_plan_step_host)");
    int rc = check_plan(p);
    if (rc) return rc;
    const void* key[4] = {q_host, nullptr, nullptr, out_host};
    const bool io_ready = p->io_exec && !p->io_append && std::equal(key, key + 4, p->io_key);
    if (io_ready || (zero_copy_enabled() && host_pinned(q_host) && host_pinned(out_host))) {
        if ((rc = ensure_io_graph(p, q_host, nullptr, nullptr, out_host))) return rc;
        CU(ctx, cudaGraphLaunch(p->io_exec, ctx->stream));
        CU(ctx, cudaStreamSynchronize(ctx->stream));
        return REATTN_OK;
    }
    CU(ctx, cudaMemcpyAsync(p->q, q_host, bytes, cudaMemcpyHostToDevice, ctx->stream));
    CU(ctx, cudaGraphLaunch(p->exec, ctx->stream));
    CU(ctx, cudaMemcpyAsync(out_host, p->out, bytes, cudaMemcpyDeviceToHost, ctx->stream));
    CU(ctx, cudaStreamSynchronize(ctx->stream));
    return REATTN_OK;
}

int reattn_plan_stats(reattn_plan* p, reattn_step_stats* st) {
    reattn_ctx* ctx = p->ctx;
    refresh_geometry(p->P, p->cache);
    ScopeHeader h;
    CU(ctx, cudaMemcpyAsync(&h, p->P.hdr, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
    CU(ctx, cudaStreamSynchronize(ctx->stream));
    return finish_step_stats(ctx, p->P, h, st, nullptr);
}

int reattn_plan_result(reattn_plan* p, reattn_step_stats* st, uint64_t* span_b_host,
                       uint64_t* span_e_host, double* entropy_host) {
    reattn_ctx* ctx = p->ctx;
    refresh_geometry(p->P, p->cache);
    ScopeHeader h;
    CU(ctx, cudaMemcpyAsync(&h, p->P.hdr, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
    CU(ctx, cudaStreamSynchronize(ctx->stream));
    int rc = finish_step_stats(ctx, p->P, h, st, entropy_host);
    if (rc) return rc;
    if (span_b_host && h.n_spans) {
        std::vector<uint32_t> b(h.n_spans), e(h.n_spans);
        CU(ctx, cudaMemcpy(b.data(), p->P.span_b, h.n_spans * 4, cudaMemcpyDeviceToHost));
        CU(ctx, cudaMemcpy(e.data(), p->P.span_e, h.n_spans * 4, cudaMemcpyDeviceToHost));
        for (uint32_t i = 0; i < h.n_spans; ++i) {
            span_b_host[i] = b[i];
            span_e_host[i] = e[i];
        }
    }
    return REATTN_OK;
}

// Decode loops that run many plans per token (one per layer) read every plan's result after
// one synchronisation: stage enqueues the copies, staged_result reads them after the caller
// synchronised the context stream.
namespace {
size_t staged_bytes(const StepPlan& P) {
    const uint64_t kp = std::max<uint64_t>(1, P.cfg.k_prime);
    return sizeof(ScopeHeader) + P.n_q * P.n_head * sizeof(double) + 2 * kp * sizeof(uint32_t);
}
}  // namespace

// one zero-copy kernel writes the header, entropies and spans into the pinned staging area
int plan_stage_result_on(reattn_plan* p, cudaStream_t s) {
    reattn_ctx* ctx = p->ctx;
    const StepPlan& P = p->P;
    if (!p->staged) CU(ctx, cudaHostAlloc(&p->staged, staged_bytes(P), cudaHostAllocDefault));
    uint8_t* h = (uint8_t*)p->staged;
    const uint64_t kp = std::max<uint64_t>(1, P.cfg.k_prime);
    const size_t ent = P.n_q * P.n_head * sizeof(double);
    const float* src[4] = {(const float*)P.hdr, (const float*)P.entropy, (const float*)P.span_b,
                           (const float*)P.span_e};
    float* dst[4] = {(float*)h, (float*)(h + sizeof(ScopeHeader)), (float*)(h + sizeof(ScopeHeader) + ent),
                     (float*)(h + sizeof(ScopeHeader) + ent + kp * 4)};
    const uint64_t n[4] = {sizeof(ScopeHeader) / 4, ent / 4, kp, kp};
    CU(ctx, launch_host_io(src, dst, n, 4, s));
    p->staged_pending = true;
    return REATTN_OK;
}

int reattn_plan_stage_result(reattn_plan* p) { return plan_stage_result_on(p, p->ctx->stream); }

int reattn_plan_staged_result(reattn_plan* p, reattn_step_stats* st, uint64_t* span_b_host,
                              uint64_t* span_e_host, double* entropy_host) {
    reattn_ctx* ctx = p->ctx;
    if (!p->staged_pending)
        return set_err(ctx, REATTN_ELOGIC, "plan: no staged result (reattn_plan_stage_result first)");
    p->staged_pending = false;
    refresh_geometry(p->P, p->cache);
    const StepPlan& P = p->P;
    const uint8_t* h = (const uint8_t*)p->staged;
    ScopeHeader hdr;
    std::memcpy(&hdr, h, sizeof(hdr));
    const double* ent = (const double*)(h + sizeof(ScopeHeader));
    const uint64_t kp = std::max<uint64_t>(1, P.cfg.k_prime);
    const uint32_t* b = (const uint32_t*)(h + sizeof(ScopeHeader) + P.n_q * P.n_head * sizeof(double));
    int rc = stats_from_host(ctx, P, hdr, ent, st, entropy_host);
    if (rc) return rc;
    if (span_b_host)
        for (uint32_t i = 0; i < std::min<uint64_t>(hdr.n_spans, kp); ++i) {
            span_b_host[i] = b[i];
            span_e_host[i] = b[kp + i];
        }
    return REATTN_OK;
}

int reattn_plan_info(const reattn_plan* p, uint64_t* kernels, uint64_t* scan_bytes,
                     uint64_t* scope_bytes) {
    const uint64_t esz = p->cache->dtype == REATTN_BF16 ? 2 : 4;
    if (kernels) *kernels = p->P.kernels;
    const uint64_t middle = p->P.dynamic ? p->cache->local_start() - p->cache->global_end() : p->P.middle;
    if (scan_bytes) *scan_bytes = p->P.select ? p->P.n_kv * middle * p->P.d * esz : 0;
    if (scope_bytes) *scope_bytes = p->P.n_kv * (uint64_t)p->P.L_upper * 2 * p->P.d * esz;
    return REATTN_OK;
}

int reattn_synth_uniform(reattn_ctx* ctx, void* dst, uint64_t n, int dtype, uint64_t seed,
                         uint64_t offset) {
    if (n == 0) return REATTN_OK;
    CU(ctx, launch_synth_uniform(dst, dtype, n, seed, offset, ctx->stream));
    CU(ctx, cudaStreamSynchronize(ctx->stream));
    return REATTN_OK;
}


// ---- batched decode: one graph over n_seq independent sequences (own caches) ---------------
// The decode scan is HBM-bound and sequences share no bytes, so batching cannot save
// traffic; it hides latency instead.  Pipelined (bf16 decode): the scans run back to back on
// num_sms - R SMs while sequence b's attention runs on the R spare SMs beside scan b+1 (side
// stream, event per sequence); only the last sequence's attention runs on the whole GPU.
struct reattn_batch_plan {
    reattn_ctx* ctx = nullptr;
    const reattn_rope* rope = nullptr;
    std::vector<const reattn_cache*> caches;
    std::vector<StepPlan> P;
    uint64_t n_head = 0, d = 0;
    void* mem = nullptr;
    float* q = nullptr;
    float* out = nullptr;
    bool pipelined = false;
    int side_sms = 0;
    cudaStream_t side = nullptr;
    std::vector<cudaEvent_t> ev;
    cudaEvent_t ev_done = nullptr;
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    uint64_t kernels = 0;
    cudaGraphExec_t io_exec = nullptr;  // zero-copy run_host for io_key's pinned buffers
    const void* io_key[2] = {nullptr, nullptr};
    ~reattn_batch_plan() {
        if (io_exec) cudaGraphExecDestroy(io_exec);
        if (exec) cudaGraphExecDestroy(exec);
        if (graph) cudaGraphDestroy(graph);
        for (auto e : ev) cudaEventDestroy(e);
        if (ev_done) cudaEventDestroy(ev_done);
        if (side) cudaStreamDestroy(side);
        if (mem) cudaFree(mem);
    }
};

int reattn_batch_plan_create(reattn_ctx* ctx, const reattn_cache* const* caches, uint32_t n_seq,
                             const reattn_rope* rope, uint64_t n_head,
                             const reattn_selection_config* cfg, int mode,
                             reattn_batch_plan** out) {
    *out = nullptr;
    if (n_seq == 0 || !caches) return set_err(ctx, REATTN_EINVAL, "batch plan: no sequences");
    auto bp = std::make_unique<reattn_batch_plan>();
    bp->ctx = ctx;
    bp->rope = rope;
    bp->caches.assign(caches, caches + n_seq);
    bp->P.resize(n_seq);
    bp->n_head = n_head;
    bp->d = caches[0]->d;
    bool pipe = n_seq > 1;
    double t_scan = 0.0, t_attn = 0.0;
    for (uint32_t b = 0; b < n_seq; ++b) {
        if (caches[b]->d != bp->d)
            return set_err(ctx, REATTN_EINVAL, "batch plan: every cache needs the same d_head");
        int rc = plan_step(ctx, caches[b], rope, 1, n_head, cfg, mode, bp->P[b], nullptr, nullptr);
        if (rc) return rc;
        StepPlan& P = bp->P[b];
        pipe = pipe && P.select && P.scan.fast && P.d == 128 && caches[b]->dtype == kBF16 &&
               P.group <= 8;
        t_scan = std::max(t_scan, (double)P.middle * P.n_kv * P.d * 2 / 5.8e6);
        t_attn = std::max(t_attn, (double)((P.L_upper + 31) / 32) * P.n_kv * 0.8);  // us x SM
    }
    if (pipe) {  // the pipeline replaces the per-sequence local-window fork
        for (auto& P : bp->P) {
            P.fork = false;
            P.scan.grid_sms = 0;
        }
        const uint64_t n_kv = bp->P[0].n_kv;
        int m = 1;
        while (m < 4 && (int)(m * n_kv) * 8 <= ctx->num_sms && t_attn / (m * n_kv) > 0.8 * t_scan) ++m;
        bp->side_sms = (int)(m * n_kv);
        for (auto& P : bp->P) P.scan.grid_sms = ctx->num_sms - bp->side_sms;
    }
    bp->pipelined = pipe;
    const uint64_t row = n_head * bp->d;
    Carver sizer{nullptr, 0, 0};
    sizer.take<float>(n_seq * row);
    sizer.take<float>(n_seq * row);
    for (uint32_t b = 0; b < n_seq; ++b) carve_step(bp->P[b], caches[b], rope, sizer);
    cudaError_t e = cudaMalloc(&bp->mem, sizer.off + 256);
    if (e == cudaSuccess) e = cudaMemset(bp->mem, 0, sizer.off + 256);
    if (e == cudaSuccess) e = cudaDeviceSynchronize();  // zeroed before any stream replays
    if (e != cudaSuccess)
        return set_err(ctx, REATTN_ECUDA, std::string("batch plan allocation: ") + cudaGetErrorString(e));
    Carver c{(uint8_t*)bp->mem, 0, sizer.off + 256};
    bp->q = c.take<float>(n_seq * row);
    bp->out = c.take<float>(n_seq * row);
    for (uint32_t b = 0; b < n_seq; ++b) carve_step(bp->P[b], caches[b], rope, c);
    CU(ctx, cudaStreamCreateWithFlags(&bp->side, cudaStreamNonBlocking));
    bp->ev.resize(n_seq, nullptr);
    for (auto& ev : bp->ev) CU(ctx, cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    CU(ctx, cudaEventCreateWithFlags(&bp->ev_done, cudaEventDisableTiming));
    // capture
    cudaStream_t cs;
    CU(ctx, cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    CU(ctx, cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
    int rc = REATTN_OK;
    for (uint32_t b = 0; b < n_seq && !rc; ++b) {
        StepPlan& P = bp->P[b];
        const float* qb = bp->q + b * row;
        float* ob = bp->out + b * row;
        if (!pipe) {
            rc = enqueue_step(ctx, P, caches[b], rope, qb, ob, cs, false);
            bp->kernels += P.kernels;
            continue;
        }
        rc = enqueue_select_part(ctx, P, caches[b], rope, qb, ob, cs, false);
        if (rc) break;
        if (b + 1 < n_seq) {  // this sequence's attention beside the next scan
            if (cudaEventRecord(bp->ev[b], cs) != cudaSuccess ||
                cudaStreamWaitEvent(bp->side, bp->ev[b], 0) != cudaSuccess) {
                rc = set_err(ctx, REATTN_ECUDA, "batch plan: event capture failed");
                break;
            }
            rc = enqueue_attn_part(ctx, P, caches[b], rope, qb, ob, bp->side, false, bp->side_sms);
        } else {
            rc = enqueue_attn_part(ctx, P, caches[b], rope, qb, ob, cs, false, 0);
        }
        bp->kernels += P.kernels;
    }
    if (!rc && pipe) {
        if (cudaEventRecord(bp->ev_done, bp->side) != cudaSuccess ||
            cudaStreamWaitEvent(cs, bp->ev_done, 0) != cudaSuccess)
            rc = set_err(ctx, REATTN_ECUDA, "batch plan: event capture failed");
    }
    cudaGraph_t g = nullptr;
    const cudaError_t ce = cudaStreamEndCapture(cs, &g);
    cudaStreamDestroy(cs);
    if (rc || ce != cudaSuccess) {
        if (g) cudaGraphDestroy(g);
        return rc ? rc : set_err(ctx, REATTN_ECUDA, std::string("graph capture: ") + cudaGetErrorString(ce));
    }
    bp->graph = g;
    e = cudaGraphInstantiate(&bp->exec, g, 0);
    if (e != cudaSuccess)
        return set_err(ctx, REATTN_ECUDA, std::string("graph instantiate: ") + cudaGetErrorString(e));
    *out = bp.release();
    return REATTN_OK;
}

void reattn_batch_plan_destroy(reattn_batch_plan* p) {
    if (!p) return;
    cudaDeviceSynchronize();
    delete p;
}

float* reattn_batch_plan_q(const reattn_batch_plan* p) { return p->q; }
float* reattn_batch_plan_out(const reattn_batch_plan* p) { return p->out; }

int reattn_batch_plan_launch(reattn_batch_plan* p) {
    CU(p->ctx, cudaGraphLaunch(p->exec, p->ctx->stream));
    return REATTN_OK;
}

int reattn_batch_plan_run_host(reattn_batch_plan* p, const float* q_host, float* out_host) {
    const size_t bytes = p->P.size() * p->n_head * p->d * sizeof(float);
    reattn_ctx* ctx = p->ctx;
    const bool io_ready = p->io_exec && p->io_key[0] == q_host && p->io_key[1] == out_host;
    if (io_ready || (zero_copy_enabled() && host_pinned(q_host) && host_pinned(out_host))) {
        if (!io_ready) {
            if (p->io_exec) cudaGraphExecDestroy(p->io_exec);
            const float* src[1] = {q_host};
            float* dst[1] = {p->q};
            const uint64_t n[1] = {bytes / sizeof(float)};
            int rc = build_io_exec(ctx, p->graph, src, dst, n, 1, p->out, out_host, n[0], &p->io_exec);
            if (rc) return rc;
            p->io_key[0] = q_host;
            p->io_key[1] = out_host;
        }
        CU(ctx, cudaGraphLaunch(p->io_exec, ctx->stream));
        CU(ctx, cudaStreamSynchronize(ctx->stream));
        return REATTN_OK;
    }
    CU(ctx, cudaMemcpyAsync(p->q, q_host, bytes, cudaMemcpyHostToDevice, ctx->stream));
    CU(ctx, cudaGraphLaunch(p->exec, ctx->stream));
    CU(ctx, cudaMemcpyAsync(out_host, p->out, bytes, cudaMemcpyDeviceToHost, ctx->stream));
    CU(ctx, cudaStreamSynchronize(ctx->stream));
    return REATTN_OK;
}

int reattn_batch_plan_stats(reattn_batch_plan* p, uint32_t seq, reattn_step_stats* st) {
    if (seq >= p->P.size()) return set_err(p->ctx, REATTN_ERANGE, "batch plan: sequence out of range");
    reattn_ctx* ctx = p->ctx;
    ScopeHeader h;
    CU(ctx, cudaMemcpyAsync(&h, p->P[seq].hdr, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
    CU(ctx, cudaStreamSynchronize(ctx->stream));
    return finish_step_stats(ctx, p->P[seq], h, st, nullptr);
}

int reattn_batch_plan_info(const reattn_batch_plan* p, uint64_t* kernels, uint64_t* scan_bytes,
                           int* side_sms) {
    uint64_t bytes = 0;
    for (size_t b = 0; b < p->P.size(); ++b) {
        const uint64_t esz = p->caches[b]->dtype == REATTN_BF16 ? 2 : 4;
        if (p->P[b].select) bytes += p->P[b].n_kv * p->P[b].middle * p->P[b].d * esz;
    }
    if (kernels) *kernels = p->kernels;
    if (scan_bytes) *scan_bytes = bytes;
    if (side_sms) *side_sms = p->pipelined ? p->side_sms : 0;
    return REATTN_OK;
}

}  // extern "C"
