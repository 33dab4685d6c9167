// C-ABI: sequence-sharded decode plans (include/reattn_cuda.h, "sequence-sharded decode").
#include <nccl.h>

#include "capi_internal.h"

using namespace reattn_impl;
using namespace reattn_capi;

struct reattn_shard_plan {
    reattn_ctx* ctx = nullptr;
    const reattn_cache* cache = nullptr;  // local: [global | shard | local]
    const reattn_rope* rope = nullptr;
    reattn_selection_config cfg{};
    uint64_t n_head = 0, n_kv = 0, d = 0, group = 0;
    // global geometry
    uint64_t g_end = 0, l_start = 0, total = 0, middle = 0, local_len = 0, window = 0;
    int world = 1, rank = 0;
    uint64_t shard_begin[65] = {};
    uint64_t shard_len = 0;
    uint64_t kk = 0;
    uint32_t L_upper = 0;
    ScanPlan scan;
    bool do_scan = false;
    // device buffers
    void* mem = nullptr;
    float* q = nullptr;
    float* out = nullptr;
    uint8_t* cand_send = nullptr;
    uint8_t* cand_recv = nullptr;
    size_t cand_bytes = 0;
    void* scan_ws = nullptr;
    uint32_t* winners = nullptr;
    uint32_t* span_b = nullptr;
    uint32_t* span_e = nullptr;
    uint32_t* scope_global = nullptr;
    uint32_t* scope_local = nullptr;
    ScopeHeader* hdr = nullptr;
    uint32_t* ranges = nullptr;   // ShardRanges of this rank (written by the select)
    void* bulk_ws = nullptr;      // decode attention workspace (tickets + per-part partials)
    double* part_send = nullptr;  // this rank's merged partial rows [n_head]
    double* part_recv = nullptr;  // all ranks' [world][n_head]
    size_t part_bytes = 0;
    double* entropy = nullptr;
    // the whole step (NCCL all-gathers included) captured by reattn_shard_capture
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
};

// An NCCL communicator over the ranks of one sharded decode (one process per GPU).  The
// library issues the two all-gathers of a step itself (reattn_shard_step), so a C++ host
// drives the whole sharded path through this ABI with no Python on it.
struct reattn_comm {
    ncclComm_t comm = nullptr;
    int world = 1, rank = 0, device = 0;
};

namespace {

void shard_bounds(uint64_t M, uint64_t m, int world, uint64_t* begin) {
    for (int r = 0; r < world; ++r) begin[r] = ((uint64_t)r * M / (uint64_t)world) / m * m;
    begin[world] = M;
    for (int r = world - 1; r >= 0; --r) begin[r] = std::min(begin[r], begin[r + 1]);
}

AttnArgs shard_attn_args(const reattn_shard_plan* p) {
    AttnArgs a;
    std::memset(&a, 0, sizeof(a));
    a.q = p->q;
    a.q_row_stride = p->n_head * p->d;
    a.n_q = 1;
    a.n_head = (int)p->n_head;
    a.n_kv = (int)p->n_kv;
    a.group = (int)p->group;
    a.d = (int)p->d;
    a.dv = (int)p->d;
    a.k_base = p->cache->keys;
    a.v_base = p->cache->values;
    a.dtype = p->cache->dtype;
    a.head_stride = p->cache->capacity;
    a.src = p->scope_local;
    a.hdr = p->hdr;
    a.rope_cos = p->rope->cos_d;
    a.rope_sin = p->rope->sin_d;
    a.causal = 1;
    a.boundary_is_tail = 1;
    a.part = p->part_send;
    a.out = p->out;
    a.entropy = p->entropy;
    return a;
}

void carve(reattn_shard_plan* p, Carver& c) {
    const uint64_t hd = p->n_head * p->d;
    p->q = c.take<float>(hd);
    p->out = c.take<float>(hd);
    p->cand_bytes = align_up(p->n_kv * p->cfg.k * 8, 256);
    p->cand_send = c.take<uint8_t>(p->cand_bytes);
    p->cand_recv = c.take<uint8_t>(p->cand_bytes * p->world);
    p->scan_ws = c.take<uint8_t>(p->scan.ws_bytes);
    const uint64_t kp = std::max<uint64_t>(1, p->cfg.k_prime);
    p->winners = c.take<uint32_t>(kp);
    p->span_b = c.take<uint32_t>(kp);
    p->span_e = c.take<uint32_t>(kp);
    p->scope_global = c.take<uint32_t>(p->L_upper);
    p->scope_local = c.take<uint32_t>(p->L_upper);
    p->hdr = c.take<ScopeHeader>(1);
    p->ranges = c.take<uint32_t>(sizeof(ShardRanges) / 4);
    AttnArgs a = shard_attn_args(p);
    p->bulk_ws = c.take<uint8_t>(decode_bulk_workspace(a, p->ctx->num_sms));
    p->part_bytes = align_up(p->n_head * kDecodePartBytes, 256);
    p->part_send = c.take<double>(p->part_bytes / 8);
    p->part_recv = c.take<double>(p->part_bytes / 8 * p->world);
    p->entropy = c.take<double>(p->n_head);
}

}  // namespace

extern "C" {

int reattn_shard_range(uint64_t M, uint64_t m, int world, int rank, uint64_t* begin,
                       uint64_t* len) {
    if (world < 1 || world > 64 || rank < 0 || rank >= world || m == 0) return REATTN_EINVAL;
    uint64_t b[65];
    shard_bounds(M, m, world, b);
    *begin = b[rank];
    *len = b[rank + 1] - b[rank];
    return REATTN_OK;
}

int reattn_shard_plan_create(reattn_ctx* ctx, const reattn_cache* cache, const reattn_rope* rope,
                             uint64_t n_head, const reattn_selection_config* cfg,
                             uint64_t global_total, int world, int rank,
                             reattn_shard_plan** out) {
    *out = nullptr;
    if (world < 1 || world > 64 || rank < 0 || rank >= world)
        return set_err(ctx, REATTN_EINVAL, "shard plan: world must be 1..64 and rank < world");
    if (n_head % cache->n_kv != 0)
        return set_err(ctx, REATTN_EINVAL, "attend_step: n_head must be a multiple of kv heads");
    if (rope->head_dim != cache->d || cache->d != 128 || cache->dtype != REATTN_BF16)
        return set_err(ctx, REATTN_EINVAL, "shard plan: decode path needs d_head == 128 and a bf16 cache");
    if (cfg->k == 0 || cfg->k > 8 || cfg->span_m == 0 || cfg->k_prime == 0)
        return set_err(ctx, REATTN_EINVAL, "shard plan: needs 1 <= k <= 8, span_m >= 1, k' >= 1");
    auto* p = new reattn_shard_plan();
    p->ctx = ctx;
    p->cache = cache;
    p->rope = rope;
    p->cfg = *cfg;
    p->n_head = n_head;
    p->n_kv = cache->n_kv;
    p->d = cache->d;
    p->group = n_head / cache->n_kv;
    p->world = world;
    p->rank = rank;
    // global geometry (kv_cache.hpp:65-67)
    p->total = global_total;
    p->g_end = std::min(global_total, cfg->l_global);
    p->l_start = global_total - std::min(global_total - p->g_end, cfg->l_local);
    p->middle = p->l_start - p->g_end;
    p->local_len = global_total - p->l_start;
    p->window = rope->max_position;
    if (p->middle == 0) {
        delete p;
        return set_err(ctx, REATTN_EINVAL, "shard plan: the global middle is empty (use a plan)");
    }
    shard_bounds(p->middle, cfg->span_m, world, p->shard_begin);
    p->shard_len = p->shard_begin[rank + 1] - p->shard_begin[rank];
    // the local cache must hold exactly [global | shard | local]
    if (cache->total != p->g_end + p->shard_len + p->local_len ||
        cache->global_end() != p->g_end || cache->local_start() != p->g_end + p->shard_len) {
        delete p;
        return set_err(ctx, REATTN_EINVAL,
                       "shard plan: local cache must hold [global | this rank's shard | local]");
    }
    p->kk = std::min<uint64_t>(cfg->k, p->middle);
    if (p->n_kv * p->kk > kSmallSelectMax) {
        delete p;
        return set_err(ctx, REATTN_EINVAL, "shard plan: n_kv * k must be <= 32 (decode)");
    }
    const uint64_t max_winners = std::min<uint64_t>(cfg->k_prime, p->n_kv * p->kk);
    const uint64_t sel_rows = std::min<uint64_t>(p->middle, max_winners * cfg->span_m);
    p->L_upper = (uint32_t)std::min<uint64_t>(p->window, p->g_end + sel_rows + p->local_len);
    // local scan over this rank's shard (the local cache's middle)
    ScanArgs& a = p->scan.a;
    a.q = nullptr;
    a.n_q = 1;
    a.n_heads = (int)n_head;
    a.n_kv = (int)p->n_kv;
    a.d = (int)p->d;
    a.keys = cache->keys;
    a.dtype = cache->dtype;
    a.head_stride = cache->capacity;
    a.row0 = p->g_end;
    a.count = (uint32_t)p->shard_len;
    a.k = (int)cfg->k;
    a.lanes = ctx->lanes;
    p->do_scan = p->shard_len > 0;
    if (p->do_scan) {
        int rc = plan_scan(ctx, p->scan);
        if (rc) {
            delete p;
            return rc;
        }
    }
    Carver sizer{nullptr, 0, 0};
    carve(p, sizer);
    cudaError_t e = cudaMalloc(&p->mem, sizer.off + 256);
    if (e == cudaSuccess) e = cudaMemset(p->mem, 0, sizer.off + 256);
    if (e == cudaSuccess) e = cudaDeviceSynchronize();  // zeroed before any stream replays
    if (e != cudaSuccess) {
        delete p;
        return set_err(ctx, REATTN_ECUDA, std::string("shard plan allocation: ") + cudaGetErrorString(e));
    }
    Carver c{(uint8_t*)p->mem, 0, sizer.off + 256};
    carve(p, c);
    *out = p;
    return REATTN_OK;
}

void reattn_shard_plan_destroy(reattn_shard_plan* p) {
    if (!p) return;
    cudaDeviceSynchronize();
    if (p->exec) cudaGraphExecDestroy(p->exec);
    if (p->graph) cudaGraphDestroy(p->graph);
    cudaFree(p->mem);
    delete p;
}

float* reattn_shard_plan_q(const reattn_shard_plan* p) { return p->q; }
float* reattn_shard_plan_out(const reattn_shard_plan* p) { return p->out; }

int reattn_shard_buffers(const reattn_shard_plan* p, void** cs, void** cr, uint64_t* cb, void** ps,
                         void** pr, uint64_t* pb) {
    if (cs) *cs = p->cand_send;
    if (cr) *cr = p->cand_recv;
    if (cb) *cb = p->cand_bytes;
    if (ps) *ps = p->part_send;
    if (pr) *pr = p->part_recv;
    if (pb) *pb = p->part_bytes;
    return REATTN_OK;
}

int reattn_shard_scan(reattn_shard_plan* p) {
    reattn_ctx* ctx = p->ctx;
    const size_t n = p->n_kv * p->cfg.k;
    // empty slots stay kNoIndex (the generic path writes only the valid prefix)
    CU(ctx, cudaMemsetAsync(p->cand_send, 0xFF, n * sizeof(uint32_t), ctx->stream));
    if (!p->do_scan) return REATTN_OK;
    p->scan.a.q = p->q;
    p->scan.a.idx_out = (uint32_t*)p->cand_send;
    p->scan.a.score_out = (float*)(p->cand_send + n * sizeof(uint32_t));
    p->scan.a.fuse_select = 0;
    return enqueue_scan(ctx, p->scan, p->scan_ws, ctx->stream, false);
}

int reattn_shard_select(reattn_shard_plan* p) {
    reattn_ctx* ctx = p->ctx;
    ShardSelectArgs s;
    std::memset(&s, 0, sizeof(s));
    const size_t n = p->n_kv * p->cfg.k;
    s.cand_idx = (const uint32_t*)p->cand_recv;
    s.cand_score = (const float*)(p->cand_recv + n * sizeof(uint32_t));
    s.src_stride = p->cand_bytes / 4;
    s.n_src = p->world;
    s.n_lists = (int)p->n_kv;
    s.k = (int)p->cfg.k;
    s.kk = (int)p->kk;
    for (int r = 0; r < p->world; ++r) s.src_offset[r] = (uint32_t)p->shard_begin[r];
    SmallSelectIO& io = s.sel;
    io.k_prime = (uint32_t)p->cfg.k_prime;
    io.span_m = (uint32_t)p->cfg.span_m;
    io.middle_len = (uint32_t)p->middle;
    io.span_mode = p->cfg.span_mode;
    io.g_end = (uint32_t)p->g_end;
    io.l_start = (uint32_t)p->l_start;
    io.total = (uint32_t)p->total;
    io.window = (uint32_t)p->window;
    io.n_q = 1;
    io.winners = p->winners;
    io.span_b = p->span_b;
    io.span_e = p->span_e;
    io.scope_src = p->scope_global;
    io.hdr = p->hdr;
    io.table_local = 1;  // the translation to local rows reads the whole global table
    s.rank = p->rank;
    s.world = p->world;
    s.ranges = p->ranges;
    s.shard_begin = (uint32_t)p->shard_begin[p->rank];
    s.shard_len = (uint32_t)p->shard_len;
    s.local_src = p->scope_local;
    CU(ctx, launch_shard_merge_select(s, ctx->stream));
    return REATTN_OK;
}

// this rank's scope rows (ShardRanges) -> one merged partial row per q head in part_send
int reattn_shard_attend(reattn_shard_plan* p) {
    AttnArgs a = shard_attn_args(p);
    CU(p->ctx, launch_attend_decode_ranges(a, p->bulk_ws, p->ctx->num_sms, p->ranges,
                                           (uint8_t*)p->part_send, p->ctx->stream));
    return REATTN_OK;
}

// the all-gathered [world][n_head] partial rows -> output + entropy (fixed rank order)
int reattn_shard_combine(reattn_shard_plan* p) {
    AttnArgs a = shard_attn_args(p);
    CU(p->ctx, launch_decode_combine_sources(a, (const uint8_t*)p->part_recv, p->world,
                                             p->part_bytes, p->ctx->stream));
    return REATTN_OK;
}

int reattn_shard_stats(reattn_shard_plan* p, reattn_step_stats* st, uint64_t* sb, uint64_t* se) {
    reattn_ctx* ctx = p->ctx;
    ScopeHeader h;
    CU(ctx, cudaMemcpyAsync(&h, p->hdr, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
    CU(ctx, cudaStreamSynchronize(ctx->stream));
    int rc = status_from_scope(ctx, h.error);
    if (rc) return rc;
    std::vector<double> ent(p->n_head);
    CU(ctx, cudaMemcpy(ent.data(), p->entropy, ent.size() * 8, cudaMemcpyDeviceToHost));
    if (st) {
        std::memset(st, 0, sizeof(*st));
        for (double e : ent) {
            st->entropy_max = std::max(st->entropy_max, e);
            st->entropy_sum += e;
        }
        st->entropy_rows = p->n_head;
        st->scope_len = h.L;
        st->max_position_used = h.L ? h.L - 1 : 0;
        st->n_spans = h.n_spans;
        st->coverage = h.coverage;
        st->coverage_total = h.coverage == p->middle ? 1 : 0;
    }
    if (sb && h.n_spans) {
        std::vector<uint32_t> b(h.n_spans), e(h.n_spans);
        CU(ctx, cudaMemcpy(b.data(), p->span_b, h.n_spans * 4, cudaMemcpyDeviceToHost));
        CU(ctx, cudaMemcpy(e.data(), p->span_e, h.n_spans * 4, cudaMemcpyDeviceToHost));
        for (uint32_t i = 0; i < h.n_spans; ++i) {
            sb[i] = b[i];
            se[i] = e[i];
        }
    }
    return REATTN_OK;
}

// ---- NCCL host path ---------------------------------------------------------------------
int reattn_comm_unique_id(uint8_t* id_out) {
    static_assert(sizeof(ncclUniqueId) == REATTN_COMM_ID_BYTES, "NCCL unique id size");
    ncclUniqueId id;
    if (ncclGetUniqueId(&id) != ncclSuccess) return REATTN_ECUDA;
    std::memcpy(id_out, &id, sizeof(id));
    return REATTN_OK;
}

int reattn_comm_create(reattn_ctx* ctx, int world, int rank, const uint8_t* id_in,
                       reattn_comm** out) {
    *out = nullptr;
    if (world < 1 || world > 64 || rank < 0 || rank >= world)
        return set_err(ctx, REATTN_EINVAL, "comm: world must be 1..64 and rank < world");
    ncclUniqueId id;
    std::memcpy(&id, id_in, sizeof(id));
    CU(ctx, cudaSetDevice(ctx->device));
    auto* c = new reattn_comm();
    c->world = world;
    c->rank = rank;
    c->device = ctx->device;
    const ncclResult_t r = ncclCommInitRank(&c->comm, world, id, rank);
    if (r != ncclSuccess) {
        delete c;
        return set_err(ctx, REATTN_ECUDA, std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
    }
    *out = c;
    return REATTN_OK;
}

void reattn_comm_destroy(reattn_comm* c) {
    if (!c) return;
    if (c->comm) ncclCommDestroy(c->comm);
    delete c;
}

namespace {
int nccl_gather(reattn_ctx* ctx, const void* send, void* recv, size_t bytes, reattn_comm* c) {
    const ncclResult_t r = ncclAllGather(send, recv, bytes, ncclUint8, c->comm, ctx->stream);
    if (r != ncclSuccess)
        return set_err(ctx, REATTN_ECUDA, std::string("ncclAllGather: ") + ncclGetErrorString(r));
    return REATTN_OK;
}

int enqueue_shard_step(reattn_shard_plan* p, reattn_comm* c) {
    if (c->world != p->world || c->rank != p->rank)
        return set_err(p->ctx, REATTN_EINVAL, "shard step: communicator world/rank != plan's");
    int rc = reattn_shard_scan(p);
    if (!rc) rc = nccl_gather(p->ctx, p->cand_send, p->cand_recv, p->cand_bytes, c);
    if (!rc) rc = reattn_shard_select(p);
    if (!rc) rc = reattn_shard_attend(p);
    if (!rc) rc = nccl_gather(p->ctx, p->part_send, p->part_recv, p->part_bytes, c);
    if (!rc) rc = reattn_shard_combine(p);
    return rc;
}
}  // namespace

int reattn_shard_step(reattn_shard_plan* p, reattn_comm* c) {
    if (p->exec) {  // a captured step replays as one graph launch
        CU(p->ctx, cudaGraphLaunch(p->exec, p->ctx->stream));
        return REATTN_OK;
    }
    return enqueue_shard_step(p, c);
}

int reattn_shard_capture(reattn_shard_plan* p, reattn_comm* c) {
    reattn_ctx* ctx = p->ctx;
    // one eager step first: NCCL connection set-up and kernel attributes happen outside capture
    int rc = enqueue_shard_step(p, c);
    if (rc) return rc;
    CU(ctx, cudaStreamSynchronize(ctx->stream));
    if (p->exec) cudaGraphExecDestroy(p->exec);
    if (p->graph) cudaGraphDestroy(p->graph);
    p->exec = nullptr;
    p->graph = nullptr;
    CU(ctx, cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
    rc = enqueue_shard_step(p, c);
    cudaGraph_t g = nullptr;
    const cudaError_t ce = cudaStreamEndCapture(ctx->stream, &g);
    if (rc || ce != cudaSuccess) {
        if (g) cudaGraphDestroy(g);
        return rc ? rc : set_err(ctx, REATTN_ECUDA, std::string("shard capture: ") + cudaGetErrorString(ce));
    }
    p->graph = g;
    CU(ctx, cudaGraphInstantiate(&p->exec, g, 0));
    return REATTN_OK;
}

int reattn_shard_run_host(reattn_shard_plan* p, reattn_comm* c, const float* q_host,
                          float* out_host) {
    reattn_ctx* ctx = p->ctx;
    const size_t bytes = p->n_head * p->d * sizeof(float);
    CU(ctx, cudaMemcpyAsync(p->q, q_host, bytes, cudaMemcpyHostToDevice, ctx->stream));
    int rc = reattn_shard_step(p, c);
    if (rc) return rc;
    CU(ctx, cudaMemcpyAsync(out_host, p->out, bytes, cudaMemcpyDeviceToHost, ctx->stream));
    CU(ctx, cudaStreamSynchronize(ctx->stream));
    return REATTN_OK;
}

}  // extern "C"
