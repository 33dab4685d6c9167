/*
 * reattn_cuda.h — the C-ABI boundary of the B200-native ReAttention hot path.
 *
 * Plain pointers and sizes only; no C++ or torch types cross this boundary.  Every
 * function returns a reattn_status; on failure reattn_last_error(ctx) holds the message,
 * worded exactly as the reference's exception (so the C++ shim in include/reattn/ can
 * rethrow the same type and text).
 *
 * Each entry point replaces one reference function of
 * /root/reference/proj/include/reattn/ (cited per declaration).  The reference has no FFI
 * of its own: its boundary is the header-only C++ API, which the headers under
 * include/reattn/ re-create on top of this ABI.
 *
 * Device pointers ("_dev") are CUDA global memory of the context's device; all work is
 * enqueued on the context's stream.  Functions documented "synchronous" return after the
 * stream drained.  The whole hot path (scan -> vote/spans/scope -> attention) runs
 * without host round trips and can be captured in a CUDA graph (reattn_plan_*).
 */
#ifndef REATTN_CUDA_H
#define REATTN_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define REATTN_ABI_VERSION 1

typedef struct reattn_ctx reattn_ctx;
typedef struct reattn_cache reattn_cache;
typedef struct reattn_rope reattn_rope;
typedef struct reattn_plan reattn_plan;

typedef enum {
    REATTN_OK = 0,
    REATTN_EINVAL = 1,   /* std::invalid_argument */
    REATTN_ERANGE = 2,   /* std::out_of_range */
    REATTN_ELOGIC = 3,   /* std::logic_error */
    REATTN_ECUDA = 4,    /* CUDA runtime / device failure */
    REATTN_ERUNTIME = 5  /* std::runtime_error */
} reattn_status;

typedef enum { REATTN_F32 = 0, REATTN_BF16 = 1 } reattn_dtype;
typedef enum { REATTN_SPAN_ALIGNED = 0, REATTN_SPAN_CENTERED = 1 } reattn_span_mode;
/* model.hpp:19 AttentionMode */
typedef enum { REATTN_MODE_FULL = 0, REATTN_MODE_WINDOW = 1, REATTN_MODE_REATTENTION = 2 } reattn_mode;
/* Lane arithmetic of the fp32 score dot (dense_matrix.hpp:41-56); the reference compiles
 * `l += a*b` either unfused or as an FMA depending on compiler/ISA/d. */
typedef enum { REATTN_LANES_UNFUSED = 0, REATTN_LANES_FMA = 1 } reattn_lanes;
/* Prefill (n_q > 1) paths, a bit mask.  TENSOR_SCAN = the tcgen05 score GEMM with
 * bounded-error windowing and exact re-scoring: indices and scores bit-identical to the
 * reference (bf16 cache, d == 128, k <= 8; other shapes take the CUDA-core scan).
 * TENSOR_ATTN = tcgen05 finite-scope attention (bf16 hi+lo operands, fp32 accumulation:
 * within 2e-4 of the reference's f64 attend in the tests, 6e-7 measured at config 3 --
 * inside north_star's bf16 bar of 1e-2; bf16 cache, d == 128).  TENSOR (both) is the
 * context default; other shapes and fp32 caches take the CUDA-core paths.  EXACT (0) = the
 * CUDA-core scan and the f64 attention everywhere (the reference's arithmetic; slow at
 * prefill sizes).  See DESIGN.md §3. */
typedef enum {
    REATTN_PREFILL_EXACT = 0,
    REATTN_PREFILL_TENSOR_SCAN = 1,
    REATTN_PREFILL_TENSOR_ATTN = 2,
    REATTN_PREFILL_TENSOR = 3
} reattn_prefill_mode;

/* selection.hpp:20-45 SelectionConfig (tile_size only bounds the reference's CPU scratch;
 * it never changes results and is ignored here). */
typedef struct {
    uint64_t k, k_prime, span_m, tile_size, l_global, l_local, l_chunk;
    int32_t span_mode;
    int32_t reserved;
} reattn_selection_config;

/* engine.hpp:23-37 RunStats (per step; the C++ shim folds it into the caller's RunStats) */
typedef struct {
    uint64_t max_position_used;
    uint64_t ood_positions;
    int32_t coverage_total;
    int32_t reserved;
    double entropy_max;
    double entropy_sum;
    uint64_t entropy_rows;
    uint64_t scope_len;
    uint64_t n_spans;
    uint64_t coverage;
    uint64_t peak_scratch_bytes;
} reattn_step_stats;

/* ---- context --------------------------------------------------------------------- */
const char* reattn_version(void);
int reattn_ctx_create(int device, reattn_ctx** out);
void reattn_ctx_destroy(reattn_ctx* ctx);
const char* reattn_last_error(const reattn_ctx* ctx);
int reattn_ctx_set_stream(reattn_ctx* ctx, void* cuda_stream);
void* reattn_ctx_stream(const reattn_ctx* ctx);
int reattn_ctx_set_lanes(reattn_ctx* ctx, int lanes);
int reattn_ctx_set_prefill(reattn_ctx* ctx, int prefill_mode);
int reattn_ctx_synchronize(reattn_ctx* ctx);
int reattn_ctx_num_sms(const reattn_ctx* ctx);
/* device memory helpers for callers without their own allocator (the C++ shim) */
int reattn_malloc(reattn_ctx* ctx, uint64_t bytes, void** out_dev);
int reattn_free(reattn_ctx* ctx, void* dev);
int reattn_memcpy_h2d(reattn_ctx* ctx, void* dst_dev, const void* src_host, uint64_t bytes);
int reattn_memcpy_d2h(reattn_ctx* ctx, void* dst_host, const void* src_dev, uint64_t bytes);

/* ---- device KV cache: kv_cache.hpp:38-118 SegmentedKvCache ------------------------ */
/* Head-major [n_kv][capacity][d] storage of `dtype` for K and V; indices are append rank. */
int reattn_cache_create(reattn_ctx* ctx, uint64_t n_kv, uint64_t d, uint64_t l_global,
                        uint64_t l_local_max, uint64_t capacity, int dtype, reattn_cache** out);
void reattn_cache_destroy(reattn_cache* cache);
/* Grow the storage to new_capacity rows per head (existing rows are kept). */
int reattn_cache_reserve(reattn_ctx* ctx, reattn_cache* cache, uint64_t new_capacity);
/* kv_cache.hpp:54-68 append: rows x (n_kv*d) fp32 in DenseMatrix layout (host or device;
 * device rows are appended in stream order, host rows synchronously). */
int reattn_cache_append(reattn_ctx* ctx, reattn_cache* cache, const float* keys,
                        const float* values, uint64_t rows, int src_on_device);
/* Declare `total` rows already written into the storage (bulk fills, e.g. benchmarks). */
int reattn_cache_set_total(reattn_ctx* ctx, reattn_cache* cache, uint64_t total);
/* kv_cache.hpp:70-87 accessors */
int reattn_cache_info(const reattn_cache* cache, uint64_t* n_kv, uint64_t* d, uint64_t* l_global,
                      uint64_t* l_local_max, uint64_t* capacity, uint64_t* total,
                      uint64_t* global_end, uint64_t* local_start, int* dtype);
void* reattn_cache_keys(const reattn_cache* cache);
void* reattn_cache_values(const reattn_cache* cache);

/* ---- RKVC cache snapshots: kv_cache.hpp:120-209 write/read_cache_snapshot ---------- */
/* open: parses and validates the whole file in the reference's read order (messages and
 * error kinds as read_cache_snapshot: runtime_error -> ERUNTIME, the SegmentedKvCache
 * constructor's invalid_argument -> EINVAL).  load_layer: a new device cache of `dtype`
 * (bf16 storage rounds the f32 payload) with capacity max(capacity, total).  write: the
 * layers' rows as f32, head-major; bf16 caches are widened exactly. */
typedef struct reattn_snapshot reattn_snapshot;
int reattn_snapshot_open(reattn_ctx* ctx, const char* path, reattn_snapshot** out);
int reattn_snapshot_info(const reattn_snapshot* snap, uint32_t* n_layers, uint32_t* n_kv,
                         uint32_t* d_head);
int reattn_snapshot_layer_info(const reattn_snapshot* snap, uint32_t layer, uint64_t* total,
                               uint64_t* l_global, uint64_t* l_local_max);
int reattn_snapshot_load_layer(reattn_ctx* ctx, reattn_snapshot* snap, uint32_t layer, int dtype,
                               uint64_t capacity, reattn_cache** out);
void reattn_snapshot_close(reattn_snapshot* snap);
int reattn_snapshot_write(reattn_ctx* ctx, const char* path, const reattn_cache* const* layers,
                          uint32_t n_layers);

/* ---- rotary table: rope.hpp:19-68 RotaryTable ----------------------------------- */
int reattn_rope_create(reattn_ctx* ctx, uint64_t head_dim, double base, uint64_t max_position,
                       reattn_rope** out);
void reattn_rope_destroy(reattn_rope* rope);
/* host copies of the float tables [max_position][head_dim/2] (may be NULL) */
int reattn_rope_tables_host(const reattn_rope* rope, float* cos_host, float* sin_host);
/* rope.hpp:70-79 rope_rotate on device rows [n_rows][head_dim]; positions on the host.
 * Synchronous.  Position >= max_position -> REATTN_ERANGE "position out of pretrained range". */
int reattn_rope_rotate(reattn_ctx* ctx, const reattn_rope* rope, float* rows_dev,
                       const uint64_t* positions_host, uint64_t n_rows);

/* ---- selection: selection.hpp:168-349 --------------------------------------------- */
/* fused_topk_scores (selection.hpp:168).  q_dev: [n_q][n_heads*d] fp32.  keys_dev: head-major
 * [n_kv][head_stride][d] of key_dtype, middle row 0 at row `row0` of every head, `count`
 * middle rows.  Outputs [n_kv][n_q][k] (score desc, index asc); *n_out = min(k, count).
 * *scratch_bytes = device workspace of the call (constant in `count`).  Synchronous. */
int reattn_fused_topk(reattn_ctx* ctx, const float* q_dev, uint64_t n_q, uint64_t n_heads,
                      const void* keys_dev, int key_dtype, uint64_t n_kv, uint64_t head_stride,
                      uint64_t row0, uint64_t count, uint64_t d, uint64_t k,
                      uint32_t* idx_out_dev, float* score_out_dev, uint64_t* n_out,
                      uint64_t* scratch_bytes);
/* naive_topk_scores (selection_reference.hpp:18-69): the same lists as reattn_fused_topk by an
 * independent route -- the full middle x n_q score matrix materialised (scratch linear in
 * `count`, the reference's point of comparison), then each row's top-k.  k <= 64.  Same
 * arguments as reattn_fused_topk.  Synchronous. */
int reattn_naive_topk(reattn_ctx* ctx, const float* q_dev, uint64_t n_q, uint64_t n_heads,
                      const void* keys_dev, int key_dtype, uint64_t n_kv, uint64_t head_stride,
                      uint64_t row0, uint64_t count, uint64_t d, uint64_t k,
                      uint32_t* idx_out_dev, float* score_out_dev, uint64_t* n_out,
                      uint64_t* scratch_bytes);
/* detail::group_mean_queries (selection.hpp:139-156): q [n_q][n_heads*d] -> [n_q][n_kv*d],
 * sequential fp32 adds times float(1/group).  Synchronous. */
int reattn_group_mean(reattn_ctx* ctx, const float* q_dev, uint64_t n_q, uint64_t n_heads,
                      uint64_t n_kv, uint64_t d, float* out_dev);
/* dot_f32 (dense_matrix.hpp:41-56) of n row pairs a[i], b[i] of length d: the reference's 8
 * lanes and tree, with the context's lane arithmetic (reattn_ctx_set_lanes).  Synchronous. */
int reattn_dot_f32(reattn_ctx* ctx, const float* a_dev, const float* b_dev, uint64_t n, uint64_t d,
                   float* out_dev);
/* dot_f64 (dense_matrix.hpp:59-74), same layout.  Synchronous. */
int reattn_dot_f64(reattn_ctx* ctx, const float* a_dev, const float* b_dev, uint64_t n, uint64_t d,
                   double* out_dev);
/* matmul (dense_matrix.hpp:77-90): c[m][n] = a[m][k] b[k][n], row-major, each element summed
 * in k order with unfused fp32 multiply-adds, as the reference.  Synchronous. */
int reattn_matmul(reattn_ctx* ctx, const float* a_dev, const float* b_dev, uint64_t m, uint64_t k,
                  uint64_t n, float* c_dev);
/* tally_candidates + vote (selection.hpp:252-286) over a flat candidate list.  Synchronous. */
int reattn_vote(reattn_ctx* ctx, const uint32_t* idx_dev, const float* score_dev, uint64_t n,
                uint64_t k_prime, uint32_t* winners_dev, uint64_t* n_winners);
/* tally_candidates (selection.hpp:252-276): every distinct index, ranked by (votes desc,
 * max score desc, index asc), with its votes and max score.  Synchronous. */
int reattn_tally(reattn_ctx* ctx, const uint32_t* idx_dev, const float* score_dev, uint64_t n,
                 uint32_t* idx_out_dev, uint32_t* votes_out_dev, float* score_out_dev,
                 uint64_t* n_unique);
/* expand_spans (selection.hpp:318-349).  Synchronous. */
int reattn_expand_spans(reattn_ctx* ctx, const uint32_t* winners_dev, uint64_t n, uint64_t span_m,
                        uint64_t middle_len, int span_mode, uint32_t* begin_dev,
                        uint32_t* end_dev, uint64_t* n_spans);

/* ---- scope + attention ------------------------------------------------------------ */
/* assemble_scope (scope.hpp:37-78).  Spans index the middle.  src_dev receives the
 * scope-row -> cache-row table (capacity >= window); keys/values_out_dev (nullable)
 * receive fp32 [n_kv][L][d] copies.  Synchronous. */
int reattn_assemble_scope(reattn_ctx* ctx, const reattn_cache* cache, const uint32_t* span_b_dev,
                          const uint32_t* span_e_dev, uint64_t n_spans, uint64_t window,
                          uint32_t* src_dev, float* keys_out_dev, float* values_out_dev,
                          uint64_t* length);
/* attend (attend.hpp:25-77).  q [n_q][d], k [L][d], v [L][dv] fp32 device rows;
 * out [n_q][dv], entropy [n_q] (f64).  Synchronous. */
int reattn_attend(reattn_ctx* ctx, const float* q_dev, uint64_t n_q, const float* k_dev,
                  const float* v_dev, uint64_t L, uint64_t d, uint64_t dv, int has_boundary,
                  uint64_t boundary, float* out_dev, double* entropy_dev);
/* attend_step (engine.hpp:43-114): selection (gated as engine.hpp:58), scope, RoPE at
 * compact positions, attention.  q_dev [n_q][n_head*d] pre-rotation; out_dev
 * [n_q][n_head*d].  span_b/e_host (nullable, capacity >= k_prime) receive the spans,
 * entropy_host (nullable, [n_q][n_head]) the row entropies.  Synchronous. */
int reattn_attend_step(reattn_ctx* ctx, const reattn_cache* cache, const reattn_rope* rope,
                       const float* q_dev, uint64_t n_q, uint64_t n_head,
                       const reattn_selection_config* cfg, int mode, float* out_dev,
                       reattn_step_stats* stats, uint64_t* span_b_host, uint64_t* span_e_host,
                       double* entropy_host);

/* ---- plans: one attend_step shape captured as a CUDA graph ------------------------ */
/* The plan owns its q/out device buffers and workspace; launching it replays the whole
 * step (scan, vote/spans/scope, attention, combine) with no host synchronisation. */
int reattn_plan_create(reattn_ctx* ctx, const reattn_cache* cache, const reattn_rope* rope,
                       uint64_t n_q, uint64_t n_head, const reattn_selection_config* cfg,
                       int mode, reattn_plan** out);
void reattn_plan_destroy(reattn_plan* plan);
float* reattn_plan_q(const reattn_plan* plan);
float* reattn_plan_out(const reattn_plan* plan);
/* asynchronous replay on the context stream.
 * A decode plan (n_q == 1, selection on the K1 fast scan with the select fused into its merger
 * CTA: every BASELINE decode config) reads the cache length from the device, so it stays valid
 * while the cache grows through reattn_cache_append / _set_total / the plan's own append node:
 * one graph serves every decode step.  Any other plan is frozen to the cache length it was
 * built for; launching it after the length changed is an error (ERUNTIME), and so is any plan
 * after reattn_cache_reserve reallocated the storage it captured. */
int reattn_plan_launch(reattn_plan* plan);
/* Append mode (decode plans only): the graph first appends the step's K and V rows
 * (kv_cache.hpp:54-68, fp32 [n_kv * d] each at reattn_plan_k_in / _v_in) at the device cache
 * length and advances it, then runs the step -- Engine::forward_block's append-then-attend
 * (engine.hpp:196-198) in one replay.  Each launch advances the cache's length by one;
 * ERUNTIME "cache append: capacity exceeded" when the storage is full. */
int reattn_plan_set_append(reattn_plan* plan, int enable);
/* 1 when the plan follows the cache length (a decode plan, see reattn_plan_launch), else 0 */
int reattn_plan_follows_cache(const reattn_plan* plan);
/* the cache storage generation the plan was captured over (a reserve bumps the cache's) */
uint64_t reattn_plan_cache_generation(const reattn_plan* plan);
float* reattn_plan_k_in(const reattn_plan* plan);
float* reattn_plan_v_in(const reattn_plan* plan);
/* end to end from host memory in append mode: H2D q, k, v; replay; D2H out; synchronise */
int reattn_plan_step_host(reattn_plan* plan, const float* q_host, const float* k_host,
                          const float* v_host, float* out_host);
/* enqueue only the plan's K-scan kernel (no graph) so callers can time it with events */
int reattn_plan_launch_scan(reattn_plan* plan);
/* end to end from host memory: H2D q, replay, D2H out, synchronise */
int reattn_plan_run_host(reattn_plan* plan, const float* q_host, float* out_host);
/* synchronise and read the last replay's stats (errors surface here) */
int reattn_plan_stats(reattn_plan* plan, reattn_step_stats* stats);
/* synchronise and read the last replay's full attend_step outputs besides `out`: stats,
 * the chosen spans (nullable, capacity >= k_prime) and the row entropies (nullable,
 * [n_q][n_head]) -- what reattn_attend_step returns through the same arguments */
int reattn_plan_result(reattn_plan* plan, reattn_step_stats* stats, uint64_t* span_b_host,
                       uint64_t* span_e_host, double* entropy_host);
/* the same outputs without a synchronisation per plan (a decoder runs one plan per layer):
 * stage enqueues their copies into pinned host memory behind the replay on the context
 * stream; after the caller synchronised that stream, staged_result reads them (ELOGIC when
 * nothing was staged) */
int reattn_plan_stage_result(reattn_plan* plan);
int reattn_plan_staged_result(reattn_plan* plan, reattn_step_stats* stats, uint64_t* span_b_host,
                              uint64_t* span_e_host, double* entropy_host);
/* Diagnostics, no reference counterpart: with REATTN_TRACE=1 in the environment when a plan
 * is built, the decode kernels stamp %globaltimer (ns) into a device trace buffer; this
 * synchronises the device and copies its first n words (n <= 4096) to the host. */
int reattn_debug_trace(uint64_t* host_out, uint64_t n);
/* model.hpp:155-178 rmsnorm and the gated feed-forward's activation, on device arrays:
 * out[r][c] = x[r][c] * float(1 / sqrt(mean_c(x^2 in f64) + 1e-5)) * w[c]; gate[i] <-
 * gate[i] / (1 + exp(-gate[i])) * up[i] (fp32, the reference's operation order). */
int reattn_rmsnorm(reattn_ctx* ctx, const float* x_dev, uint64_t rows, uint64_t cols, const float* w_dev,
                   float* out_dev);
int reattn_silu_mul(reattn_ctx* ctx, float* gate_dev, const float* up_dev, uint64_t n);
/* softmax.hpp:13-36 stable_softmax (max-subtracted, f64 sums) and attention_entropy of one
 * device vector; entropy_out: one double on the device. */
int reattn_stable_softmax(reattn_ctx* ctx, const float* logits_dev, uint64_t n, float* out_dev);
int reattn_attention_entropy(reattn_ctx* ctx, const float* weights_dev, uint64_t n, double* entropy_out_dev);
/* Diagnostics: the decoder's fp32 GEMV (y[N] = x[K] . W[K][N] + beta y) on the context
 * stream, for benchmarking the projection kernel alone (tools/bench_gemv.py); ws is a device
 * workspace of reattn_debug_gemv_workspace(N) bytes, zeroed once. */
size_t reattn_debug_gemv_workspace(uint64_t n);
int reattn_debug_gemv(reattn_ctx* ctx, const float* x, const float* w, uint64_t ldw, uint64_t n,
                      uint64_t k, float* y, float beta, void* ws);
/* kernels per replay, and the algorithmic bytes of the dominant kernel (the K scan) */
int reattn_plan_info(const reattn_plan* plan, uint64_t* kernels_per_step,
                     uint64_t* scan_bytes, uint64_t* scope_bytes);

/* ---- batched decode (one graph over n_seq sequences with their own caches) ----------- */
/* Batch > 1 is a reference non-goal; each sequence's result is exactly its own
 * attend_step (engine.hpp:43, n_q = 1).  bf16 decode with a middle: the scans run back to
 * back while sequence b's attention runs beside scan b+1 on `side_sms` spare SMs.
 * q / out: [n_seq][n_head * d] fp32 on the device. */
typedef struct reattn_batch_plan reattn_batch_plan;
int reattn_batch_plan_create(reattn_ctx* ctx, const reattn_cache* const* caches, uint32_t n_seq,
                             const reattn_rope* rope, uint64_t n_head,
                             const reattn_selection_config* cfg, int mode,
                             reattn_batch_plan** out);
void reattn_batch_plan_destroy(reattn_batch_plan* plan);
float* reattn_batch_plan_q(const reattn_batch_plan* plan);
float* reattn_batch_plan_out(const reattn_batch_plan* plan);
int reattn_batch_plan_launch(reattn_batch_plan* plan);
int reattn_batch_plan_run_host(reattn_batch_plan* plan, const float* q_host, float* out_host);
int reattn_batch_plan_stats(reattn_batch_plan* plan, uint32_t seq, reattn_step_stats* stats);
int reattn_batch_plan_info(const reattn_batch_plan* plan, uint64_t* kernels_per_step,
                           uint64_t* scan_bytes, int* side_sms);

/* ---- sequence-sharded decode ---------------------------------------- */
/* Rank `rank` of `world` holds [global | its middle shard | local] in `local_cache` (same
 * l_global / l_local as the unsharded cache; the shard is the local cache's middle).  The
 * middle of the GLOBAL cache (`global_total` rows) is split at multiples of span_m:
 * shard r = [floor(r*M/world/m)*m, floor((r+1)*M/world/m)*m) (last shard ends at M).
 * A step is four asynchronous stages on the context stream with two all-gathers between
 * them, done by the caller's collective library (NCCL):
 *   scan -> all_gather(cand) -> select -> attend -> all_gather(part) -> combine.
 * Every rank ends with the full output. */
typedef struct reattn_shard_plan reattn_shard_plan;
int reattn_shard_plan_create(reattn_ctx* ctx, const reattn_cache* local_cache,
                             const reattn_rope* rope, uint64_t n_head,
                             const reattn_selection_config* cfg, uint64_t global_total,
                             int world, int rank, reattn_shard_plan** out);
void reattn_shard_plan_destroy(reattn_shard_plan* plan);
/* shard boundaries in middle coordinates (rank r: [begin, begin + len)) */
int reattn_shard_range(uint64_t middle_len, uint64_t span_m, int world, int rank,
                       uint64_t* begin, uint64_t* len);
float* reattn_shard_plan_q(const reattn_shard_plan* plan);    /* [1][n_head*d] */
float* reattn_shard_plan_out(const reattn_shard_plan* plan);  /* [1][n_head*d] */
/* device buffers for the two all-gathers: this rank's send block and the world-sized
 * receive buffer (rank r's block at recv + r * bytes) */
int reattn_shard_buffers(const reattn_shard_plan* plan, void** cand_send, void** cand_recv,
                         uint64_t* cand_bytes, void** part_send, void** part_recv,
                         uint64_t* part_bytes);
int reattn_shard_scan(reattn_shard_plan* plan);     /* local K scan -> cand_send */
int reattn_shard_select(reattn_shard_plan* plan);   /* cand_recv -> vote/spans/scopes */
int reattn_shard_attend(reattn_shard_plan* plan);   /* owned scope rows -> part_send */
int reattn_shard_combine(reattn_shard_plan* plan);  /* part_recv -> out */
/* synchronise; header errors surface here */
int reattn_shard_stats(reattn_shard_plan* plan, reattn_step_stats* stats, uint64_t* span_b_host,
                       uint64_t* span_e_host);

/* NCCL host path: the library owns an NCCL communicator and issues both all-gathers of a
 * step itself, so a C++ (or any FFI) host runs the sharded decode with no collective
 * library of its own.  Rank 0 creates the id (reattn_comm_unique_id) and ships the 128
 * bytes to every rank out of band (e.g. the launcher's store); every rank then calls
 * reattn_comm_create collectively.  reattn_shard_step enqueues scan -> ncclAllGather ->
 * select -> attend -> ncclAllGather -> combine on the context stream (or replays the
 * graph captured by reattn_shard_capture, which must also be called collectively). */
#define REATTN_COMM_ID_BYTES 128
typedef struct reattn_comm reattn_comm;
int reattn_comm_unique_id(uint8_t* id_out /* REATTN_COMM_ID_BYTES */);
int reattn_comm_create(reattn_ctx* ctx, int world, int rank, const uint8_t* id, reattn_comm** out);
void reattn_comm_destroy(reattn_comm* comm);
int reattn_shard_step(reattn_shard_plan* plan, reattn_comm* comm);
int reattn_shard_capture(reattn_shard_plan* plan, reattn_comm* comm);
/* end to end from host memory: H2D q, step, D2H out, synchronise */
int reattn_shard_run_host(reattn_shard_plan* plan, reattn_comm* comm, const float* q_host,
                          float* out_host);

/* ---- decoder model + generation engine (reference model.hpp, engine.hpp:119-216) ------
 * The toy decoder the reference's Engine drives: pre-norm blocks x += attn(norm(x)),
 * x += ffn(norm(x)), greedy decode.  Weights live on the device (fp32, the reference's
 * layout: projections input-major, d_in x d_out).  Projections run as fp32 GEMMs
 * (cuBLAS, no TF32); the K/V projections of an fp32 cache write straight into the cache
 * rows; attention is the reattn_attend_step pipeline.  Errors carry the reference's
 * exception kinds and messages (model config / weights file / engine). */
typedef struct {
    uint64_t n_layer, n_head, n_kv_head, d_model, d_head, d_ff, vocab_size, pretrain_window;
    double rope_base;
    int32_t attention_mode; /* reattn_mode: 0 full, 1 window, 2 reattention */
    int32_t reserved;
} reattn_model_config;

/* LayerWeights / ModelWeights tensors (model.hpp:66-84); layer is ignored for globals */
typedef enum {
    REATTN_W_EMBEDDING = 0, /* vocab x d_model */
    REATTN_W_WQ = 1,        /* d_model x n_head*d_head */
    REATTN_W_WK = 2,        /* d_model x n_kv_head*d_head */
    REATTN_W_WV = 3,
    REATTN_W_WO = 4,        /* d_model x d_model */
    REATTN_W_GATE = 5,      /* d_model x d_ff */
    REATTN_W_UP = 6,
    REATTN_W_DOWN = 7,      /* d_ff x d_model */
    REATTN_W_NORM_ATTN = 8, /* d_model */
    REATTN_W_NORM_FFN = 9,
    REATTN_W_NORM_FINAL = 10,
    REATTN_W_LM_HEAD = 11   /* d_model x vocab */
} reattn_weight_kind;

typedef struct reattn_weights reattn_weights;
/* ModelConfig::validate (model.hpp:51-61) */
int reattn_model_config_validate(reattn_ctx* ctx, const reattn_model_config* cfg);
/* zero projections, unit norms */
int reattn_weights_create(reattn_ctx* ctx, const reattn_model_config* cfg, reattn_weights** out);
/* init_random (model.hpp:120-152): the same mt19937_64 Box-Muller stream, std 0.02 */
int reattn_weights_init_random(reattn_ctx* ctx, const reattn_model_config* cfg, uint64_t seed,
                               reattn_weights** out);
/* benchmarking only, no reference counterpart: projections, embedding and lm_head filled on
 * the device with splitmix64 uniform values times 0.02, unit norms (init_random draws its
 * Gaussian stream on the host, minutes for an 8B-parameter shape) */
int reattn_weights_synth(reattn_ctx* ctx, const reattn_model_config* cfg, uint64_t seed,
                         reattn_weights** out);
/* RATW weight files (model.hpp:204-339 save_weights / load_weights) */
int reattn_weights_load(reattn_ctx* ctx, const char* path, reattn_weights** out);
int reattn_weights_save(reattn_ctx* ctx, const reattn_weights* w, const char* path);
int reattn_weights_config(const reattn_weights* w, reattn_model_config* cfg);
int reattn_weights_shape(const reattn_weights* w, int kind, uint64_t* rows, uint64_t* cols);
int reattn_weights_upload(reattn_ctx* ctx, reattn_weights* w, int kind, uint64_t layer,
                          const float* host, uint64_t n);
int reattn_weights_download(reattn_ctx* ctx, const reattn_weights* w, int kind, uint64_t layer,
                            float* host, uint64_t n);
void reattn_weights_destroy(reattn_weights* w);

/* RunStats accumulated over an engine's steps (engine.hpp:23-37) */
typedef struct {
    uint64_t max_position_used;
    uint64_t ood_positions;
    int32_t coverage_total;
    int32_t reserved;
    double entropy_max;
    double entropy_sum;
    uint64_t entropy_rows;
    uint64_t scope_len_max;
    uint64_t peak_scratch_bytes;
    uint64_t chunks_processed;
    uint64_t decode_steps;
} reattn_run_stats;

typedef struct reattn_engine reattn_engine;
/* Engine(weights, sel, mode) (engine.hpp:121-132): `w` must outlive the engine.
 * cache_dtype: REATTN_F32 (the reference's storage) or REATTN_BF16. */
int reattn_engine_create(reattn_ctx* ctx, const reattn_weights* w, const reattn_selection_config* sel,
                         int mode, int cache_dtype, reattn_engine** out);
int reattn_engine_reset(reattn_engine* e);
/* prefill (engine.hpp:147-160): first l_global + l_local tokens, then l_chunk strides; the
 * final chunk's hidden states stay on the device (rows -> *rows_out) */
int reattn_engine_prefill(reattn_engine* e, const uint32_t* tokens_host, uint64_t n,
                          uint64_t* rows_out);
/* the hidden states of the last forward block, rows x d_model */
int reattn_engine_hidden(reattn_engine* e, float* host, uint64_t n);
/* logits(hidden) (engine.hpp:177-179): final norm + lm_head of host rows x d_model */
int reattn_engine_logits(reattn_engine* e, const float* hidden_host, uint64_t rows,
                         float* logits_host);
/* decode_step (engine.hpp:163-174): one token in, greedy next token out */
int reattn_engine_decode_step(reattn_engine* e, uint32_t last_token, uint32_t* next_token);
int reattn_engine_last_logits(reattn_engine* e, float* host, uint64_t n);
int reattn_engine_stats(const reattn_engine* e, reattn_run_stats* st);
/* decode_latency_ms entries (up to cap); *n = how many exist */
int reattn_engine_decode_latencies(const reattn_engine* e, double* out, uint64_t cap, uint64_t* n);
/* spans chosen by the layer's most recent attend_step (engine.hpp:183-184) */
int reattn_engine_last_spans(const reattn_engine* e, uint64_t layer, uint64_t* begin,
                             uint64_t* end, uint64_t cap, uint64_t* n);
const reattn_cache* reattn_engine_cache(const reattn_engine* e, uint64_t layer);
/* benchmarking only: every layer's cache holds `total` synthetic rows (as if a prompt of that
 * length had been prefilled), so decode throughput can be measured at long contexts */
int reattn_engine_synth_context(reattn_engine* e, uint64_t total, uint64_t seed);
void reattn_engine_destroy(reattn_engine* e);

/* ---- synthetic inputs (tests and benchmarks; not on the hot path) ---------------- */
/* dst[i] = splitmix64(seed, offset+i) mapped to [-1, 1) (24 significant bits), stored as
 * fp32 or bf16 (round to nearest even). */
int reattn_synth_uniform(reattn_ctx* ctx, void* dst_dev, uint64_t n, int dtype, uint64_t seed,
                         uint64_t offset);

#ifdef __cplusplus
}
#endif
#endif /* REATTN_CUDA_H */
