// Host-side launch interface of the sm_100a kernels (internal; the public boundary is
// include/reattn_cuda.h).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

namespace reattn_impl {

enum DType { kF32 = 0, kBF16 = 1 };

// Scope descriptor written on the device by the vote/span/scope kernel and read by the
// attention kernels, so a whole attend_step runs without a host round trip.
struct ScopeHeader {
    uint32_t L;          // scope length L'
    uint32_t n_spans;
    uint32_t coverage;   // rows selected from the middle
    uint32_t n_winners;
    int32_t error;       // 0 ok, see kScopeErr*
    uint32_t pad[3];
};
enum {
    kScopeOk = 0,
    kScopeErrWindow = 1,      // "scope exceeds pretrain window"
    kScopeErrSpanRange = 2,   // "assemble_scope: span outside middle"
    kScopeErrQueryLong = 3,   // "attend_step: query block longer than scope"
    kScopeErrWinnerRange = 4, // "expand_spans: winner outside middle"
    kScopeErrTooMany = 5,     // candidate count beyond the device vote capacity
};

// Inputs/outputs of the warp-level vote + spans + scope routine (select_small.cuh), used
// standalone and fused into the K-scan's merger CTA (CTA 0).
struct SmallSelectIO {
    uint32_t k_prime, span_m, middle_len;
    int span_mode;
    uint32_t g_end, l_start, total, window, n_q;
    uint32_t* winners;
    uint32_t* span_b;
    uint32_t* span_e;
    uint32_t* scope_src;
    ScopeHeader* hdr;
    // 0: the table's local rows are not needed (the decode fork attends the local window
    // straight from the cache and the head launch reads rows [0, L' - n_local) only)
    int table_local = 1;
};
constexpr uint32_t kSmallSelectMax = 32;

// ---- K1: decode scan + top-k (selection.hpp:168-248) -------------------------------
struct ScanArgs {
    const float* q;        // [n_q][n_heads*d] pre-rotation queries
    int n_q, n_heads, n_kv, d;
    const void* keys;      // head 0, row 0 of a head-major [n_kv][head_stride][d] array
    int dtype;
    uint64_t head_stride;  // rows between heads
    uint64_t row0;         // middle row 0 inside each head
    uint32_t count;        // middle length
    int k;
    int lanes;             // kLanesUnfused / kLanesFma
    uint32_t* idx_out;     // [n_kv][n_q][k]
    float* score_out;
    // fast path only: run vote + spans + scope in the merger CTA (n_kv * min(k, count) <= 32)
    int fuse_select = 0;
    SmallSelectIO sel = {};
    // fast path: keep the adaptive tile partition in the workspace (private, zero-initialised
    // plan workspaces only)
    int balance = 0;
    // fast path: a device-resident cache length (plans that survive cache growth).  When set,
    // count / row0 and the fused select's geometry come from it (kv_cache.hpp:65-67 with
    // l_global / l_local), and the grid is the full num_sms.
    const uint32_t* dev_total = nullptr;
    uint32_t l_global = 0, l_local = 0;
};

// Fast path: TMA-staged, one thread per key row, q in registers, register top-k.
// Requires d == 128, n_q == 1, k <= 8.
bool scan_fast_supported(const ScanArgs& a);
size_t scan_fast_workspace(const ScanArgs& a, int num_sms);
// `kmap` is a 2-D tiled tensor map over [n_kv*head_stride rows][d] with a 128-byte box
// width and SWIZZLE_128B (built by make_key_tensor_map).
cudaError_t launch_scan_fast(const ScanArgs& a, const CUtensorMap& kmap, void* workspace,
                             int num_sms, cudaStream_t s);
bool make_key_tensor_map(CUtensorMap* map, const void* base, int dtype, uint64_t d,
                         uint64_t rows, int box_rows);
int scan_fast_box_rows(int dtype);

// Prefill path on tcgen05 (prefill_tc.cu): one bf16 score GEMM of the group-mean query with
// a bounded error, streaming approximate top-(k+4) lists, exact dot_f32 re-scoring of the
// keys inside the error window.  d == 128, bf16 keys, k <= 8.  Bit-exact with the reference.
bool prefill_tc_supported(const ScanArgs& a);
size_t prefill_tc_workspace(const ScanArgs& a);
int prefill_tc_key_box_rows();
cudaError_t launch_prefill_tc(const ScanArgs& a, const CUtensorMap& kmap, void* workspace,
                              cudaStream_t s);

// Generic path: any d, n_q, k (k <= kGenericMaxK), streaming threshold buffer + bitonic
// compaction in shared memory; one CTA per (query, kv head).
constexpr int kGenericMaxK = 7936;
cudaError_t launch_scan_generic(const ScanArgs& a, cudaStream_t s);

// ---- K3: vote + spans + scope (selection.hpp:252-349, scope.hpp:37-78) ----------
struct SelectArgs {
    const uint32_t* cand_idx;  // n_lists lists of list_len valid entries, list stride
    const float* cand_score;
    uint32_t n_lists, list_len, list_stride;
    uint32_t k_prime;
    uint32_t span_m;
    uint32_t middle_len;
    int span_mode;
    // scope build (skipped when build_scope == 0)
    int build_scope;
    uint32_t g_end, l_start, total, window, n_q;
    // external winners / spans (bypass stages): used by the standalone APIs
    const uint32_t* winners_in;  // if non-null: skip the vote, use these n_winners_in
    uint32_t n_winners_in;
    const uint32_t* n_winners_dev;  // if non-null: the winner count, read on the device
    const uint32_t* span_b_in;   // if non-null: skip vote + expand, use these spans
    const uint32_t* span_e_in;
    uint32_t n_spans_in;
    // outputs
    uint32_t* winners;   // [k_prime]
    uint32_t* rank_votes;  // optional [k_prime]: votes of each winner (tally API)
    float* rank_score;     // optional [k_prime]: max score of each winner
    uint32_t* span_b;    // [k_prime]
    uint32_t* span_e;
    uint32_t* scope_src; // [window]
    ScopeHeader* hdr;
};
constexpr uint32_t kVoteMaxSmem = 8192;
size_t select_smem_bytes(uint32_t n_cand, uint32_t k_prime);
cudaError_t launch_select(const SelectArgs& a, cudaStream_t s);
// > kVoteMaxSmem candidates: device-wide radix-sort vote (vote_large.cu), then spans+scope
// bounded path (middle_len > 0, k' <= 1024): the workspace must be zeroed once (it stays
// clean across launches)
size_t vote_large_workspace(uint32_t n_cand, uint32_t middle_len, uint32_t k_prime);
uint32_t vote_large_kernels(uint32_t n_cand, uint32_t middle_len, uint32_t k_prime);
cudaError_t launch_vote_large(const SelectArgs& a, void* workspace, cudaStream_t s);

// ---- K4+K5: gather + RoPE + finite-scope attention (attend.hpp, engine.hpp:71-107)
struct AttnArgs {
    const float* q;          // query rows, q_row_stride floats apart; head h at +h*d
    uint64_t q_row_stride;
    int n_q, n_head, n_kv, group, d, dv;
    const void* k_base;      // [n_kv][head_stride][d]
    const void* v_base;      // [n_kv][head_stride][dv]
    int dtype;
    uint64_t head_stride;
    const uint32_t* src;     // scope row -> cache row (nullptr: identity)
    const ScopeHeader* hdr;  // L from the device header (nullptr: use L_host)
    uint32_t L_host;
    const float* rope_cos;   // [max_pos][d/2] (nullptr: no rotation)
    const float* rope_sin;
    int causal;              // 1: row i sees [0, boundary+i+1)
    int boundary_is_tail;    // 1: boundary = L - n_q (attend_step), else boundary_host
    uint32_t boundary_host;
    double* part;            // workspace, see attend_workspace
    float* out;              // [n_q][n_head*dv]
    double* entropy;         // [n_q][n_head]
};
constexpr int kAttnSplit = 64;
size_t attend_workspace(const AttnArgs& a, uint32_t L_max);
cudaError_t launch_attend(const AttnArgs& a, uint32_t L_max, cudaStream_t s);
int attend_kernel_count(const AttnArgs& a, uint32_t L_max);
// decode attention with a bulk-copy ring and fused combine (attend_decode.cu): n_q == 1,
// d == dv == 128, bf16 cache.  ws = a.part: per-kv-head tickets (zero before the
// first launch; the kernel re-arms them) + partial rows.  The tickets take
// decode_ticket_bytes(n_kv) (one uint32 per kv head, rounded up to 256 B).
bool decode_bulk_eligible(const AttnArgs& a);
size_t decode_ticket_bytes(int n_kv);
size_t decode_bulk_workspace(const AttnArgs& a, int num_sms);
cudaError_t launch_attend_decode_bulk(const AttnArgs& a, void* ws, int num_sms, cudaStream_t s);
// same on `num_sms` SMs' worth of CTAs, with or without programmatic dependent launch
cudaError_t launch_attend_decode_bulk_ex(const AttnArgs& a, void* ws, int num_sms, cudaStream_t s,
                                         bool pdl);
// Local-window fork: the last n_local scope rows are the cache's local segment, independent of
// the selection (RoPE is relative, so they can be attended at positions 0..n_local-1 with the
// query at n_local-1).  The local launch runs beside the scan on local_parts CTAs per kv head
// (partials only); the head launch attends scope rows [0, L'-n_local) after the select and
// merges both.  Same workspace as launch_attend_decode_bulk.
struct DecodeFork {
    uint32_t n_local;     // local segment rows (cache total - local start)
    uint32_t local_row0;  // cache row of local row 0
    int local_parts;      // CTAs per kv head for the local launch (1..kMaxLocalParts)
    int heads_per_cta;    // kv heads each local CTA processes in turn (divides n_kv)
    int post;             // 1: the local launch follows the scan on the same stream (PDL): its
                          // CTAs fill the SMs the scan CTAs release while the scan's merger CTA
                          // runs its tail, and it completes only after the scan (so the head
                          // launch's griddepcontrol.wait covers both); 0: beside the scan on
                          // local_parts * n_kv lent SMs (side stream)
    // growing caches: n_local / local_row0 from the device-resident cache length (null: above)
    const uint32_t* dev_total = nullptr;
    uint32_t l_global = 0, l_local = 0;
};
constexpr int kMaxLocalParts = 32;
cudaError_t launch_attend_decode_local(const AttnArgs& a, void* ws, int num_sms, const DecodeFork& f,
                                       cudaStream_t s);
cudaError_t launch_attend_decode_head(const AttnArgs& a, void* ws, int num_sms, const DecodeFork& f,
                                      cudaStream_t s, bool pdl);
// prefill attention on tcgen05 (attend_tc.cu): d == dv == 128, bf16 cache; bf16 hi+lo split
// operands, fp32 TMEM accumulation (bf16 tolerance).  ws: attend_tc_workspace bytes.
bool attend_tc_supported(const AttnArgs& a);
size_t attend_tc_workspace(const AttnArgs& a, uint32_t L_max);
cudaError_t launch_attend_tc(const AttnArgs& a, uint32_t L_max, void* ws, cudaStream_t s);
// sharded decode halves (n_q == 1, d == 128): partial states, then the multi-source combine
bool attend_decode_supported(const AttnArgs& a, uint32_t L_max);
size_t attend_decode_partial_bytes(const AttnArgs& a, uint32_t L_max);  // per source
cudaError_t launch_attend_decode_partials(const AttnArgs& a, uint32_t L_max, cudaStream_t s);
cudaError_t launch_attend_decode_combine(const AttnArgs& a, uint32_t L_max, int n_src,
                                         cudaStream_t s);

// ---- sharded decode: merge gathered candidates, vote/spans/scope, local ownership ------
struct ShardSelectArgs {
    // source s, list l, rank j at [s * src_stride + l * k + j]; indices are shard-local
    // middle indices (kNoIndex = empty slot)
    const uint32_t* cand_idx;
    const float* cand_score;
    size_t src_stride;
    int n_src, n_lists, k, kk;  // kk = min(k, global middle length)
    uint32_t src_offset[64];    // shard_begin of each source rank
    SmallSelectIO sel;          // global geometry; sel.scope_src receives the GLOBAL table
    int rank, world;
    uint32_t shard_begin, shard_len;
    uint32_t* local_src;        // [L'] local cache row, or kNoIndex (a middle row held elsewhere)
    uint32_t* ranges;           // ShardRanges: the scope rows this rank attends
};
cudaError_t launch_shard_merge_select(const ShardSelectArgs& a, cudaStream_t s);
// Scope rows (index ranges [begin, end) in scope order) attended by one rank of a sharded
// decode step: rank 0 the global rows, every rank its own span rows and a 32-row aligned
// 1/world slice of the local window.  Written on the device by the shard select.
struct ShardRanges {
    uint32_t n;
    uint32_t begin[3], end[3];
};
// Sharded decode attention: the bulk decode kernel over the rank's ShardRanges; the parts of
// each kv head are merged on the device into ONE partial row per q head at `merged`
// ([n_head] rows of kDecodePartBytes: f64 m (log2), A, B, pad; fp32 acc[128]).  ws as
// decode_bulk_workspace.
constexpr int kDecodePartBytes = 32 + 128 * 4;
cudaError_t launch_attend_decode_ranges(const AttnArgs& a, void* ws, int num_sms,
                                        const uint32_t* ranges, uint8_t* merged, cudaStream_t s);
// Final merge of n_src ranks' merged partial rows (rank s at parts + s * src_stride bytes,
// [n_head] rows each) -> out + entropy.
cudaError_t launch_decode_combine_sources(const AttnArgs& a, const uint8_t* parts, int n_src,
                                          size_t src_stride, cudaStream_t s);

// ---- dense numerics of the drop-in API (dense.cu) ------------------------------------
cudaError_t launch_dot_f32(const float* a, const float* b, uint64_t n, uint64_t d, int lanes,
                           float* out, cudaStream_t s);
cudaError_t launch_dot_f64(const float* a, const float* b, uint64_t n, uint64_t d, double* out,
                           cudaStream_t s);
cudaError_t launch_matmul(const float* a, const float* b, uint64_t m, uint64_t k, uint64_t n,
                          float* c, cudaStream_t s);
cudaError_t launch_group_mean(const float* q, uint64_t n_q, uint64_t n_heads, uint64_t n_kv,
                              uint64_t d, float* out, cudaStream_t s);
// naive_topk_scores (selection_reference.hpp:18-69): materialised scores, then row top-k
// (k <= 64); ws: naive_topk_workspace bytes
size_t naive_topk_workspace(uint64_t n_q, uint64_t n_kv, uint64_t count, uint64_t d);
cudaError_t launch_naive_topk(const ScanArgs& a, void* ws, cudaStream_t s);

// ---- misc kernels ------------------------------------------------------------------
// rows x (n_kv*d) fp32 (DenseMatrix layout) -> head-major [n_kv][head_stride][d] at row0.
cudaError_t launch_cache_append(const float* src, void* dst, int dtype, uint64_t rows,
                                uint64_t n_kv, uint64_t d, uint64_t head_stride, uint64_t row0,
                                cudaStream_t s);
// one row per head (rows = 1, [n_kv * d] fp32 K and V) at the device cache length *dev_total,
// which the kernel then advances by one (a decode step's append inside a plan's graph)
cudaError_t launch_cache_append_step(const float* k_in, const float* v_in, void* keys, void* values,
                                     int dtype, uint64_t n_kv, uint64_t d, uint64_t head_stride,
                                     uint32_t* dev_total, cudaStream_t s);
cudaError_t launch_set_u32(uint32_t* p, uint32_t v, cudaStream_t s);
// copies count (<= 4) arrays src[i] -> dst[i] of n[i] floats (pinned host <-> device, zero-copy)
cudaError_t launch_host_io(const float* const* src, float* const* dst, const uint64_t* n, int count,
                           cudaStream_t s);
// scope gather to fp32 [n_kv][L][d] (assemble_scope's copies, scope.hpp:63-76).
cudaError_t launch_gather(const void* base, int dtype, uint64_t n_kv, uint64_t d,
                          uint64_t head_stride, const uint32_t* src, uint32_t L, float* out,
                          cudaStream_t s);
cudaError_t launch_rope_rotate(float* rows, const uint32_t* pos, uint64_t n_rows, uint64_t d,
                               const float* cos_t, const float* sin_t, cudaStream_t s);
cudaError_t launch_synth_uniform(void* dst, int dtype, uint64_t n, uint64_t seed,
                                 uint64_t offset, cudaStream_t s);
// entropy stats reduction in the reference's order (engine.hpp:100-106): for h, for i.
cudaError_t launch_entropy_stats(const double* entropy, int n_q, int n_head, double* out2,
                                 cudaStream_t s);

// ---- decoder block around attend_step (model.cu; reference model.hpp) ----------------------
cudaError_t launch_embed(const uint32_t* tokens, uint64_t rows, const float* emb, uint64_t d_model,
                         float* out, cudaStream_t s);
cudaError_t launch_rmsnorm(const float* x, uint64_t rows, uint64_t cols, const float* w, float* out,
                           cudaStream_t s);
cudaError_t launch_silu_mul(float* gate, const float* up, uint64_t n, cudaStream_t s);
// softmax.hpp utilities (scratch: n doubles)
cudaError_t launch_stable_softmax(const float* l, uint64_t n, float* out, double* scratch, cudaStream_t s);
cudaError_t launch_attention_entropy(const float* w, uint64_t n, double* out, double* scratch, cudaStream_t s);
cudaError_t launch_argmax(const float* v, uint64_t n, uint32_t* out, cudaStream_t s);
cudaError_t launch_scale(float* x, uint64_t n, float a, cudaStream_t s);
// decode projections: y[N] = x[K] . W[K][N] (+ beta y), workspace sized for N <= n_max
// (zeroed once: the split tickets reset themselves)
size_t gemv_workspace_bytes(uint64_t n_max);
bool gemv_supported(uint64_t N, uint64_t K, uint64_t ldw, const void* x, const void* W, const void* y);
cudaError_t launch_gemv(const float* x, const float* W, uint64_t ldw, uint64_t N, uint64_t K, float* y,
                        float beta, void* ws, uint64_t n_max, cudaStream_t s);
struct GemvDesc {
    const float* W;
    uint64_t ldw, N;
    float* y;
    float beta;
    int kind;              // 0: y dense fp32; 1 / 2: y is a bf16 / fp32 cache's K or V base and
    uint64_t d, row;       //   column c lands in head c / d, element c % d of cache row `row`
    uint64_t head_stride;  //   (the cache capacity)
};
// a plain (unswizzled) 2-D tensor map: `outer` rows of `inner` elements, row_bytes apart
bool make_tensor_map_2d(CUtensorMap* map, const void* base, int dtype, uint64_t inner, uint64_t outer,
                        uint64_t row_bytes, uint32_t box_inner, uint32_t box_outer);
// the GEMV's weight tile map (64 rows x 128 fp32 columns) for W[K][N] with row stride ldw
bool gemv_weight_map(CUtensorMap* map, const float* W, uint64_t ldw, uint64_t N, uint64_t K);
// up to 3 matrices sharing x in one launch; silu_pair: mats = {gate, up}, gate <- silu(g) * u;
// maps (optional, one per matrix, from gemv_weight_map): the TMA-fed kernel when K fits;
// total_ptr (optional): written with total_val by the launch (a cache's device length)
cudaError_t launch_gemv_batch(const float* x, uint64_t K, const GemvDesc* mats, int count, bool silu_pair,
                              void* ws, uint64_t n_max, cudaStream_t s, uint32_t* total_ptr = nullptr,
                              uint32_t total_val = 0, const CUtensorMap* maps = nullptr);

// ---- timeline trace (diagnostics): REATTN_TRACE=1 at plan / launch time makes the decode
// kernels stamp %globaltimer into a device buffer (layout in misc.cu); null otherwise.
constexpr int kTraceWords = 4096;
uint64_t* trace_buffer();

}  // namespace reattn_impl
