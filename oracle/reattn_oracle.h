/*
 * TEST INFRASTRUCTURE ONLY — CPU restatement of the reference ReAttention hot path.
 *
 * This is the parity oracle for the B200 kernels in paper_2407_15176_b200/csrc.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may load it,
 * and only as the checker.  The product path never links or calls it.
 *
 * Every function restates one reference function, cited as file:line under
 * /root/reference/proj/include/reattn/.  Arithmetic is compiled with
 * -ffp-contract=off so the fp32 score lanes are "multiply, round, add, round",
 * the variant SURVEY.md §8(c) found in the reference's fused_topk_scores build.
 * Pinned against: oracle/_ref (the reference headers compiled in place, see
 * oracle/Makefile) and the golden fixtures in tests/golden/.
 */
#ifndef REATTN_ORACLE_H
#define REATTN_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORACLE_OK = 0, ORACLE_INVALID_ARGUMENT = 1, ORACLE_OUT_OF_RANGE = 2, ORACLE_LOGIC = 3 };
enum { ORACLE_SPAN_ALIGNED = 0, ORACLE_SPAN_CENTERED = 1 };
enum { ORACLE_LANES_UNFUSED = 0, ORACLE_LANES_FMA = 1 };
enum { ORACLE_MODE_FULL = 0, ORACLE_MODE_WINDOW = 1, ORACLE_MODE_REATTENTION = 2 };

typedef struct {
    size_t k, k_prime, span_m, tile_size, l_global, l_local, l_chunk;
    int span_mode;
} oracle_selection_config;

typedef struct {
    size_t max_position_used;
    size_t ood_positions;
    int coverage_total;
    double entropy_max;
    double entropy_sum;
    size_t entropy_rows;
    size_t scope_len_max;
    size_t scope_len;      /* this step's L' */
    size_t n_spans;
    size_t coverage;
} oracle_step_stats;

/* Lane arithmetic of dot_f32 (process-global; default ORACLE_LANES_UNFUSED). */
void oracle_set_lane_mode(int mode);
int oracle_get_lane_mode(void);
/* dense_matrix.hpp:41-56 — 8 fp32 lanes over j, j+8, ..., fixed tree. */
float oracle_dot_f32(const float* a, const float* b, size_t d);
/* dense_matrix.hpp:59-74 */
double oracle_dot_f64(const float* a, const float* b, size_t d);

/* selection.hpp:139-156: out[n_q][n_kv*d], sequential fp32 add, times float(1/group). */
void oracle_group_mean(const float* q, size_t n_q, size_t n_heads, size_t n_kv, size_t d,
                       float* mq);

/* selection.hpp:168-248 (fused_topk_scores).  keys[h] points at middle row 0 of kv head h,
 * rows are row_stride floats apart.  Output [n_kv][n_q][k] (score desc, index asc);
 * *n_out = min(k, count).  Returns ORACLE_INVALID_ARGUMENT on head mismatch. */
int oracle_topk(const float* q, size_t n_q, size_t n_heads, const float* const* keys, size_t n_kv,
                size_t count, size_t d, size_t row_stride, size_t k, uint64_t* idx_out,
                float* score_out, size_t* n_out);

/* selection.hpp:252-286 (tally_candidates + vote) over a flat candidate list. */
int oracle_vote(const uint64_t* idx, const float* score, size_t n, size_t k_prime,
                uint64_t* winners, size_t* n_winners);

/* selection.hpp:318-349.  Returns ORACLE_OUT_OF_RANGE for a winner >= middle_len. */
int oracle_expand_spans(const uint64_t* winners, size_t n, size_t span_m, size_t middle_len,
                        int mode, uint64_t* begin, uint64_t* end, size_t* n_spans);

/* rope.hpp:21-40: float tables [max_position][d/2] computed in double. */
void oracle_rope_table(size_t d, double base, size_t max_position, float* cos_t, float* sin_t);
/* rope.hpp:49-60 (table row already selected). */
void oracle_rotate_row(float* v, size_t d, const float* c, const float* s);

/* attend.hpp:25-77.  q [n_q][d], k [L][d], v [L][dv]; entropy [n_q]. */
int oracle_attend(const float* q, size_t n_q, const float* k, const float* v, size_t L, size_t d,
                  size_t dv, int has_boundary, size_t boundary, float* out, double* entropy);

/* kv_cache.hpp:65-67 boundary arithmetic. */
void oracle_cache_bounds(size_t total, size_t l_global, size_t l_local_max, size_t* global_end,
                         size_t* local_start);

/* scope.hpp:37-78: source indices for global ++ spans ++ local.  Returns
 * ORACLE_OUT_OF_RANGE (span outside middle) or ORACLE_INVALID_ARGUMENT (> window). */
int oracle_scope_indices(size_t total, size_t l_global, size_t l_local_max, const uint64_t* sb,
                         const uint64_t* se, size_t n_spans, size_t pretrain_window,
                         uint64_t* source_indices, size_t* length);

/* engine.hpp:43-114 (attend_step).  Cache K/V are head-major [n_kv][cap][d] fp32 with
 * `total` rows appended.  out [n_q][n_head*d].  spans_begin/end sized >= k_prime (may be
 * NULL).  rope tables from oracle_rope_table(d, base, max_position). */
int oracle_attend_step(const float* q_pre, size_t n_q, size_t n_head, const float* cache_k,
                       const float* cache_v, size_t n_kv, size_t d, size_t cap, size_t total,
                       const oracle_selection_config* cfg, const float* rope_cos,
                       const float* rope_sin, size_t max_position, int mode, float* out,
                       oracle_step_stats* stats, uint64_t* spans_begin, uint64_t* spans_end);

/* ---- storage-generic, multi-threaded variants (full-size parity tests) ---------------
 * Same arithmetic as above; keys / values are fp32 (ORACLE_DTYPE_F32) or bf16 words
 * (ORACLE_DTYPE_BF16, widened exactly).  n_threads worker threads (>= 1). */
enum { ORACLE_DTYPE_F32 = 0, ORACLE_DTYPE_BF16 = 1 };
int oracle_topk_ex(const float* q, size_t n_q, size_t n_heads, const void* const* keys, int dtype,
                   size_t n_kv, size_t count, size_t d, size_t row_stride, size_t k,
                   int n_threads, uint64_t* idx_out, float* score_out, size_t* n_out);
/* attend_step over a head-major [n_kv][cap][d] cache of `dtype`.  entropy (nullable):
 * [n_q][n_head] row entropies; winners_out (nullable, >= k_prime): the voted winners;
 * cand_idx_out / cand_score_out (nullable, [n_kv][n_q][k]): the per-head top-k lists. */
int oracle_attend_step_ex(const float* q_pre, size_t n_q, size_t n_head, const void* cache_k,
                          const void* cache_v, int dtype, size_t n_kv, size_t d, size_t cap,
                          size_t total, const oracle_selection_config* cfg,
                          const float* rope_cos, const float* rope_sin, size_t max_position,
                          int mode, int n_threads, float* out, double* entropy,
                          oracle_step_stats* stats, uint64_t* spans_begin, uint64_t* spans_end,
                          uint64_t* winners_out, size_t* n_winners_out, uint64_t* cand_idx_out,
                          float* cand_score_out);

/* bf16 round-to-nearest-even of an fp32 value, returned as fp32 (test input helper). */
float oracle_round_bf16(float x);
/* splitmix64(seed, offset+i) -> [-1, 1) (24 significant bits), optionally bf16-rounded;
 * identical to the library's reattn_synth_uniform (test/bench input generator). */
void oracle_synth_uniform(uint64_t seed, uint64_t offset, uint64_t n, float* out, int bf16);

#ifdef __cplusplus
}
#endif
#endif
