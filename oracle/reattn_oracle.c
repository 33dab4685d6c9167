/*
 * TEST INFRASTRUCTURE ONLY — see reattn_oracle.h.  CPU restatement of the reference
 * hot path (/root/reference/proj/include/reattn), compiled with -ffp-contract=off.
 * Never linked into the product library.
 */
#include "reattn_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ---- dense_matrix.hpp:41-56 ---------------------------------------------------- */
/* The reference's lane update `l += a*b` is contracted to an FMA or not depending on
 * the compiler, -march and d (ref_fma_selfcheck measures it per build).
 * Both variants are restated; ORACLE_LANES_UNFUSED is the d=128 reference build. */
static int g_lane_mode = ORACLE_LANES_UNFUSED;
void oracle_set_lane_mode(int mode) { g_lane_mode = mode; }
int oracle_get_lane_mode(void) { return g_lane_mode; }

float oracle_dot_f32(const float* a, const float* b, size_t d) {
    float l[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    size_t j = 0;
    if (g_lane_mode == ORACLE_LANES_FMA) {
        for (; j + 8 <= d; j += 8)
            for (int t = 0; t < 8; ++t) l[t] = fmaf(a[j + t], b[j + t], l[t]);
        for (; j < d; ++j) l[0] = fmaf(a[j], b[j], l[0]);
    } else {
        for (; j + 8 <= d; j += 8)
            for (int t = 0; t < 8; ++t) l[t] += a[j + t] * b[j + t];
        for (; j < d; ++j) l[0] += a[j] * b[j];
    }
    return ((l[0] + l[1]) + (l[2] + l[3])) + ((l[4] + l[5]) + (l[6] + l[7]));
}

/* ---- dense_matrix.hpp:59-74 ---------------------------------------------------- */
double oracle_dot_f64(const float* a, const float* b, size_t d) {
    double l[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    size_t j = 0;
    for (; j + 8 <= d; j += 8)
        for (int t = 0; t < 8; ++t) l[t] += (double)a[j + t] * (double)b[j + t];
    for (; j < d; ++j) l[0] += (double)a[j] * (double)b[j];
    return ((l[0] + l[1]) + (l[2] + l[3])) + ((l[4] + l[5]) + (l[6] + l[7]));
}

/* ---- selection.hpp:139-156 ----------------------------------------------------- */
void oracle_group_mean(const float* q, size_t n_q, size_t n_heads, size_t n_kv, size_t d,
                       float* mq) {
    const size_t group = n_heads / n_kv;
    const float inv = 1.0f / (float)group;
    for (size_t r = 0; r < n_q; ++r) {
        const float* src = q + r * n_heads * d;
        float* dst = mq + r * n_kv * d;
        for (size_t kv = 0; kv < n_kv; ++kv)
            for (size_t c = 0; c < d; ++c) {
                float acc = 0.0f;
                for (size_t g = 0; g < group; ++g) acc += src[(kv * group + g) * d + c];
                dst[kv * d + c] = acc * inv;
            }
    }
}

/* ---- selection.hpp:81-135 + 275-355 -------------------------------------------- */
/* Running exact top-k: candidates arrive in ascending index order; a score equal to
 * the current worst never displaces it (selection.hpp:124), so ties keep the lower
 * index.  The buffer is kept sorted (score desc, index asc), which is what
 * TopkBuffer::sorted() returns (selection.hpp:127-134). */
int oracle_topk(const float* q, size_t n_q, size_t n_heads, const float* const* keys, size_t n_kv,
                size_t count, size_t d, size_t row_stride, size_t k, uint64_t* idx_out,
                float* score_out, size_t* n_out) {
    if (n_kv == 0 || n_heads % n_kv != 0) return ORACLE_INVALID_ARGUMENT;
    const size_t kk = count < k ? count : k;
    *n_out = kk;
    if (count == 0 || n_q == 0) return ORACLE_OK;
    float* mq = (float*)malloc(sizeof(float) * n_q * n_kv * d);
    oracle_group_mean(q, n_q, n_heads, n_kv, d, mq);
    for (size_t kv = 0; kv < n_kv; ++kv)
        for (size_t qq = 0; qq < n_q; ++qq) {
            uint64_t* bi = idx_out + (kv * n_q + qq) * k;
            float* bs = score_out + (kv * n_q + qq) * k;
            size_t filled = 0;
            const float* qrow = mq + qq * n_kv * d + kv * d;
            for (size_t i = 0; i < count; ++i) {
                const float s = oracle_dot_f32(qrow, keys[kv] + i * row_stride, d);
                if (filled == kk && !(s > bs[kk - 1])) continue;
                size_t p = filled < kk ? filled : kk - 1;  /* slot to fill/replace */
                while (p > 0 && s > bs[p - 1]) {
                    bs[p] = bs[p - 1];
                    bi[p] = bi[p - 1];
                    --p;
                }
                bs[p] = s;
                bi[p] = i;
                if (filled < kk) ++filled;
            }
        }
    free(mq);
    return ORACLE_OK;
}

/* ---- selection.hpp:252-286 ----------------------------------------------------- */
typedef struct {
    uint64_t idx;
    float score;
    size_t votes;
} cand_t;

static int cmp_idx(const void* a, const void* b) {
    const cand_t* x = (const cand_t*)a;
    const cand_t* y = (const cand_t*)b;
    return x->idx < y->idx ? -1 : (x->idx > y->idx ? 1 : 0);
}
static int cmp_rank(const void* a, const void* b) {
    const cand_t* x = (const cand_t*)a;
    const cand_t* y = (const cand_t*)b;
    if (x->votes != y->votes) return x->votes > y->votes ? -1 : 1;
    if (x->score != y->score) return x->score > y->score ? -1 : 1;
    return x->idx < y->idx ? -1 : (x->idx > y->idx ? 1 : 0);
}

int oracle_vote(const uint64_t* idx, const float* score, size_t n, size_t k_prime,
                uint64_t* winners, size_t* n_winners) {
    *n_winners = 0;
    if (k_prime == 0 || n == 0) return ORACLE_OK;
    cand_t* flat = (cand_t*)malloc(sizeof(cand_t) * n);
    for (size_t i = 0; i < n; ++i) flat[i] = (cand_t){idx[i], score[i], 1};
    qsort(flat, n, sizeof(cand_t), cmp_idx);
    size_t u = 0;
    for (size_t i = 0; i < n; ++i) {
        if (u > 0 && flat[u - 1].idx == flat[i].idx) {
            flat[u - 1].votes += 1;
            /* std::max(a, b) keeps a unless a < b */
            if (flat[u - 1].score < flat[i].score) flat[u - 1].score = flat[i].score;
        } else {
            flat[u++] = flat[i];
        }
    }
    qsort(flat, u, sizeof(cand_t), cmp_rank);
    const size_t m = u < k_prime ? u : k_prime;
    for (size_t i = 0; i < m; ++i) winners[i] = flat[i].idx;
    *n_winners = m;
    free(flat);
    return ORACLE_OK;
}

/* ---- selection.hpp:318-349 ----------------------------------------------------- */
typedef struct {
    uint64_t b, e;
} span_t;
static int cmp_span(const void* a, const void* b) {
    const span_t* x = (const span_t*)a;
    const span_t* y = (const span_t*)b;
    if (x->b != y->b) return x->b < y->b ? -1 : 1;
    if (x->e != y->e) return x->e < y->e ? -1 : 1;
    return 0;
}

int oracle_expand_spans(const uint64_t* winners, size_t n, size_t span_m, size_t middle_len,
                        int mode, uint64_t* begin, uint64_t* end, size_t* n_spans) {
    *n_spans = 0;
    if (n == 0 || middle_len == 0) return ORACLE_OK;
    span_t* raw = (span_t*)malloc(sizeof(span_t) * n);
    for (size_t i = 0; i < n; ++i) {
        const uint64_t w = winners[i];
        if (w >= middle_len) {
            free(raw);
            return ORACLE_OUT_OF_RANGE;
        }
        uint64_t start;
        if (mode == ORACLE_SPAN_ALIGNED) {
            start = (w / span_m) * span_m;
        } else {
            start = w > span_m / 2 ? w - span_m / 2 : 0;
            if (start + span_m > middle_len) start = middle_len > span_m ? middle_len - span_m : 0;
        }
        const uint64_t e = start + span_m < middle_len ? start + span_m : middle_len;
        raw[i] = (span_t){start, e};
    }
    qsort(raw, n, sizeof(span_t), cmp_span);
    size_t m = 0;
    for (size_t i = 0; i < n; ++i) {
        if (m > 0 && raw[i].b <= end[m - 1] && mode == ORACLE_SPAN_CENTERED) {
            if (raw[i].e > end[m - 1]) end[m - 1] = raw[i].e;
        } else if (m > 0 && raw[i].b == begin[m - 1] && raw[i].e == end[m - 1]) {
            continue;
        } else {
            begin[m] = raw[i].b;
            end[m] = raw[i].e;
            ++m;
        }
    }
    *n_spans = m;
    free(raw);
    return ORACLE_OK;
}

/* ---- rope.hpp:21-60 ---------------------------------------------------------- */
void oracle_rope_table(size_t d, double base, size_t max_position, float* cos_t, float* sin_t) {
    const size_t half = d / 2;
    double* inv_freq = (double*)malloc(sizeof(double) * half);
    for (size_t i = 0; i < half; ++i) inv_freq[i] = pow(base, -2.0 * (double)i / (double)d);
    for (size_t p = 0; p < max_position; ++p)
        for (size_t i = 0; i < half; ++i) {
            const double angle = (double)p * inv_freq[i];
            cos_t[p * half + i] = (float)cos(angle);
            sin_t[p * half + i] = (float)sin(angle);
        }
    free(inv_freq);
}

void oracle_rotate_row(float* v, size_t d, const float* c, const float* s) {
    for (size_t i = 0; i < d / 2; ++i) {
        const float x = v[2 * i];
        const float y = v[2 * i + 1];
        v[2 * i] = x * c[i] - y * s[i];
        v[2 * i + 1] = x * s[i] + y * c[i];
    }
}

/* ---- attend.hpp:25-77 -------------------------------------------------------- */
int oracle_attend(const float* q, size_t n_q, const float* k, const float* v, size_t L, size_t d,
                  size_t dv, int has_boundary, size_t boundary, float* out, double* entropy) {
    if (L == 0) return ORACLE_INVALID_ARGUMENT;
    const double scale = 1.0 / sqrt((double)d);
    double* acc = (double*)malloc(sizeof(double) * (dv ? dv : 1));
    for (size_t i = 0; i < n_q; ++i) {
        size_t visible = L;
        if (has_boundary && boundary + i + 1 < visible) visible = boundary + i + 1;
        const float* qrow = q + i * d;
        double m = -INFINITY, denom = 0.0, ent = 0.0;
        for (size_t c = 0; c < dv; ++c) acc[c] = 0.0;
        for (size_t j = 0; j < visible; ++j) {
            const double s = oracle_dot_f64(qrow, k + j * d, d) * scale;
            const float* vrow = v + j * dv;
            if (s <= m) {
                const double w = exp(s - m);
                denom += w;
                ent += (s - m) * w;
                for (size_t c = 0; c < dv; ++c) acc[c] += w * (double)vrow[c];
            } else if (denom == 0.0) {
                m = s;
                denom = 1.0;
                for (size_t c = 0; c < dv; ++c) acc[c] = (double)vrow[c];
            } else {
                const double r = exp(m - s);
                ent = r * (ent + (m - s) * denom);
                denom = denom * r + 1.0;
                for (size_t c = 0; c < dv; ++c) acc[c] = acc[c] * r + (double)vrow[c];
                m = s;
            }
        }
        for (size_t c = 0; c < dv; ++c) out[i * dv + c] = (float)(acc[c] / denom);
        const double h = log(denom) - ent / denom;
        entropy[i] = h < 0.0 ? 0.0 : h;
    }
    free(acc);
    return ORACLE_OK;
}

/* ---- kv_cache.hpp:65-67 -------------------------------------------------------- */
void oracle_cache_bounds(size_t total, size_t l_global, size_t l_local_max, size_t* global_end,
                         size_t* local_start) {
    const size_t g = total < l_global ? total : l_global;
    const size_t rest = total - g;
    *global_end = g;
    *local_start = total - (rest < l_local_max ? rest : l_local_max);
}

/* ---- scope.hpp:37-78 (index part) -------------------------------------------- */
int oracle_scope_indices(size_t total, size_t l_global, size_t l_local_max, const uint64_t* sb,
                         const uint64_t* se, size_t n_spans, size_t pretrain_window,
                         uint64_t* source_indices, size_t* length) {
    size_t g_end, l_start;
    oracle_cache_bounds(total, l_global, l_local_max, &g_end, &l_start);
    const size_t middle_len = l_start - g_end;
    size_t selected = 0;
    for (size_t s = 0; s < n_spans; ++s) {
        if (se[s] > middle_len) return ORACLE_OUT_OF_RANGE;
        selected += se[s] - sb[s];
    }
    const size_t L = g_end + selected + (total - l_start);
    *length = L;
    if (L > pretrain_window) return ORACLE_INVALID_ARGUMENT;
    if (source_indices) {
        size_t r = 0;
        for (size_t i = 0; i < g_end; ++i) source_indices[r++] = i;
        for (size_t s = 0; s < n_spans; ++s)
            for (uint64_t i = sb[s]; i < se[s]; ++i) source_indices[r++] = g_end + i;
        for (size_t i = l_start; i < total; ++i) source_indices[r++] = i;
    }
    return ORACLE_OK;
}

/* ---- engine.hpp:43-114 -------------------------------------------------------- */
int oracle_attend_step(const float* q_pre, size_t n_q, size_t n_head, const float* cache_k,
                       const float* cache_v, size_t n_kv, size_t d, size_t cap, size_t total,
                       const oracle_selection_config* cfg, const float* rope_cos,
                       const float* rope_sin, size_t max_position, int mode, float* out,
                       oracle_step_stats* stats, uint64_t* spans_begin, uint64_t* spans_end) {
    if (n_head % n_kv != 0) return ORACLE_INVALID_ARGUMENT;
    const size_t group = n_head / n_kv;
    size_t g_end, l_start;
    oracle_cache_bounds(total, cfg->l_global, cfg->l_local, &g_end, &l_start);
    const size_t middle_len = l_start - g_end;

    size_t n_spans = 0;
    uint64_t* sb = (uint64_t*)malloc(sizeof(uint64_t) * (cfg->k_prime + 1));
    uint64_t* se = (uint64_t*)malloc(sizeof(uint64_t) * (cfg->k_prime + 1));
    int rc = ORACLE_OK;
    if (mode == ORACLE_MODE_REATTENTION && cfg->k_prime > 0 && middle_len > 0) {
        const float** heads = (const float**)malloc(sizeof(float*) * n_kv);
        for (size_t h = 0; h < n_kv; ++h) heads[h] = cache_k + (h * cap + g_end) * d;
        const size_t kk = cfg->k;
        uint64_t* ci = (uint64_t*)malloc(sizeof(uint64_t) * n_kv * n_q * kk);
        float* cs = (float*)malloc(sizeof(float) * n_kv * n_q * kk);
        size_t nk = 0;
        rc = oracle_topk(q_pre, n_q, n_head, heads, n_kv, middle_len, d, d, kk, ci, cs, &nk);
        /* flatten [kv][q][0..nk) as tally_candidates does (selection.hpp:254-256) */
        size_t nf = 0;
        for (size_t l = 0; l < n_kv * n_q; ++l)
            for (size_t j = 0; j < nk; ++j) {
                ci[nf] = ci[l * kk + j];
                cs[nf] = cs[l * kk + j];
                ++nf;
            }
        uint64_t* winners = (uint64_t*)malloc(sizeof(uint64_t) * (cfg->k_prime + 1));
        size_t nw = 0;
        if (rc == ORACLE_OK) rc = oracle_vote(ci, cs, nf, cfg->k_prime, winners, &nw);
        if (rc == ORACLE_OK)
            rc = oracle_expand_spans(winners, nw, cfg->span_m, middle_len, cfg->span_mode, sb, se,
                                     &n_spans);
        free(winners);
        free(ci);
        free(cs);
        free(heads);
    }
    if (rc != ORACLE_OK) {
        free(sb);
        free(se);
        return rc;
    }
    size_t coverage = 0;
    for (size_t s = 0; s < n_spans; ++s) coverage += se[s] - sb[s];
    if (stats && coverage != middle_len) stats->coverage_total = 0;
    if (spans_begin)
        for (size_t s = 0; s < n_spans; ++s) {
            spans_begin[s] = sb[s];
            spans_end[s] = se[s];
        }

    size_t L = 0;
    rc = oracle_scope_indices(total, cfg->l_global, cfg->l_local, sb, se, n_spans, max_position,
                              NULL, &L);
    if (rc != ORACLE_OK) {
        free(sb);
        free(se);
        return rc;
    }
    uint64_t* src = (uint64_t*)malloc(sizeof(uint64_t) * (L ? L : 1));
    oracle_scope_indices(total, cfg->l_global, cfg->l_local, sb, se, n_spans, max_position, src,
                         &L);
    free(sb);
    free(se);
    if (n_q > L) {
        free(src);
        return ORACLE_LOGIC;
    }
    const size_t half = d / 2;
    float* krot = (float*)malloc(sizeof(float) * n_kv * L * d + 1);
    float* vmat = (float*)malloc(sizeof(float) * n_kv * L * d + 1);
    for (size_t kv = 0; kv < n_kv; ++kv)
        for (size_t i = 0; i < L; ++i) {
            memcpy(krot + (kv * L + i) * d, cache_k + (kv * cap + src[i]) * d, d * sizeof(float));
            memcpy(vmat + (kv * L + i) * d, cache_v + (kv * cap + src[i]) * d, d * sizeof(float));
            if (stats && i >= max_position) ++stats->ood_positions;
            oracle_rotate_row(krot + (kv * L + i) * d, d, rope_cos + i * half, rope_sin + i * half);
        }
    float* qh = (float*)malloc(sizeof(float) * n_q * d + 1);
    float* oh = (float*)malloc(sizeof(float) * n_q * d + 1);
    double* ent = (double*)malloc(sizeof(double) * n_q + 1);
    for (size_t h = 0; h < n_head; ++h) {
        const size_t kv = h / group;
        for (size_t i = 0; i < n_q; ++i) {
            memcpy(qh + i * d, q_pre + i * n_head * d + h * d, d * sizeof(float));
            const size_t pos = L - n_q + i;
            if (stats && pos >= max_position) ++stats->ood_positions;
            oracle_rotate_row(qh + i * d, d, rope_cos + pos * half, rope_sin + pos * half);
        }
        oracle_attend(qh, n_q, krot + kv * L * d, vmat + kv * L * d, L, d, d, 1, L - n_q, oh, ent);
        for (size_t i = 0; i < n_q; ++i)
            memcpy(out + i * n_head * d + h * d, oh + i * d, d * sizeof(float));
        if (stats) {
            for (size_t i = 0; i < n_q; ++i) {
                if (ent[i] > stats->entropy_max) stats->entropy_max = ent[i];
                stats->entropy_sum += ent[i];
            }
            stats->entropy_rows += n_q;
        }
    }
    if (stats) {
        if (L > stats->scope_len_max) stats->scope_len_max = L;
        if (L - 1 > stats->max_position_used) stats->max_position_used = L - 1;
        stats->scope_len = L;
        stats->n_spans = n_spans;
        stats->coverage = coverage;
    }
    free(src);
    free(krot);
    free(vmat);
    free(qh);
    free(oh);
    free(ent);
    return ORACLE_OK;
}

/* Host twin of the library's synthetic generator (misc.cu synth_value). */
void oracle_synth_uniform(uint64_t seed, uint64_t offset, uint64_t n, float* out, int bf16) {
    for (uint64_t e = 0; e < n; ++e) {
        uint64_t z = seed * 0x9E3779B97F4A7C15ull + (offset + e) + 0x632BE59BD9B4E019ull;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        z ^= z >> 31;
        const float v = (float)(z >> 40) * (1.0f / 8388608.0f) - 1.0f;
        out[e] = bf16 ? oracle_round_bf16(v) : v;
    }
}

float oracle_round_bf16(float x) {
    uint32_t u;
    memcpy(&u, &x, 4);
    if ((u & 0x7f800000u) == 0x7f800000u) { /* inf / nan: truncate */
        u &= 0xffff0000u;
    } else {
        u += 0x7fffu + ((u >> 16) & 1u);
        u &= 0xffff0000u;
    }
    float y;
    memcpy(&y, &u, 4);
    return y;
}
