/*
 * TEST INFRASTRUCTURE ONLY — see reattn_oracle.h.  CPU restatement of the reference
 * hot path (/root/reference/proj/include/reattn), compiled with -ffp-contract=off.
 * Never linked into the product library.
 */
#include "reattn_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdatomic.h>
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


/* =================================================================================== *
 * Storage-generic, multi-threaded entry points for the full-size parity tests.        *
 * Keys / values may be fp32 rows or bf16 rows (uint16 words, widened exactly), so a   *
 * 1M-4M token device cache is checked from its own bf16 bytes without an fp32 copy.   *
 * The arithmetic is the single-threaded restatement above, unchanged: the top-k is    *
 * split over (kv head, key range) and the per-range lists are merged under the same   *
 * total order (score desc, index asc; selection.hpp:81-135), which selects exactly    *
 * the keys the sequential TopkBuffer keeps; attention runs one head per work item.    *
 * =================================================================================== */

static void load_row(const void* base, int dtype, size_t row, size_t d, float* out) {
    if (dtype == ORACLE_DTYPE_F32) {
        memcpy(out, (const float*)base + row * d, d * sizeof(float));
    } else {
        const uint16_t* p = (const uint16_t*)base + row * d;
        for (size_t c = 0; c < d; ++c) {
            const uint32_t u = (uint32_t)p[c] << 16;
            memcpy(out + c, &u, 4);
        }
    }
}

typedef struct {
    atomic_size_t next;
    size_t n_items;
    void (*fn)(void*, size_t);
    void* arg;
} par_t;

static void* par_worker(void* p) {
    par_t* P = (par_t*)p;
    for (;;) {
        const size_t i = atomic_fetch_add(&P->next, 1);
        if (i >= P->n_items) break;
        P->fn(P->arg, i);
    }
    return NULL;
}

static void par_for(int n_threads, size_t n_items, void (*fn)(void*, size_t), void* arg) {
    par_t P;
    atomic_init(&P.next, 0);
    P.n_items = n_items;
    P.fn = fn;
    P.arg = arg;
    if (n_threads < 1) n_threads = 1;
    if ((size_t)n_threads > n_items) n_threads = (int)(n_items ? n_items : 1);
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * n_threads);
    int started = 0;
    for (int t = 1; t < n_threads; ++t)
        if (pthread_create(&th[t], NULL, par_worker, &P) == 0) ++started, th[started] = th[t];
    par_worker(&P);
    for (int t = 1; t <= started; ++t) pthread_join(th[t], NULL);
    free(th);
}

/* dot_f32 (dense_matrix.hpp:41-56) for d % 8 == 0 with unfused lanes, written on 8-wide
 * vectors: lane t of the vector accumulator IS the reference's lane l_t (element-wise IEEE
 * mul then add, -ffp-contract=off), then the same fixed tree -- bit-identical to
 * oracle_dot_f32, several times faster (used by the bulk paths below). */
typedef float v8f __attribute__((vector_size(32)));
static inline float dot_f32_v8(const float* a, const float* b, size_t d) {
    v8f l = {0, 0, 0, 0, 0, 0, 0, 0};
    for (size_t j = 0; j < d; j += 8) {
        v8f x, y;
        memcpy(&x, a + j, 32);
        memcpy(&y, b + j, 32);
        l = l + x * y;
    }
    return ((l[0] + l[1]) + (l[2] + l[3])) + ((l[4] + l[5]) + (l[6] + l[7]));
}
static inline float dot_fast(const float* a, const float* b, size_t d) {
    if (g_lane_mode == ORACLE_LANES_UNFUSED && d % 8 == 0) return dot_f32_v8(a, b, d);
    return oracle_dot_f32(a, b, d);
}

static int better_entry(float sa, uint64_t ia, float sb, uint64_t ib) {
    return sa > sb || (sa == sb && ia < ib);
}

/* insert (s, i) into a sorted (score desc, index asc) list of capacity kk holding *filled */
static void list_offer(float* bs, uint64_t* bi, size_t kk, size_t* filled, float s, uint64_t i) {
    if (*filled == kk && !better_entry(s, i, bs[kk - 1], bi[kk - 1])) return;
    size_t p = *filled < kk ? *filled : kk - 1;
    while (p > 0 && better_entry(s, i, bs[p - 1], bi[p - 1])) {
        bs[p] = bs[p - 1];
        bi[p] = bi[p - 1];
        --p;
    }
    bs[p] = s;
    bi[p] = i;
    if (*filled < kk) ++*filled;
}

typedef struct {
    const float* mq;  /* [n_q][n_kv*d] */
    const void* const* keys;
    int dtype;
    size_t n_q, n_kv, count, d, row_stride, kk, chunk, n_chunks;
    float* ls;        /* [n_kv][n_chunks][n_q][kk] */
    uint64_t* li;
    size_t* lf;       /* [n_kv][n_chunks][n_q] */
} topk_job;

static void topk_item(void* p, size_t item) {
    topk_job* J = (topk_job*)p;
    const size_t kv = item / J->n_chunks, ch = item % J->n_chunks;
    const size_t r0 = ch * J->chunk, r1 = r0 + J->chunk < J->count ? r0 + J->chunk : J->count;
    const size_t d = J->d;
    enum { RB = 64 };
    float* rows = (float*)malloc(sizeof(float) * RB * d);
    float* ls = J->ls + (kv * J->n_chunks + ch) * J->n_q * J->kk;
    uint64_t* li = J->li + (kv * J->n_chunks + ch) * J->n_q * J->kk;
    size_t* lf = J->lf + (kv * J->n_chunks + ch) * J->n_q;
    for (size_t q = 0; q < J->n_q; ++q) lf[q] = 0;
    for (size_t b0 = r0; b0 < r1; b0 += RB) {
        const size_t nb = b0 + RB < r1 ? RB : r1 - b0;
        for (size_t r = 0; r < nb; ++r)
            if (J->dtype == ORACLE_DTYPE_F32)
                memcpy(rows + r * d, (const float*)J->keys[kv] + (b0 + r) * J->row_stride,
                       d * sizeof(float));
            else
                load_row((const uint16_t*)J->keys[kv] + (b0 + r) * J->row_stride, ORACLE_DTYPE_BF16,
                         0, d, rows + r * d);
        for (size_t q = 0; q < J->n_q; ++q) {
            const float* qrow = J->mq + q * J->n_kv * d + kv * d;
            float* bs = ls + q * J->kk;
            uint64_t* bi = li + q * J->kk;
            for (size_t r = 0; r < nb; ++r) {
                const float sc = dot_fast(qrow, rows + r * d, d);
                /* rows arrive in ascending index order: once full, only a strictly larger
                 * score can enter (selection.hpp:230-236) */
                if (lf[q] == J->kk && !(sc > bs[J->kk - 1])) continue;
                list_offer(bs, bi, J->kk, &lf[q], sc, b0 + r);
            }
        }
    }
    free(rows);
}

int oracle_topk_ex(const float* q, size_t n_q, size_t n_heads, const void* const* keys, int dtype,
                   size_t n_kv, size_t count, size_t d, size_t row_stride, size_t k,
                   int n_threads, uint64_t* idx_out, float* score_out, size_t* n_out) {
    if (n_kv == 0 || n_heads % n_kv != 0) return ORACLE_INVALID_ARGUMENT;
    const size_t kk = count < k ? count : k;
    *n_out = kk;
    if (count == 0 || n_q == 0) return ORACLE_OK;
    float* mq = (float*)malloc(sizeof(float) * n_q * n_kv * d);
    oracle_group_mean(q, n_q, n_heads, n_kv, d, mq);
    topk_job J;
    J.mq = mq;
    J.keys = keys;
    J.dtype = dtype;
    J.n_q = n_q;
    J.n_kv = n_kv;
    J.count = count;
    J.d = d;
    J.row_stride = row_stride;
    J.kk = kk;
    /* enough items to keep every thread busy, ranges of >= 2048 rows */
    size_t want = (size_t)(n_threads > 1 ? n_threads : 1) * 4 / n_kv + 1;
    size_t chunk = (count + want - 1) / want;
    if (chunk < 2048) chunk = 2048;
    J.chunk = chunk;
    J.n_chunks = (count + chunk - 1) / chunk;
    J.ls = (float*)malloc(sizeof(float) * n_kv * J.n_chunks * n_q * kk);
    J.li = (uint64_t*)malloc(sizeof(uint64_t) * n_kv * J.n_chunks * n_q * kk);
    J.lf = (size_t*)malloc(sizeof(size_t) * n_kv * J.n_chunks * n_q);
    par_for(n_threads, n_kv * J.n_chunks, topk_item, &J);
    for (size_t kv = 0; kv < n_kv; ++kv)
        for (size_t qq = 0; qq < n_q; ++qq) {
            uint64_t* bi = idx_out + (kv * n_q + qq) * k;
            float* bs = score_out + (kv * n_q + qq) * k;
            size_t filled = 0;
            for (size_t ch = 0; ch < J.n_chunks; ++ch) {
                const size_t base = (kv * J.n_chunks + ch) * n_q + qq;
                for (size_t e = 0; e < J.lf[base]; ++e)
                    list_offer(bs, bi, kk, &filled, J.ls[base * kk + e], J.li[base * kk + e]);
            }
        }
    free(J.ls);
    free(J.li);
    free(J.lf);
    free(mq);
    return ORACLE_OK;
}

typedef struct {
    const float* q_pre;
    size_t n_q, n_head, n_kv, d, L, group;
    const float* krot;  /* [n_kv][L][d] rotated */
    const float* vmat;
    const float* rope_cos;
    const float* rope_sin;
    float* out;
    double* ent;        /* [n_head][n_q] */
} attn_job;

static void attn_item(void* p, size_t h) {
    attn_job* J = (attn_job*)p;
    const size_t d = J->d, n_q = J->n_q, half = d / 2, kv = h / J->group;
    float* qh = (float*)malloc(sizeof(float) * n_q * d + 1);
    float* oh = (float*)malloc(sizeof(float) * n_q * d + 1);
    for (size_t i = 0; i < n_q; ++i) {
        memcpy(qh + i * d, J->q_pre + i * J->n_head * d + h * d, d * sizeof(float));
        const size_t pos = J->L - n_q + i;
        oracle_rotate_row(qh + i * d, d, J->rope_cos + pos * half, J->rope_sin + pos * half);
    }
    oracle_attend(qh, n_q, J->krot + kv * J->L * d, J->vmat + kv * J->L * d, J->L, d, d, 1,
                  J->L - n_q, oh, J->ent + h * n_q);
    for (size_t i = 0; i < n_q; ++i)
        memcpy(J->out + i * J->n_head * d + h * d, oh + i * d, d * sizeof(float));
    free(qh);
    free(oh);
}

int oracle_attend_step_ex(const float* q_pre, size_t n_q, size_t n_head, const void* cache_k,
                          const void* cache_v, int dtype, size_t n_kv, size_t d, size_t cap,
                          size_t total, const oracle_selection_config* cfg,
                          const float* rope_cos, const float* rope_sin, size_t max_position,
                          int mode, int n_threads, float* out, double* entropy,
                          oracle_step_stats* stats, uint64_t* spans_begin, uint64_t* spans_end,
                          uint64_t* winners_out, size_t* n_winners_out, uint64_t* cand_idx_out,
                          float* cand_score_out) {
    if (n_head % n_kv != 0) return ORACLE_INVALID_ARGUMENT;
    const size_t group = n_head / n_kv;
    const size_t esz = dtype == ORACLE_DTYPE_F32 ? 4 : 2;
    size_t g_end, l_start;
    oracle_cache_bounds(total, cfg->l_global, cfg->l_local, &g_end, &l_start);
    const size_t middle_len = l_start - g_end;
    size_t n_spans = 0;
    uint64_t* sb = (uint64_t*)malloc(sizeof(uint64_t) * (cfg->k_prime + 1));
    uint64_t* se = (uint64_t*)malloc(sizeof(uint64_t) * (cfg->k_prime + 1));
    int rc = ORACLE_OK;
    if (n_winners_out) *n_winners_out = 0;
    /* engine.hpp:58-63 */
    if (mode == ORACLE_MODE_REATTENTION && cfg->k_prime > 0 && middle_len > 0) {
        const void** heads = (const void**)malloc(sizeof(void*) * n_kv);
        for (size_t h = 0; h < n_kv; ++h)
            heads[h] = (const uint8_t*)cache_k + (h * cap + g_end) * d * esz;
        const size_t kk = cfg->k;
        uint64_t* ci = (uint64_t*)malloc(sizeof(uint64_t) * n_kv * n_q * kk);
        float* cs = (float*)malloc(sizeof(float) * n_kv * n_q * kk);
        size_t nk = 0;
        rc = oracle_topk_ex(q_pre, n_q, n_head, heads, dtype, n_kv, middle_len, d, d, kk,
                            n_threads, ci, cs, &nk);
        if (rc == ORACLE_OK && cand_idx_out) { /* [n_kv][n_q][k] lists, min(k, middle) valid */
            memcpy(cand_idx_out, ci, sizeof(uint64_t) * n_kv * n_q * kk);
            memcpy(cand_score_out, cs, sizeof(float) * n_kv * n_q * kk);
        }
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
        if (rc == ORACLE_OK && winners_out) {
            memcpy(winners_out, winners, nw * sizeof(uint64_t));
            *n_winners_out = nw;
        }
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
    /* scope.hpp:63-76 copies, engine.hpp:78-81 key rotation at compact i */
    const size_t half = d / 2;
    float* krot = (float*)malloc(sizeof(float) * n_kv * L * d + 1);
    float* vmat = (float*)malloc(sizeof(float) * n_kv * L * d + 1);
    for (size_t kv = 0; kv < n_kv; ++kv)
        for (size_t i = 0; i < L; ++i) {
            load_row(cache_k, dtype, kv * cap + src[i], d, krot + (kv * L + i) * d);
            load_row(cache_v, dtype, kv * cap + src[i], d, vmat + (kv * L + i) * d);
            oracle_rotate_row(krot + (kv * L + i) * d, d, rope_cos + i * half, rope_sin + i * half);
        }
    double* ent = (double*)malloc(sizeof(double) * n_head * n_q + 1);
    attn_job A = {q_pre, n_q, n_head, n_kv, d, L, group, krot, vmat, rope_cos, rope_sin, out, ent};
    par_for(n_threads, n_head, attn_item, &A);
    /* engine.hpp:100-112 statistics, accumulated in the reference's (h, i) order */
    if (stats) {
        for (size_t h = 0; h < n_head; ++h) {
            for (size_t i = 0; i < n_q; ++i) {
                const double e = ent[h * n_q + i];
                if (e > stats->entropy_max) stats->entropy_max = e;
                stats->entropy_sum += e;
            }
            stats->entropy_rows += n_q;
        }
        for (size_t i = 0; i < L; ++i)
            if (i >= max_position) ++stats->ood_positions;
        for (size_t i = 0; i < n_q; ++i)
            if (L - n_q + i >= max_position) stats->ood_positions += n_head;
        if (L > stats->scope_len_max) stats->scope_len_max = L;
        if (L - 1 > stats->max_position_used) stats->max_position_used = L - 1;
        stats->scope_len = L;
        stats->n_spans = n_spans;
        stats->coverage = coverage;
    }
    if (entropy)  /* [n_q][n_head], the layout of the library's entropy rows */
        for (size_t h = 0; h < n_head; ++h)
            for (size_t i = 0; i < n_q; ++i) entropy[i * n_head + h] = ent[h * n_q + i];
    free(ent);
    free(src);
    free(krot);
    free(vmat);
    return ORACLE_OK;
}
