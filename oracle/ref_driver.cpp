// TEST INFRASTRUCTURE ONLY.  Thin extern "C" shim around the UNMODIFIED reference
// headers, compiled in place from /root/reference/proj/include (see oracle/Makefile);
// the output library lives in oracle/_ref/ and is git-ignored.  Used to pin the C
// restatement (oracle/reattn_oracle.c), to generate tests/golden fixtures, and as the
// "reference" CPU arm of bench.py.  No reference source is copied into this repo.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <optional>
#include <random>
#include <stdexcept>
#include <span>
#include <string>
#include <vector>

#include "reattn/attend.hpp"
#include "reattn/engine.hpp"
#include "reattn/full_attention.hpp"
#include "reattn/model.hpp"
#include "reattn/window_reference.hpp"
#include "reattn/kv_cache.hpp"
#include "reattn/rope.hpp"
#include "reattn/scope.hpp"
#include "reattn/selection.hpp"
#include "reattn/selection_reference.hpp"

using namespace reattn;

namespace {
thread_local std::string g_err;
int fail(const std::exception& e, int code) {
    g_err = e.what();
    return code;
}
#define REF_TRY(body)                                          \
    try {                                                      \
        body;                                                  \
    } catch (const std::out_of_range& e) {                     \
        return fail(e, 2);                                     \
    } catch (const std::invalid_argument& e) {                 \
        return fail(e, 1);                                     \
    } catch (const std::logic_error& e) {                      \
        return fail(e, 3);                                     \
    } catch (const std::exception& e) {                        \
        return fail(e, 5);                                     \
    }                                                          \
    return 0;

DenseMatrix to_matrix(const float* p, std::size_t r, std::size_t c) {
    DenseMatrix m(r, c);
    if (r * c) std::memcpy(m.values.data(), p, r * c * sizeof(float));
    return m;
}

void write_topk(const PerHeadTopk& res, std::size_t k, uint64_t* idx, float* score,
                std::size_t* n_out) {
    std::size_t n = 0;
    for (std::size_t kv = 0; kv < res.size(); ++kv)
        for (std::size_t q = 0; q < res[kv].size(); ++q) {
            n = res[kv][q].size();
            for (std::size_t j = 0; j < n; ++j) {
                idx[(kv * res[kv].size() + q) * k + j] = res[kv][q][j].index;
                score[(kv * res[kv].size() + q) * k + j] = res[kv][q][j].score;
            }
        }
    *n_out = n;
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// selection.hpp:168 fused_topk_scores.  keys[h]: middle rows of head h (row_stride == d).
int ref_fused_topk(const float* q, std::size_t n_q, std::size_t n_heads, const float* const* keys,
                   std::size_t n_kv, std::size_t count, std::size_t d, std::size_t k,
                   std::size_t tile, uint64_t* idx, float* score, std::size_t* n_out,
                   std::size_t* peak_scratch) {
    REF_TRY({
        std::vector<KeySegmentView> views;
        for (std::size_t h = 0; h < n_kv; ++h) views.push_back(KeySegmentView{keys[h], count, d});
        SelectionConfig cfg;
        cfg.k = k;
        cfg.tile_size = tile;
        ScratchMeter meter;
        const PerHeadTopk res =
            fused_topk_scores(to_matrix(q, n_q, n_heads * d), n_heads, views, cfg, &meter);
        write_topk(res, k, idx, score, n_out);
        if (peak_scratch) *peak_scratch = meter.peak;
    })
}

// selection_reference.hpp:18 naive_topk_scores.
int ref_naive_topk(const float* q, std::size_t n_q, std::size_t n_heads, const float* const* keys,
                   std::size_t n_kv, std::size_t count, std::size_t d, std::size_t k,
                   uint64_t* idx, float* score, std::size_t* n_out, std::size_t* peak_scratch) {
    REF_TRY({
        std::vector<KeySegmentView> views;
        for (std::size_t h = 0; h < n_kv; ++h) views.push_back(KeySegmentView{keys[h], count, d});
        SelectionConfig cfg;
        cfg.k = k;
        ScratchMeter meter;
        const PerHeadTopk res =
            naive_topk_scores(to_matrix(q, n_q, n_heads * d), n_heads, views, cfg, &meter);
        write_topk(res, k, idx, score, n_out);
        if (peak_scratch) *peak_scratch = meter.peak;
    })
}

// selection.hpp:278 vote over one flat list (one (kv,q) slot per candidate is enough:
// tally_candidates flattens anyway).
int ref_vote(const uint64_t* idx, const float* score, std::size_t n, std::size_t k_prime,
             uint64_t* winners, std::size_t* n_winners) {
    REF_TRY({
        PerHeadTopk ph(1, std::vector<std::vector<TopkEntry>>(1));
        for (std::size_t i = 0; i < n; ++i) ph[0][0].push_back(TopkEntry{idx[i], score[i]});
        const auto w = vote(ph, k_prime);
        for (std::size_t i = 0; i < w.size(); ++i) winners[i] = w[i];
        *n_winners = w.size();
    })
}

// selection.hpp:318 expand_spans.
int ref_expand_spans(const uint64_t* winners, std::size_t n, std::size_t span_m,
                     std::size_t middle_len, int mode, uint64_t* begin, uint64_t* end,
                     std::size_t* n_spans) {
    REF_TRY({
        std::vector<std::size_t> w(winners, winners + n);
        const SpanSet s = expand_spans(w, span_m, middle_len,
                                       mode == 0 ? SpanMode::Aligned : SpanMode::Centered);
        for (std::size_t i = 0; i < s.spans.size(); ++i) {
            begin[i] = s.spans[i].begin;
            end[i] = s.spans[i].end;
        }
        *n_spans = s.spans.size();
    })
}

// rope.hpp:21 RotaryTable tables.
int ref_rope_table(std::size_t d, double base, std::size_t max_position, float* cos_t,
                   float* sin_t) {
    REF_TRY({
        const RotaryTable t(d, base, max_position);
        for (std::size_t p = 0; p < max_position; ++p) {
            std::memcpy(cos_t + p * (d / 2), t.cos_row(p), (d / 2) * sizeof(float));
            std::memcpy(sin_t + p * (d / 2), t.sin_row(p), (d / 2) * sizeof(float));
        }
    })
}

// attend.hpp:25 attend.
int ref_attend(const float* q, std::size_t n_q, const float* k, const float* v, std::size_t L,
               std::size_t d, std::size_t dv, int has_boundary, std::size_t boundary, float* out,
               double* entropy) {
    REF_TRY({
        std::optional<std::size_t> b;
        if (has_boundary) b = boundary;
        const AttendResult r =
            attend(to_matrix(q, n_q, d), to_matrix(k, L, d), to_matrix(v, L, dv), b);
        std::memcpy(out, r.output.values.data(), n_q * dv * sizeof(float));
        std::memcpy(entropy, r.row_entropy.data(), n_q * sizeof(double));
    })
}

// Cache boundary + assemble_scope source indices (kv_cache.hpp:54-68, scope.hpp:37).
int ref_scope_indices(std::size_t total, std::size_t l_global, std::size_t l_local_max,
                      const uint64_t* sb, const uint64_t* se, std::size_t n_spans,
                      std::size_t window, uint64_t* src, std::size_t* length) {
    REF_TRY({
        SegmentedKvCache cache(1, 2, l_global, l_local_max);
        cache.append(DenseMatrix(total, 2), DenseMatrix(total, 2));
        SpanSet spans;
        for (std::size_t i = 0; i < n_spans; ++i) spans.spans.push_back(Span{sb[i], se[i]});
        const AttentionScope s = assemble_scope(cache, spans, window);
        for (std::size_t i = 0; i < s.length; ++i) src[i] = s.source_indices[i];
        *length = s.length;
    })
}

// A long-lived reference cache so the CPU baseline can time attend_step alone.
struct RefCache {
    SegmentedKvCache cache;
};

// keys/values: head-major [n_kv][total][d] fp32 (same layout as the device cache).
void* ref_cache_create(std::size_t n_kv, std::size_t d, std::size_t l_global,
                       std::size_t l_local_max, const float* keys, const float* values,
                       std::size_t total) {
    try {
        auto* rc = new RefCache{SegmentedKvCache(n_kv, d, l_global, l_local_max)};
        const std::size_t chunk = 65536;
        for (std::size_t r0 = 0; r0 < total; r0 += chunk) {
            const std::size_t rows = std::min(chunk, total - r0);
            DenseMatrix k(rows, n_kv * d), v(rows, n_kv * d);
            for (std::size_t r = 0; r < rows; ++r)
                for (std::size_t h = 0; h < n_kv; ++h) {
                    std::memcpy(k.row(r) + h * d, keys + (h * total + r0 + r) * d,
                                d * sizeof(float));
                    std::memcpy(v.row(r) + h * d, values + (h * total + r0 + r) * d,
                                d * sizeof(float));
                }
            rc->cache.append(k, v);
        }
        return rc;
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}

void ref_cache_destroy(void* p) { delete static_cast<RefCache*>(p); }

// kv_cache.hpp:143-166 write_cache_snapshot over caches built by ref_cache_create.
int ref_snapshot_write(const char* path, void* const* caches, std::size_t n) {
    REF_TRY({
        std::vector<SegmentedKvCache> layers;
        for (std::size_t i = 0; i < n; ++i) layers.push_back(static_cast<RefCache*>(caches[i])->cache);
        write_cache_snapshot(path, std::span<const SegmentedKvCache>(layers));
    })
}

// kv_cache.hpp:168-209 read_cache_snapshot: the layer count, and for `layer` its geometry
// (n_kv, d, total, l_global, l_local_max) and head-major payloads when they fit `cap` floats.
int ref_snapshot_read(const char* path, std::size_t layer, std::size_t* n_layers, uint64_t* info5,
                      float* keys, float* values, std::size_t cap) {
    REF_TRY({
        const auto layers = read_cache_snapshot(path);
        *n_layers = layers.size();
        if (layer < layers.size()) {
            const auto& c = layers[layer];
            info5[0] = c.n_kv_heads();
            info5[1] = c.d_head();
            info5[2] = c.total();
            info5[3] = c.l_global();
            info5[4] = c.l_local_max();
            const std::size_t per = c.total() * c.d_head();
            if (keys && values && per * c.n_kv_heads() <= cap && c.total())
                for (std::size_t h = 0; h < c.n_kv_heads(); ++h) {
                    std::memcpy(keys + h * per, c.key(h, 0), per * sizeof(float));
                    std::memcpy(values + h * per, c.value(h, 0), per * sizeof(float));
                }
        }
    })
}

struct RefStats {
    std::size_t max_position_used, ood_positions;
    int coverage_total;
    double entropy_max, entropy_sum;
    std::size_t entropy_rows, scope_len_max, scope_len, n_spans, coverage;
};

// engine.hpp:43 attend_step on a ref cache.
int ref_attend_step(void* cache_p, const float* q_pre, std::size_t n_q, std::size_t n_head,
                    std::size_t k, std::size_t k_prime, std::size_t span_m, std::size_t tile,
                    std::size_t l_global, std::size_t l_local, std::size_t l_chunk, int span_mode,
                    double rope_base, std::size_t max_position, int mode, float* out,
                    RefStats* st, uint64_t* sb, uint64_t* se) {
    REF_TRY({
        const auto& cache = static_cast<RefCache*>(cache_p)->cache;
        SelectionConfig cfg;
        cfg.k = k;
        cfg.k_prime = k_prime;
        cfg.span_m = span_m;
        cfg.tile_size = tile;
        cfg.l_global = l_global;
        cfg.l_local = l_local;
        cfg.l_chunk = l_chunk;
        cfg.span_mode = span_mode == 0 ? SpanMode::Aligned : SpanMode::Centered;
        static thread_local std::unique_ptr<RotaryTable> rope;
        if (!rope || rope->head_dim() != cache.d_head() || rope->base() != rope_base ||
            rope->max_position() != max_position)
            rope = std::make_unique<RotaryTable>(cache.d_head(), rope_base, max_position);
        RunStats stats;
        ScratchMeter meter;
        SpanSet spans;
        const DenseMatrix o =
            attend_step(to_matrix(q_pre, n_q, n_head * cache.d_head()), n_head, cache, cfg, *rope,
                        static_cast<AttentionMode>(mode), &stats, &meter, &spans);
        std::memcpy(out, o.values.data(), o.values.size() * sizeof(float));
        if (st) {
            st->max_position_used = stats.max_position_used;
            st->ood_positions = stats.ood_positions;
            st->coverage_total = stats.coverage_total;
            st->entropy_max = stats.entropy_max;
            st->entropy_sum = stats.entropy_sum;
            st->entropy_rows = stats.entropy_rows;
            st->scope_len_max = stats.scope_len_max;
            st->scope_len = stats.scope_len_max;
            st->n_spans = spans.spans.size();
            st->coverage = spans.coverage();
        }
        if (sb)
            for (std::size_t i = 0; i < spans.spans.size(); ++i) {
                sb[i] = spans.spans[i].begin;
                se[i] = spans.spans[i].end;
            }
    })
}

// SURVEY §8(c) arithmetic self-check: which fp32 lane variant did this build's
// fused_topk_scores compile to?  Returns 0 = unfused (mul, round, add), 1 = FMA lanes,
// 2 = neither; counts per-variant matches over `trials` random (query, key) pairs.
int ref_fma_selfcheck(std::size_t d, std::size_t trials, std::size_t* unfused_hits,
                      std::size_t* fma_hits) {
    std::uint64_t s = 0x9E3779B97F4A7C15ull;
    auto rnd = [&s]() {
        s ^= s << 13;
        s ^= s >> 7;
        s ^= s << 17;
        return float(double(s >> 11) / double(1ull << 53) * 2.0 - 1.0);
    };
    std::size_t un = 0, fm = 0;
    std::vector<float> keys(trials * d), q(d);
    for (float& v : q) v = rnd();
    for (float& v : keys) v = rnd();
    KeySegmentView view{keys.data(), trials, d};
    SelectionConfig cfg;
    cfg.k = trials;
    const PerHeadTopk res = fused_topk_scores(to_matrix(q.data(), 1, d), 1,
                                              std::span<const KeySegmentView>(&view, 1), cfg);
    for (const TopkEntry& e : res[0][0]) {
        const float* b = keys.data() + e.index * d;
        volatile float l[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        float f[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        std::size_t j = 0;
        for (; j + 8 <= d; j += 8)
            for (int t = 0; t < 8; ++t) {
                volatile float p = q[j + t] * b[j + t];
                l[t] = l[t] + p;
                f[t] = std::fma(q[j + t], b[j + t], f[t]);
            }
        for (; j < d; ++j) {
            volatile float p = q[j] * b[j];
            l[0] = l[0] + p;
            f[0] = std::fma(q[j], b[j], f[0]);
        }
        volatile float a01 = l[0] + l[1], a23 = l[2] + l[3], a45 = l[4] + l[5], a67 = l[6] + l[7];
        volatile float a03 = a01 + a23, a47 = a45 + a67;
        volatile float u = a03 + a47;
        const float fmv = ((f[0] + f[1]) + (f[2] + f[3])) + ((f[4] + f[5]) + (f[6] + f[7]));
        if (u == e.score) ++un;
        if (fmv == e.score) ++fm;
    }
    *unfused_hits = un;
    *fma_hits = fm;
    if (un == trials) return 0;
    if (fm == trials) return 1;
    return 2;
}


// ---- decoder model / engine (model.hpp, engine.hpp:119-216, full_attention.hpp) ----
// cfg8: n_layer, n_head, n_kv_head, d_model, d_head, d_ff, vocab_size, pretrain_window
void* ref_model_init(const uint64_t* cfg8, double rope_base, int mode, uint64_t seed) {
    try {
        ModelConfig c;
        c.n_layer = cfg8[0];
        c.n_head = cfg8[1];
        c.n_kv_head = cfg8[2];
        c.d_model = cfg8[3];
        c.d_head = cfg8[4];
        c.d_ff = cfg8[5];
        c.vocab_size = cfg8[6];
        c.pretrain_window = cfg8[7];
        c.rope_base = rope_base;
        c.attention_mode = static_cast<AttentionMode>(mode);
        return new ModelWeights(init_random(c, seed));
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}

void* ref_model_load(const char* path) {
    try {
        return new ModelWeights(load_weights(path));
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}

int ref_model_save(void* w, const char* path) { REF_TRY(save_weights(*static_cast<ModelWeights*>(w), path)) }

void ref_model_destroy(void* w) { delete static_cast<ModelWeights*>(w); }

// tensor kinds as reattn_weight_kind (include/reattn_cuda.h)
int ref_model_tensor(void* wp, int kind, std::size_t layer, float* out, std::size_t n) {
    REF_TRY({
        const ModelWeights& w = *static_cast<ModelWeights*>(wp);
        const std::vector<float>* v = nullptr;
        const LayerWeights* L = kind >= 1 && kind <= 9 ? &w.layers.at(layer) : nullptr;
        switch (kind) {
            case 0: v = &w.embedding.values; break;
            case 1: v = &L->wq.values; break;
            case 2: v = &L->wk.values; break;
            case 3: v = &L->wv.values; break;
            case 4: v = &L->wo.values; break;
            case 5: v = &L->w_gate.values; break;
            case 6: v = &L->w_up.values; break;
            case 7: v = &L->w_down.values; break;
            case 8: v = &L->norm_attn; break;
            case 9: v = &L->norm_ffn; break;
            case 10: v = &w.norm_final; break;
            case 11: v = &w.lm_head.values; break;
            default: throw std::invalid_argument("bad kind");
        }
        if (v->size() != n) throw std::invalid_argument("size mismatch");
        std::memcpy(out, v->data(), n * sizeof(float));
    })
}

// forward_full (full_attention.hpp:21-69): logits n x vocab
int ref_forward_full(void* w, const uint32_t* tokens, std::size_t n, float* logits) {
    REF_TRY({
        const DenseMatrix o = forward_full(std::span<const uint32_t>(tokens, n), *static_cast<ModelWeights*>(w));
        std::memcpy(logits, o.values.data(), o.values.size() * sizeof(float));
    })
}

struct RefEngine {
    std::unique_ptr<Engine> eng;
    std::unique_ptr<WindowReference> win;
};

// sel7: k, k_prime, span_m, tile, l_global, l_local, l_chunk.  kind 0 = Engine(mode),
// 1 = WindowReference(w, l_global, l_local, l_chunk)
void* ref_engine_create(void* w, const uint64_t* sel7, int span_mode, int mode, int kind) {
    try {
        SelectionConfig s;
        s.k = sel7[0];
        s.k_prime = sel7[1];
        s.span_m = sel7[2];
        s.tile_size = sel7[3];
        s.l_global = sel7[4];
        s.l_local = sel7[5];
        s.l_chunk = sel7[6];
        s.span_mode = span_mode == 0 ? SpanMode::Aligned : SpanMode::Centered;
        auto* r = new RefEngine();
        const ModelWeights& mw = *static_cast<ModelWeights*>(w);
        if (kind == 0)
            r->eng = std::make_unique<Engine>(mw, s, static_cast<AttentionMode>(mode));
        else
            r->win = std::make_unique<WindowReference>(mw, s.l_global, s.l_local, s.l_chunk);
        return r;
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}

void ref_engine_destroy(void* e) { delete static_cast<RefEngine*>(e); }

// prefill: hidden of the final chunk (rows x d_model) into `hidden` (capacity cap floats)
int ref_engine_prefill(void* ep, const uint32_t* tokens, std::size_t n, float* hidden,
                       std::size_t cap, std::size_t* rows) {
    REF_TRY({
        auto* r = static_cast<RefEngine*>(ep);
        const DenseMatrix h = r->eng ? r->eng->prefill(std::span<const uint32_t>(tokens, n))
                                     : r->win->prefill(std::span<const uint32_t>(tokens, n));
        if (h.values.size() > cap) throw std::invalid_argument("hidden capacity");
        std::memcpy(hidden, h.values.data(), h.values.size() * sizeof(float));
        *rows = h.rows;
    })
}

int ref_engine_logits(void* ep, const float* hidden, std::size_t rows, std::size_t d_model,
                      float* out) {
    REF_TRY({
        auto* r = static_cast<RefEngine*>(ep);
        if (!r->eng) throw std::invalid_argument("logits: engine only");
        const DenseMatrix l = r->eng->logits(to_matrix(hidden, rows, d_model));
        std::memcpy(out, l.values.data(), l.values.size() * sizeof(float));
    })
}

// decode_step: next token + last logits (vocab floats)
int ref_engine_decode(void* ep, uint32_t tok, uint32_t* next, float* logits, std::size_t vocab) {
    REF_TRY({
        auto* r = static_cast<RefEngine*>(ep);
        *next = r->eng ? r->eng->decode_step(tok) : r->win->decode_step(tok);
        std::span<const float> l = r->eng ? r->eng->last_logits() : r->win->last_logits();
        if (l.size() != vocab) throw std::invalid_argument("vocab mismatch");
        std::memcpy(logits, l.data(), vocab * sizeof(float));
    })
}

// RunStats: out10 = max_position_used, ood_positions, coverage_total, entropy_max,
// entropy_sum, entropy_rows, scope_len_max, peak_scratch_bytes, chunks_processed, decode_steps
int ref_engine_stats(void* ep, double* out10) {
    REF_TRY({
        auto* r = static_cast<RefEngine*>(ep);
        if (!r->eng) throw std::invalid_argument("stats: engine only");
        const RunStats& s = r->eng->stats();
        out10[0] = double(s.max_position_used);
        out10[1] = double(s.ood_positions);
        out10[2] = double(s.coverage_total);
        out10[3] = s.entropy_max;
        out10[4] = s.entropy_sum;
        out10[5] = double(s.entropy_rows);
        out10[6] = double(s.scope_len_max);
        out10[7] = double(s.peak_scratch_bytes);
        out10[8] = double(s.chunks_processed);
        out10[9] = double(s.decode_steps);
    })
}


// the reference tests' random_tokens (test_engine.cpp:50-56): std::mt19937 +
// uniform_int_distribution<uint32_t>(0, vocab - 1), this build's standard library
void ref_random_tokens(std::size_t n, uint32_t vocab, uint32_t seed, uint32_t* out) {
    std::mt19937 rng(seed);
    std::uniform_int_distribution<std::uint32_t> dist(0, vocab - 1);
    for (std::size_t i = 0; i < n; ++i) out[i] = dist(rng);
}

// greedy_decode_full (full_attention.hpp:72-84)
int ref_greedy_decode_full(void* w, const uint32_t* prompt, std::size_t n, std::size_t steps,
                           uint32_t* out) {
    REF_TRY({
        const std::vector<std::uint32_t> g = greedy_decode_full(
            std::span<const uint32_t>(prompt, n), *static_cast<ModelWeights*>(w), steps);
        std::copy(g.begin(), g.end(), out);
    })
}

}  // extern "C"
