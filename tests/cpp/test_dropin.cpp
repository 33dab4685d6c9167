// The reference's own hot-path unit tests (proj/tests/test_selection.cpp, test_scope.cpp,
// test_numerics.cpp, acceptance_test.cpp C01/C04/C09), ported onto the drop-in headers
// (include/reattn/*.hpp -> C-ABI -> sm_100a kernels).  Oracles: the reference tests' own
// independent oracles where they are self-contained, and the C restatement in oracle/
// (TEST INFRASTRUCTURE ONLY, linked here as the checker).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <map>
#include <random>
#include <set>
#include <string>
#include <vector>

#include <unistd.h>

#include "../../oracle/reattn_oracle.h"
#include "reattn/reattn.hpp"

using namespace reattn;

static int g_fail = 0, g_checks = 0;
#define CHECK(cond, ...)                                                      \
    do {                                                                      \
        ++g_checks;                                                           \
        if (!(cond)) {                                                        \
            ++g_fail;                                                         \
            std::printf("FAIL %s:%d: %s ", __FILE__, __LINE__, #cond);         \
            std::printf(__VA_ARGS__);                                         \
            std::printf("\n");                                                \
        }                                                                     \
    } while (0)
template <typename E, typename F>
static bool throws(F&& f, const char* msg = nullptr) {
    try {
        f();
    } catch (const E& e) {
        return !msg || std::string(e.what()).find(msg) != std::string::npos;
    } catch (...) {
        return false;
    }
    return false;
}

static DenseMatrix random_rows(std::size_t r, std::size_t c, std::mt19937& rng) {
    std::uniform_real_distribution<float> dist(-1.0f, 1.0f);
    DenseMatrix m(r, c);
    for (float& v : m.values) v = dist(rng);
    return m;
}

// oracle top-k for host views
static PerHeadTopk oracle_topk(const DenseMatrix& q, std::size_t n_heads,
                               const std::vector<std::vector<float>>& heads, std::size_t count,
                               std::size_t d, std::size_t k) {
    const std::size_t n_kv = heads.size(), n_q = q.rows;
    std::vector<const float*> ptrs;
    for (auto& h : heads) ptrs.push_back(h.data());
    std::vector<uint64_t> idx(std::max<std::size_t>(1, n_kv * n_q * k));
    std::vector<float> sc(idx.size());
    size_t n_out = 0;
    oracle_topk(q.values.data(), n_q, n_heads, ptrs.data(), n_kv, count, d, d, k, idx.data(),
                sc.data(), &n_out);
    PerHeadTopk out(n_kv, std::vector<std::vector<TopkEntry>>(n_q));
    for (std::size_t kv = 0; kv < n_kv; ++kv)
        for (std::size_t qq = 0; qq < n_q; ++qq)
            for (std::size_t j = 0; j < n_out; ++j)
                out[kv][qq].push_back(TopkEntry{idx[(kv * n_q + qq) * k + j], sc[(kv * n_q + qq) * k + j]});
    return out;
}

static void test_fused_topk() {
    // test_selection.cpp:105-131
    std::mt19937 rng(31);
    const std::size_t d = 32;
    for (std::size_t len : {0u, 1u, 3u, 4u, 5u, 127u, 1000u, 2047u, 2048u, 2049u, 10000u})
        for (std::size_t tile : {16u, 100u, 2048u})
            for (std::size_t k : {1u, 4u, 8u}) {
                const std::size_t n_kv = 1 + len % 2, n_heads = n_kv * 2, n_q = 1 + (len + tile) % 5;
                std::vector<std::vector<float>> heads(n_kv, std::vector<float>(len * d));
                std::uniform_real_distribution<float> dist(-1.0f, 1.0f);
                for (auto& h : heads)
                    for (float& v : h) v = dist(rng);
                std::vector<KeySegmentView> views;
                for (auto& h : heads) views.push_back(KeySegmentView{h.data(), len, d});
                const DenseMatrix q = random_rows(n_q, n_heads * d, rng);
                SelectionConfig cfg;
                cfg.k = k;
                cfg.tile_size = tile;
                const PerHeadTopk got = fused_topk_scores(q, n_heads, views, cfg);
                const PerHeadTopk want = oracle_topk(q, n_heads, heads, len, d, k);
                bool eq = got.size() == want.size();
                for (std::size_t kv = 0; eq && kv < got.size(); ++kv)
                    for (std::size_t qq = 0; eq && qq < got[kv].size(); ++qq) {
                        eq = got[kv][qq].size() == want[kv][qq].size();
                        for (std::size_t i = 0; eq && i < got[kv][qq].size(); ++i)
                            eq = got[kv][qq][i].index == want[kv][qq][i].index &&
                                 got[kv][qq][i].score == want[kv][qq][i].score;
                    }
                CHECK(eq, "fused vs oracle len=%zu tile=%zu k=%zu", len, tile, k);
            }
    // :168-191 ties keep the lower index
    const std::size_t dd = 8, L = 64;
    std::vector<float> data(L * dd, 0.0f);
    for (std::size_t i : {0u, 7u, 15u, 16u, 17u, 31u, 32u, 49u, 62u, 63u})
        for (std::size_t c = 0; c < dd; ++c) data[i * dd + c] = 0.5f;
    KeySegmentView view{data.data(), L, dd};
    DenseMatrix q(1, dd);
    for (std::size_t c = 0; c < dd; ++c) q.at(0, c) = 1.0f;
    SelectionConfig cfg;
    const PerHeadTopk got = fused_topk_scores(q, 1, std::span<const KeySegmentView>(&view, 1), cfg);
    CHECK(got[0][0].size() == 4 && got[0][0][0].index == 0 && got[0][0][1].index == 7 &&
              got[0][0][2].index == 15 && got[0][0][3].index == 16, "ties");
    // :210-231 scratch independent of the middle length
    std::size_t peaks[2];
    for (int i = 0; i < 2; ++i) {
        const std::size_t len = i ? 262144 : 4096;
        std::vector<float> h(len * 32);
        std::uniform_real_distribution<float> dist(-1.0f, 1.0f);
        for (float& v : h) v = dist(rng);
        KeySegmentView v{h.data(), len, 32};
        ScratchMeter m;
        fused_topk_scores(random_rows(4, 32, rng), 1, std::span<const KeySegmentView>(&v, 1), cfg, &m);
        peaks[i] = m.peak;
    }
    CHECK(peaks[0] == peaks[1] && peaks[0] > 0, "scratch %zu vs %zu", peaks[0], peaks[1]);
    // :401-407 head mismatch throws
    std::vector<std::vector<float>> mid(3, std::vector<float>(10 * 8, 0.f));
    std::vector<KeySegmentView> mv;
    for (auto& h : mid) mv.push_back(KeySegmentView{h.data(), 10, 8});
    CHECK(throws<std::invalid_argument>([&] { fused_topk_scores(random_rows(1, 32, rng), 4, mv, cfg); }),
          "head mismatch");
}

static void test_vote_spans() {
    // test_selection.cpp:233-270 map oracle
    std::mt19937 rng(53);
    std::uniform_int_distribution<std::size_t> idx(0, 49);
    std::uniform_real_distribution<float> score(-1.0f, 1.0f);
    for (int iter = 0; iter < 200; ++iter) {
        PerHeadTopk per_head(8, std::vector<std::vector<TopkEntry>>(4));
        std::map<std::size_t, std::pair<std::size_t, float>> tally;
        for (auto& head : per_head)
            for (auto& query : head) {
                std::set<std::size_t> seen;
                for (int j = 0; j < 4; ++j) {
                    std::size_t i = idx(rng);
                    while (seen.count(i)) i = idx(rng);
                    seen.insert(i);
                    const float s = score(rng);
                    query.push_back(TopkEntry{i, s});
                    auto it = tally.find(i);
                    if (it == tally.end())
                        tally[i] = {1, s};
                    else {
                        it->second.first += 1;
                        it->second.second = std::max(it->second.second, s);
                    }
                }
            }
        std::vector<std::pair<std::size_t, std::pair<std::size_t, float>>> ranked(tally.begin(), tally.end());
        std::sort(ranked.begin(), ranked.end(), [](const auto& a, const auto& b) {
            if (a.second.first != b.second.first) return a.second.first > b.second.first;
            if (a.second.second != b.second.second) return a.second.second > b.second.second;
            return a.first < b.first;
        });
        const std::size_t k_prime = 1 + iter % 20;
        const auto got = vote(per_head, k_prime);
        bool ok = got.size() == std::min(k_prime, ranked.size());
        for (std::size_t i = 0; ok && i < got.size(); ++i) ok = got[i] == ranked[i].first;
        CHECK(ok, "vote iter %d", iter);
        if (iter == 0) {
            const auto t = tally_candidates(per_head);
            bool tok = t.size() == ranked.size();
            for (std::size_t i = 0; tok && i < t.size(); ++i)
                tok = t[i].middle_index == ranked[i].first && t[i].votes == ranked[i].second.first &&
                      t[i].score == ranked[i].second.second;
            CHECK(tok, "tally");
        }
    }
    {  // :281-292 agreement outranks score
        PerHeadTopk ph(1, std::vector<std::vector<TopkEntry>>(2));
        ph[0][0] = {TopkEntry{7, 0.1f}, TopkEntry{3, 9.0f}};
        ph[0][1] = {TopkEntry{7, 0.2f}, TopkEntry{5, 0.05f}};
        const auto w = vote(ph, 3);
        CHECK(w.size() == 3 && w[0] == 7 && w[1] == 3 && w[2] == 5, "agreement");
        CHECK(vote(ph, 0).empty(), "k'=0");
    }
    // :300-323 aligned blocks from the set oracle; :339-371 centered vs interval oracle
    for (int iter = 0; iter < 100; ++iter) {
        const std::size_t m = 1 + iter % 64;
        const std::size_t len = 1 + std::uniform_int_distribution<std::size_t>(0, 100000)(rng);
        std::vector<std::size_t> winners(120);
        std::uniform_int_distribution<std::size_t> pick(0, len - 1);
        for (auto& w : winners) w = pick(rng);
        const SpanSet got = expand_spans(winners, m, len);
        std::set<std::size_t> blocks;
        for (std::size_t w : winners) blocks.insert(w / m);
        bool ok = got.spans.size() == blocks.size();
        std::size_t i = 0;
        for (std::size_t b : blocks) {
            if (!ok) break;
            ok = got.spans[i].begin == b * m && got.spans[i].end == std::min(b * m + m, len);
            ++i;
        }
        CHECK(ok, "aligned iter %d", iter);
        const std::size_t mc = 2 + iter % 63;
        const std::size_t lc = mc + std::uniform_int_distribution<std::size_t>(0, 5000)(rng);
        std::vector<std::size_t> wc(40);
        std::uniform_int_distribution<std::size_t> pc(0, lc - 1);
        for (auto& w : wc) w = pc(rng);
        const SpanSet gc = expand_spans(wc, mc, lc, SpanMode::Centered);
        std::vector<uint64_t> w64(wc.begin(), wc.end()), ob(wc.size()), oe(wc.size());
        size_t on = 0;
        oracle_expand_spans(w64.data(), w64.size(), mc, lc, ORACLE_SPAN_CENTERED, ob.data(), oe.data(), &on);
        bool okc = gc.spans.size() == on;
        for (std::size_t j = 0; okc && j < on; ++j) okc = gc.spans[j].begin == ob[j] && gc.spans[j].end == oe[j];
        CHECK(okc, "centered iter %d", iter);
    }
    CHECK(expand_spans(std::vector<std::size_t>{5, 20}, 32, 100).spans == (std::vector<Span>{{0, 32}}), "5,20");
    CHECK(expand_spans(std::vector<std::size_t>{98}, 32, 100).spans == (std::vector<Span>{{96, 100}}), "98");
    CHECK(throws<std::out_of_range>([] { expand_spans(std::vector<std::size_t>{100}, 32, 100); },
                                    "expand_spans: winner outside middle"), "winner range");
    CHECK(expand_spans(std::vector<std::size_t>{}, 32, 100).empty(), "empty");
}

static void check_scope(const AttentionScope& scope, const SegmentedKvCache& cache, const SpanSet& spans,
                        const char* label) {
    const auto segs = cache.views();
    std::vector<std::size_t> want;
    for (std::size_t i = segs.global.begin; i < segs.global.end; ++i) want.push_back(i);
    for (const Span& s : spans.spans)
        for (std::size_t i = s.begin; i < s.end; ++i) want.push_back(segs.middle.begin + i);
    for (std::size_t i = segs.local.begin; i < segs.local.end; ++i) want.push_back(i);
    bool ok = scope.length == want.size() && scope.source_indices == want;
    for (std::size_t kv = 0; ok && kv < cache.n_kv_heads(); ++kv)
        for (std::size_t r = 0; ok && r < scope.length; ++r)
            ok = std::equal(scope.key_row(kv, r), scope.key_row(kv, r) + cache.d_head(), cache.key(kv, want[r])) &&
                 std::equal(scope.value_row(kv, r), scope.value_row(kv, r) + cache.d_head(), cache.value(kv, want[r]));
    CHECK(ok, "%s", label);
}

static void test_scope() {
    // test_scope.cpp:53-132
    std::mt19937 rng(71);
    for (int iter = 0; iter < 30; ++iter) {
        const std::size_t g = std::uniform_int_distribution<std::size_t>(0, 40)(rng);
        const std::size_t loc = std::uniform_int_distribution<std::size_t>(1, 64)(rng);
        const std::size_t total = std::uniform_int_distribution<std::size_t>(1, 2000)(rng);
        SegmentedKvCache cache(2, 8, g, loc);
        cache.append(random_rows(total, 16, rng), random_rows(total, 16, rng));
        SpanSet spans;
        if (cache.middle_len() > 0) {
            std::vector<std::size_t> winners(8);
            std::uniform_int_distribution<std::size_t> pick(0, cache.middle_len() - 1);
            for (auto& w : winners) w = pick(rng);
            spans = expand_spans(winners, 16, cache.middle_len());
        }
        check_scope(assemble_scope(cache, spans, 1 << 20), cache, spans, "gather oracle");
    }
    {
        SegmentedKvCache cache(1, 4, 4, 8);
        cache.append(random_rows(50, 4, rng), random_rows(50, 4, rng));
        const AttentionScope s = assemble_window_scope(cache, 4096);
        CHECK(s.length == 12 && s.source_indices[0] == 0 && s.source_indices[4] == 42, "window");
    }
    {
        SegmentedKvCache cache(1, 4, 4, 8);
        cache.append(random_rows(12, 4, rng), random_rows(12, 4, rng));
        CHECK(throws<std::invalid_argument>([&] { assemble_scope(cache, SpanSet{}, 11); },
                                            "scope exceeds pretrain window"), "overflow");
        CHECK(assemble_scope(cache, SpanSet{}, 12).length == 12, "fits");
    }
    {
        SegmentedKvCache cache(1, 4, 4, 8);
        cache.append(random_rows(20, 4, rng), random_rows(20, 4, rng));
        SpanSet spans;
        spans.spans.push_back(Span{4, 9});
        CHECK(throws<std::out_of_range>([&] { assemble_scope(cache, spans, 4096); }), "span range");
    }
    {  // C01: the budget fills the window exactly
        SegmentedKvCache cache(1, 2, 32, 4096);
        cache.append(random_rows(9000, 2, rng), random_rows(9000, 2, rng));
        std::vector<std::size_t> winners;
        for (std::size_t b = 0; b < 127; ++b) winners.push_back(b * 32);
        const SpanSet spans = expand_spans(winners, 32, cache.middle_len());
        CHECK(spans.coverage() == 127u * 32u, "coverage");
        const AttentionScope s = assemble_scope(cache, spans, 8192);
        CHECK(s.length == 8192 && s.length == SelectionConfig{}.budget(), "budget 8192");
        check_scope(s, cache, spans, "budget gather");
    }
}

static void test_rope_attend() {
    std::mt19937 rng(3);
    {  // test_numerics.cpp:150-237
        const RotaryTable t(8, 10000.0, 16);
        const DenseMatrix m = random_rows(4, 8, rng);
        const std::vector<std::size_t> pos(4, 0);
        CHECK(rope_rotate(m, pos, t).values == m.values, "pos 0 identity");
        const RotaryTable t2(2, 10000.0, 64);
        for (std::size_t p : {1u, 5u, 63u}) {
            DenseMatrix v(1, 2);
            v.at(0, 0) = 1.0f;
            const std::vector<std::size_t> pp{p};
            const DenseMatrix r = rope_rotate(v, pp, t2);
            CHECK(std::abs(r.at(0, 0) - std::cos(double(p))) < 1e-6 && std::abs(r.at(0, 1) - std::sin(double(p))) < 1e-6,
                  "angle %zu", p);
        }
        const RotaryTable t3(8, 10000.0, 100);
        DenseMatrix z(1, 8);
        CHECK(throws<std::out_of_range>([&] { t3.rotate_row(z.row(0), 100); }, "position out of pretrained range"),
              "ood");
        CHECK(throws<std::invalid_argument>([] { RotaryTable(7, 10000.0, 16); }), "odd dim");
        CHECK(throws<std::invalid_argument>([] { RotaryTable(8, -1.0, 16); }), "base");
        CHECK(throws<std::invalid_argument>([] { RotaryTable(8, 10000.0, 0); }), "max pos");
        // table bytes equal the oracle restatement (rope.hpp:27-39)
        const RotaryTable t4(128, 500000.0, 8192);
        std::vector<float> oc(8192 * 64), os(8192 * 64);
        oracle_rope_table(128, 500000.0, 8192, oc.data(), os.data());
        CHECK(std::equal(oc.begin(), oc.end(), t4.cos_row(0)) && std::equal(os.begin(), os.end(), t4.sin_row(0)),
              "table");
    }
    {  // :281-320 attend vs oracle, causal boundary, single key, empty set
        std::uniform_int_distribution<std::size_t> nq(1, 8), len(1, 512), dim(4, 64);
        for (int iter = 0; iter < 200; ++iter) {
            const std::size_t n_q = nq(rng), L = len(rng), d = dim(rng) & ~1ull;
            const DenseMatrix q = random_rows(n_q, d, rng), k = random_rows(L, d, rng), v = random_rows(L, d, rng);
            std::optional<std::size_t> b;
            if (iter % 2 == 0 && L >= n_q) b = L - n_q;
            const AttendResult got = attend(q, k, v, b);
            std::vector<float> out(n_q * d);
            std::vector<double> ent(n_q);
            oracle_attend(q.values.data(), n_q, k.values.data(), v.values.data(), L, d, d, b.has_value(),
                          b.value_or(0), out.data(), ent.data());
            double md = 0, me = 0;
            for (std::size_t i = 0; i < out.size(); ++i) md = std::max(md, std::abs(double(out[i]) - got.output.values[i]));
            for (std::size_t i = 0; i < n_q; ++i) me = std::max(me, std::abs(ent[i] - got.row_entropy[i]));
            CHECK(md <= 1e-6 && me <= 1e-9, "attend iter %d md=%g me=%g", iter, md, me);
        }
        DenseMatrix q(2, 4), k(3, 4), v(3, 4);
        for (std::size_t c = 0; c < 4; ++c) {
            q.at(0, c) = q.at(1, c) = 1.0f;
            k.at(2, c) = 100.0f;
            v.at(0, c) = 5.0f;
            v.at(1, c) = 9.0f;
            v.at(2, c) = -50.0f;
        }
        const AttendResult r = attend(q, k, v, 0);
        CHECK(r.output.at(0, 0) == 5.0f && std::abs(r.output.at(1, 0) - 7.0f) < 1e-6, "causal boundary");
        DenseMatrix e(0, 8);
        CHECK(throws<std::invalid_argument>([&] { attend(DenseMatrix(1, 8), e, e); }, "empty key set"), "empty");
    }
}

static void test_attend_step() {
    // engine.hpp attend_step vs the oracle restatement, toy + LLaMA geometries, both modes
    std::mt19937 rng(7);
    struct Case { std::size_t n_kv, nh, d, total, n_q, window; SelectionConfig cfg; AttentionMode mode; };
    std::vector<Case> cases;
    SelectionConfig toy;
    toy.l_global = 16; toy.l_local = 256; toy.l_chunk = 128; toy.span_m = 16; toy.k = 4; toy.k_prime = 64;
    cases.push_back({2, 4, 16, 2000, 1, 2048, toy, AttentionMode::ReAttention});
    cases.push_back({2, 4, 16, 3000, 64, 2048, toy, AttentionMode::ReAttention});
    SelectionConfig cen = toy;
    cen.span_mode = SpanMode::Centered;
    cases.push_back({2, 4, 16, 5000, 8, 2048, cen, AttentionMode::ReAttention});
    cases.push_back({2, 4, 16, 900, 32, 2048, toy, AttentionMode::Window});
    cases.push_back({8, 32, 128, 12000, 1, 8192, SelectionConfig{}, AttentionMode::ReAttention});
    for (const Case& c : cases) {
        SegmentedKvCache cache(c.n_kv, c.d, c.cfg.l_global, c.cfg.l_local);
        const DenseMatrix K = random_rows(c.total, c.n_kv * c.d, rng), V = random_rows(c.total, c.n_kv * c.d, rng);
        cache.append(K, V);
        const RotaryTable rope(c.d, 10000.0, c.window);
        const DenseMatrix q = random_rows(c.n_q, c.nh * c.d, rng);
        RunStats st;
        SpanSet spans;
        const DenseMatrix out = attend_step(q, c.nh, cache, c.cfg, rope, c.mode, &st, nullptr, &spans);
        // oracle on the head-major copy
        std::vector<float> hk(c.n_kv * c.total * c.d), hv(hk.size());
        for (std::size_t h = 0; h < c.n_kv; ++h)
            for (std::size_t r = 0; r < c.total; ++r)
                for (std::size_t e = 0; e < c.d; ++e) {
                    hk[(h * c.total + r) * c.d + e] = K.at(r, h * c.d + e);
                    hv[(h * c.total + r) * c.d + e] = V.at(r, h * c.d + e);
                }
        std::vector<float> oc(c.window * c.d / 2), os(oc.size()), oout(c.n_q * c.nh * c.d);
        oracle_rope_table(c.d, 10000.0, c.window, oc.data(), os.data());
        oracle_selection_config ocfg{c.cfg.k, c.cfg.k_prime, c.cfg.span_m, c.cfg.tile_size, c.cfg.l_global,
                                     c.cfg.l_local, c.cfg.l_chunk, c.cfg.span_mode == SpanMode::Aligned ? 0 : 1};
        oracle_step_stats ost{};
        ost.coverage_total = 1;
        std::vector<uint64_t> sb(c.cfg.k_prime + 1), se(c.cfg.k_prime + 1);
        const int rc = oracle_attend_step(q.values.data(), c.n_q, c.nh, hk.data(), hv.data(), c.n_kv, c.d, c.total,
                                          c.total, &ocfg, oc.data(), os.data(), c.window, (int)c.mode, oout.data(),
                                          &ost, sb.data(), se.data());
        double md = 0;
        for (std::size_t i = 0; i < oout.size(); ++i) md = std::max(md, std::abs(double(oout[i]) - out.values[i]));
        bool spans_eq = spans.spans.size() == ost.n_spans;
        for (std::size_t i = 0; spans_eq && i < ost.n_spans; ++i)
            spans_eq = spans.spans[i].begin == sb[i] && spans.spans[i].end == se[i];
        CHECK(rc == 0 && md <= 1e-6 && spans_eq && st.scope_len_max == ost.scope_len &&
                  std::abs(st.entropy_max - ost.entropy_max) <= 1e-6 && st.coverage_total == (bool)ost.coverage_total,
              "attend_step total=%zu n_q=%zu md=%g dH=%g L=%zu/%zu", c.total, c.n_q, md,
              std::abs(st.entropy_max - ost.entropy_max), st.scope_len_max, ost.scope_len);
    }
    {  // errors: engine.hpp:51-53, scope.hpp:51-52, engine.hpp:69
        SelectionConfig cfg;
        cfg.l_global = 4; cfg.l_local = 8; cfg.k_prime = 2; cfg.span_m = 4;
        SegmentedKvCache cache(1, 4, 4, 8);
        cache.append(random_rows(12, 4, rng), random_rows(12, 4, rng));
        CHECK(throws<std::invalid_argument>([&] { attend_step(DenseMatrix(1, 4), 1, cache, cfg, RotaryTable(4, 1e4, 11),
                                                              AttentionMode::ReAttention); },
                                            "scope exceeds pretrain window"), "window");
        CHECK(throws<std::logic_error>([&] { attend_step(DenseMatrix(13, 4), 1, cache, cfg, RotaryTable(4, 1e4, 64),
                                                         AttentionMode::ReAttention); },
                                       "query block longer than scope"), "query long");
        CHECK(throws<std::invalid_argument>([&] { attend_step(DenseMatrix(1, 10), 3, cache, cfg, RotaryTable(4, 1e4, 64),
                                                              AttentionMode::ReAttention); },
                                            "query width"), "width");
    }
}

// kv_cache.hpp:120-209 snapshot round trip through the drop-in API, plus the reference's
// failure messages (runtime_error / invalid_argument) for corrupt files.
static void test_snapshot() {
    std::mt19937 rng(91);
    std::vector<SegmentedKvCache> layers;
    const std::size_t totals[3] = {70, 0, 5};
    for (std::size_t t : totals) {
        SegmentedKvCache c(2, 16, 4, 32);
        if (t) c.append(random_rows(t, 32, rng), random_rows(t, 32, rng));
        layers.push_back(std::move(c));
    }
    const std::string path = "/tmp/reattn_dropin_snapshot_" + std::to_string(::getpid()) + ".rkvc";
    write_cache_snapshot(path, std::span<const SegmentedKvCache>(layers));
    for (auto storage : {SegmentedKvCache::Storage::F32, SegmentedKvCache::Storage::BF16}) {
        auto back = read_cache_snapshot(path, storage);
        bool ok = back.size() == 3;
        for (std::size_t l = 0; ok && l < 3; ++l) {
            ok = back[l].total() == layers[l].total() && back[l].l_global() == 4 &&
                 back[l].l_local_max() == 32 && back[l].n_kv_heads() == 2 && back[l].d_head() == 16;
            for (std::size_t h = 0; ok && h < 2; ++h)
                for (std::size_t e = 0; ok && e < layers[l].total() * 16; ++e) {
                    const float want = layers[l].key(h, 0)[e], wv = layers[l].value(h, 0)[e];
                    const float gk = back[l].key(h, 0)[e], gv = back[l].value(h, 0)[e];
                    if (storage == SegmentedKvCache::Storage::F32)
                        ok = gk == want && gv == wv;
                    else
                        ok = gk == oracle_round_bf16(want) && gv == oracle_round_bf16(wv);
                    if (!ok)
                        std::printf("snapshot mismatch layer %zu head %zu elem %zu: key %g/%g value %g/%g\n",
                                    l, h, e, gk, want, gv, wv);
                }
            if (!ok && l < back.size())
                std::printf("snapshot layer %zu: total %zu/%zu g %zu local %zu\n", l, back[l].total(),
                            layers[l].total(), back[l].l_global(), back[l].l_local_max());
        }
        CHECK(ok, "snapshot round trip storage=%d", (int)storage);
    }
    {
        FILE* f = std::fopen(path.c_str(), "wb");
        std::fwrite("RKVX", 1, 4, f);
        std::fclose(f);
        CHECK(throws<std::runtime_error>([&] { read_cache_snapshot(path); },
                                         "not a cache snapshot (bad magic)"),
              "snapshot bad magic");
        CHECK(throws<std::runtime_error>([&] { read_cache_snapshot("/tmp/no/such.rkvc"); },
                                         "cannot open /tmp/no/such.rkvc"),
              "snapshot missing file");
        CHECK(throws<std::invalid_argument>(
                  [&] { write_cache_snapshot(path, std::span<const SegmentedKvCache>()); },
                  "cache snapshot: no layers"),
              "snapshot no layers");
    }
    std::remove(path.c_str());
}

// test_engine.cpp (reference) on the drop-in Engine / ModelWeights / forward_full /
// WindowReference headers.  Parity against the reference build itself is in
// tests/test_engine_gpu.py; here the API surface, its identities and its errors.
static ModelConfig toy_config() {
    ModelConfig cfg;
    cfg.n_layer = 2;
    cfg.n_head = 4;
    cfg.n_kv_head = 2;
    cfg.d_model = 64;
    cfg.d_head = 16;
    cfg.d_ff = 128;
    cfg.vocab_size = 128;
    cfg.pretrain_window = 2048;
    return cfg;
}

static SelectionConfig toy_selection() {
    SelectionConfig sel;
    sel.l_global = 16;
    sel.l_local = 256;
    sel.l_chunk = 128;
    sel.span_m = 16;
    sel.k = 4;
    sel.k_prime = 64;
    sel.tile_size = 512;
    return sel;
}

static std::vector<std::uint32_t> tokens_of(std::size_t n, std::uint32_t vocab, std::uint32_t seed) {
    std::mt19937 rng(seed);
    std::uniform_int_distribution<std::uint32_t> dist(0, vocab - 1);
    std::vector<std::uint32_t> out(n);
    for (auto& t : out) t = dist(rng);
    return out;
}

static void test_engine() {
    const ModelWeights w = init_random(toy_config(), 22);
    CHECK(w.layers.size() == 2 && w.embedding.rows == 128 && w.lm_head.cols == 128, "shapes");
    CHECK(w.layers[0].norm_attn.size() == 64 && w.layers[0].norm_attn[0] == 1.0f, "unit norms");
    // constructor checks (test_engine.cpp:57-66)
    CHECK(throws<std::invalid_argument>([&] { Engine(w, toy_selection(), AttentionMode::Full); },
                                        "full attention is the reference path"), "full mode");
    SelectionConfig big = toy_selection();
    big.k_prime = 1000;
    CHECK(throws<std::invalid_argument>([&] { Engine(w, big, AttentionMode::ReAttention); },
                                        "exceeds pretrain window"), "budget");
    // single-token prefill == decode on an empty cache (test_engine.cpp:68-78), bitwise
    {
        Engine a(w, toy_selection(), AttentionMode::ReAttention);
        Engine b(w, toy_selection(), AttentionMode::ReAttention);
        const std::vector<std::uint32_t> one{42};
        const DenseMatrix la = a.logits(a.prefill(one));
        b.decode_step(42);
        bool same = la.cols == b.last_logits().size();
        for (std::size_t i = 0; same && i < la.cols; ++i) same = la.at(0, i) == b.last_logits()[i];
        CHECK(same, "prefill == decode");
    }
    // full coverage vs forward_full (test_engine.cpp:80-110), 1e-4
    {
        const auto toks = tokens_of(372, 128, 220);
        SelectionConfig sel = toy_selection();
        sel.k = 100;
        sel.k_prime = 100;
        Engine eng(w, sel, AttentionMode::ReAttention);
        const DenseMatrix got = eng.logits(eng.prefill(toks));
        CHECK(eng.stats().coverage_total, "coverage");
        const DenseMatrix full = forward_full(toks, w);
        double md = 0;
        for (std::size_t r = 0; r < got.rows; ++r)
            for (std::size_t c = 0; c < got.cols; ++c)
                md = std::max(md, std::abs(double(got.at(r, c)) - double(full.at(372 - got.rows + r, c))));
        CHECK(got.rows == 100 && md <= 1e-4, "md %g", md);
    }
    // selection off == WindowReference, bitwise on the device (C03), and window mode
    {
        const auto toks = tokens_of(900, 128, 230);
        SelectionConfig off = toy_selection();
        off.k_prime = 0;
        Engine eng(w, off, AttentionMode::ReAttention);
        WindowReference ref(w, off.l_global, off.l_local, off.l_chunk);
        const DenseMatrix a = eng.prefill(toks), b = ref.prefill(toks);
        CHECK(a.values == b.values, "window reference");
        for (int s = 0; s < 3; ++s) CHECK(eng.decode_step(s) == ref.decode_step(s), "decode %d", s);
        CHECK(throws<std::invalid_argument>([&] { WindowReference(w, 16, 0, 1); },
                                            "window reference: bad local/chunk sizes"), "wr");
    }
    // stats (test_engine.cpp:219-231)
    {
        Engine eng(w, toy_selection(), AttentionMode::ReAttention);
        eng.prefill(tokens_of(700, 128, 280));
        CHECK(eng.stats().chunks_processed == 5, "chunks %zu", eng.stats().chunks_processed);
        eng.decode_step(1);
        eng.decode_step(2);
        CHECK(eng.stats().decode_steps == 2 && eng.stats().decode_latency_ms.size() == 2, "steps");
        CHECK(eng.last_spans().size() == 2, "spans");
        CHECK(throws<std::out_of_range>([&] { eng.decode_step(500); }, "token id outside vocabulary"),
              "vocab");
    }
    // weights file round trip + load errors (model.hpp:259-339)
    {
        char path[] = "/tmp/reattn_dropin_w_XXXXXX";
        const int fd = mkstemp(path);
        close(fd);
        save_weights(w, path);
        const ModelWeights back = load_weights(path);
        CHECK(back.embedding.values == w.embedding.values && back.lm_head.values == w.lm_head.values &&
                  back.layers[1].w_down.values == w.layers[1].w_down.values,
              "round trip");
        FILE* f = std::fopen(path, "ab");
        std::fputc(0, f);
        std::fclose(f);
        CHECK(throws<std::runtime_error>([&] { load_weights(path); },
                                         "weights file: trailing bytes after lm_head"), "trailing");
        std::remove(path);
        CHECK(throws<std::runtime_error>([&] { load_weights(path); }, "cannot open weights file"), "missing");
    }
}

static void test_dense_and_naive() {
    std::mt19937 rng(1234);
    std::uniform_real_distribution<float> dist(-1.0f, 1.0f);
    // dense_matrix.hpp:41-74 dot lanes (test_numerics.cpp:335-347 style), bit for bit
    for (std::size_t d : {1, 5, 8, 16, 31, 64, 128, 200}) {
        std::vector<float> a(d), b(d);
        for (auto& v : a) v = dist(rng);
        for (auto& v : b) v = dist(rng);
        const float f = dot_f32(a.data(), b.data(), d), fo = oracle_dot_f32(a.data(), b.data(), d);
        CHECK(std::memcmp(&f, &fo, 4) == 0 || (f == 0.0f && fo == 0.0f), "dot_f32 d=%zu %g %g", d, f, fo);
        const double g = dot_f64(a.data(), b.data(), d), go = oracle_dot_f64(a.data(), b.data(), d);
        CHECK(g == go, "dot_f64 d=%zu %.17g %.17g", d, g, go);
    }
    // dense_matrix.hpp:77-90 matmul: k-ordered unfused sums, bit for bit
    {
        const DenseMatrix A = random_rows(7, 33, rng), B = random_rows(33, 5, rng);
        const DenseMatrix C = matmul(A, B);
        bool same = C.rows == 7 && C.cols == 5;
        for (std::size_t i = 0; i < 7 && same; ++i)
            for (std::size_t j = 0; j < 5; ++j) {
                float acc = 0.0f;
                for (std::size_t kk = 0; kk < 33; ++kk) {
                    const float p = A.at(i, kk) * B.at(kk, j);
                    acc = acc + p;
                }
                same = same && acc == C.at(i, j);
            }
        CHECK(same, "matmul differs from the k-ordered sum");
        CHECK(throws<std::invalid_argument>([&] { matmul(A, A); }, "inner dimensions differ"), "matmul shapes");
    }
    // selection.hpp:139-156 group means (groups 1, 3, 4)
    for (std::size_t g : {1, 3, 4}) {
        const std::size_t n_kv = 2, d = 16, nh = n_kv * g;
        const DenseMatrix q = random_rows(3, nh * d, rng);
        const DenseMatrix mq = detail::group_mean_queries(q, nh, n_kv, d);
        std::vector<float> want(3 * n_kv * d);
        oracle_group_mean(q.values.data(), 3, nh, n_kv, d, want.data());
        CHECK(std::memcmp(mq.values.data(), want.data(), want.size() * 4) == 0, "group mean g=%zu", g);
    }
    // selection.hpp:81-135 TopkBuffer: ties keep the lower index (test_selection.cpp:168-191)
    {
        detail::TopkBuffer buf;
        buf.init(4);
        for (std::size_t i = 0; i < 64; ++i) {
            const bool tied = i == 0 || i == 7 || i == 15 || i == 16 || i == 17 || i == 31;
            buf.offer(i, tied ? 1.0f : -1.0f);
        }
        const auto s = buf.sorted();
        CHECK(s.size() == 4 && s[0].index == 0 && s[1].index == 7 && s[2].index == 15 && s[3].index == 16,
              "TopkBuffer tie order");
        // against the oracle's top-k on random scores offered in index order
        const std::size_t d = 16, count = 3000;
        std::vector<std::vector<float>> heads(1, std::vector<float>(count * d));
        for (auto& v : heads[0]) v = dist(rng);
        const DenseMatrix q = random_rows(1, d, rng);
        const PerHeadTopk want = oracle_topk(q, 1, heads, count, d, 5);
        detail::TopkBuffer b2;
        b2.init(5);
        for (std::size_t i = 0; i < count; ++i) b2.offer(i, oracle_dot_f32(q.values.data(), heads[0].data() + i * d, d));
        const auto got = b2.sorted();
        bool same = got.size() == want[0][0].size();
        for (std::size_t j = 0; same && j < got.size(); ++j)
            same = got[j].index == want[0][0][j].index && got[j].score == want[0][0][j].score;
        CHECK(same, "TopkBuffer vs oracle");
    }
    // selection_reference.hpp:18-69 naive scorer == fused scorer == oracle, bit for bit
    // (test_selection.cpp:89-103); its scratch grows with the middle, the fused one's does not
    std::size_t naive_small = 0, naive_large = 0, fused_small = 0, fused_large = 0;
    for (std::size_t count : {0, 1, 4, 5, 127, 1000, 2049, 10000}) {
        for (std::size_t k : {1, 4, 8, 100}) {  // k > 64: the naive select has no capacity limit
            const std::size_t n_kv = 2, nh = 4, d = 32;
            std::vector<std::vector<float>> heads(n_kv, std::vector<float>(std::max<std::size_t>(1, count) * d));
            for (auto& h : heads)
                for (auto& v : h) v = dist(rng);
            std::vector<KeySegmentView> views;
            for (auto& h : heads) views.push_back(KeySegmentView{h.data(), count, d});
            const DenseMatrix q = random_rows(3, nh * d, rng);
            SelectionConfig cfg;
            cfg.k = k;
            ScratchMeter mn, mf;
            const PerHeadTopk naive = naive_topk_scores(q, nh, views, cfg, &mn);
            const PerHeadTopk fused = fused_topk_scores(q, nh, views, cfg, &mf);
            const PerHeadTopk want = oracle_topk(q, nh, heads, count, d, k);
            bool same = naive.size() == n_kv;
            for (std::size_t kv = 0; same && kv < n_kv; ++kv)
                for (std::size_t qq = 0; same && qq < 3; ++qq) {
                    same = naive[kv][qq].size() == want[kv][qq].size() &&
                           fused[kv][qq].size() == want[kv][qq].size();
                    for (std::size_t j = 0; same && j < want[kv][qq].size(); ++j)
                        same = naive[kv][qq][j].index == want[kv][qq][j].index &&
                               naive[kv][qq][j].score == want[kv][qq][j].score &&
                               fused[kv][qq][j].index == want[kv][qq][j].index &&
                               fused[kv][qq][j].score == want[kv][qq][j].score;
                }
            CHECK(same, "naive/fused/oracle top-k count=%zu k=%zu", count, k);
            if (count == 1000 && k == 4) naive_small = mn.peak, fused_small = mf.peak;
            if (count == 10000 && k == 4) naive_large = mn.peak, fused_large = mf.peak;
        }
    }
    CHECK(naive_large > 5 * naive_small, "naive scratch grows with the middle (%zu %zu)", naive_small, naive_large);
    CHECK(fused_large == fused_small, "fused scratch is flat (%zu %zu)", fused_small, fused_large);
    CHECK(throws<std::invalid_argument>([&] {
              std::vector<float> h(32 * 10);
              std::vector<KeySegmentView> v{KeySegmentView{h.data(), 10, 32}, KeySegmentView{h.data(), 10, 32}};
              naive_topk_scores(random_rows(1, 3 * 32, rng), 3, v, SelectionConfig{});
          }, "naive_topk_scores: n_heads must be a multiple of kv heads"),
          "naive head mismatch");
}

static void test_sharded_world1() {
    // include/reattn/sharded.hpp at world 1: the library's own NCCL communicator (one rank on
    // this GPU) and the captured sharded step equal the single-GPU attend_step
    std::mt19937 rng(17);
    const std::size_t n_kv = 8, nh = 32, d = 128, total = 20000;
    SegmentedKvCache cache(n_kv, d, 32, 4096, SegmentedKvCache::Storage::BF16, total);
    DenseMatrix K = random_rows(total, n_kv * d, rng), V = random_rows(total, n_kv * d, rng);
    for (float* m : {K.values.data(), V.values.data()})
        for (std::size_t i = 0; i < K.values.size(); ++i) m[i] = oracle_round_bf16(m[i]);
    cache.append(K, V);
    const RotaryTable rope(d, 500000.0, 8192);
    const SelectionConfig cfg;
    ShardedDecoder dec(cache, rope, nh, cfg, total, 1, 0, ShardedDecoder::new_comm_id());
    for (int rep = 0; rep < 3; ++rep) {
        if (rep == 1) dec.capture();
        const DenseMatrix q = random_rows(1, nh * d, rng);
        RunStats st;
        const DenseMatrix want = attend_step(q, nh, cache, cfg, rope, AttentionMode::ReAttention, &st);
        const DenseMatrix got = dec.step(q);
        double md = 0;
        for (std::size_t i = 0; i < got.values.size(); ++i)
            md = std::max(md, std::abs(double(got.values[i]) - want.values[i]));
        const reattn_step_stats ss = dec.stats();
        CHECK(md <= 1e-6 && ss.scope_len == st.scope_len_max, "sharded world-1 rep %d md=%g L=%llu/%zu", rep,
              md, (unsigned long long)ss.scope_len, st.scope_len_max);
    }
}

// REATTN_TEST_GARBAGE=1: fill (and free) most device memory with 0xFF bytes first, so later
// allocations start from garbage -- surfaces reads of memory a test never wrote.
static void fill_device_garbage() {
    std::vector<unsigned char> host(64u << 20, 0xFF);
    std::vector<void*> blocks;
    for (int i = 0; i < 24; ++i) {
        void* p = nullptr;
        if (reattn_malloc(gpu::context(), 4ull << 30, &p) != REATTN_OK) break;
        for (std::size_t o = 0; o < (4ull << 30); o += host.size())
            reattn_memcpy_h2d(gpu::context(), (char*)p + o, host.data(), host.size());
        blocks.push_back(p);
    }
    for (void* p : blocks) reattn_free(gpu::context(), p);
}

int main() {
    if (std::getenv("REATTN_TEST_GARBAGE")) fill_device_garbage();
    test_snapshot();
    test_dense_and_naive();
    test_sharded_world1();
    test_fused_topk();
    test_vote_spans();
    test_scope();
    test_rope_attend();
    test_attend_step();
    test_engine();
    std::printf("%d checks, %d failures\n", g_checks, g_fail);
    return g_fail ? 1 : 0;
}
