// Drop-in for reattn/selection.hpp (reference selection.hpp:16-349): same names, types,
// defaults, exceptions; the computation runs in the sm_100a kernels (K1 scan + top-k,
// K3 vote/spans) through include/reattn_cuda.h.
#pragma once

#include <algorithm>
#include <cstdint>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "reattn/dense_matrix.hpp"
#include "reattn/kv_cache.hpp"
#include "reattn/runtime.hpp"

namespace reattn {

enum class SpanMode { Aligned, Centered };

// selection.hpp:20-45 (identical defaults: budget 32 + 127*32 + 4096 = 8192).
struct SelectionConfig {
    std::size_t k = 4;
    std::size_t k_prime = 127;
    std::size_t span_m = 32;
    std::size_t tile_size = 2048;  // bounds the reference's CPU scratch only; ignored here
    std::size_t l_global = 32;
    std::size_t l_local = 4096;
    std::size_t l_chunk = 512;
    SpanMode span_mode = SpanMode::Aligned;

    std::size_t budget() const { return l_global + k_prime * span_m + l_local; }

    void validate(std::size_t pretrain_window) const {
        if (k == 0) throw std::invalid_argument("selection: k must be >= 1");
        if (span_m == 0) throw std::invalid_argument("selection: span_m must be >= 1");
        if (tile_size == 0) throw std::invalid_argument("selection: tile_size must be >= 1");
        if (l_chunk == 0) throw std::invalid_argument("selection: l_chunk must be >= 1");
        if (l_chunk > l_local)
            throw std::invalid_argument("selection: l_chunk must not exceed l_local");
        if (budget() > pretrain_window)
            throw std::invalid_argument(
                "selection: budget l_global + k_prime*span_m + l_local = " +
                std::to_string(budget()) + " exceeds pretrain window " +
                std::to_string(pretrain_window));
    }

    reattn_selection_config to_c() const {
        reattn_selection_config c{};
        c.k = k;
        c.k_prime = k_prime;
        c.span_m = span_m;
        c.tile_size = tile_size;
        c.l_global = l_global;
        c.l_local = l_local;
        c.l_chunk = l_chunk;
        c.span_mode = span_mode == SpanMode::Aligned ? REATTN_SPAN_ALIGNED : REATTN_SPAN_CENTERED;
        return c;
    }
};

// selection.hpp:49-58: counts the transient DEVICE workspace the scorer uses (constant in
// the middle length, the reference's scratch contract).
struct ScratchMeter {
    std::size_t current = 0;
    std::size_t peak = 0;
    void add(std::size_t n) {
        current += n;
        peak = std::max(peak, current);
    }
    void sub(std::size_t n) { current -= n; }
    void reset() { current = peak = 0; }
};

struct TopkEntry {
    std::size_t index;
    float score;
};

struct ScoredCandidate {
    std::size_t middle_index;
    float score;
    std::size_t votes;
};

using PerHeadTopk = std::vector<std::vector<std::vector<TopkEntry>>>;

namespace detail {

// selection.hpp:81-135: the running top-k buffer (host; the device scans keep the same rule in
// registers).  Filled unsorted; once full, the worst entry -- lowest score, then highest
// index -- is cached, and only a strictly greater score replaces it, so equal scores keep the
// lower (earlier) index.  sorted() orders by score desc, index asc.
struct TopkBuffer {
    std::vector<TopkEntry> entries;
    std::size_t cap = 0;
    std::size_t worst = 0;
    float threshold = 0.0f;

    void init(std::size_t k) {
        cap = k;
        entries.clear();
        entries.reserve(k);
        worst = 0;
        threshold = 0.0f;
    }
    bool full() const { return entries.size() == cap; }
    void refresh_worst() {
        std::size_t w = 0;
        for (std::size_t i = 1; i < entries.size(); ++i) {
            const bool lower = entries[i].score < entries[w].score;
            const bool tie_later = entries[i].score == entries[w].score && entries[i].index > entries[w].index;
            if (lower || tie_later) w = i;
        }
        worst = w;
        threshold = entries.empty() ? 0.0f : entries[w].score;
    }
    void fill(std::size_t index, float score) {
        entries.push_back(TopkEntry{index, score});
        if (full()) refresh_worst();
    }
    void replace_worst(std::size_t index, float score) {  // caller checked score > threshold
        entries[worst] = TopkEntry{index, score};
        refresh_worst();
    }
    void offer(std::size_t index, float score) {
        if (!full())
            fill(index, score);
        else if (score > threshold)
            replace_worst(index, score);
    }
    std::vector<TopkEntry> sorted() const {
        std::vector<TopkEntry> out(entries);
        std::stable_sort(out.begin(), out.end(), [](const TopkEntry& x, const TopkEntry& y) {
            return x.score != y.score ? x.score > y.score : x.index < y.index;
        });
        return out;
    }
};

// selection.hpp:139-156 on the device (csrc/dense.cu): each kv group's mean query, a sequential
// fp32 sum times float(1 / group).
inline DenseMatrix group_mean_queries(const DenseMatrix& queries, std::size_t n_heads,
                                      std::size_t n_kv_heads, std::size_t d) {
    DenseMatrix mq(queries.rows, n_kv_heads * d);
    if (n_kv_heads == 0 || n_heads % n_kv_heads != 0)
        throw std::invalid_argument("fused_topk_scores: n_heads must be a multiple of kv heads");
    if (mq.values.empty()) return mq;
    gpu::DeviceBuffer<float> q, out(mq.values.size());
    q.upload(queries.values.data(), queries.values.size());
    gpu::check(reattn_group_mean(gpu::context(), q.get(), queries.rows, n_heads, n_kv_heads, d,
                                 out.get()));
    mq.values = out.to_vector(mq.values.size());
    return mq;
}

}  // namespace detail

// fused_topk_scores on a device view (no copy of the middle).
inline PerHeadTopk fused_topk_scores(const DenseMatrix& queries, std::size_t n_heads,
                                     const DeviceKeySegmentView& mid, const SelectionConfig& cfg,
                                     ScratchMeter* meter = nullptr) {
    const std::size_t n_kv = mid.n_kv;
    if (n_kv == 0 || n_heads % n_kv != 0)
        throw std::invalid_argument("fused_topk_scores: n_heads must be a multiple of kv heads");
    if (queries.cols != n_heads * mid.dim)
        throw std::invalid_argument("fused_topk_scores: query width != n_heads * d");
    const std::size_t n_q = queries.rows, k = cfg.k;
    PerHeadTopk result(n_kv, std::vector<std::vector<TopkEntry>>(n_q));
    gpu::DeviceBuffer<float> q;
    q.upload(queries.values.data(), queries.values.size());
    gpu::DeviceBuffer<std::uint32_t> idx(n_kv * n_q * k);
    gpu::DeviceBuffer<float> sc(n_kv * n_q * k);
    std::uint64_t n_out = 0, scratch = 0;
    gpu::check(reattn_fused_topk(gpu::context(), q.get(), n_q, n_heads, mid.base, mid.dtype, n_kv,
                                 mid.head_stride, mid.row0, mid.count, mid.dim, k, idx.get(),
                                 sc.get(), &n_out, &scratch));
    if (meter) {
        meter->add(scratch);
        meter->sub(scratch);
    }
    if (mid.count == 0 || n_q == 0) return result;
    const auto hi = idx.to_vector(n_kv * n_q * k);
    const auto hs = sc.to_vector(n_kv * n_q * k);
    for (std::size_t kv = 0; kv < n_kv; ++kv)
        for (std::size_t qq = 0; qq < n_q; ++qq)
            for (std::size_t j = 0; j < n_out; ++j) {
                const std::size_t o = (kv * n_q + qq) * k + j;
                result[kv][qq].push_back(TopkEntry{hi[o], hs[o]});
            }
    return result;
}

// selection.hpp:168 signature: host views (copied to the device for the call).
inline PerHeadTopk fused_topk_scores(const DenseMatrix& queries, std::size_t n_heads,
                                     std::span<const KeySegmentView> middle,
                                     const SelectionConfig& cfg, ScratchMeter* meter = nullptr) {
    const std::size_t n_kv = middle.size();
    if (n_kv == 0 || n_heads % n_kv != 0)
        throw std::invalid_argument("fused_topk_scores: n_heads must be a multiple of kv heads");
    const std::size_t d = middle[0].dim, count = middle[0].count;
    if (queries.cols != n_heads * d)
        throw std::invalid_argument("fused_topk_scores: query width != n_heads * d");
    std::vector<float> packed(n_kv * count * d);
    for (std::size_t h = 0; h < n_kv; ++h)
        if (count) std::copy(middle[h].data, middle[h].data + count * d, packed.begin() + h * count * d);
    gpu::DeviceBuffer<float> keys;
    keys.upload(packed.data(), packed.size());
    return fused_topk_scores(queries, n_heads,
                             DeviceKeySegmentView{keys.get(), REATTN_F32, n_kv, count, 0, count, d},
                             cfg, meter);
}

namespace detail {
inline void flatten(const PerHeadTopk& per_head, std::vector<std::uint32_t>& idx,
                    std::vector<float>& score) {
    for (const auto& head : per_head)
        for (const auto& query : head)
            for (const TopkEntry& e : query) {
                if (e.index > 0xFFFFFFFFull) throw std::out_of_range("vote: index beyond 32 bits");
                idx.push_back(static_cast<std::uint32_t>(e.index));
                score.push_back(e.score);
            }
}
}  // namespace detail

// selection.hpp:252-276 (on the device).
inline std::vector<ScoredCandidate> tally_candidates(const PerHeadTopk& per_head) {
    std::vector<std::uint32_t> idx;
    std::vector<float> score;
    detail::flatten(per_head, idx, score);
    std::vector<ScoredCandidate> out;
    if (idx.empty()) return out;
    gpu::DeviceBuffer<std::uint32_t> di, oi(idx.size()), ov(idx.size());
    gpu::DeviceBuffer<float> ds, os(idx.size());
    di.upload(idx.data(), idx.size());
    ds.upload(score.data(), score.size());
    std::uint64_t n = 0;
    gpu::check(reattn_tally(gpu::context(), di.get(), ds.get(), idx.size(), oi.get(), ov.get(),
                            os.get(), &n));
    const auto hi = oi.to_vector(n);
    const auto hv = ov.to_vector(n);
    const auto hs = os.to_vector(n);
    for (std::size_t i = 0; i < n; ++i) out.push_back(ScoredCandidate{hi[i], hs[i], hv[i]});
    return out;
}

// selection.hpp:278-286 (on the device).
inline std::vector<std::size_t> vote(const PerHeadTopk& per_head, std::size_t k_prime) {
    std::vector<std::size_t> winners;
    if (k_prime == 0) return winners;
    std::vector<std::uint32_t> idx;
    std::vector<float> score;
    detail::flatten(per_head, idx, score);
    if (idx.empty()) return winners;
    gpu::DeviceBuffer<std::uint32_t> di, dw(std::min(k_prime, idx.size()));
    gpu::DeviceBuffer<float> ds;
    di.upload(idx.data(), idx.size());
    ds.upload(score.data(), score.size());
    std::uint64_t n = 0;
    gpu::check(reattn_vote(gpu::context(), di.get(), ds.get(), idx.size(), k_prime, dw.get(), &n));
    for (std::uint32_t w : dw.to_vector(n)) winners.push_back(w);
    return winners;
}

struct Span {
    std::size_t begin = 0;
    std::size_t end = 0;
    std::size_t size() const { return end - begin; }
    bool operator==(const Span&) const = default;
};

struct SpanSet {
    std::vector<Span> spans;
    std::size_t coverage() const {
        std::size_t c = 0;
        for (const Span& s : spans) c += s.size();
        return c;
    }
    bool contains(std::size_t idx) const {
        for (const Span& s : spans)
            if (idx >= s.begin && idx < s.end) return true;
        return false;
    }
    bool empty() const { return spans.empty(); }
};

// selection.hpp:318-349 (on the device).
inline SpanSet expand_spans(std::span<const std::size_t> winners, std::size_t span_m,
                            std::size_t middle_len, SpanMode mode = SpanMode::Aligned) {
    SpanSet out;
    if (winners.empty() || middle_len == 0) return out;
    if (middle_len > 0xFFFFFFFFull) throw std::out_of_range("expand_spans: middle beyond 32 bits");
    std::vector<std::uint32_t> w;
    for (std::size_t x : winners) {
        if (x >= middle_len) throw std::out_of_range("expand_spans: winner outside middle");
        w.push_back(static_cast<std::uint32_t>(x));
    }
    gpu::DeviceBuffer<std::uint32_t> dw, db(w.size()), de(w.size());
    dw.upload(w.data(), w.size());
    std::uint64_t n = 0;
    gpu::check(reattn_expand_spans(gpu::context(), dw.get(), w.size(), span_m, middle_len,
                                   mode == SpanMode::Aligned ? REATTN_SPAN_ALIGNED
                                                             : REATTN_SPAN_CENTERED,
                                   db.get(), de.get(), &n));
    const auto hb = db.to_vector(n);
    const auto he = de.to_vector(n);
    for (std::size_t i = 0; i < n; ++i) out.spans.push_back(Span{hb[i], he[i]});
    return out;
}

}  // namespace reattn
