// Drop-in for reattn/engine.hpp: RunStats (engine.hpp:23-37), attend_step (engine.hpp:43-114)
// and the generation Engine (engine.hpp:119-216).  attend_step -- selection gated as the
// reference, vote, spans, scope, RoPE at compact positions, attention -- is one device
// pipeline (reattn_attend_step); the Engine runs every layer of the decoder on the device
// (reattn_engine_*): projections, cache appends, attend_step, FFN, logits, greedy pick.
#pragma once

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <stdexcept>
#include <vector>

#include "reattn/attend.hpp"
#include "reattn/kv_cache.hpp"
#include "reattn/model.hpp"
#include "reattn/rope.hpp"
#include "reattn/runtime.hpp"
#include "reattn/scope.hpp"
#include "reattn/selection.hpp"

namespace reattn {

struct RunStats {
    std::size_t max_position_used = 0;
    std::size_t ood_positions = 0;
    bool coverage_total = true;
    double entropy_max = 0.0;
    double entropy_sum = 0.0;
    std::size_t entropy_rows = 0;
    std::size_t scope_len_max = 0;
    std::size_t peak_scratch_bytes = 0;
    std::size_t chunks_processed = 0;
    std::size_t decode_steps = 0;
    std::vector<double> decode_latency_ms;
    double entropy_mean() const { return entropy_rows ? entropy_sum / entropy_rows : 0.0; }
};

inline DenseMatrix attend_step(const DenseMatrix& q_pre, std::size_t n_head,
                               const SegmentedKvCache& cache, const SelectionConfig& cfg,
                               const RotaryTable& rope, AttentionMode mode,
                               RunStats* stats = nullptr, ScratchMeter* meter = nullptr,
                               SpanSet* spans_out = nullptr) {
    const std::size_t d = cache.d_head();
    if (n_head % cache.n_kv_heads() != 0)
        throw std::invalid_argument("attend_step: n_head must be a multiple of kv heads");
    if (q_pre.cols != n_head * d)
        throw std::invalid_argument("attend_step: query width != n_head * d_head");
    const std::size_t n_q = q_pre.rows;
    gpu::DeviceBuffer<float> dq, dout(std::max<std::size_t>(1, n_q * n_head * d));
    dq.upload(q_pre.values.data(), q_pre.values.size());
    const reattn_selection_config c = cfg.to_c();
    reattn_step_stats st{};
    std::vector<std::uint64_t> sb(std::max<std::size_t>(1, cfg.k_prime)),
        se(std::max<std::size_t>(1, cfg.k_prime));
    gpu::check(reattn_attend_step(gpu::context(), cache.device(), rope.device(), dq.get(), n_q,
                                  n_head, &c, static_cast<int>(mode), dout.get(), &st, sb.data(),
                                  se.data(), nullptr));
    DenseMatrix out(n_q, n_head * d);
    dout.download(out.values.data(), out.values.size());
    if (meter) {
        meter->add(st.peak_scratch_bytes);
        meter->sub(st.peak_scratch_bytes);
    }
    if (spans_out) {
        spans_out->spans.clear();
        for (std::size_t i = 0; i < st.n_spans; ++i) spans_out->spans.push_back(Span{sb[i], se[i]});
    }
    if (stats) {  // engine.hpp:64, :100-112 accumulation semantics
        if (!st.coverage_total) stats->coverage_total = false;
        stats->ood_positions += st.ood_positions;
        stats->entropy_max = std::max(stats->entropy_max, st.entropy_max);
        stats->entropy_sum += st.entropy_sum;
        stats->entropy_rows += st.entropy_rows;
        stats->scope_len_max = std::max<std::size_t>(stats->scope_len_max, st.scope_len);
        stats->max_position_used = std::max<std::size_t>(stats->max_position_used, st.max_position_used);
        stats->peak_scratch_bytes = std::max<std::size_t>(stats->peak_scratch_bytes, st.peak_scratch_bytes);
    }
    return out;
}

// Engine (engine.hpp:119-216): per-layer device caches, chunked prefill (first l_global +
// l_local tokens, then l_chunk strides), greedy decode.  Holds `weights` by reference as the
// reference does, plus its device copy.  caches() is not mirrored (the device caches are
// reachable through reattn_engine_cache); everything else keeps the reference's semantics.
class Engine {
public:
    Engine(const ModelWeights& weights, const SelectionConfig& sel, AttentionMode mode)
        : w_(weights), sel_(sel), mode_(mode), dev_(detail::DeviceWeights::from_host(weights)) {
        const reattn_selection_config c = sel.to_c();
        gpu::check(reattn_engine_create(gpu::context(), dev_.get(), &c, static_cast<int>(mode),
                                        REATTN_F32, &e_));
        last_spans_.assign(weights.config.n_layer, SpanSet{});
    }
    Engine(const Engine&) = delete;
    Engine& operator=(const Engine&) = delete;
    ~Engine() {
        if (e_) reattn_engine_destroy(e_);
    }

    void reset() {
        gpu::check(reattn_engine_reset(e_));
        last_spans_.assign(w_.config.n_layer, SpanSet{});
        last_logits_.clear();
        refresh();
    }

    DenseMatrix prefill(std::span<const std::uint32_t> tokens) {
        std::uint64_t rows = 0;
        gpu::check(reattn_engine_prefill(e_, tokens.data(), tokens.size(), &rows));
        DenseMatrix h(rows, w_.config.d_model);
        gpu::check(reattn_engine_hidden(e_, h.values.data(), h.values.size()));
        refresh();
        return h;
    }

    std::uint32_t decode_step(std::uint32_t last_token) {
        std::uint32_t next = 0;
        gpu::check(reattn_engine_decode_step(e_, last_token, &next));
        last_logits_.resize(w_.config.vocab_size);
        gpu::check(reattn_engine_last_logits(e_, last_logits_.data(), last_logits_.size()));
        refresh();
        return next;
    }

    DenseMatrix logits(const DenseMatrix& hidden) const {
        DenseMatrix out(hidden.rows, w_.config.vocab_size);
        if (hidden.cols != w_.config.d_model) throw std::invalid_argument("rmsnorm: weight width mismatch");
        gpu::check(reattn_engine_logits(e_, hidden.values.data(), hidden.rows, out.values.data()));
        return out;
    }

    const RunStats& stats() const { return stats_; }
    const std::vector<SpanSet>& last_spans() const { return last_spans_; }
    const ModelWeights& weights() const { return w_; }
    const SelectionConfig& selection_config() const { return sel_; }
    AttentionMode mode() const { return mode_; }
    std::span<const float> last_logits() const { return last_logits_; }
    const reattn_cache* cache_handle(std::size_t layer) const { return reattn_engine_cache(e_, layer); }

private:
    void refresh() {
        reattn_run_stats s{};
        gpu::check(reattn_engine_stats(e_, &s));
        stats_.max_position_used = s.max_position_used;
        stats_.ood_positions = s.ood_positions;
        stats_.coverage_total = s.coverage_total != 0;
        stats_.entropy_max = s.entropy_max;
        stats_.entropy_sum = s.entropy_sum;
        stats_.entropy_rows = s.entropy_rows;
        stats_.scope_len_max = s.scope_len_max;
        stats_.peak_scratch_bytes = s.peak_scratch_bytes;
        stats_.chunks_processed = s.chunks_processed;
        stats_.decode_steps = s.decode_steps;
        std::uint64_t n = 0;
        gpu::check(reattn_engine_decode_latencies(e_, nullptr, 0, &n));
        stats_.decode_latency_ms.resize(n);
        gpu::check(reattn_engine_decode_latencies(e_, stats_.decode_latency_ms.data(), n, &n));
        for (std::size_t l = 0; l < last_spans_.size(); ++l) {
            std::uint64_t k = 0;
            gpu::check(reattn_engine_last_spans(e_, l, nullptr, nullptr, 0, &k));
            std::vector<std::uint64_t> b(k), e(k);
            gpu::check(reattn_engine_last_spans(e_, l, b.data(), e.data(), k, &k));
            last_spans_[l].spans.clear();
            for (std::size_t i = 0; i < k; ++i) last_spans_[l].spans.push_back(Span{b[i], e[i]});
        }
    }

    const ModelWeights& w_;
    SelectionConfig sel_;
    AttentionMode mode_;
    detail::DeviceWeights dev_;
    reattn_engine* e_ = nullptr;
    RunStats stats_;
    std::vector<SpanSet> last_spans_;
    std::vector<float> last_logits_;
};

}  // namespace reattn
