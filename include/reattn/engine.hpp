// Drop-in for the hot-path part of reattn/engine.hpp: AttentionMode (model.hpp:19),
// RunStats (engine.hpp:23-37) and attend_step (engine.hpp:43-114 in the survey's
// numbering; :501-572 in the file).  The whole step — selection gated as the reference,
// vote, spans, scope, RoPE at compact positions, attention — is one device pipeline
// (reattn_attend_step).  The toy-model Engine around it is out of scope.
#pragma once

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <stdexcept>
#include <vector>

#include "reattn/attend.hpp"
#include "reattn/kv_cache.hpp"
#include "reattn/rope.hpp"
#include "reattn/runtime.hpp"
#include "reattn/scope.hpp"
#include "reattn/selection.hpp"

namespace reattn {

enum class AttentionMode : std::uint32_t { Full = 0, Window = 1, ReAttention = 2 };

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
    if (stats) {  // engine.hpp:522, :558-570 accumulation semantics
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

}  // namespace reattn
