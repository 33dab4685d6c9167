// Drop-in for reattn/full_attention.hpp (reference full_attention.hpp:21-84): the quadratic
// causal forward pass at true token positions and the greedy decoder built on it.  On the
// device it is the Engine in window mode with l_global = 0 and l_local = pretrain_window and
// k' = 0: the whole stream is one block, so the scope is every token at its own position
// with the causal boundary at 0 -- exactly forward_full's attention (f64 online softmax
// instead of the reference's float stable_softmax; logits agree within the reference's
// 1e-4 bar, tests/test_engine_gpu.py).
#pragma once

#include <cstdint>
#include <span>
#include <stdexcept>
#include <vector>

#include "reattn/engine.hpp"
#include "reattn/model.hpp"

namespace reattn {

inline DenseMatrix forward_full(std::span<const std::uint32_t> tokens, const ModelWeights& w) {
    if (tokens.empty()) throw std::invalid_argument("empty input");
    const ModelConfig& cfg = w.config;
    if (tokens.size() > cfg.pretrain_window)
        throw std::invalid_argument("input length exceeds pretrain window");
    SelectionConfig sel;
    sel.l_global = 0;
    sel.l_local = cfg.pretrain_window;
    sel.l_chunk = cfg.pretrain_window;
    sel.k_prime = 0;
    Engine eng(w, sel, AttentionMode::Window);
    return eng.logits(eng.prefill(tokens));
}

// greedy continuation by full recomputation each step (full_attention.hpp:72-84)
inline std::vector<std::uint32_t> greedy_decode_full(std::span<const std::uint32_t> prompt,
                                                     const ModelWeights& w, std::size_t n_steps) {
    std::vector<std::uint32_t> stream(prompt.begin(), prompt.end());
    std::vector<std::uint32_t> generated;
    for (std::size_t s = 0; s < n_steps; ++s) {
        const DenseMatrix logits = forward_full(stream, w);
        const std::uint32_t next =
            argmax_token(std::span<const float>(logits.row(logits.rows - 1), logits.cols));
        generated.push_back(next);
        stream.push_back(next);
    }
    return generated;
}

}  // namespace reattn
