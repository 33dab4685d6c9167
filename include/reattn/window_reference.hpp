// Drop-in for reattn/window_reference.hpp (reference window_reference.hpp:21-140): global
// prefix + local suffix attention with the reference's constructor checks and messages.
// On the device this is the Engine in window mode (no selection), which the reference's own
// C03 criterion proves bit-identical to its independent WindowReference.
#pragma once

#include <cstdint>
#include <memory>
#include <span>
#include <stdexcept>

#include "reattn/engine.hpp"
#include "reattn/model.hpp"

namespace reattn {

class WindowReference {
public:
    WindowReference(const ModelWeights& weights, std::size_t l_global, std::size_t l_local,
                    std::size_t l_chunk)
        : w_(weights) {
        if (l_local == 0 || l_chunk == 0 || l_chunk > l_local)
            throw std::invalid_argument("window reference: bad local/chunk sizes");
        if (l_global + l_local > weights.config.pretrain_window)
            throw std::invalid_argument("window reference: window budget exceeds pretrain range");
        SelectionConfig sel;
        sel.l_global = l_global;
        sel.l_local = l_local;
        sel.l_chunk = l_chunk;
        sel.k_prime = 0;
        eng_ = std::make_unique<Engine>(weights, sel, AttentionMode::Window);
    }

    DenseMatrix prefill(std::span<const std::uint32_t> tokens) { return eng_->prefill(tokens); }
    std::uint32_t decode_step(std::uint32_t last_token) { return eng_->decode_step(last_token); }
    DenseMatrix logits(const DenseMatrix& hidden) const { return eng_->logits(hidden); }
    std::span<const float> last_logits() const { return eng_->last_logits(); }

private:
    const ModelWeights& w_;
    std::unique_ptr<Engine> eng_;
};

}  // namespace reattn
