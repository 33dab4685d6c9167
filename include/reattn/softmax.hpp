// Drop-in for reattn/softmax.hpp (reference softmax.hpp:13-36): the max-subtracted softmax with
// f64 sums and the Shannon entropy of a probability vector, computed on the device
// (reattn_stable_softmax / reattn_attention_entropy) with the reference's element-order sums.
#pragma once

#include <span>
#include <stdexcept>
#include <vector>

#include "reattn/runtime.hpp"

namespace reattn {

inline std::vector<float> stable_softmax(std::span<const float> logits) {
    if (logits.empty()) throw std::invalid_argument("empty logits");
    gpu::DeviceBuffer<float> d, out(logits.size());
    d.upload(logits.data(), logits.size());
    gpu::check(reattn_stable_softmax(gpu::context(), d.get(), logits.size(), out.get()));
    return out.to_vector(logits.size());
}

inline double attention_entropy(std::span<const float> weights) {
    gpu::DeviceBuffer<float> d;
    gpu::DeviceBuffer<double> h(1);
    if (!weights.empty()) d.upload(weights.data(), weights.size());
    gpu::check(reattn_attention_entropy(gpu::context(), weights.empty() ? nullptr : d.get(), weights.size(),
                                        h.get()));
    return h.to_vector(1)[0];
}

}  // namespace reattn
