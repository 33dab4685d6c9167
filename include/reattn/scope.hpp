// Drop-in for reattn/scope.hpp (reference scope.hpp:17-85): scope assembly on the device
// (index table + K/V gather); the hot path (attend_step) never materialises these copies.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <vector>

#include "reattn/kv_cache.hpp"
#include "reattn/runtime.hpp"
#include "reattn/selection.hpp"

namespace reattn {

struct AttentionScope {
    std::size_t n_kv_heads = 0;
    std::size_t d_head = 0;
    std::size_t length = 0;
    std::vector<std::vector<float>> keys;    // [kv][length * d_head]
    std::vector<std::vector<float>> values;  // [kv][length * d_head]
    std::vector<std::size_t> source_indices;
    const float* key_row(std::size_t kv, std::size_t i) const { return keys[kv].data() + i * d_head; }
    const float* value_row(std::size_t kv, std::size_t i) const {
        return values[kv].data() + i * d_head;
    }
};

inline AttentionScope assemble_scope(const SegmentedKvCache& cache, const SpanSet& spans,
                                     std::size_t pretrain_window) {
    AttentionScope scope;
    scope.n_kv_heads = cache.n_kv_heads();
    scope.d_head = cache.d_head();
    std::vector<std::uint32_t> b, e;
    for (const Span& s : spans.spans) {
        if (s.end > 0xFFFFFFFFull) throw std::out_of_range("assemble_scope: span outside middle");
        b.push_back(static_cast<std::uint32_t>(s.begin));
        e.push_back(static_cast<std::uint32_t>(s.end));
    }
    gpu::DeviceBuffer<std::uint32_t> db, de;
    db.upload(b.data(), b.size());
    de.upload(e.data(), e.size());
    // upper bound on L: the whole cache (the device checks the window)
    const std::size_t cap = std::min<std::size_t>(cache.total(), pretrain_window) + 1;
    gpu::DeviceBuffer<std::uint32_t> src(cap);
    gpu::DeviceBuffer<float> k(cache.n_kv_heads() * cap * cache.d_head()),
        v(cache.n_kv_heads() * cap * cache.d_head());
    std::uint64_t L = 0;
    gpu::check(reattn_assemble_scope(gpu::context(), cache.device(), b.empty() ? nullptr : db.get(),
                                     e.empty() ? nullptr : de.get(), b.size(), pretrain_window,
                                     src.get(), k.get(), v.get(), &L));
    scope.length = L;
    for (std::uint32_t s : src.to_vector(L)) scope.source_indices.push_back(s);
    const std::size_t per = L * scope.d_head;
    const auto hk = k.to_vector(scope.n_kv_heads * per);
    const auto hv = v.to_vector(scope.n_kv_heads * per);
    scope.keys.resize(scope.n_kv_heads);
    scope.values.resize(scope.n_kv_heads);
    for (std::size_t h = 0; h < scope.n_kv_heads; ++h) {
        scope.keys[h].assign(hk.begin() + h * per, hk.begin() + (h + 1) * per);
        scope.values[h].assign(hv.begin() + h * per, hv.begin() + (h + 1) * per);
    }
    return scope;
}

inline AttentionScope assemble_window_scope(const SegmentedKvCache& cache,
                                            std::size_t pretrain_window) {
    return assemble_scope(cache, SpanSet{}, pretrain_window);
}

}  // namespace reattn
