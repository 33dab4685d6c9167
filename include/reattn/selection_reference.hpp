// Drop-in for reattn/selection_reference.hpp (reference selection_reference.hpp:18-69):
// naive_topk_scores, the unfused scorer the reference keeps for equivalence tests and its
// memory benchmark.  Here an independent device route (csrc/dense.cu): the whole middle x n_q
// score matrix is materialised in device memory (scratch linear in the middle length, as the
// reference's), then each row's top-k is selected; the lists equal fused_topk_scores'.
#pragma once

#include <span>
#include <stdexcept>
#include <vector>

#include "reattn/selection.hpp"

namespace reattn {

inline PerHeadTopk naive_topk_scores(const DenseMatrix& queries, std::size_t n_heads,
                                     const DeviceKeySegmentView& mid, const SelectionConfig& cfg,
                                     ScratchMeter* meter = nullptr) {
    const std::size_t n_kv = mid.n_kv;
    if (n_kv == 0 || n_heads % n_kv != 0)
        throw std::invalid_argument("naive_topk_scores: n_heads must be a multiple of kv heads");
    if (queries.cols != n_heads * mid.dim)
        throw std::invalid_argument("naive_topk_scores: query width != n_heads * d");
    const std::size_t n_q = queries.rows, k = cfg.k;
    PerHeadTopk result(n_kv, std::vector<std::vector<TopkEntry>>(n_q));
    gpu::DeviceBuffer<float> q;
    q.upload(queries.values.data(), queries.values.size());
    gpu::DeviceBuffer<std::uint32_t> idx(n_kv * n_q * k);
    gpu::DeviceBuffer<float> sc(n_kv * n_q * k);
    std::uint64_t n_out = 0, scratch = 0;
    gpu::check(reattn_naive_topk(gpu::context(), q.get(), n_q, n_heads, mid.base, mid.dtype, n_kv,
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

// selection_reference.hpp:18-20 signature: host views (copied to the device for the call).
inline PerHeadTopk naive_topk_scores(const DenseMatrix& queries, std::size_t n_heads,
                                     std::span<const KeySegmentView> middle,
                                     const SelectionConfig& cfg, ScratchMeter* meter = nullptr) {
    const std::size_t n_kv = middle.size();
    if (n_kv == 0 || n_heads % n_kv != 0)
        throw std::invalid_argument("naive_topk_scores: n_heads must be a multiple of kv heads");
    const std::size_t d = middle[0].dim, count = middle[0].count;
    if (queries.cols != n_heads * d)
        throw std::invalid_argument("naive_topk_scores: query width != n_heads * d");
    std::vector<float> packed(n_kv * count * d);
    for (std::size_t h = 0; h < n_kv; ++h)
        if (count) std::copy(middle[h].data, middle[h].data + count * d, packed.begin() + h * count * d);
    gpu::DeviceBuffer<float> keys;
    keys.upload(packed.data(), packed.size());
    return naive_topk_scores(queries, n_heads,
                             DeviceKeySegmentView{keys.get(), REATTN_F32, n_kv, count, 0, count, d},
                             cfg, meter);
}

}  // namespace reattn
