// Drop-in for reattn/attend.hpp (reference attend.hpp:14-77): finite-scope attention on the
// device with f64 softmax state (m, denominator, entropy numerator, accumulator).
#pragma once

#include <optional>
#include <stdexcept>
#include <vector>

#include "reattn/dense_matrix.hpp"
#include "reattn/runtime.hpp"

namespace reattn {

struct AttendResult {
    DenseMatrix output;               // n_q x dv
    std::vector<double> row_entropy;  // nats, one per query row
};

inline AttendResult attend(const DenseMatrix& q, const DenseMatrix& k, const DenseMatrix& v,
                           std::optional<std::size_t> causal_boundary = std::nullopt) {
    if (k.rows == 0) throw std::invalid_argument("empty key set");
    if (q.cols != k.cols) throw std::invalid_argument("attend: q/k width mismatch");
    if (k.rows != v.rows) throw std::invalid_argument("attend: k/v length mismatch");
    AttendResult res;
    res.output = DenseMatrix(q.rows, v.cols);
    res.row_entropy.assign(q.rows, 0.0);
    if (q.rows == 0) return res;
    gpu::DeviceBuffer<float> dq, dk, dv, dout(q.rows * v.cols);
    gpu::DeviceBuffer<double> dent(q.rows);
    dq.upload(q.values.data(), q.values.size());
    dk.upload(k.values.data(), k.values.size());
    dv.upload(v.values.data(), v.values.size());
    gpu::check(reattn_attend(gpu::context(), dq.get(), q.rows, dk.get(), dv.get(), k.rows, q.cols,
                             v.cols, causal_boundary.has_value() ? 1 : 0,
                             causal_boundary.value_or(0), dout.get(), dent.get()));
    dout.download(res.output.values.data(), res.output.values.size());
    dent.download(res.row_entropy.data(), q.rows);
    return res;
}

}  // namespace reattn
