// Drop-in for reattn/rope.hpp (reference rope.hpp:19-79): rotary tables built exactly as
// the reference (double -> float, :27-39) and resident on the device; rotations run on
// the device (unfused fp32 ops, :55-58).
#pragma once

#include <cstddef>
#include <cstdint>
#include <memory>
#include <span>
#include <stdexcept>
#include <vector>

#include "reattn/dense_matrix.hpp"
#include "reattn/runtime.hpp"

namespace reattn {

class RotaryTable {
public:
    RotaryTable(std::size_t head_dim, double base, std::size_t max_position)
        : head_dim_(head_dim), max_position_(max_position), base_(base) {
        reattn_rope* r = nullptr;
        gpu::check(reattn_rope_create(gpu::context(), head_dim, base, max_position, &r));
        dev_ = std::shared_ptr<reattn_rope>(r, Del{});
        cos_.resize(max_position * (head_dim / 2));
        sin_.resize(max_position * (head_dim / 2));
        gpu::check(reattn_rope_tables_host(r, cos_.data(), sin_.data()));
    }

    std::size_t head_dim() const { return head_dim_; }
    std::size_t max_position() const { return max_position_; }
    double base() const { return base_; }
    const float* cos_row(std::size_t pos) const { return cos_.data() + pos * (head_dim_ / 2); }
    const float* sin_row(std::size_t pos) const { return sin_.data() + pos * (head_dim_ / 2); }

    void rotate_row(float* v, std::size_t pos) const {
        gpu::DeviceBuffer<float> d;
        d.upload(v, head_dim_);
        const std::uint64_t p = pos;
        gpu::check(reattn_rope_rotate(gpu::context(), dev_.get(), d.get(), &p, 1));
        d.download(v, head_dim_);
    }
    const reattn_rope* device() const { return dev_.get(); }

private:
    struct Del {
        void operator()(reattn_rope* r) const { reattn_rope_destroy(r); }
    };
    std::size_t head_dim_, max_position_;
    double base_;
    std::vector<float> cos_, sin_;
    std::shared_ptr<reattn_rope> dev_{nullptr, Del{}};
};

// rope.hpp:70-79
inline DenseMatrix rope_rotate(const DenseMatrix& vectors, std::span<const std::size_t> positions,
                               const RotaryTable& table) {
    if (vectors.cols != table.head_dim())
        throw std::invalid_argument("rope_rotate: row width != head_dim");
    if (positions.size() != vectors.rows)
        throw std::invalid_argument("rope_rotate: one position per row required");
    DenseMatrix out = vectors;
    if (out.rows == 0) return out;
    gpu::DeviceBuffer<float> d;
    d.upload(out.values.data(), out.values.size());
    std::vector<std::uint64_t> p(positions.begin(), positions.end());
    gpu::check(reattn_rope_rotate(gpu::context(), table.device(), d.get(), p.data(), out.rows));
    d.download(out.values.data(), out.values.size());
    return out;
}

}  // namespace reattn
