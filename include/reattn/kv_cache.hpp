// Drop-in for reattn/kv_cache.hpp (reference kv_cache.hpp:17-118): the segmented,
// position-free KV cache, now resident on the device (head-major [n_kv][capacity][d],
// fp32 by default or bf16), with the reference's FIFO boundary arithmetic (:65-67).
// A host shadow of the appended rows backs the reference's zero-copy host accessors
// (key(), value(), middle_keys()); compute never reads it.
#pragma once

#include <algorithm>
#include <cstddef>
#include <cstdint>
#include <cstring>
#include <span>
#include <string>
#include <memory>
#include <stdexcept>
#include <utility>
#include <vector>

#include "reattn/dense_matrix.hpp"
#include "reattn/runtime.hpp"

namespace reattn {

struct SegmentView {
    std::size_t begin = 0;
    std::size_t end = 0;
    std::size_t size() const { return end - begin; }
    bool empty() const { return begin == end; }
};

// Contiguous slice of one KV head's key storage on the HOST (reference kv_cache.hpp:25-30).
struct KeySegmentView {
    const float* data = nullptr;
    std::size_t count = 0;
    std::size_t dim = 0;
    const float* row(std::size_t i) const { return data + i * dim; }
};

// The same slice on the DEVICE: rows `row0 .. row0+count` of every head of a head-major
// [n_kv][head_stride][dim] array (what the kernels consume without a copy).
struct DeviceKeySegmentView {
    const void* base = nullptr;
    int dtype = REATTN_F32;
    std::size_t n_kv = 0, head_stride = 0, row0 = 0, count = 0, dim = 0;
};

class SegmentedKvCache {
public:
    enum class Storage { F32 = REATTN_F32, BF16 = REATTN_BF16 };

    SegmentedKvCache(std::size_t n_kv_heads, std::size_t d_head, std::size_t l_global,
                     std::size_t l_local_max, Storage storage = Storage::F32,
                     std::size_t initial_capacity = 1024, bool host_shadow = true)
        : n_kv_(n_kv_heads), d_(d_head), g_(l_global), local_(l_local_max),
          shadow_(host_shadow), keys_(n_kv_heads), values_(n_kv_heads) {
        if (n_kv_heads == 0 || d_head == 0)
            throw std::invalid_argument("cache needs at least one head and a positive head dim");
        if (l_local_max == 0) throw std::invalid_argument("l_local_max must be positive");
        reattn_cache* c = nullptr;
        gpu::check(reattn_cache_create(gpu::context(), n_kv_heads, d_head, l_global, l_local_max,
                                       std::max<std::size_t>(initial_capacity, 1),
                                       static_cast<int>(storage), &c));
        dev_.reset(c);
    }

    // new_keys / new_values: rows = entries, cols = n_kv_heads * d_head (kv_cache.hpp:54).
    void append(const DenseMatrix& new_keys, const DenseMatrix& new_values) {
        if (new_keys.cols != n_kv_ * d_ || !new_keys.same_shape(new_values))
            throw std::invalid_argument("cache append: shape mismatch");
        if (new_keys.rows == 0) return;
        std::uint64_t cap = 0, total = 0;
        reattn_cache_info(dev_.get(), nullptr, nullptr, nullptr, nullptr, &cap, &total, nullptr,
                          nullptr, nullptr);
        if (total + new_keys.rows > cap)
            gpu::check(reattn_cache_reserve(gpu::context(), dev_.get(),
                                            std::max<std::uint64_t>(2 * cap, total + new_keys.rows)));
        gpu::check(reattn_cache_append(gpu::context(), dev_.get(), new_keys.values.data(),
                                       new_values.values.data(), new_keys.rows, 0));
        if (shadow_) {
            for (std::size_t r = 0; r < new_keys.rows; ++r)
                for (std::size_t h = 0; h < n_kv_; ++h) {
                    keys_[h].insert(keys_[h].end(), new_keys.row(r) + h * d_,
                                    new_keys.row(r) + (h + 1) * d_);
                    values_[h].insert(values_[h].end(), new_values.row(r) + h * d_,
                                      new_values.row(r) + (h + 1) * d_);
                }
        }
        total_ += new_keys.rows;
    }

    std::size_t total() const { return total_; }
    std::size_t n_kv_heads() const { return n_kv_; }
    std::size_t d_head() const { return d_; }
    std::size_t l_global() const { return g_; }
    std::size_t l_local_max() const { return local_; }

    struct Views {
        SegmentView global;
        SegmentView middle;
        SegmentView local;
    };
    Views views() const {
        const std::size_t ge = std::min(total_, g_);
        const std::size_t ls = total_ - std::min(total_ - ge, local_);
        return Views{SegmentView{0, ge}, SegmentView{ge, ls}, SegmentView{ls, total_}};
    }
    std::size_t middle_len() const { return views().middle.size(); }

    const float* key(std::size_t head, std::size_t idx) const {
        need_shadow();
        return keys_[head].data() + idx * d_;
    }
    const float* value(std::size_t head, std::size_t idx) const {
        need_shadow();
        return values_[head].data() + idx * d_;
    }
    KeySegmentView middle_keys(std::size_t head) const {
        need_shadow();
        return KeySegmentView{keys_[head].data() + views().global.end * d_, middle_len(), d_};
    }
    std::vector<KeySegmentView> middle_keys_all() const {
        std::vector<KeySegmentView> out;
        for (std::size_t h = 0; h < n_kv_; ++h) out.push_back(middle_keys(h));
        return out;
    }

    // device-side views (no copies)
    DeviceKeySegmentView device_middle_keys() const {
        std::uint64_t cap = 0;
        int dt = 0;
        reattn_cache_info(dev_.get(), nullptr, nullptr, nullptr, nullptr, &cap, nullptr, nullptr,
                          nullptr, &dt);
        return DeviceKeySegmentView{reattn_cache_keys(dev_.get()), dt, n_kv_, cap,
                                    views().global.end, middle_len(), d_};
    }
    const reattn_cache* device() const { return dev_.get(); }

    // Adopt a device cache created by the C-ABI (snapshot load); with host_shadow the rows
    // are read back once for the reference's host accessors (bf16 widened exactly).
    static SegmentedKvCache adopt(reattn_cache* c, bool host_shadow = true) {
        std::uint64_t n_kv = 0, d = 0, g = 0, loc = 0, cap = 0, total = 0;
        int dt = 0;
        reattn_cache_info(c, &n_kv, &d, &g, &loc, &cap, &total, nullptr, nullptr, &dt);
        SegmentedKvCache out(c, n_kv, d, g, loc, host_shadow);
        out.total_ = total;
        if (host_shadow && total) {
            const std::size_t esz = dt == REATTN_BF16 ? 2 : 4;
            std::vector<std::uint8_t> raw(total * d * esz);
            for (int part = 0; part < 2; ++part) {
                const auto* base = static_cast<const std::uint8_t*>(part ? reattn_cache_values(c)
                                                                         : reattn_cache_keys(c));
                for (std::size_t h = 0; h < n_kv; ++h) {
                    gpu::check(reattn_memcpy_d2h(gpu::context(), raw.data(), base + h * cap * d * esz,
                                                 raw.size()));
                    auto& dst = part ? out.values_[h] : out.keys_[h];
                    dst.resize(total * d);
                    for (std::size_t e = 0; e < total * d; ++e) {
                        if (esz == 4) {
                            std::memcpy(&dst[e], raw.data() + 4 * e, 4);
                        } else {
                            std::uint16_t b;
                            std::memcpy(&b, raw.data() + 2 * e, 2);
                            const std::uint32_t w = std::uint32_t(b) << 16;
                            std::memcpy(&dst[e], &w, 4);
                        }
                    }
                }
            }
        }
        return out;
    }

private:
    SegmentedKvCache(reattn_cache* c, std::size_t n_kv, std::size_t d, std::size_t g,
                     std::size_t loc, bool host_shadow)
        : n_kv_(n_kv), d_(d), g_(g), local_(loc), shadow_(host_shadow), keys_(n_kv),
          values_(n_kv) {
        dev_.reset(c);
    }
    void need_shadow() const {
        if (!shadow_)
            throw std::logic_error("SegmentedKvCache: host accessors need host_shadow = true");
    }
    struct Del {
        void operator()(reattn_cache* c) const { reattn_cache_destroy(c); }
    };
    std::size_t n_kv_, d_, g_, local_, total_ = 0;
    bool shadow_;
    std::vector<std::vector<float>> keys_, values_;
    std::unique_ptr<reattn_cache, Del> dev_;
};

// RKVC snapshot container (reference kv_cache.hpp:120-209): magic "RKVC", u32 version,
// u32 n_layers / n_kv_heads / d_head, per layer u64 {total, l_global, l_local_max} and raw
// f32 key and value payloads, head-major.  Same signatures, messages and exception types;
// the payloads stream straight between the file and device storage.
inline void write_cache_snapshot(const std::string& path, std::span<const SegmentedKvCache> layers) {
    std::vector<const reattn_cache*> dev;
    for (const auto& l : layers) dev.push_back(l.device());
    gpu::check(reattn_snapshot_write(gpu::context(), path.c_str(), dev.data(),
                                     static_cast<std::uint32_t>(dev.size())));
}

inline std::vector<SegmentedKvCache> read_cache_snapshot(
    const std::string& path, SegmentedKvCache::Storage storage = SegmentedKvCache::Storage::F32,
    bool host_shadow = true) {
    reattn_snapshot* s = nullptr;
    gpu::check(reattn_snapshot_open(gpu::context(), path.c_str(), &s));
    std::unique_ptr<reattn_snapshot, void (*)(reattn_snapshot*)> guard(s, reattn_snapshot_close);
    std::uint32_t n_layers = 0;
    reattn_snapshot_info(s, &n_layers, nullptr, nullptr);
    std::vector<SegmentedKvCache> layers;
    layers.reserve(n_layers);
    for (std::uint32_t l = 0; l < n_layers; ++l) {
        reattn_cache* c = nullptr;
        gpu::check(reattn_snapshot_load_layer(gpu::context(), s, l, static_cast<int>(storage), 0, &c));
        layers.push_back(SegmentedKvCache::adopt(c, host_shadow));
    }
    return layers;
}

}  // namespace reattn
