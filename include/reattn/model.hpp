// Drop-in for reattn/model.hpp (reference model.hpp:19-341): the decoder's configuration and
// host-side weights, with the reference's names, defaults and error messages.  The weight
// stream of init_random (mt19937_64 Box-Muller, model.hpp:90-152) and the RATW file format
// (model.hpp:204-339) are produced by the library (reattn_weights_*), so the C-ABI and this
// header share one implementation; the host ModelWeights is a copy of the device tensors.
#pragma once

#include <cstdint>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "reattn/dense_matrix.hpp"
#include "reattn/runtime.hpp"

namespace reattn {

enum class AttentionMode : std::uint32_t { Full = 0, Window = 1, ReAttention = 2 };

inline const char* mode_name(AttentionMode m) {
    switch (m) {
        case AttentionMode::Full: return "full";
        case AttentionMode::Window: return "window";
        case AttentionMode::ReAttention: return "reattention";
    }
    throw std::invalid_argument("unknown attention mode");
}

inline AttentionMode parse_mode(const std::string& s) {
    if (s == "full") return AttentionMode::Full;
    if (s == "window") return AttentionMode::Window;
    if (s == "reattention") return AttentionMode::ReAttention;
    throw std::invalid_argument("unknown attention mode: " + s);
}

// model.hpp:39-61 (toy defaults)
struct ModelConfig {
    std::size_t n_layer = 2;
    std::size_t n_head = 4;
    std::size_t n_kv_head = 2;
    std::size_t d_model = 128;
    std::size_t d_head = 32;
    std::size_t d_ff = 512;
    std::size_t vocab_size = 512;
    std::size_t pretrain_window = 4096;
    double rope_base = 10000.0;
    AttentionMode attention_mode = AttentionMode::ReAttention;

    reattn_model_config to_c() const {
        reattn_model_config c{};
        c.n_layer = n_layer;
        c.n_head = n_head;
        c.n_kv_head = n_kv_head;
        c.d_model = d_model;
        c.d_head = d_head;
        c.d_ff = d_ff;
        c.vocab_size = vocab_size;
        c.pretrain_window = pretrain_window;
        c.rope_base = rope_base;
        c.attention_mode = static_cast<int32_t>(attention_mode);
        return c;
    }
    static ModelConfig from_c(const reattn_model_config& c) {
        ModelConfig m;
        m.n_layer = c.n_layer;
        m.n_head = c.n_head;
        m.n_kv_head = c.n_kv_head;
        m.d_model = c.d_model;
        m.d_head = c.d_head;
        m.d_ff = c.d_ff;
        m.vocab_size = c.vocab_size;
        m.pretrain_window = c.pretrain_window;
        m.rope_base = c.rope_base;
        m.attention_mode = static_cast<AttentionMode>(c.attention_mode);
        return m;
    }
    void validate() const {
        const reattn_model_config c = to_c();
        gpu::check(reattn_model_config_validate(gpu::context(), &c));
    }
};

// model.hpp:66-84: projections input-major (d_in x d_out)
struct LayerWeights {
    DenseMatrix wq, wk, wv, wo, w_gate, w_up, w_down;
    std::vector<float> norm_attn, norm_ffn;
};

struct ModelWeights {
    ModelConfig config;
    DenseMatrix embedding;
    std::vector<LayerWeights> layers;
    std::vector<float> norm_final;
    DenseMatrix lm_head;
};

namespace detail {

// Owning handle of device weights (reattn_weights).
class DeviceWeights {
public:
    explicit DeviceWeights(reattn_weights* w) : w_(w) {}
    DeviceWeights(const DeviceWeights&) = delete;
    DeviceWeights& operator=(const DeviceWeights&) = delete;
    ~DeviceWeights() {
        if (w_) reattn_weights_destroy(w_);
    }
    reattn_weights* get() const { return w_; }

    // device -> host ModelWeights
    ModelWeights to_host() const {
        reattn_model_config c{};
        gpu::check(reattn_weights_config(w_, &c));
        ModelWeights m;
        m.config = ModelConfig::from_c(c);
        m.embedding = matrix(REATTN_W_EMBEDDING, 0);
        m.layers.resize(c.n_layer);
        for (std::size_t l = 0; l < c.n_layer; ++l) {
            LayerWeights& L = m.layers[l];
            L.wq = matrix(REATTN_W_WQ, l);
            L.wk = matrix(REATTN_W_WK, l);
            L.wv = matrix(REATTN_W_WV, l);
            L.wo = matrix(REATTN_W_WO, l);
            L.w_gate = matrix(REATTN_W_GATE, l);
            L.w_up = matrix(REATTN_W_UP, l);
            L.w_down = matrix(REATTN_W_DOWN, l);
            L.norm_attn = matrix(REATTN_W_NORM_ATTN, l).values;
            L.norm_ffn = matrix(REATTN_W_NORM_FFN, l).values;
        }
        m.norm_final = matrix(REATTN_W_NORM_FINAL, 0).values;
        m.lm_head = matrix(REATTN_W_LM_HEAD, 0);
        return m;
    }

    // host ModelWeights -> new device weights
    static reattn_weights* from_host(const ModelWeights& m) {
        const reattn_model_config c = m.config.to_c();
        reattn_weights* w = nullptr;
        gpu::check(reattn_weights_create(gpu::context(), &c, &w));
        DeviceWeights guard(w);
        auto up = [&](int kind, std::size_t layer, const std::vector<float>& v) {
            gpu::check(reattn_weights_upload(gpu::context(), w, kind, layer, v.data(), v.size()));
        };
        up(REATTN_W_EMBEDDING, 0, m.embedding.values);
        if (m.layers.size() != m.config.n_layer)
            throw std::invalid_argument("model weights: layer count != config.n_layer");
        for (std::size_t l = 0; l < m.layers.size(); ++l) {
            const LayerWeights& L = m.layers[l];
            up(REATTN_W_WQ, l, L.wq.values);
            up(REATTN_W_WK, l, L.wk.values);
            up(REATTN_W_WV, l, L.wv.values);
            up(REATTN_W_WO, l, L.wo.values);
            up(REATTN_W_GATE, l, L.w_gate.values);
            up(REATTN_W_UP, l, L.w_up.values);
            up(REATTN_W_DOWN, l, L.w_down.values);
            up(REATTN_W_NORM_ATTN, l, L.norm_attn);
            up(REATTN_W_NORM_FFN, l, L.norm_ffn);
        }
        up(REATTN_W_NORM_FINAL, 0, m.norm_final);
        up(REATTN_W_LM_HEAD, 0, m.lm_head.values);
        guard.w_ = nullptr;
        return w;
    }

private:
    DenseMatrix matrix(int kind, std::size_t layer) const {
        std::uint64_t r = 0, c = 0;
        gpu::check(reattn_weights_shape(w_, kind, &r, &c));
        DenseMatrix m(r, c);
        gpu::check(reattn_weights_download(gpu::context(), w_, kind, layer, m.values.data(),
                                           m.values.size()));
        return m;
    }
    reattn_weights* w_;
};

}  // namespace detail

// init_random (model.hpp:120-152): the same pinned Gaussian stream, std 0.02, unit norms
inline ModelWeights init_random(const ModelConfig& cfg, std::uint64_t seed) {
    const reattn_model_config c = cfg.to_c();
    reattn_weights* w = nullptr;
    gpu::check(reattn_weights_init_random(gpu::context(), &c, seed, &w));
    ModelWeights m = detail::DeviceWeights(w).to_host();
    m.config = cfg;
    return m;
}

// save_weights / load_weights (model.hpp:259-339): the RATW format, same messages
inline void save_weights(const ModelWeights& w, const std::string& path) {
    detail::DeviceWeights d(detail::DeviceWeights::from_host(w));
    gpu::check(reattn_weights_save(gpu::context(), d.get(), path.c_str()));
}

inline ModelWeights load_weights(const std::string& path) {
    reattn_weights* w = nullptr;
    gpu::check(reattn_weights_load(gpu::context(), path.c_str(), &w));
    return detail::DeviceWeights(w).to_host();
}

// rmsnorm (model.hpp:155-167): the mean square in f64, then two fp32 multiplies per element
inline DenseMatrix rmsnorm(const DenseMatrix& x, std::span<const float> weight) {
    if (x.cols != weight.size()) throw std::invalid_argument("rmsnorm: weight width mismatch");
    DenseMatrix out(x.rows, x.cols);
    if (out.values.empty()) return out;
    gpu::DeviceBuffer<float> dx, dw, dout(out.values.size());
    dx.upload(x.values.data(), x.values.size());
    dw.upload(weight.data(), weight.size());
    gpu::check(reattn_rmsnorm(gpu::context(), dx.get(), x.rows, x.cols, dw.get(), dout.get()));
    out.values = dout.to_vector(out.values.size());
    return out;
}

// feed_forward (model.hpp:169-178): (silu(x Wg) * (x Wu)) Wd with the reference's k-ordered
// matmul and fp32 activation
inline DenseMatrix feed_forward(const DenseMatrix& x, const LayerWeights& layer) {
    DenseMatrix gate = matmul(x, layer.w_gate);
    const DenseMatrix up = matmul(x, layer.w_up);
    if (!gate.values.empty()) {
        gpu::DeviceBuffer<float> dg, du;
        dg.upload(gate.values.data(), gate.values.size());
        du.upload(up.values.data(), up.values.size());
        gpu::check(reattn_silu_mul(gpu::context(), dg.get(), du.get(), gate.values.size()));
        gate.values = dg.to_vector(gate.values.size());
    }
    return matmul(gate, layer.w_down);
}

// embed (model.hpp:181-190)
inline DenseMatrix embed(std::span<const std::uint32_t> tokens, const ModelWeights& w) {
    DenseMatrix out(tokens.size(), w.config.d_model);
    for (std::size_t i = 0; i < tokens.size(); ++i) {
        if (tokens[i] >= w.config.vocab_size) throw std::out_of_range("token id outside vocabulary");
        const float* src = w.embedding.row(tokens[i]);
        std::copy(src, src + w.config.d_model, out.row(i));
    }
    return out;
}

// argmax_token (model.hpp:193-199): greedy pick, ties to the lowest token id
inline std::uint32_t argmax_token(std::span<const float> logits) {
    if (logits.empty()) throw std::invalid_argument("empty logits");
    std::size_t best = 0;
    for (std::size_t i = 1; i < logits.size(); ++i)
        if (logits[i] > logits[best]) best = i;
    return std::uint32_t(best);
}

}  // namespace reattn
