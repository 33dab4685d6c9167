// Runtime glue of the drop-in C++ API: the process-wide device context, status -> exception
// translation (same exception types and messages as the reference) and RAII device
// buffers.  Everything that computes goes through include/reattn_cuda.h (sm_100a kernels);
// there is no CPU fallback.
#pragma once

#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "../reattn_cuda.h"

namespace reattn {
namespace gpu {

// The context used by every drop-in call (device 0 unless REATTN_DEVICE is set).
inline reattn_ctx* context() {
    static reattn_ctx* ctx = [] {
        int dev = 0;
        if (const char* e = std::getenv("REATTN_DEVICE")) dev = std::atoi(e);
        reattn_ctx* c = nullptr;
        if (reattn_ctx_create(dev, &c) != REATTN_OK || !c)
            throw std::runtime_error("reattn: no CUDA device available (B200 / sm_100a required)");
        return c;
    }();
    return ctx;
}

// Rethrow a C-ABI status as the reference's exception type with its message.
inline void check(int rc) {
    if (rc == REATTN_OK) return;
    const std::string msg = reattn_last_error(context());
    switch (rc) {
        case REATTN_EINVAL: throw std::invalid_argument(msg);
        case REATTN_ERANGE: throw std::out_of_range(msg);
        case REATTN_ELOGIC: throw std::logic_error(msg);
        default: throw std::runtime_error(msg);
    }
}

template <typename T>
class DeviceBuffer {
public:
    DeviceBuffer() = default;
    explicit DeviceBuffer(std::size_t n) { resize(n); }
    DeviceBuffer(const DeviceBuffer&) = delete;
    DeviceBuffer& operator=(const DeviceBuffer&) = delete;
    DeviceBuffer(DeviceBuffer&& o) noexcept : p_(o.p_), n_(o.n_) { o.p_ = nullptr, o.n_ = 0; }
    DeviceBuffer& operator=(DeviceBuffer&& o) noexcept {
        std::swap(p_, o.p_);
        std::swap(n_, o.n_);
        return *this;
    }
    ~DeviceBuffer() {
        if (p_) reattn_free(context(), p_);
    }
    void resize(std::size_t n) {
        if (n <= n_ && p_) return;
        if (p_) reattn_free(context(), p_);
        p_ = nullptr;
        void* p = nullptr;
        check(reattn_malloc(context(), std::max<std::size_t>(n, 1) * sizeof(T), &p));
        p_ = static_cast<T*>(p);
        n_ = n;
    }
    void upload(const T* src, std::size_t n) {
        resize(n);
        if (n) check(reattn_memcpy_h2d(context(), p_, src, n * sizeof(T)));
    }
    void download(T* dst, std::size_t n) const {
        if (n) check(reattn_memcpy_d2h(context(), dst, p_, n * sizeof(T)));
    }
    std::vector<T> to_vector(std::size_t n) const {
        std::vector<T> v(n);
        download(v.data(), n);
        return v;
    }
    T* get() const { return p_; }

private:
    T* p_ = nullptr;
    std::size_t n_ = 0;
};

}  // namespace gpu
}  // namespace reattn
