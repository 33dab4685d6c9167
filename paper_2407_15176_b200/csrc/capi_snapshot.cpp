// RKVC cache snapshots (reference kv_cache.hpp:120-209, write_cache_snapshot /
// read_cache_snapshot) straight to and from device caches.
//
// Format: magic "RKVC", u32 version (1), u32 n_layers, n_kv_heads, d_head; per layer u64
// {total, l_global, l_local_max} then the keys and the values as raw little-endian f32,
// head-major ([head][entry][d]).  The head-major payload is the device cache's own layout,
// so a layer loads as one streamed copy per head (chunked through pinned memory, converted
// to the cache dtype on the device); bf16 caches are written back as f32 (exact).
//
// Validation follows the reference's read order and messages: bad magic / version, per
// layer the three u64 fields ("cache snapshot truncated at <field>"), the SegmentedKvCache
// constructor checks (kv_cache.hpp:40-51), then the key and value payloads.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "capi_internal.h"

using namespace reattn_impl;
using namespace reattn_capi;

struct reattn_snapshot {
    std::string path;
    FILE* f = nullptr;
    uint32_t n_layers = 0, n_kv = 0, d = 0;
    struct Layer {
        uint64_t total, l_global, l_local_max, offset;  // offset: first key byte
    };
    std::vector<Layer> layers;
    ~reattn_snapshot() {
        if (f) std::fclose(f);
    }
};

namespace {

constexpr char kMagic[4] = {'R', 'K', 'V', 'C'};
constexpr uint32_t kVersion = 1;
constexpr size_t kChunkBytes = 32u << 20;  // pinned staging per direction

template <typename T>
bool read_pod(FILE* f, T* v) {
    return std::fread(v, sizeof(T), 1, f) == 1;
}

bool mul_ok(uint64_t a, uint64_t b, uint64_t* out) { return !__builtin_mul_overflow(a, b, out); }

struct Pinned {
    void* p = nullptr;
    ~Pinned() {
        if (p) cudaFreeHost(p);
    }
};

}  // namespace

extern "C" {

int reattn_snapshot_open(reattn_ctx* ctx, const char* path, reattn_snapshot** out) {
    *out = nullptr;
    auto s = std::make_unique<reattn_snapshot>();
    s->path = path ? path : "";
    s->f = std::fopen(s->path.c_str(), "rb");
    if (!s->f) return set_err(ctx, REATTN_ERUNTIME, "cannot open " + s->path);
    char magic[4];
    if (std::fread(magic, 1, 4, s->f) != 4 || std::memcmp(magic, kMagic, 4) != 0)
        return set_err(ctx, REATTN_ERUNTIME, "not a cache snapshot (bad magic): " + s->path);
    uint32_t version = 0;
    if (!read_pod(s->f, &version))
        return set_err(ctx, REATTN_ERUNTIME, "cache snapshot truncated at version");
    if (version != kVersion)
        return set_err(ctx, REATTN_ERUNTIME,
                       "unsupported cache snapshot version " + std::to_string(version));
    if (!read_pod(s->f, &s->n_layers))
        return set_err(ctx, REATTN_ERUNTIME, "cache snapshot truncated at n_layers");
    if (!read_pod(s->f, &s->n_kv))
        return set_err(ctx, REATTN_ERUNTIME, "cache snapshot truncated at n_kv_heads");
    if (!read_pod(s->f, &s->d))
        return set_err(ctx, REATTN_ERUNTIME, "cache snapshot truncated at d_head");
    if (fseeko(s->f, 0, SEEK_END) != 0) return set_err(ctx, REATTN_ERUNTIME, "cannot open " + s->path);
    const uint64_t fsize = (uint64_t)ftello(s->f);
    uint64_t pos = 4 + 4 * sizeof(uint32_t);
    for (uint32_t l = 0; l < s->n_layers; ++l) {
        reattn_snapshot::Layer L{};
        uint64_t* fields[3] = {&L.total, &L.l_global, &L.l_local_max};
        const char* names[3] = {"layer entry count", "l_global", "l_local_max"};
        for (int i = 0; i < 3; ++i) {
            if (pos + 8 > fsize)
                return set_err(ctx, REATTN_ERUNTIME,
                               std::string("cache snapshot truncated at ") + names[i]);
            fseeko(s->f, (off_t)pos, SEEK_SET);
            if (!read_pod(s->f, fields[i]))
                return set_err(ctx, REATTN_ERUNTIME,
                               std::string("cache snapshot truncated at ") + names[i]);
            pos += 8;
        }
        // SegmentedKvCache(n_kv, d, l_global, l_local_max) (kv_cache.hpp:40-51)
        if (s->n_kv == 0 || s->d == 0)
            return set_err(ctx, REATTN_EINVAL, "cache needs at least one head and a positive head dim");
        if (L.l_local_max == 0) return set_err(ctx, REATTN_EINVAL, "l_local_max must be positive");
        uint64_t per = 0, payload = 0;
        const bool ok = mul_ok(L.total, (uint64_t)s->d * 4, &per) && mul_ok(per, s->n_kv, &payload);
        L.offset = pos;
        if (!ok || pos + payload > fsize)
            return set_err(ctx, REATTN_ERUNTIME, "cache snapshot truncated at layer keys");
        pos += payload;
        if (pos + payload > fsize)
            return set_err(ctx, REATTN_ERUNTIME, "cache snapshot truncated at layer values");
        pos += payload;
        s->layers.push_back(L);
    }
    *out = s.release();
    return REATTN_OK;
}

int reattn_snapshot_info(const reattn_snapshot* s, uint32_t* n_layers, uint32_t* n_kv,
                         uint32_t* d_head) {
    if (!s) return REATTN_EINVAL;
    if (n_layers) *n_layers = s->n_layers;
    if (n_kv) *n_kv = s->n_kv;
    if (d_head) *d_head = s->d;
    return REATTN_OK;
}

int reattn_snapshot_layer_info(const reattn_snapshot* s, uint32_t layer, uint64_t* total,
                               uint64_t* l_global, uint64_t* l_local_max) {
    if (!s || layer >= s->n_layers) return REATTN_ERANGE;
    const auto& L = s->layers[layer];
    if (total) *total = L.total;
    if (l_global) *l_global = L.l_global;
    if (l_local_max) *l_local_max = L.l_local_max;
    return REATTN_OK;
}

int reattn_snapshot_load_layer(reattn_ctx* ctx, reattn_snapshot* s, uint32_t layer, int dtype,
                               uint64_t capacity, reattn_cache** out) {
    *out = nullptr;
    if (!s || layer >= s->n_layers) return set_err(ctx, REATTN_ERANGE, "snapshot layer out of range");
    const auto& L = s->layers[layer];
    reattn_cache* c = nullptr;
    int rc = reattn_cache_create(ctx, s->n_kv, s->d, L.l_global, L.l_local_max,
                                 std::max<uint64_t>(std::max<uint64_t>(capacity, L.total), 1), dtype, &c);
    if (rc) return rc;
    std::unique_ptr<reattn_cache, void (*)(reattn_cache*)> guard(c, reattn_cache_destroy);
    if (L.total) {
        Pinned host;
        CU(ctx, cudaMallocHost(&host.p, kChunkBytes));
        rc = ensure_arena(ctx, kChunkBytes + 256);
        if (rc) return rc;
        float* dev = (float*)ctx->arena;
        const uint64_t row_bytes = (uint64_t)s->d * 4;
        const uint64_t rows_per_chunk = std::max<uint64_t>(1, kChunkBytes / row_bytes);
        const uint64_t esz = dtype == REATTN_BF16 ? 2 : 4;
        fseeko(s->f, (off_t)L.offset, SEEK_SET);
        for (int kvpart = 0; kvpart < 2; ++kvpart) {
            uint8_t* base = (uint8_t*)(kvpart ? c->values : c->keys);
            for (uint32_t h = 0; h < s->n_kv; ++h) {
                void* head = base + (uint64_t)h * c->capacity * s->d * esz;
                for (uint64_t r0 = 0; r0 < L.total; r0 += rows_per_chunk) {
                    const uint64_t n = std::min(rows_per_chunk, L.total - r0);
                    if (std::fread(host.p, row_bytes, n, s->f) != n)
                        return set_err(ctx, REATTN_ERUNTIME,
                                       kvpart ? "cache snapshot truncated at layer values"
                                              : "cache snapshot truncated at layer keys");
                    CU(ctx, cudaMemcpyAsync(dev, host.p, n * row_bytes, cudaMemcpyHostToDevice,
                                            ctx->stream));
                    // one head's rows [r0, r0+n): the append kernel with n_kv = 1
                    CU(ctx, launch_cache_append(dev, head, dtype, n, 1, s->d, c->capacity, r0,
                                                ctx->stream));
                    CU(ctx, cudaStreamSynchronize(ctx->stream));  // staging reuse
                }
            }
        }
        c->total = L.total;
        int rc = cache_sync_total(ctx, c, ctx->stream);
        if (rc) return rc;
    }
    *out = guard.release();
    return REATTN_OK;
}

void reattn_snapshot_close(reattn_snapshot* s) { delete s; }

int reattn_snapshot_write(reattn_ctx* ctx, const char* path, const reattn_cache* const* layers,
                          uint32_t n_layers) {
    const std::string p = path ? path : "";
    if (n_layers == 0 || !layers) return set_err(ctx, REATTN_EINVAL, "cache snapshot: no layers");
    CU(ctx, cudaStreamSynchronize(ctx->stream));  // rows appended on the context stream
    FILE* f = std::fopen(p.c_str(), "wb");
    if (!f) return set_err(ctx, REATTN_ERUNTIME, "cannot open " + p + " for writing");
    std::unique_ptr<FILE, int (*)(FILE*)> fg(f, std::fclose);
    bool good = std::fwrite(kMagic, 1, 4, f) == 4;
    const uint32_t hdr[4] = {kVersion, n_layers, (uint32_t)layers[0]->n_kv, (uint32_t)layers[0]->d};
    good = good && std::fwrite(hdr, sizeof(hdr), 1, f) == 1;
    Pinned host;
    CU(ctx, cudaMallocHost(&host.p, 2 * kChunkBytes));
    float* out = (float*)host.p;
    uint16_t* raw = (uint16_t*)((uint8_t*)host.p + kChunkBytes);
    for (uint32_t l = 0; l < n_layers && good; ++l) {
        const reattn_cache* c = layers[l];
        const uint64_t lh[3] = {c->total, c->l_global, c->l_local_max};
        good = std::fwrite(lh, sizeof(lh), 1, f) == 1;
        if (!c->total) continue;
        const uint64_t esz = c->dtype == REATTN_BF16 ? 2 : 4;
        const uint64_t rows_per_chunk = std::max<uint64_t>(1, kChunkBytes / (c->d * 4));
        for (int kvpart = 0; kvpart < 2 && good; ++kvpart) {
            const uint8_t* base = (const uint8_t*)(kvpart ? c->values : c->keys);
            for (uint64_t h = 0; h < c->n_kv && good; ++h) {
                const uint8_t* head = base + h * c->capacity * c->d * esz;
                for (uint64_t r0 = 0; r0 < c->total && good; r0 += rows_per_chunk) {
                    const uint64_t n = std::min(rows_per_chunk, c->total - r0);
                    const uint64_t elems = n * c->d;
                    if (esz == 4) {
                        CU(ctx, cudaMemcpy(out, head + r0 * c->d * 4, elems * 4, cudaMemcpyDeviceToHost));
                    } else {
                        CU(ctx, cudaMemcpy(raw, head + r0 * c->d * 2, elems * 2, cudaMemcpyDeviceToHost));
                        for (uint64_t e = 0; e < elems; ++e) {  // bf16 -> f32 is exact
                            const uint32_t w = (uint32_t)raw[e] << 16;
                            std::memcpy(&out[e], &w, 4);
                        }
                    }
                    good = std::fwrite(out, 4, elems, f) == elems;
                }
            }
        }
    }
    if (!good || std::fflush(f) != 0) return set_err(ctx, REATTN_ERUNTIME, "write failed: " + p);
    return REATTN_OK;
}

}  // extern "C"
