// oscar_kv.hpp -- header-only C++ host wrapper over the C-ABI (oscar_kv.h)
// that re-exposes the reference's class and method names
// (/root/reference/proj/include/oscar/kv_cache.hpp:61-123) and its exception
// types (std::invalid_argument / std::logic_error / std::runtime_error), so
// reference call sites change only their include and constructor arguments.
// See INTEGRATION.md.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "oscar_kv.h"

namespace oscar_b200 {

// status -> the reference's exception types (kv_cache.cpp:51-67, 225-227, 471)
inline void check(int rc) {
    if (rc == 0) return;
    const std::string msg = oscar_last_error();
    if (rc == 1) throw std::invalid_argument(msg);
    if (rc == 2) throw std::logic_error(msg);
    throw std::runtime_error(msg);
}

enum class Method : int32_t { Fp = OSCAR_FP, Kivi = OSCAR_KIVI, RotateOnly = OSCAR_ROTATE_ONLY,
                              ScaleOnly = OSCAR_SCALE_ONLY, Oscar = OSCAR_OSCAR };
enum class Scaling : int32_t { L2 = OSCAR_L2, Rsqrt = OSCAR_RSQRT, Max = OSCAR_MAX, MeanAbs = OSCAR_MEAN_ABS };

// PipelineConfig (kv_cache.hpp:19-32) with the same defaults, plus rotate_v.
struct PipelineConfig {
    Method method = Method::Oscar;
    int bits = 2;
    int64_t group_size = 32;
    int64_t residual_len = 128;
    Scaling scaling = Scaling::L2;
    int64_t head_dim = 128;
    int64_t heads = 1;
    bool rotate_v = false;

    oscar_kv_config c() const {
        oscar_kv_config x{};
        x.method = static_cast<int32_t>(method);
        x.bits = bits;
        x.group_size = group_size;
        x.residual_len = residual_len;
        x.scaling = static_cast<int32_t>(scaling);
        x.rotate_v = rotate_v ? 1 : 0;
        x.head_dim = head_dim;
        x.heads = heads;
        return x;
    }
    void validate() const {  // PipelineConfig::validate (kv_cache.cpp:51-67)
        const oscar_kv_config x = c();
        check(oscar_kv_config_validate(&x));
    }
};

// Tensor3 (tensor.hpp:11-33): dense [token][head][channel] fp64, channel fastest.
struct Tensor3 {
    int64_t tokens = 0, heads = 0, channels = 0;
    std::vector<double> data;
    Tensor3() = default;
    Tensor3(int64_t s, int64_t h, int64_t c) : tokens(s), heads(h), channels(c), data((size_t)(s * h * c), 0.0) {}
    Tensor3(int64_t s, int64_t h, int64_t c, std::vector<double> v) : tokens(s), heads(h), channels(c), data(std::move(v)) {
        if ((int64_t)data.size() != s * h * c) throw std::invalid_argument("Tensor3: data size does not match shape");
    }
    double &at(int64_t t, int64_t h, int64_t c) { return data[(size_t)((t * heads + h) * channels + c)]; }
    double at(int64_t t, int64_t h, int64_t c) const { return data[(size_t)((t * heads + h) * channels + c)]; }
    double *row(int64_t t, int64_t h) { return data.data() + (t * heads + h) * channels; }
    const double *row(int64_t t, int64_t h) const { return data.data() + (t * heads + h) * channels; }
};

// Device KvCache for `batch` sequences x cfg.heads KV heads.  Single writer
// (kv_cache.hpp:58-60); every call enqueues on `stream` (a cudaStream_t).
class KvCache {
public:
    KvCache(const PipelineConfig &cfg, int64_t batch, int64_t q_heads, int64_t max_tokens, int device = 0,
            bool keep_exact = true)
        : cfg_(cfg), batch_(batch) {
        const oscar_kv_config x = cfg.c();
        check(oscar_kv_create(&x, batch, q_heads, max_tokens, device, keep_exact ? 1 : 0, &h_));
    }
    KvCache(const KvCache &) = delete;
    KvCache &operator=(const KvCache &) = delete;
    KvCache(KvCache &&o) noexcept : cfg_(o.cfg_), batch_(o.batch_), h_(std::exchange(o.h_, nullptr)) {}
    ~KvCache() {
        if (h_) oscar_kv_destroy(h_);
    }

    // buffer_quant_k + buffer_quant_v (kv_cache.cpp:194-292) on RAW bf16 keys
    // [batch, n, heads, d]: the key transform of apply_method runs on device.
    void buffer_quant(const void *k, const void *v, int64_t n_tokens, void *stream = nullptr) {
        check(oscar_kv_append(h_, k, v, n_tokens, stream));
    }
    // The reference's own call shapes (kv_cache.hpp:80-84) for a one-sequence cache,
    // host fp64 rows: buffer_quant_k(K_u, norms) -- keys ALREADY transformed by
    // apply_method -- and buffer_quant_v(v).  Bit-exact vs the reference; one input
    // form per cache (these or buffer_quant above).
    void buffer_quant_k(const Tensor3 &new_k, const std::vector<double> &norms, void *stream = nullptr) {
        one_sequence("buffer_quant_k");
        if (new_k.tokens > 0 && (new_k.heads != cfg_.heads || new_k.channels != cfg_.head_dim))
            throw std::invalid_argument("buffer_quant_k: tensor shape does not match config");
        if ((int64_t)norms.size() != new_k.tokens * new_k.heads)
            throw std::invalid_argument("buffer_quant_k: one norm per (token, head) required");
        check(oscar_kv_append_k(h_, new_k.data.data(), norms.data(), new_k.tokens, stream));
    }
    void buffer_quant_v(const Tensor3 &new_v, void *stream = nullptr) {
        one_sequence("buffer_quant_v");
        if (new_v.tokens > 0 && (new_v.heads != cfg_.heads || new_v.channels != cfg_.head_dim))
            throw std::invalid_argument("buffer_quant_v: tensor shape does not match config");
        check(oscar_kv_append_v(h_, new_v.data.data(), new_v.tokens, stream));
    }
    // batched device-pointer forms: k_t fp64 [batch, n, heads, d], norms [batch, n, heads]
    void buffer_quant_k(const double *k_t, const double *norms, int64_t n_tokens, void *stream = nullptr) {
        check(oscar_kv_append_k(h_, k_t, norms, n_tokens, stream));
    }
    void buffer_quant_v(const double *v, int64_t n_tokens, void *stream = nullptr) {
        check(oscar_kv_append_v(h_, v, n_tokens, stream));
    }
    // decode_step with the current token in that form (device pointers)
    void decode_step_f64(const void *q, const double *k_t, const double *norms, const double *v, float *out,
                         float *lse = nullptr, void *stream = nullptr) {
        check(oscar_kv_decode_step_f64(h_, q, k_t, norms, v, out, lse, stream));
    }

    // decode_step body (pipeline.cpp:292-323) without the projections.
    void decode_step(const void *q, const void *k, const void *v, float *out, float *lse = nullptr,
                     void *stream = nullptr) {
        check(oscar_kv_decode_step(h_, q, k, v, out, lse, stream));
    }
    void attend(const void *q, float *out, float *lse, void *stream = nullptr) {
        check(oscar_kv_attend(h_, q, out, lse, stream));
    }

    int64_t packed_tokens() const { return stats().packed; }
    int64_t residual_tokens() const { return stats().residual; }
    int64_t total_tokens() const {
        const Stats s = stats();
        return s.packed + s.residual;
    }
    int64_t flush_count() const { return stats().flushes; }
    // device-side flags since the last clear (OSCAR_STATUS_*; synchronises)
    int32_t status(bool clear = false) {
        int32_t f = 0;
        check(oscar_kv_status(h_, &f, clear ? 1 : 0));
        return f;
    }

    oscar_kv_memory_report_t memory_report() const {
        oscar_kv_memory_report_t r{};
        check(oscar_kv_memory_report(h_, &r));
        return r;
    }
    // KvCache::dump (kv_cache.cpp:469-507) of sequence b
    void dump(int64_t b, const std::string &path) { check(oscar_kv_dump(h_, b, path.c_str())); }
    // KvCache::load (kv_cache.cpp:509-549) into sequence b
    void load(int64_t b, const std::string &path) { check(oscar_kv_load(h_, b, path.c_str())); }
    // static KvCache::load(path) (kv_cache.hpp:95): a one-sequence cache with the
    // file's config, holding its contents (q_heads: the GQA query heads to attend with)
    static KvCache load(const std::string &path, int64_t q_heads, int64_t max_tokens = 0, int device = 0) {
        oscar_kv_config c{};
        int64_t tokens = 0;
        check(oscar_kvc1_read_config(path.c_str(), &c, &tokens));
        PipelineConfig cfg;
        cfg.method = static_cast<Method>(c.method);
        cfg.bits = c.bits;
        cfg.group_size = c.group_size;
        cfg.residual_len = c.residual_len;
        cfg.scaling = static_cast<Scaling>(c.scaling);
        cfg.head_dim = c.head_dim;
        cfg.heads = c.heads;
        KvCache k(cfg, 1, q_heads, max_tokens > 0 ? max_tokens : tokens + c.residual_len, device);
        k.load(0, path);
        return k;
    }
    // materialize_k / materialize_v (kv_cache.cpp:327-381) of sequence b, fp64 [total, H, d]
    std::pair<std::vector<double>, std::vector<double>> materialize(int64_t b) {
        const size_t n = (size_t)(total_tokens() * cfg_.heads * cfg_.head_dim);
        std::vector<double> k(n), v(n);
        check(oscar_kv_materialize(h_, b, k.data(), v.data()));
        return {std::move(k), std::move(v)};
    }

    // materialize_k / materialize_v (kv_cache.cpp:327-381) of sequence b as Tensor3
    Tensor3 materialize_k(int64_t b = 0) { return materialized(b, true); }
    Tensor3 materialize_v(int64_t b = 0) { return materialized(b, false); }

    oscar_kv_handle *handle() const { return h_; }
    const PipelineConfig &config() const { return cfg_; }

private:
    void one_sequence(const char *what) const {
        if (batch_ != 1)
            throw std::invalid_argument(std::string(what) + ": the Tensor3 form is per sequence (batch 1 caches); "
                                                            "use the device-pointer form for batches");
    }
    Tensor3 materialized(int64_t b, bool keys) {
        auto kv = materialize(b);
        const int64_t n = total_tokens();
        return Tensor3(n, cfg_.heads, cfg_.head_dim, keys ? std::move(kv.first) : std::move(kv.second));
    }
    struct Stats {
        int64_t packed = 0, residual = 0, flushes = 0;
    };
    Stats stats() const {
        Stats s;
        check(oscar_kv_stats(h_, &s.packed, &s.residual, &s.flushes));
        return s;
    }
    PipelineConfig cfg_;
    int64_t batch_ = 1;
    oscar_kv_handle *h_ = nullptr;
};

}  // namespace oscar_b200
