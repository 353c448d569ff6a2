// host_ref.h -- host-side fp64 transforms used by the export path.
//
// oscar_kv_export must return the residual window as the reference holds it:
// transformed K_u rows + norms (kv_cache.cpp:219-224).  The device keeps the
// raw bf16 rows (exact), so the export recomputes the deterministic fp64
// transform here with the reference's operation order.  This translation
// unit is compiled with -ffp-contract=off (no FMA), like the reference.
#pragma once
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>

namespace osk {
namespace host {

// hadamard.cpp:10-26
inline void fht(double *v, int64_t d) {
    for (int64_t half = 1; half < d; half <<= 1)
        for (int64_t base = 0; base < d; base += half << 1)
            for (int64_t i = base; i < base + half; ++i) {
                const double a = v[i], b = v[i + half];
                v[i] = a + b;
                v[i + half] = a - b;
            }
    const double scale = 1.0 / std::sqrt(static_cast<double>(d));
    for (int64_t i = 0; i < d; ++i) v[i] *= scale;
}

// pipeline.cpp:80-88
inline double fast_rsqrt(double x) {
    const float xf = static_cast<float>(x);
    if (xf <= 0.0f || !std::isfinite(xf)) return 1.0 / std::sqrt(x);
    double y = static_cast<double>(1.0f / std::sqrt(xf));
    y = y * (1.5 - 0.5 * x * y * y);
    return y;
}

// pipeline.cpp:90-148 on one (token, head) row, in place; returns the norm
inline double token_scale(double *x, int64_t d, int strategy) {
    bool zero = true;
    for (int64_t c = 0; c < d; ++c)
        if (x[c] != 0.0) zero = false;
    double s, inv;
    if (zero) {
        s = 1e-12;
        inv = 1.0 / 1e-12;
    } else if (strategy == 0 || strategy == 1) {
        double ss = 0.0;
        for (int64_t c = 0; c < d; ++c) ss += x[c] * x[c];
        if (strategy == 0) {
            s = std::sqrt(ss);
            inv = 1.0 / s;
        } else {
            inv = fast_rsqrt(ss);
            s = 1.0 / inv;
        }
    } else if (strategy == 2) {
        double m = 0.0;
        for (int64_t c = 0; c < d; ++c) m = std::max(m, std::fabs(x[c]));
        s = m;
        inv = 1.0 / s;
    } else {
        double m = 0.0;
        for (int64_t c = 0; c < d; ++c) m += std::fabs(x[c]);
        s = m / static_cast<double>(d);
        inv = 1.0 / s;
    }
    for (int64_t c = 0; c < d; ++c) x[c] = x[c] * inv;
    return s;
}

inline double bf16_to_double(uint16_t b) {
    const uint32_t u = static_cast<uint32_t>(b) << 16;
    float f;
    std::memcpy(&f, &u, 4);
    return static_cast<double>(f);
}

// quant.cpp:21-47 from the kept (lo, hi): delta, zero point, constant
inline void params_from_lohi(double lo, double hi, int bits, double &delta, int64_t &zp, double &constant) {
    if (hi == lo) {
        delta = 0.0;
        zp = 0;
        constant = lo;
        return;
    }
    delta = (hi - lo) / static_cast<double>((int64_t{1} << bits) - 1);
    zp = std::llround(-lo / delta);
    constant = lo;
}

}  // namespace host
}  // namespace osk
