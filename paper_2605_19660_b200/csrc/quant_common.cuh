// quant_common.cuh -- the fp64 group quantiser shared by the raw-bf16 append
// path (quantize.cu) and the reference-form fp64 path (f64_path.cu).  Both
// translation units are compiled with -fmad=false and every arithmetic op is an
// explicit round-to-nearest intrinsic, so the operation order is the
// reference's.
#pragma once
#include <cuda_fp16.h>
#include <stdint.h>

#include "kernels.h"

namespace osk {

__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }

// quant.cpp:21-47 on 32 values in index order; returns delta, zp, lo, hi
struct GroupQ {
    double lo, hi, delta;
    long long zp;
};
// UNR: unroll factor of the element loops (32: register-array getters; a smaller one
// keeps the code of shared-memory getters compact)
template <int UNR = 32, typename Get>
__device__ __forceinline__ GroupQ group_params(Get get, int bits) {
    GroupQ p;
    double lo = get(0), hi = lo;
#pragma unroll(UNR)
    for (int i = 0; i < 32; ++i) {
        const double x = get(i);
        lo = (x < lo) ? x : lo;  // std::min(lo, x)
        hi = (hi < x) ? x : hi;  // std::max(hi, x)
    }
    p.lo = lo;
    p.hi = hi;
    if (hi == lo) {
        p.delta = 0.0;
        p.zp = 0;
    } else {
        p.delta = ddiv(dsub(hi, lo), (double)((1 << bits) - 1));
        p.zp = llround(ddiv(-lo, p.delta));
    }
    return p;
}

// quant.cpp:53-57 over one group: q = clamp(llround(x / delta) + zp, 0, 2^b-1).
// x / delta is taken as x * (1/delta) -- within 2 ulp of the IEEE quotient --
// and rounded branch-free; an element whose product lies within 1e-9 of a
// half-integer (where the two could round apart; 2 ulp < 1e-9 while
// |x/delta| < 2^20, checked once per group) is redone with the exact IEEE
// division afterwards.  The codes are bit-identical to the reference's.
template <int UNR = 32, typename Get, typename Put>
__device__ __forceinline__ void quantize_group(Get get, const GroupQ &p, int bits, Put put) {
    const int mx = (1 << bits) - 1;
    if (p.delta == 0.0) {
#pragma unroll
        for (int i = 0; i < 32; ++i) put(i, 0);
        return;
    }
    const double inv = ddiv(1.0, p.delta);
    const bool fast = dmul(fmax(fabs(p.lo), fabs(p.hi)), inv) < 1048576.0;
    // codes saturate, so a zero point beyond +-2^30 acts like +-2^30
    const int zp = p.zp > (1ll << 30) ? (1 << 30) : (p.zp < -(1ll << 30) ? -(1 << 30) : (int)p.zp);
    unsigned tie = 0;
#pragma unroll(UNR)
    for (int i = 0; i < 32; ++i) {
        const double y = dmul(get(i), inv);
        const double fl = floor(y);
        const double fr = dsub(y, fl);
        tie |= (fabs(dsub(fr, 0.5)) <= 1e-9 ? 1u : 0u) << i;
        const int q = (int)fl + (fr > 0.5 ? 1 : 0) + zp;
        put(i, q < 0 ? 0 : (q > mx ? mx : q));
    }
    if (!fast || tie) {  // rare: exact division for the flagged elements
        for (int i = 0; i < 32; ++i) {
            if (fast && !((tie >> i) & 1u)) continue;
            long long q = llround(ddiv(get(i), p.delta)) + p.zp;
            put(i, (int)(q < 0 ? 0 : (q > mx ? mx : q)));
        }
    }
}

// affine fp16 form used by the attention kernel: x = a*code + b
__device__ __forceinline__ void affine16(const GroupQ &p, __half &a, __half &b) {
    if (p.delta == 0.0) {
        a = __double2half(0.0);
        b = __double2half(p.lo);
    } else {
        a = __double2half(p.delta);
        b = __double2half(dmul(p.delta, -(double)p.zp));
    }
}

// device status (QuantizeArgs::status): record overflow / non-finite input
__device__ __forceinline__ void flag_status(int *status, const GroupQ &p, __half ha, __half hb) {
    if (!status) return;
    // (non-finite inputs are flagged where they are loaded)
    if (isfinite(p.lo) && isfinite(p.hi) && (__hisinf(ha) || __hisinf(hb))) atomicOr(status, STATUS_FP16_OVERFLOW);
}

__device__ __forceinline__ void flag_nonfinite(int *status) {
    if (status) atomicOr(status, STATUS_NONFINITE_INPUT);
}

}  // namespace osk
