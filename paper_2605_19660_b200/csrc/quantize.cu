// quantize.cu -- the quantize/append kernel: Canalized Rotation + Omni-Token
// Scaling + KIVI-style group quantisation + bit packing, in fp64 with the
// reference's exact operation order (compiled with -fmad=false; every
// arithmetic op is an explicit IEEE round-to-nearest intrinsic on top).
//
// Reference semantics reproduced bit-for-bit:
//   fht_inplace        hadamard.cpp:10-26   butterfly stages half=1..64, then *1/sqrt(d)
//   omni_token_scale   pipeline.cpp:90-148  zero test, sequential FMA-free sum of squares
//   fast_rsqrt         pipeline.cpp:80-88
//   quant_params       quant.cpp:21-47      lo/hi in index order, delta, llround zp (unclamped)
//   quantize_one       quant.cpp:53-57
//   flush_k_block      kv_cache.cpp:101-129 per-channel groups of G tokens
//   flush_v_block      kv_cache.cpp:131-157 per-token groups of G channels
//
// One CTA = one R-block of one (sequence, head): 128 threads, processed one
// 32-token group at a time.  Thread (token tl, quarter q) owns 32 channels
// of one token; the Hadamard butterfly runs 5 stages in registers and the
// last 2 across the 4-lane quad with shuffles; the l2 sum of squares is a
// sequential chain handed across the quad so the addition order is the
// reference's c = 0..127.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "device_common.cuh"
#include "kernels.h"
#include "layout.h"
#include "quant_common.cuh"

namespace osk {

namespace {

constexpr int QT = 128;  // threads per CTA
constexpr int KU_ROW = 4 * 33;  // doubles per token row of the K_u tile (4 quarters of 32, padded to 33)
// shared code tiles hold one code per nibble (codes <= 15), two per byte, so that
// four prefill CTAs fit per SM (53.75 KB each, 16 warps: the kernel is latency-bound):
//   K: [token pair][channel] bytes, row stride KC_STRIDE (the low nibble is the even token)
//   V: [token][channel pair] bytes, row stride VC_STRIDE (the low nibble is the even channel),
//      16-byte chunks XOR-swizzled by (token >> 1) & 3 (vc_swz): the pack loop's gathers
//      (4 token pairs 128 B apart per warp) hit distinct banks
constexpr int KC_STRIDE = D + 4;
constexpr int VC_STRIDE = D / 2;
__device__ __forceinline__ int vc_swz(int t) { return ((t >> 1) & 3) << 4; }

// a thread's 32 codes of one group as nibbles of two 64-bit registers (any write order)
struct Nib32 {
    uint64_t lo = 0, hi = 0;
    __device__ __forceinline__ void put(int i, int code) {
        const int sh = 4 * (i & 15);
        const uint64_t m = ~(0xFull << sh), v = (uint64_t)(uint32_t)code << sh;
        if (i < 16) lo = (lo & m) | v;
        else hi = (hi & m) | v;
    }
    __device__ __forceinline__ uint32_t byte(int k) const {  // nibbles 2k, 2k+1
        return (uint32_t)((k < 8 ? lo >> (8 * k) : hi >> (8 * (k - 8))) & 0xFF);
    }
};

// 32 bf16 -> fp64 (exact); bit 15 / 31 of `bad` flags non-finite inputs
__device__ __forceinline__ void load32(const __nv_bfloat16 *p, double (&x)[32], uint32_t &bad) {
    const uint4 *p4 = reinterpret_cast<const uint4 *>(p);
#pragma unroll
    for (int v = 0; v < 4; ++v) {
        uint4 u = p4[v];
        uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            x[v * 8 + 2 * e] = (double)__uint_as_float(w[e] << 16);
            x[v * 8 + 2 * e + 1] = (double)__uint_as_float(w[e] & 0xffff0000u);
            // a half is non-finite iff its exponent is all ones: adding 0x0080 to the
            // masked exponent then carries into bit 15 (no carry across halves)
            bad |= (w[e] & 0x7F807F80u) + 0x00800080u;
        }
    }
}
__device__ __forceinline__ double bf16_bits_to_double(uint16_t u, uint32_t &bad) {
    bad |= ((uint32_t)u & 0x7F80u) + 0x0080u;  // bit 15 set iff non-finite
    return (double)__uint_as_float((uint32_t)u << 16);
}

// hadamard.cpp:10-26 on a 128-vector spread over a 4-lane quad (32 per lane)
__device__ __forceinline__ void fht128_quad(double (&x)[32], int q) {
#pragma unroll
    for (int half = 1; half < 32; half <<= 1) {
#pragma unroll
        for (int base = 0; base < 32; base += 2 * half) {
#pragma unroll
            for (int i = base; i < base + half; ++i) {
                const double a = x[i], b = x[i + half];
                x[i] = dadd(a, b);
                x[i + half] = dsub(a, b);
            }
        }
    }
    // half = 32: partner quarter q^1; half = 64: partner quarter q^2
#pragma unroll
    for (int xm = 1; xm <= 2; xm <<= 1) {
        // lower lane: a + b; upper lane: a - b with a = partner, b = own value:
        // fma(+-1, own, partner) rounds once, exactly like dadd / dsub
        const double sgn = (q & xm) ? -1.0 : 1.0;
#pragma unroll
        for (int i = 0; i < 32; ++i) {
            const double o = __shfl_xor_sync(0xffffffffu, x[i], xm);
            x[i] = __fma_rn(sgn, x[i], o);
        }
    }
    const double scale = ddiv(1.0, __dsqrt_rn(128.0));
#pragma unroll
    for (int i = 0; i < 32; ++i) x[i] = dmul(x[i], scale);
}

// pipeline.cpp:80-88
__device__ __forceinline__ double fast_rsqrt_ref(double x) {
    const float xf = __double2float_rn(x);
    if (xf <= 0.0f || !isfinite(xf)) return ddiv(1.0, __dsqrt_rn(x));
    double y = (double)__fdiv_rn(1.0f, __fsqrt_rn(xf));
    // y * (1.5 - 0.5 * x * y * y), left to right
    const double t = dmul(dmul(dmul(0.5, x), y), y);
    return dmul(y, dsub(1.5, t));
}

#ifndef OSK_QC_ROLL
#define OSK_QC_ROLL 1  // the quad chain's step loop rolled: smaller code, prefill -3 % (ab_quant_occupancy)
#endif
#ifndef OSK_KROLL
#define OSK_KROLL 32  // unroll factor of the K-side (shared-memory) group loops
#endif
// sequential chain over the quad: acc_{c+1} = acc_c (+) f(x_c), c = 0..127
template <typename F>
__device__ __forceinline__ double quad_chain(const double (&x)[32], int q, int lane, F f) {
    double acc = 0.0;
#if OSK_QC_ROLL
#pragma unroll 1
#else
#pragma unroll
#endif
    for (int step = 0; step < 4; ++step) {
        if (q == step) {
#pragma unroll
            for (int i = 0; i < 32; ++i) acc = dadd(acc, f(x[i]));
        }
        acc = __shfl_sync(0xffffffffu, acc, (lane & ~3) | step);
    }
    return acc;
}

// group_params for values that are exactly representable in fp32
__device__ __forceinline__ GroupQ group_params_f32(const double (&y)[32], int bits) {
    float lo = (float)y[0], hi = lo;
#pragma unroll
    for (int i = 1; i < 32; ++i) {
        lo = fminf(lo, (float)y[i]);
        hi = fmaxf(hi, (float)y[i]);
    }
    if (lo == 0.0f || hi == 0.0f) return group_params([&](int i) { return y[i]; }, bits);
    GroupQ p;
    p.lo = (double)lo;
    p.hi = (double)hi;
    if (p.hi == p.lo) {
        p.delta = 0.0;
        p.zp = 0;
    } else {
        p.delta = ddiv(dsub(p.hi, p.lo), (double)((1 << bits) - 1));
        p.zp = llround(ddiv(-p.lo, p.delta));
    }
    return p;
}

// GPAR 32-token groups of the block are processed concurrently by GPAR
// 128-thread quarters of the CTA (GPAR = 1: prefill, throughput; GPAR = 4:
// the single-block flush, latency).
template <int BITS, int GPAR>
__global__ void __launch_bounds__(QT * GPAR, GPAR == 1 ? 4 : 1) quantize_kernel(const QuantizeArgs a) {
    using Blk = Block<BITS>;
    extern __shared__ __align__(16) uint8_t smem[];
    double *ku = reinterpret_cast<double *>(smem) + (threadIdx.x / QT) * 32 * KU_ROW;  // [GPAR][32][4][33]
    uint8_t *ck = smem + GPAR * 32 * KU_ROW * 8;                  // [64][KC_STRIDE] K code nibbles
    uint8_t *cv = ck + (R / 2) * KC_STRIDE;                       // [128][64] V code nibbles
    // params + norms staged in record order: K tail [a][b][norms] (K_PART - KA_OFF
    // bytes), then V tail [a][b] (BYTES - VA_OFF bytes)
    uint8_t *prm = cv + R * VC_STRIDE;
    __half *ka = reinterpret_cast<__half *>(prm);
    __half *kb = ka + D * NGRP;
    float *nrm = reinterpret_cast<float *>(kb + D * NGRP);
    __half *va = reinterpret_cast<__half *>(nrm + R);
    __half *vb = va + R * NGC;

    const int tid = threadIdx.x % QT, lane = tid & 31, q = tid & 3, tl = tid >> 2;
    const int bh = blockIdx.y, b = bh / a.H, h = bh % a.H;
    const int64_t blk = blockIdx.x;
    const __nv_bfloat16 *kin = reinterpret_cast<const __nv_bfloat16 *>(a.k) + b * a.sb + h * a.sh;
    const __nv_bfloat16 *vin = reinterpret_cast<const __nv_bfloat16 *>(a.v) + b * a.sb + h * a.sh;
    // block 0 may start with a.rtok tokens of the open residual window (rings):
    // token t of block blk is ring row t if blk == 0 && t < rtok, else input token
    // tok0 + blk*R + t - rtok
    const int64_t tok_base = a.tok0 + blk * R - a.rtok;
    const uint16_t *rk = a.rk ? reinterpret_cast<const uint16_t *>(a.rk) + (int64_t)bh * R * D : nullptr;
    const uint16_t *rv = a.rv ? reinterpret_cast<const uint16_t *>(a.rv) + (int64_t)bh * R * D : nullptr;
    const int64_t out_blk = (int64_t)bh * a.max_blocks + a.blk0 + blk;
    double *shadow = a.shadow ? a.shadow + out_blk * SHADOW_DOUBLES : nullptr;
    const TransformCfg tc = a.tc;

    for (int gi = threadIdx.x / QT; gi < NGRP; gi += GPAR) {
        const int t = gi * G + tl;  // token within the block
        // ---------------- K: rotate, scale (apply_method) ----------------
        double x[32];
        uint32_t bad = 0;  // non-finite K or V inputs of this thread's row
        const bool from_ring = blk == 0 && t < a.rtok;
        load32(from_ring ? reinterpret_cast<const __nv_bfloat16 *>(rk) + (int64_t)t * D + q * 32
                         : kin + (tok_base + t) * a.st + q * 32,
               x, bad);
        if (tc.rotates) fht128_quad(x, q);
        double s = 1.0, inv = 1.0;
        if (tc.scales) {
            bool nz = false;
#pragma unroll
            for (int i = 0; i < 32; ++i) nz |= (x[i] != 0.0);
            // zero test over all 128 channels (pipeline.cpp:99-102; -0.0 counts as zero)
            const unsigned ballot = __ballot_sync(0xffffffffu, nz);
            const bool quad_zero = ((ballot >> (lane & ~3)) & 0xFu) == 0;
            if (quad_zero) {
                s = 1e-12;
                inv = ddiv(1.0, 1e-12);
            } else if (tc.scaling == 0 || tc.scaling == 1) {
                const double ss = quad_chain(x, q, lane, [](double v) { return dmul(v, v); });
                if (tc.scaling == 0) {
                    s = __dsqrt_rn(ss);
                    inv = ddiv(1.0, s);
                } else {
                    inv = fast_rsqrt_ref(ss);
                    s = ddiv(1.0, inv);
                }
            } else if (tc.scaling == 2) {
                double m = 0.0;
#pragma unroll
                for (int i = 0; i < 32; ++i) {
                    const double av = fabs(x[i]);
                    m = (m < av) ? av : m;
                }
                m = fmax(m, __shfl_xor_sync(0xffffffffu, m, 1));
                m = fmax(m, __shfl_xor_sync(0xffffffffu, m, 2));
                s = m;
                inv = ddiv(1.0, s);
            } else {
                const double sa = quad_chain(x, q, lane, [](double v) { return fabs(v); });
                s = ddiv(sa, 128.0);
                inv = ddiv(1.0, s);
            }
#pragma unroll
            for (int i = 0; i < 32; ++i) x[i] = dmul(x[i], inv);
        }
        if (q == 0) {
            // attention-facing copy pre-multiplied by log2(e)/sqrt(d) (logits in log2 units)
            nrm[norm_index(t)] = __double2float_rn(dmul(s, 0.12751743074202186));
            if (shadow) shadow[SHADOW_K_DOUBLES + SHADOW_V_DOUBLES + t] = s;
        }
#pragma unroll
        for (int i = 0; i < 32; ++i) ku[tl * KU_ROW + q * 33 + i] = x[i];

        // ---------------- V: optional rotation, per-token groups ----------------
        {
            double y[32];
            if (from_ring) {  // the residual V ring (tile-major)
#pragma unroll
                for (int i = 0; i < 32; ++i) y[i] = bf16_bits_to_double(rv[vring_index(q * 32 + i, t)], bad);
            } else if (a.vsc == 1) {
                load32(vin + (tok_base + t) * a.vst + q * 32, y, bad);
            } else {  // a residual V ring (tile-major, vring_index): the flush
                const uint16_t *vp = reinterpret_cast<const uint16_t *>(vin);
#pragma unroll
                for (int i = 0; i < 32; ++i) y[i] = bf16_bits_to_double(vp[vring_index(q * 32 + i, (int)(tok_base + t))], bad);
            }
            if ((bad & 0x80008000u) && a.status) atomicOr(a.status, STATUS_NONFINITE_INPUT);
            if (tc.rotate_v) fht128_quad(y, q);
            // raw (bf16-valued) V: the group range in fp32 is exact, one FMNMX per
            // element; a zero extreme re-runs the sequential std::min/max so the
            // sign of a zero constant matches quant.cpp:26-34
            const GroupQ p = tc.rotate_v ? group_params([&](int i) { return y[i]; }, BITS)
                                         : group_params_f32(y, BITS);
#pragma unroll
            Nib32 nv;
            quantize_group([&](int i) { return y[i]; }, p, BITS, [&](int i, int code) { nv.put(i, code); });
            // channels q*32 .. q*32+31 of token t: 16 contiguous bytes, one 128-bit store
            *reinterpret_cast<uint4 *>(cv + t * VC_STRIDE + ((q * 16) ^ vc_swz(t))) =
                make_uint4((uint32_t)nv.lo, (uint32_t)(nv.lo >> 32), (uint32_t)nv.hi, (uint32_t)(nv.hi >> 32));
            __half ha, hb;
            affine16(p, ha, hb);
            flag_status(a.status, p, ha, hb);
            va[va_index(t, q)] = ha;
            vb[vb_index(t, q)] = hb;
            if (shadow) {
                shadow[SHADOW_K_DOUBLES + (t * NGC + q) * 2] = p.lo;
                shadow[SHADOW_K_DOUBLES + (t * NGC + q) * 2 + 1] = p.hi;
            }
        }
        __syncthreads();
        // ---------------- K: per-channel group of G tokens ----------------
        {
            const int c = tid;  // channel
            const int cc = (c >> 5) * 33 + (c & 31);
            const GroupQ p = group_params<OSK_KROLL>([&](int i) { return ku[i * KU_ROW + cc]; }, BITS);
            Nib32 nk;
            quantize_group<OSK_KROLL>([&](int i) { return ku[i * KU_ROW + cc]; }, p, BITS,
                                      [&](int i, int code) { nk.put(i, code); });
#pragma unroll
            for (int k = 0; k < 16; ++k) ck[(gi * (G / 2) + k) * KC_STRIDE + c] = (uint8_t)nk.byte(k);
            // keys use the same affine form as values, x = a*code + b with
            // b = -delta*zp (a constant group is a = 0, b = lo: its codes are 0,
            // quant.cpp:37-42, 65-68); the attention kernel folds b into one
            // MMA per k-step against the rotated query
            __half ha, hb;
            affine16(p, ha, hb);
            flag_status(a.status, p, ha, hb);
            ka[ka_index(c, gi)] = ha;
            kb[kb_index(c, gi)] = hb;
            if (shadow) {
                shadow[(c * NGRP + gi) * 2] = p.lo;
                shadow[(c * NGRP + gi) * 2 + 1] = p.hi;
            }
        }
        __syncthreads();
    }

    // ---------------- assemble the permuted code words ----------------
    uint8_t *out = a.blocks + out_blk * (int64_t)Blk::BYTES;
    constexpr int NWORDS = R * D * BITS / 32;
    constexpr int TPW = 16 / BITS;
    // four consecutive code words per thread -> one 128-bit store each for K and V
    for (int w4 = threadIdx.x; w4 < NWORDS / 4; w4 += QT * GPAR) {
        uint32_t wk[4], wv[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const int w = 4 * w4 + e;
            wk[e] = wv[e] = 0;
#pragma unroll
            for (int hi = 0; hi < 2; ++hi) {
                // field f of a K word is token +16f of field 0, of a V word channel +16f
                int tk, ckn, tv, cvn;
                k_word_coords(BITS, w, 0, hi, tk, ckn);
                v_word_coords(BITS, w, 0, hi, tv, cvn);
                // field f: K token tk + 16f (same nibble parity), V channel cvn + 16f
                const uint8_t *pk = ck + (tk >> 1) * KC_STRIDE + ckn;
                const uint8_t *pv = cv + tv * VC_STRIDE;
                const int bv = cvn >> 1, sv = vc_swz(tv);
                const int shk = (tk & 1) * 4, shv = (cvn & 1) * 4;
#pragma unroll
                for (int f = 0; f < TPW; ++f) {
                    wk[e] |= (((uint32_t)pk[8 * f * KC_STRIDE] >> shk) & 0xFu) << (hi * 16 + f * BITS);
                    wv[e] |= (((uint32_t)pv[(bv + 8 * f) ^ sv] >> shv) & 0xFu) << (hi * 16 + f * BITS);
                }
            }
        }
        reinterpret_cast<uint4 *>(out + Blk::K_OFF)[w4] = make_uint4(wk[0], wk[1], wk[2], wk[3]);
        reinterpret_cast<uint4 *>(out + Blk::V_OFF)[w4] = make_uint4(wv[0], wv[1], wv[2], wv[3]);
    }
    // params + norms: the K tail [a][b][norms] and the V tail [a][b] of the record
    constexpr int KTAIL = Blk::K_PART - Blk::KA_OFF, VTAIL = Blk::BYTES - Blk::VA_OFF;
    static_assert(KTAIL % 16 == 0 && VTAIL % 16 == 0, "128-bit tail stores");
    for (int i = threadIdx.x; i < (KTAIL + VTAIL) / 16; i += QT * GPAR) {
        const uint4 x = reinterpret_cast<const uint4 *>(prm)[i];
        if (i < KTAIL / 16) reinterpret_cast<uint4 *>(out + Blk::KA_OFF)[i] = x;
        else reinterpret_cast<uint4 *>(out + Blk::VA_OFF)[i - KTAIL / 16] = x;
    }
}

// bits == 0 / method fp: the record is raw bf16, four 32-token quarters of
// [K 8 KB][V 8 KB] in A-fragment order (layout.h, bf16_k_coords / bf16_v_coords)
__global__ void __launch_bounds__(QT) raw_block_kernel_dyn(const QuantizeArgs a) {
    extern __shared__ __align__(16) uint8_t smem[];
    uint16_t *sk = reinterpret_cast<uint16_t *>(smem);
    uint16_t *sv = sk + R * D;
    const int bh = blockIdx.y, b = bh / a.H, h = bh % a.H;
    const int64_t blk = blockIdx.x;
    const int64_t out_blk = (int64_t)bh * a.max_blocks + a.blk0 + blk;
    uint8_t *out = a.blocks + out_blk * (int64_t)BF16_BLOCK_BYTES;
    const uint16_t *kin = reinterpret_cast<const uint16_t *>(a.k) + b * a.sb + h * a.sh;
    const uint16_t *vin = reinterpret_cast<const uint16_t *>(a.v) + b * a.sb + h * a.sh;
    const int64_t tok_base = a.tok0 + blk * R - a.rtok;
    const uint16_t *rk = a.rk ? reinterpret_cast<const uint16_t *>(a.rk) + (int64_t)bh * R * D : nullptr;
    const uint16_t *rv = a.rv ? reinterpret_cast<const uint16_t *>(a.rv) + (int64_t)bh * R * D : nullptr;
    for (int i = threadIdx.x; i < R * 16; i += QT) {
        const int t = i >> 4, part = i & 15;
        if (blk == 0 && t < a.rtok) {  // open residual window: K row-major ring, V tile-major ring
            reinterpret_cast<uint4 *>(sk)[i] = *reinterpret_cast<const uint4 *>(rk + (int64_t)t * D + part * 8);
#pragma unroll
            for (int e = 0; e < 8; ++e) sv[t * D + part * 8 + e] = rv[vring_index(part * 8 + e, t)];
            continue;
        }
        reinterpret_cast<uint4 *>(sk)[i] = *reinterpret_cast<const uint4 *>(kin + (tok_base + t) * a.st + part * 8);
        if (a.vsc == 1) {
            reinterpret_cast<uint4 *>(sv)[i] = *reinterpret_cast<const uint4 *>(vin + (tok_base + t) * a.vst + part * 8);
        } else {
#pragma unroll
            for (int e = 0; e < 8; ++e) sv[t * D + part * 8 + e] = vin[vring_index(part * 8 + e, (int)(tok_base + t))];
        }
    }
    __syncthreads();
    constexpr int QW = BF16_QUARTER_BYTES / 2 / 4;  // 32-bit words per tensor per quarter (2048)
    for (int i = threadIdx.x; i < 4 * QW; i += QT) {
        const int qu = i / QW, w = i % QW;
        int t0, c0, t1, c1;
        bf16_k_coords(w, 0, t0, c0);
        bf16_k_coords(w, 1, t1, c1);
        const uint32_t kw = (uint32_t)sk[(qu * 32 + t0) * D + c0] | ((uint32_t)sk[(qu * 32 + t1) * D + c1] << 16);
        bf16_v_coords(w, 0, t0, c0);
        bf16_v_coords(w, 1, t1, c1);
        const uint32_t vw = (uint32_t)sv[(qu * 32 + t0) * D + c0] | ((uint32_t)sv[(qu * 32 + t1) * D + c1] << 16);
        uint32_t *qo = reinterpret_cast<uint32_t *>(out + qu * BF16_QUARTER_BYTES);
        qo[w] = kw;
        qo[QW + w] = vw;
    }
}

__global__ void ring_copy_kernel(const RingCopyArgs a) {
    const int bh = blockIdx.y, b = bh / a.H, h = bh % a.H;
    const int64_t t = blockIdx.x;
    const uint16_t *kin = reinterpret_cast<const uint16_t *>(a.k) + b * a.sb + h * a.sh + (a.tok0 + t) * a.st;
    const uint16_t *vin = reinterpret_cast<const uint16_t *>(a.v) + b * a.sb + h * a.sh + (a.tok0 + t) * a.st;
    uint16_t *rk = reinterpret_cast<uint16_t *>(a.ring_k) + ((int64_t)bh * R + a.slot0 + t) * D;
    uint16_t *rv = reinterpret_cast<uint16_t *>(a.ring_v) + (int64_t)bh * R * D;
    const int slot = (int)(a.slot0 + t);
    const int i = threadIdx.x;  // 32 threads: 16 B of K each (row-major), 4 V channels each (tile-major ring)
    if (i < 16) reinterpret_cast<uint4 *>(rk)[i] = reinterpret_cast<const uint4 *>(kin)[i];
    const uint2 vv = reinterpret_cast<const uint2 *>(vin)[i];
    rv[vring_index(4 * i + 0, slot)] = (uint16_t)(vv.x & 0xffffu);
    rv[vring_index(4 * i + 1, slot)] = (uint16_t)(vv.x >> 16);
    rv[vring_index(4 * i + 2, slot)] = (uint16_t)(vv.y & 0xffffu);
    rv[vring_index(4 * i + 3, slot)] = (uint16_t)(vv.y >> 16);
}

}  // namespace

template <int BITS, int GPAR>
cudaError_t launch_q(const QuantizeArgs &a, dim3 grid, cudaStream_t st) {
    const int smem = GPAR * 32 * KU_ROW * 8 + (R / 2) * KC_STRIDE + R * VC_STRIDE + (Block<BITS>::K_PART - Block<BITS>::KA_OFF) +
                     (Block<BITS>::BYTES - Block<BITS>::VA_OFF);
    static std::atomic<uint64_t> attr_done{0};
    if (cudaError_t e = ensure_smem_attr(quantize_kernel<BITS, GPAR>, smem, attr_done); e != cudaSuccess) return e;
    quantize_kernel<BITS, GPAR><<<grid, QT * GPAR, smem, st>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_quantize(const QuantizeArgs &a, cudaStream_t st) {
    if (a.n_blocks <= 0) return cudaSuccess;
    dim3 grid((unsigned)a.n_blocks, (unsigned)(a.B * a.H));
    if (a.tc.bits == 0) {
        static std::atomic<uint64_t> attr_done{0};
        if (cudaError_t e = ensure_smem_attr(raw_block_kernel_dyn, 2 * R * D * 2, attr_done); e != cudaSuccess)
            return e;
        raw_block_kernel_dyn<<<grid, QT, 2 * R * D * 2, st>>>(a);
        return cudaGetLastError();
    }
    // few blocks (the flush; short streaming chunks): 4 groups in parallel per CTA
    // for latency; bulk prefill: one group at a time, more CTAs per SM
    const bool flush = a.n_blocks * a.B * a.H <= 2 * 148;
    if (a.tc.bits == 2) return flush ? launch_q<2, 4>(a, grid, st) : launch_q<2, 1>(a, grid, st);
    return flush ? launch_q<4, 4>(a, grid, st) : launch_q<4, 1>(a, grid, st);
}

cudaError_t launch_ring_copy(const RingCopyArgs &a, cudaStream_t st) {
    if (a.n <= 0) return cudaSuccess;
    dim3 grid((unsigned)a.n, (unsigned)(a.B * a.H));
    ring_copy_kernel<<<grid, 32, 0, st>>>(a);
    return cudaGetLastError();
}

}  // namespace osk
