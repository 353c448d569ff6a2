// f64_path.cu -- the reference-form append path: keys that are ALREADY
// transformed (apply_method's rotated + scaled rows K_u, fp64) with their
// norms, and fp64 value rows, exactly what KvCache::buffer_quant_k(new_k,
// norms) / buffer_quant_v(new_v) receive (kv_cache.cpp:194-292).  The raw
// bf16 path (quantize.cu) fuses the transform; this one starts after it.
//
//   quantize_f64_kernel  flush_k_block / flush_v_block (kv_cache.cpp:101-157) of
//                        one R-block: the K part (per-channel groups of G tokens,
//                        norms) OR the V part (per-token groups of G channels) of
//                        the record + the exact fp64 shadow, bit-exact vs the
//                        reference (same fp64 operation order as quantize.cu)
//   window_f64_kernel    residual-window append: the fp64 rows into the exact
//                        residual shadow (export, flush) and their fp16 image into
//                        the attention rings (the decode kernel's residual tiles
//                        attend raw q . raw k, so the key ring holds
//                        FHT(K_u * norm) -- apply_method inverted -- in fp16)
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "device_common.cuh"
#include "kernels.h"
#include "layout.h"
#include "quant_common.cuh"

namespace osk {

namespace {

constexpr int FT = 128;  // threads per CTA
constexpr int CSTRIDE = D + 4;  // padded code-tile row (as quantize.cu)

// element (b, h, t, c) of a strided fp64 source
__device__ __forceinline__ const double *row_ptr(const F64Src &s, int b, int h, int64_t t) {
    return s.p + b * s.sb + h * s.sh + t * s.st;
}

template <int BITS>
__global__ void __launch_bounds__(FT) quantize_f64_kernel(const QuantizeF64Args a) {
    using Blk = Block<BITS>;
    __shared__ uint8_t codes[R * CSTRIDE];                 // [token][channel]
    __shared__ __align__(16) uint8_t prm[Blk::K_PART - Blk::KA_OFF > Blk::BYTES - Blk::VA_OFF
                                             ? Blk::K_PART - Blk::KA_OFF
                                             : Blk::BYTES - Blk::VA_OFF];
    const int tid = threadIdx.x;
    const int bh = blockIdx.y, b = bh / a.H, h = bh % a.H;
    const int64_t blk = blockIdx.x;
    const int64_t out_blk = (int64_t)bh * a.max_blocks + a.blk0 + blk;
    uint8_t *out = a.blocks + out_blk * (int64_t)Blk::BYTES;
    double *shadow = a.shadow + out_blk * SHADOW_DOUBLES;
    const int64_t t0 = a.tok0 + blk * R;  // first source token of the block
    if (a.part == 0) {
        // ---- K part: channel c = tid, groups of G tokens (kv_cache.cpp:101-129) ----
        __half *ka = reinterpret_cast<__half *>(prm);
        __half *kb = ka + D * NGRP;
        float *nrm = reinterpret_cast<float *>(kb + D * NGRP);
        const int c = tid;
        for (int grp = 0; grp < NGRP; ++grp) {
            double x[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) x[i] = row_ptr(a.src, b, h, t0 + grp * G + i)[c];
            const GroupQ p = group_params([&](int i) { return x[i]; }, BITS);
            quantize_group([&](int i) { return x[i]; }, p, BITS,
                           [&](int i, int code) { codes[(grp * G + i) * CSTRIDE + c] = (uint8_t)code; });
            __half ha, hb;
            affine16(p, ha, hb);
            flag_status(a.status, p, ha, hb);
            if (!isfinite(p.lo) || !isfinite(p.hi)) flag_nonfinite(a.status);
            ka[ka_index(c, grp)] = ha;
            kb[kb_index(c, grp)] = hb;
            shadow[(c * NGRP + grp) * 2] = p.lo;
            shadow[(c * NGRP + grp) * 2 + 1] = p.hi;
        }
        {
            const int t = tid;  // norms, token t (the record's fp32 copy is pre-multiplied by log2(e)/sqrt(d))
            const double s = a.norms.p[b * a.norms.sb + h * a.norms.sh + (t0 + t) * a.norms.st];
            nrm[norm_index(t)] = __double2float_rn(__dmul_rn(s, 0.12751743074202186));
            shadow[SHADOW_K_DOUBLES + SHADOW_V_DOUBLES + t] = s;
        }
    } else {
        // ---- V part: token t = tid, groups of G channels (kv_cache.cpp:131-157) ----
        __half *va = reinterpret_cast<__half *>(prm);
        __half *vb = va + R * NGC;
        const int t = tid;
        const double *row = row_ptr(a.src, b, h, t0 + t);
        for (int gc = 0; gc < NGC; ++gc) {
            double y[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) y[i] = row[gc * G + i];
            const GroupQ p = group_params([&](int i) { return y[i]; }, BITS);
            quantize_group([&](int i) { return y[i]; }, p, BITS,
                           [&](int i, int code) { codes[t * CSTRIDE + gc * G + i] = (uint8_t)code; });
            __half ha, hb;
            affine16(p, ha, hb);
            flag_status(a.status, p, ha, hb);
            if (!isfinite(p.lo) || !isfinite(p.hi)) flag_nonfinite(a.status);
            va[va_index(t, gc)] = ha;
            vb[vb_index(t, gc)] = hb;
            shadow[SHADOW_K_DOUBLES + (t * NGC + gc) * 2] = p.lo;
            shadow[SHADOW_K_DOUBLES + (t * NGC + gc) * 2 + 1] = p.hi;
        }
    }
    __syncthreads();
    // ---- the permuted code words of this part (layout.h), 128-bit stores ----
    constexpr int NWORDS = R * D * BITS / 32;
    constexpr int TPW = 16 / BITS;
    uint8_t *dst = out + (a.part == 0 ? Blk::K_OFF : Blk::V_OFF);
    for (int w4 = tid; w4 < NWORDS / 4; w4 += FT) {
        uint32_t wd[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const int w = 4 * w4 + e;
            wd[e] = 0;
#pragma unroll
            for (int hi = 0; hi < 2; ++hi) {
                int t, c;
                if (a.part == 0) k_word_coords(BITS, w, 0, hi, t, c);
                else v_word_coords(BITS, w, 0, hi, t, c);
                // field f of a K word is token +16f, of a V word channel +16f
                const uint8_t *pc = codes + t * CSTRIDE + c;
#pragma unroll
                for (int f = 0; f < TPW; ++f)
                    wd[e] |= (uint32_t)pc[a.part == 0 ? 16 * f * CSTRIDE : 16 * f] << (hi * 16 + f * BITS);
            }
        }
        reinterpret_cast<uint4 *>(dst)[w4] = make_uint4(wd[0], wd[1], wd[2], wd[3]);
    }
    // the part's params (+ norms): K tail [a][b][norms] or V tail [a][b]
    const int tail = a.part == 0 ? Blk::K_PART - Blk::KA_OFF : Blk::BYTES - Blk::VA_OFF;
    uint8_t *tdst = out + (a.part == 0 ? Blk::KA_OFF : Blk::VA_OFF);
    for (int i = tid; i < tail / 16; i += FT) reinterpret_cast<uint4 *>(tdst)[i] = reinterpret_cast<const uint4 *>(prm)[i];
}

// normalised FHT of a 128-vector, 4 per lane, fp64 in the reference's stage
// order (hadamard.cpp:10-26: half = 1, 2 in the lane, then 4..64 across lanes)
__device__ __forceinline__ void fht128_lanes(double (&x)[4], int lane) {
    double a = x[0], b = x[1];
    x[0] = __dadd_rn(a, b);
    x[1] = __dsub_rn(a, b);
    a = x[2];
    b = x[3];
    x[2] = __dadd_rn(a, b);
    x[3] = __dsub_rn(a, b);
    a = x[0];
    b = x[2];
    x[0] = __dadd_rn(a, b);
    x[2] = __dsub_rn(a, b);
    a = x[1];
    b = x[3];
    x[1] = __dadd_rn(a, b);
    x[3] = __dsub_rn(a, b);
#pragma unroll
    for (int xm = 1; xm < 32; xm <<= 1) {
        const bool upper = (lane & xm) != 0;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const double o = __shfl_xor_sync(0xffffffffu, x[e], xm);
            x[e] = upper ? __dsub_rn(o, x[e]) : __dadd_rn(x[e], o);
        }
    }
    const double sc = __ddiv_rn(1.0, __dsqrt_rn(128.0));
#pragma unroll
    for (int e = 0; e < 4; ++e) x[e] = __dmul_rn(x[e], sc);
}

// the fp16 image of an fp64 ring value, round to nearest (the host load path
// rounds the same way: double_to_half_rn)
__device__ __forceinline__ uint16_t ring_image(double x) {
    const __half v = __double2half(x);
    return *reinterpret_cast<const uint16_t *>(&v);
}

// one warp per (token, bh): K (part 0) or V (part 1) rows of the window
__global__ void window_f64_kernel(const WindowF64Args a) {
    const int lane = threadIdx.x;
    const int64_t t = blockIdx.x;
    const int bh = blockIdx.y, b = bh / a.H, h = bh % a.H;
    const int slot = (int)(a.slot0 + t);
    const double *row = row_ptr(a.src, b, h, a.tok0 + t);
    double x[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) x[e] = row[4 * lane + e];
    if (a.part == 0) {
        const double s = a.norms.p[b * a.norms.sb + h * a.norms.sh + (a.tok0 + t) * a.norms.st];
        double *rk = a.res_k + ((int64_t)bh * R + slot) * D;
#pragma unroll
        for (int e = 0; e < 4; ++e) rk[4 * lane + e] = x[e];
        if (lane == 0) a.res_n[(int64_t)bh * R + slot] = s;
        // the raw key the decode kernel attends: apply_method inverted (K_u * s, then
        // the Hadamard transform again -- it is its own inverse), rounded to bf16
        double y[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) y[e] = a.scales ? __dmul_rn(x[e], s) : x[e];
        if (a.rotates) fht128_lanes(y, lane);
        uint16_t *ring = reinterpret_cast<uint16_t *>(a.ring_k) + ((int64_t)bh * R + slot) * D;
        reinterpret_cast<uint2 *>(ring)[lane] = make_uint2((uint32_t)ring_image(y[0]) | ((uint32_t)ring_image(y[1]) << 16),
                                                           (uint32_t)ring_image(y[2]) | ((uint32_t)ring_image(y[3]) << 16));
    } else {
        double *rv = a.res_v + ((int64_t)bh * R + slot) * D;
#pragma unroll
        for (int e = 0; e < 4; ++e) rv[4 * lane + e] = x[e];
        uint16_t *ring = reinterpret_cast<uint16_t *>(a.ring_v) + (int64_t)bh * R * D;  // tile-major (vring_index)
#pragma unroll
        for (int e = 0; e < 4; ++e) ring[vring_index(4 * lane + e, slot)] = ring_image(x[e]);
    }
}

}  // namespace

cudaError_t launch_quantize_f64(const QuantizeF64Args &a, cudaStream_t st) {
    if (a.n_blocks <= 0) return cudaSuccess;
    dim3 grid((unsigned)a.n_blocks, (unsigned)(a.B * a.H));
    if (a.bits == 2) quantize_f64_kernel<2><<<grid, FT, 0, st>>>(a);
    else if (a.bits == 4) quantize_f64_kernel<4><<<grid, FT, 0, st>>>(a);
    else return cudaErrorInvalidValue;
    return cudaGetLastError();
}

cudaError_t launch_window_f64(const WindowF64Args &a, cudaStream_t st) {
    if (a.n <= 0) return cudaSuccess;
    dim3 grid((unsigned)a.n, (unsigned)(a.B * a.H));
    window_f64_kernel<<<grid, 32, 0, st>>>(a);
    return cudaGetLastError();
}

}  // namespace osk
