// logits.cu -- StepOutput.logits of the reference's decode_step
// (pipeline.hpp:54-58; written by attend_one at pipeline.cpp:158-165 and
// returned at pipeline.cpp:314-318): for every query head the attention logit
// q.k/sqrt(d) (natural units) of every context token, head-major.
//
// A debug / fidelity output, not the hot path: the decode-attention kernel
// never materialises logits.  This kernel reads the SAME device records the
// attention kernel streams (fp16 step a and offset b per group, fp32 norm per
// token, the permuted code words) and evaluates
//   packed token t:  logit = ||k_t|| / sqrt(d) * sum_c Qrot[c] * (a * code + b)
//   window / current token:  logit = q . k_raw / sqrt(d)   (bf16 rows)
// in fp32, one thread per token, so it reports what the device cache holds.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "kernels.h"
#include "layout.h"

namespace osk {

namespace {

constexpr float LN2 = 0.6931471805599453f;
constexpr float INV_SQRT_D = 0.08838834764831845f;

__device__ __forceinline__ float bf16_at(const void *base, int64_t idx) {
    const uint16_t u = reinterpret_cast<const uint16_t *>(base)[idx];
    return __uint_as_float((uint32_t)u << 16);
}

// grid (tiles, BH): tile < nb -> packed R-block `tile`; tile == nb -> the
// residual window + current token (ntok <= R tokens).  128 threads = tokens.
template <int BITS>
__global__ void __launch_bounds__(128) logits_kernel(const LogitsArgs a) {
    __shared__ float qs[8][D];
    const int bh = blockIdx.y, tile = blockIdx.x, tid = threadIdx.x;
    const int b = bh / a.Hkv, kvh = bh % a.Hkv, g = a.g;
    const bool packed = tile < a.nb;
    // this (b, kv head)'s query rows; rotated (normalised FHT, the Q side of
    // apply_method, pipeline.cpp:224-236) for the packed part of a rotating cache
    for (int j = 0; j < g; ++j)
        qs[j][tid] = bf16_at(a.q, ((int64_t)b * a.Hq + kvh * g + j) * D + tid);
    __syncthreads();
    if (packed && a.rotates) {
        for (int half = 1; half < D; half <<= 1) {  // hadamard.cpp:14-23 stage order
            for (int j = 0; j < g; ++j) {
                float x = 0.f;
                const int partner = tid ^ half;
                const float mine = qs[j][tid], other = qs[j][partner];
                x = (tid & half) ? other - mine : mine + other;
                __syncthreads();
                qs[j][tid] = x;
                __syncthreads();
            }
        }
        for (int j = 0; j < g; ++j) qs[j][tid] *= INV_SQRT_D;
        __syncthreads();
    }
    float acc[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] = 0.f;
    int64_t tok;
    float scale;
    if (packed) {
        const uint8_t *rec = a.blocks + ((int64_t)bh * a.max_blocks + tile) * (int64_t)a.block_bytes;
        const int t = tid;
        tok = (int64_t)tile * R + t;
        if (BITS == 0) {
            for (int c = 0; c < D; ++c) {
                const uint16_t u = *reinterpret_cast<const uint16_t *>(rec + bf16_k_byte(t, c));
                const float kv = __uint_as_float((uint32_t)u << 16);
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    if (j < g) acc[j] += qs[j][c] * kv;
            }
            scale = INV_SQRT_D;  // raw q . raw k (the bf16 record holds untransformed rows)
        } else {
            using Blk = Block<BITS == 0 ? 2 : BITS>;
            const uint32_t *kw = reinterpret_cast<const uint32_t *>(rec + Blk::K_OFF);
            const __half *ka = reinterpret_cast<const __half *>(rec + Blk::KA_OFF);
            const __half *kb = reinterpret_cast<const __half *>(rec + Blk::KB_OFF);
            const float *nr = reinterpret_cast<const float *>(rec + Blk::NORM_OFF);
            const int grp = t / G;
            for (int c = 0; c < D; ++c) {
                int w, sh;
                k_code_loc(BITS, t, c, w, sh);
                const float code = (float)((kw[w] >> sh) & ((1u << BITS) - 1u));
                const float kv = __half2float(ka[ka_index(c, grp)]) * code + __half2float(kb[kb_index(c, grp)]);
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    if (j < g) acc[j] += qs[j][c] * kv;
            }
            scale = nr[norm_index(t)] * LN2;  // record norm = ||k|| * log2(e) / sqrt(d)
        }
    } else {
        const int ntok = a.r + (a.kcur ? 1 : 0);
        if (tid >= ntok) return;
        tok = (int64_t)a.nb * R + tid;
        const void *krow = nullptr;
        int64_t off = 0;
        if (tid < a.r) {
            krow = a.ring_k;
            off = ((int64_t)bh * R + tid) * D;
        } else {
            krow = a.kcur;
            off = (int64_t)bh * D;
        }
        const bool f16 = a.ring_f16 && tid < a.r;
        for (int c = 0; c < D; ++c) {
            const float kv = f16 ? __half2float(reinterpret_cast<const __half *>(krow)[off + c]) : bf16_at(krow, off + c);
#pragma unroll
            for (int j = 0; j < 8; ++j)
                if (j < g) acc[j] += qs[j][c] * kv;
        }
        scale = INV_SQRT_D;
    }
    for (int j = 0; j < g; ++j)
        a.logits[((int64_t)b * a.Hq + kvh * g + j) * a.s_total + tok] = acc[j] * scale;
}

}  // namespace

cudaError_t launch_logits(int bits, const LogitsArgs &a, cudaStream_t st) {
    const int ntok = a.r + (a.kcur ? 1 : 0);
    const int64_t tiles = a.nb + (ntok > 0 ? 1 : 0);
    if (tiles == 0 || a.BH == 0) return cudaSuccess;
    dim3 grid((unsigned)tiles, (unsigned)a.BH);
    switch (bits) {
        case 2: logits_kernel<2><<<grid, 128, 0, st>>>(a); break;
        case 4: logits_kernel<4><<<grid, 128, 0, st>>>(a); break;
        case 0: logits_kernel<0><<<grid, 128, 0, st>>>(a); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

}  // namespace osk
