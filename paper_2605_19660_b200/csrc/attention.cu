// attention.cu -- fused-dequant split-KV decode attention over the packed
// OScaR cache (replaces materialize_k + materialize_v + the attend_one loop,
// pipeline.cpp:294-319 / kv_cache.cpp:327-381).
//
// Persistent, stream-K style: one CTA per SM gets an equal contiguous range
// of the global (sequence*KV-head, R-block) space, so every SM streams the
// same number of bytes.  All NCW warps consume (12 for INT2, 8 for INT4 and
// bf16): unit p of the range (one R-block record of 12.8 KB INT2 / 21 KB
// INT4, or a 16 KB quarter of a bf16 record, see layout.h) is streamed HBM ->
// shared memory by ONE cp.async.bulk (TMA engine, L2 evict-first) into stage
// p % NST of an mbarrier ring and processed by warp p % NCW, which then
// refills that same stage with unit p + NST -- no producer warp, no empty
// barriers.
// Per block a consumer runs QK^T and P.V on the tensor cores
// (mma.sync m16n8k16, fp16 in / fp32 accumulate) straight from the packed
// codes: every loaded 32-bit word ANDed with a field mask IS an A register
// holding fp16 subnormals code*2^(f*BITS-24); the per-group step a is folded
// into the B operand (Q*aK for keys, P*aV for values), the per-group offset b
// into one extra MMA per block, the per-token key norm into the fp32
// epilogue.  Online softmax in log2 units; partials are merged per CTA in
// shared memory and across CTAs by the last-arriving CTA of each (b, kv-head)
// (atomic ticket).  The residual window (< R full-precision tokens) plus the
// current token are attended on the bf16 tensor cores, one 16-token tile per
// warp of the CTA that owns the last packed block of the sequence; the tile
// holding the current token also writes it into the residual ring.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <math_constants.h>
#include <stdlib.h>

#include "device_common.cuh"
#include "kernels.h"
#include "layout.h"
#include "peer.cuh"
#include "split.h"

namespace osk {

namespace {

// phase-cycle counters (OSCAR_PROF) exist only in the profiling build
// (make PROF=1 -> liboscar_b200_prof.so): the timers cost ~30 issue slots per unit
#ifndef OSK_PROF
#define OSK_PROF 0
#endif
constexpr bool kProf = OSK_PROF != 0;
// partials per batch of the ticket-form final merge (one L2 round trip each)
#ifndef OSK_TICKET_FB
#define OSK_TICKET_FB 32
#endif

constexpr int MERGE_FLOATS = 8 * D + 16 + D;  // per-warp partial: O[8][128], m[8], l[8] + 128 scratch
constexpr float LOG2E = 1.4426950408889634f;
constexpr float LN2 = 0.6931471805599453f;
#ifndef OSK_RESCALE_SLACK
#define OSK_RESCALE_SLACK 3
#endif
constexpr float RESCALE_SLACK = (float)OSK_RESCALE_SLACK;  // log2 units
// Cost experiments for the accuracy/speed table (results are NOT
// correct in these builds): OSK_COST_EXTRA extra record bytes per unit,
// OSK_COST_KB_HILO a second key-offset MMA per k-step (hi/lo fp16 split of b),
// OSK_COST_K_HILO a second code MMA + q*a_lo product per key tile (hi/lo split of q*a)
#ifndef OSK_SKIP_TILES  // experiment: residual tiles not computed (results not correct)
#define OSK_SKIP_TILES 0
#endif
#ifndef OSK_COST_EXTRA
#define OSK_COST_EXTRA 0
#endif
#ifndef OSK_COST_KB_HILO
#define OSK_COST_KB_HILO 0
#endif
#ifndef OSK_COST_K_HILO
#define OSK_COST_K_HILO 0
#endif

constexpr int MAXSEG_SMEM = 64;  // max segments (b, kv heads) per CTA range
constexpr int NCW_MAX = 16;
constexpr int QH_STRIDE = 136;  // padded fp16 row of a q tile (conflict-free; 16-B aligned rows)
constexpr int QSEG = 4;         // segment q tiles held in shared memory (one wave)

template <int BITS, int NCW_ = ((BITS == 4) ? 8 : 12), bool TILES_ = false>
struct AttnCfg {
    // one pipeline stage: a whole INT2/INT4 record, or a 32-token quarter of a bf16 record
    static constexpr int BYTES = (BITS == 0) ? BF16_BLOCK_BYTES : Block<BITS == 0 ? 2 : BITS>::BYTES;
    static constexpr int SUB = (BITS == 0) ? 4 : 1;
    // (OSK_COST_EXTRA: cost experiments only -- every stage also streams that many
    //  bytes past its record, as a wider record would)
    static constexpr int STAGE = BYTES / SUB + (BITS == 0 ? 0 : OSK_COST_EXTRA);
    static constexpr int NCW = NCW_;  // warps per CTA, all consumers
    static constexpr int NTHREADS = NCW * 32;
    static constexpr int QH_OFF = 0;                                   // QSEG segment q tiles
    static constexpr int SEG_OFF = QH_OFF + QSEG * 8 * QH_STRIDE * 2;  // lastflag[MAXSEG_SMEM]
    static constexpr int TAB_OFF = ((SEG_OFF + MAXSEG_SMEM * 4 + 7) / 8) * 8;  // last-segment slot per warp
    static constexpr int WALK_OFF = TAB_OFF + NCW_MAX * 8;  // per-warp refill walker (tile units)
    static constexpr int BAR_OFF = WALK_OFF + (TILES_ ? NCW_MAX * 16 : 0);
    // shared ring of NST stages: as many whole stages as fit in 227 KB
    static constexpr int NST = (232448 - BAR_OFF - 1024) / STAGE;
    static constexpr int CNT_OFF = BAR_OFF + NST * 8;  // consumed-round counter per stage
    static constexpr int RING_OFF = ((CNT_OFF + NST * 4 + 127) / 128) * 128;
    static constexpr int SMEM = RING_OFF + NST * STAGE;
    static_assert(SMEM <= 232448, "shared memory budget");
};

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// normalized FHT of a 128-vector held 4 per lane (channel lane*4+e), fp32
__device__ __forceinline__ void fht128_warp(float (&x)[4], int lane) {
    // half = 1, 2 inside the lane
    {
        float a = x[0], b = x[1];
        x[0] = a + b;
        x[1] = a - b;
        a = x[2];
        b = x[3];
        x[2] = a + b;
        x[3] = a - b;
        a = x[0];
        b = x[2];
        x[0] = a + b;
        x[2] = a - b;
        a = x[1];
        b = x[3];
        x[1] = a + b;
        x[3] = a - b;
    }
#pragma unroll
    for (int xm = 1; xm < 32; xm <<= 1) {
        const bool upper = (lane & xm) != 0;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const float o = __shfl_xor_sync(0xffffffffu, x[e], xm);
            x[e] = upper ? (o - x[e]) : (x[e] + o);
        }
    }
    const float sc = 0.08838834764831845f;  // 1/sqrt(128)
#pragma unroll
    for (int e = 0; e < 4; ++e) x[e] *= sc;
}

__device__ __forceinline__ void load_bf16x4(const __nv_bfloat16 *p, float (&x)[4]) {
    const uint2 u = *reinterpret_cast<const uint2 *>(p);
    x[0] = __uint_as_float(u.x << 16);
    x[1] = __uint_as_float(u.x & 0xffff0000u);
    x[2] = __uint_as_float(u.y << 16);
    x[3] = __uint_as_float(u.y & 0xffff0000u);
}


// ----------------------------------------------------------------------------
// per-warp accumulator state (fragment layouts, see layout.h)
struct WarpState {
    float o[8][4];   // P.V accumulators: m-tile mm, (row gq|gq+8) x (head 2tq|2tq+1)
    float ob[4];     // V-offset accumulators: row gq = channel group, even k-steps
    float ob2[4];    //   rows gq+8 = channel group, odd k-steps (paired b-param quads)
    float m[2], l[2];
};

__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ long long clk() {
    long long c;
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(c));
    return c;
}

// qsm: this lane's row of the segment's rotated-q tile in shared memory (fp16,
// row gq, offset 2tq); the B fragments are re-read per k-step instead of being
// held in 16 registers across the block
template <int BITS>
__device__ __forceinline__ void process_block(const uint8_t *__restrict__ sb, WarpState &st,
                                              const __half *__restrict__ qsm, int lane, float c0,
                                              long long *tm = nullptr) {
    long long t0 = tm ? clk() : 0;
    using Blk = Block<BITS>;
    constexpr int TPW = 16 / BITS;   // m-tiles per half-word
    constexpr int WPF = 8 / TPW;     // words per fragment family per k-step
    constexpr int HALFT = TPW / 2;   // fields reachable without a shift
    constexpr uint32_t FMASK = (BITS == 2) ? 0x00030003u : 0x000F000Fu;
    const int gq = lane >> 2, tq = lane & 3;

    // ---- key offsets as A (row gq = group): bias[grp][head] = sum_c b[c,grp] * Qrot[head][c]
    //      (x = a*code + b, the value form of dequantize_one, quant.cpp:65-68) -- one
    //      MMA per k-step; row gq < 4 (= group) is read back, rows 4..15 are don't-care
    const uint4 *bkp = reinterpret_cast<const uint4 *>(sb + Blk::KB_OFF + ((gq & 3) * 4 + tq) * 16);
    float kbias[4], kbias2[4];  // rows gq: even k-steps; rows gq+8: odd k-steps
    uint4 zk;

    // ---- QK^T --------------------------------------------------------------------
    float sacc[8][4];
#pragma unroll
    for (int s = 0; s < 8; ++s) {
        uint32_t kw[4 * WPF], kwh[4 * WPF];
        {
            const uint4 *p = reinterpret_cast<const uint4 *>(sb + Blk::K_OFF + (s * 32 + lane) * 16 * WPF);
#pragma unroll
            for (int v = 0; v < WPF; ++v) {
                const uint4 u = p[v];
                kw[4 * v] = u.x;
                kw[4 * v + 1] = u.y;
                kw[4 * v + 2] = u.z;
                kw[4 * v + 3] = u.w;
            }
#pragma unroll
            for (int v = 0; v < 4 * WPF; ++v) kwh[v] = shr8(kw[v]);
        }
        uint32_t qf[8][2];  // only [s] is live
        qf[s][0] = *reinterpret_cast<const uint32_t *>(qsm + 16 * s);
        qf[s][1] = *reinterpret_cast<const uint32_t *>(qsm + 16 * s + 8);
        uint32_t bq[4][2];
        {
            const uint4 *p = reinterpret_cast<const uint4 *>(sb + Blk::KA_OFF + (s * 4 + tq) * 32);
            const uint4 a01 = p[0], a23 = p[1];
            bq[0][0] = hmul2_u32(qf[s][0], a01.x);
            bq[0][1] = hmul2_u32(qf[s][1], a01.y);
            bq[1][0] = hmul2_u32(qf[s][0], a01.z);
            bq[1][1] = hmul2_u32(qf[s][1], a01.w);
            bq[2][0] = hmul2_u32(qf[s][0], a23.x);
            bq[2][1] = hmul2_u32(qf[s][1], a23.y);
            bq[3][0] = hmul2_u32(qf[s][0], a23.z);
            bq[3][1] = hmul2_u32(qf[s][1], a23.w);
        }
        {
            // one quad per k-step pair (layout.h kb_index): rows gq = group gq & 3 at
            // k-step s (even), rows gq+8 = the same group at s+1; the other rows of
            // each product are don't-care (lanes gq >= 4 duplicate groups 0-3)
            if ((s & 1) == 0) zk = bkp[(s >> 1) * 16];
            if (s == 0) mma16816_zc(kbias, zk.x, zk.y, zk.z, zk.w, qf[s][0], qf[s][1]);
            else if (s == 1) mma16816_zc(kbias2, zk.x, zk.y, zk.z, zk.w, qf[s][0], qf[s][1]);
            else if ((s & 1) == 0) mma16816(kbias, zk.x, zk.y, zk.z, zk.w, qf[s][0], qf[s][1]);
            else mma16816(kbias2, zk.x, zk.y, zk.z, zk.w, qf[s][0], qf[s][1]);
            if (OSK_COST_KB_HILO) {  // cost experiment: the b_lo half of a split offset
                if ((s & 1) == 0) mma16816(kbias, zk.y, zk.x, zk.w, zk.z, qf[s][0], qf[s][1]);
                else mma16816(kbias2, zk.y, zk.x, zk.w, zk.z, qf[s][0], qf[s][1]);
            }
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int half = i / TPW, f = i % TPW;
            const int fs = f % HALFT;
            const uint32_t mask = FMASK << (BITS * fs);
            const uint32_t *src = (f < HALFT) ? kw : kwh;
            // word of family fam, half `half`: index fam*WPF + half
            if (s == 0)
                mma16816_zc(sacc[i], src[0 * WPF + half] & mask, src[1 * WPF + half] & mask,
                            src[2 * WPF + half] & mask, src[3 * WPF + half] & mask, bq[i >> 1][0], bq[i >> 1][1]);
            else
                mma16816(sacc[i], src[0 * WPF + half] & mask, src[1 * WPF + half] & mask,
                         src[2 * WPF + half] & mask, src[3 * WPF + half] & mask, bq[i >> 1][0], bq[i >> 1][1]);
            if (OSK_COST_K_HILO) {  // cost experiment: the (q*a)_lo half of a split B operand
                const uint32_t l0 = hmul2_u32(bq[i >> 1][0], 0x11001100u), l1 = hmul2_u32(bq[i >> 1][1], 0x11001100u);
                mma16816(sacc[i], src[0 * WPF + half] & mask, src[1 * WPF + half] & mask,
                         src[2 * WPF + half] & mask, src[3 * WPF + half] & mask, l0, l1);
            }
        }
    }

    long long t1 = tm ? clk() : 0;
    // ---- logits (log2 units) ------------------------------------------------------------
    float nrm[16];
    {
        const uint4 *p = reinterpret_cast<const uint4 *>(sb + Blk::NORM_OFF + gq * 64);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const uint4 u = p[i];
            nrm[4 * i] = __uint_as_float(u.x);
            nrm[4 * i + 1] = __uint_as_float(u.y);
            nrm[4 * i + 2] = __uint_as_float(u.z);
            nrm[4 * i + 3] = __uint_as_float(u.w);
        }
    }
    float kb0[4], kb1[4];
#pragma unroll
    for (int grp = 0; grp < 4; ++grp) {
        kb0[grp] = __shfl_sync(0xffffffffu, kbias[0] + kbias2[2], grp * 4 + tq);
        kb1[grp] = __shfl_sync(0xffffffffu, kbias[1] + kbias2[3], grp * 4 + tq);
    }
    // logits relative to the running max, y = logit - m (one FFMA with the key
    // norm); first block of a segment: m = -inf, measure against 0 instead
    const float r0 = (st.m[0] == -CUDART_INF_F) ? 0.f : st.m[0];
    const float r1 = (st.m[1] == -CUDART_INF_F) ? 0.f : st.m[1];
    float bm0 = -CUDART_INF_F, bm1 = -CUDART_INF_F;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int fs = (i % TPW) % HALFT;
        const float sc = __int_as_float((127 + 24 - BITS * fs) << 23);  // 2^(24 - BITS*fs)
        const int grp = i >> 1;
        sacc[i][0] = fmaf(fmaf(sacc[i][0], sc, kb0[grp]), nrm[2 * i], -r0);
        sacc[i][1] = fmaf(fmaf(sacc[i][1], sc, kb1[grp]), nrm[2 * i], -r1);
        sacc[i][2] = fmaf(fmaf(sacc[i][2], sc, kb0[grp]), nrm[2 * i + 1], -r0);
        sacc[i][3] = fmaf(fmaf(sacc[i][3], sc, kb1[grp]), nrm[2 * i + 1], -r1);
        bm0 = fmaxf(bm0, fmaxf(sacc[i][0], sacc[i][2]));
        bm1 = fmaxf(bm1, fmaxf(sacc[i][1], sacc[i][3]));
    }
    // lazy rescale: the reference only moves when some lane's block max exceeds
    // it by more than RESCALE_SLACK (then reduce and rescale to the exact max);
    // in between, P = 2^(logit - m) may reach 2^RESCALE_SLACK (fp16-safe: the
    // P*a fold stays finite for value-group ranges below 65504 * 3 / 2^SLACK)
    if (!__all_sync(0xffffffffu, bm0 <= RESCALE_SLACK && bm1 <= RESCALE_SLACK && st.m[0] != -CUDART_INF_F &&
                                     st.m[1] != -CUDART_INF_F)) {
#pragma unroll
        for (int o = 4; o < 32; o <<= 1) {
            bm0 = fmaxf(bm0, __shfl_xor_sync(0xffffffffu, bm0, o));
            bm1 = fmaxf(bm1, __shfl_xor_sync(0xffffffffu, bm1, o));
        }
        // new max = r + d with d = max(block max - r, old max - r)
        const float d0 = fmaxf(bm0, st.m[0] - r0), d1 = fmaxf(bm1, st.m[1] - r1);
        const float mn0 = r0 + d0, mn1 = r1 + d1;
        const float al0 = fast_exp2(st.m[0] - mn0), al1 = fast_exp2(st.m[1] - mn1);
        st.m[0] = mn0;
        st.m[1] = mn1;
#pragma unroll
        for (int mm = 0; mm < 8; ++mm) {
            st.o[mm][0] *= al0;
            st.o[mm][1] *= al1;
            st.o[mm][2] *= al0;
            st.o[mm][3] *= al1;
        }
        st.ob[0] *= al0;
        st.ob[1] *= al1;
        st.ob2[2] *= al0;
        st.ob2[3] *= al1;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            sacc[i][0] -= d0;
            sacc[i][1] -= d1;
            sacc[i][2] -= d0;
            sacc[i][3] -= d1;
        }
    }
    // P = 2^y in fp32 (MUFU.EX2), packed to the fp16 pairs the P.V B operand needs
    // (an ex2.f16x2 of the fp16-rounded y measured 1 % slower at C2: it issues two
    // MUFU.EX2.F16 plus a PRMT per pair).  The softmax denominator is not summed
    // here: the value-offset MMA's spare A row 4 is all ones, so it accumulates
    // sum_t P per head (see P.V below).
    uint32_t P01[8], P23[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        P01[i] = pack_half2(fast_exp2(sacc[i][0]), fast_exp2(sacc[i][1]));
        P23[i] = pack_half2(fast_exp2(sacc[i][2]), fast_exp2(sacc[i][3]));
    }

    long long t2 = tm ? clk() : 0;
    // ---- P.V ---------------------------------------------------------------------------
    // value offsets as A: row gq (< 4) = channel group, k = tokens
    //      (rows 4 / 12, lanes gq == 4: all ones -> the running sum_t P per head)
    const uint4 *vbp = reinterpret_cast<const uint4 *>(sb + Blk::VB_OFF + ((gq & 3) * 4 + tq) * 16);
    constexpr uint32_t ONES = 0x3C003C00u;  // half2(1, 1)
    uint4 zv = make_uint4(ONES, ONES, ONES, ONES);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        // P of tokens 16j..16j+15 as the B operand: the accumulator rows (tokens) x
        // cols (heads 2tq, 2tq+1), transposed per 8x8 half by movmatrix, is exactly
        // the B fragment (k = tokens 2tq, 2tq+1 | 2tq+8, 2tq+9; n = head gq)
        const uint32_t bp0 = movmatrix_t(P01[j]);
        const uint32_t bp1 = movmatrix_t(P23[j]);
        uint32_t bv[4][2];
        {
            const uint4 *p = reinterpret_cast<const uint4 *>(sb + Blk::VA_OFF + (j * 4 + tq) * 32);
            const uint4 a01 = p[0], a23 = p[1];
            bv[0][0] = hmul2_u32(bp0, a01.x);
            bv[0][1] = hmul2_u32(bp1, a01.y);
            bv[1][0] = hmul2_u32(bp0, a01.z);
            bv[1][1] = hmul2_u32(bp1, a01.w);
            bv[2][0] = hmul2_u32(bp0, a23.x);
            bv[2][1] = hmul2_u32(bp1, a23.y);
            bv[3][0] = hmul2_u32(bp0, a23.z);
            bv[3][1] = hmul2_u32(bp1, a23.w);
        }
        uint32_t vw[4 * WPF], vwh[4 * WPF];
        {
            const uint4 *p = reinterpret_cast<const uint4 *>(sb + Blk::V_OFF + (j * 32 + lane) * 16 * WPF);
#pragma unroll
            for (int v = 0; v < WPF; ++v) {
                const uint4 u = p[v];
                vw[4 * v] = u.x;
                vw[4 * v + 1] = u.y;
                vw[4 * v + 2] = u.z;
                vw[4 * v + 3] = u.w;
            }
#pragma unroll
            for (int v = 0; v < 4 * WPF; ++v) vwh[v] = shr8(vw[v]);
        }
#pragma unroll
        for (int mm = 0; mm < 8; ++mm) {
            const int half = mm / TPW, f = mm % TPW;
            const int fs = f % HALFT;
            const uint32_t mask = FMASK << (BITS * fs);
            const uint32_t *src = (f < HALFT) ? vw : vwh;
            mma16816(st.o[mm], src[0 * WPF + half] & mask, src[1 * WPF + half] & mask,
                     src[2 * WPF + half] & mask, src[3 * WPF + half] & mask, bv[mm >> 1][0], bv[mm >> 1][1]);
        }
        {
            // paired quads as for the keys: even j -> rows gq of ob, odd j -> rows gq+8 of ob2
            if ((j & 1) == 0) {
                if (gq != 4) zv = vbp[(j >> 1) * 16];
                mma16816(st.ob, zv.x, zv.y, zv.z, zv.w, bp0, bp1);
            } else {
                mma16816(st.ob2, zv.x, zv.y, zv.z, zv.w, bp0, bp1);
            }
        }
    }
    if (tm) {
        const float keep = st.o[0][0] + st.o[7][3];  // order the timer after the MMAs issued
        asm volatile("" ::"f"(keep));
        const long long t3 = clk();
        tm[1] += t1 - t0;
        tm[2] += t2 - t1;
        tm[3] += t3 - t2;
    }
}

// bf16 baseline: one 32-token quarter of a raw bf16 record, [K 8 KB][V 8 KB]
// already in A-fragment order (layout.h) -> one LDS.128 per MMA, no dequant.
__device__ __forceinline__ void process_quarter_bf16(const uint8_t *__restrict__ sb, WarpState &st,
                                                     const uint32_t (&qf)[8][2], int lane, float c0) {
    const int gq = lane >> 2, tq = lane & 3;
    const uint4 *K = reinterpret_cast<const uint4 *>(sb);
    const uint4 *V = reinterpret_cast<const uint4 *>(sb + BF16_QUARTER_BYTES / 2);
    float sacc[2][4];
#pragma unroll
    for (int i = 0; i < 2; ++i) sacc[i][0] = sacc[i][1] = sacc[i][2] = sacc[i][3] = 0.f;
#pragma unroll
    for (int s = 0; s < 8; ++s) {
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            const uint4 a = K[(i * 8 + s) * 32 + lane];
            mma16816_bf16(sacc[i], a.x, a.y, a.z, a.w, qf[s][0], qf[s][1]);
        }
    }
    float bm0 = -CUDART_INF_F, bm1 = -CUDART_INF_F;
#pragma unroll
    for (int i = 0; i < 2; ++i) {
#pragma unroll
        for (int e = 0; e < 4; ++e) sacc[i][e] *= c0;
        bm0 = fmaxf(bm0, fmaxf(sacc[i][0], sacc[i][2]));
        bm1 = fmaxf(bm1, fmaxf(sacc[i][1], sacc[i][3]));
    }
#pragma unroll
    for (int o = 4; o < 32; o <<= 1) {
        bm0 = fmaxf(bm0, __shfl_xor_sync(0xffffffffu, bm0, o));
        bm1 = fmaxf(bm1, __shfl_xor_sync(0xffffffffu, bm1, o));
    }
    const float mn0 = fmaxf(st.m[0], bm0), mn1 = fmaxf(st.m[1], bm1);
    const float al0 = fast_exp2(st.m[0] - mn0), al1 = fast_exp2(st.m[1] - mn1);
    st.m[0] = mn0;
    st.m[1] = mn1;
    float ls0 = 0.f, ls1 = 0.f;
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        sacc[i][0] = fast_exp2(sacc[i][0] - mn0);
        sacc[i][1] = fast_exp2(sacc[i][1] - mn1);
        sacc[i][2] = fast_exp2(sacc[i][2] - mn0);
        sacc[i][3] = fast_exp2(sacc[i][3] - mn1);
        ls0 += sacc[i][0] + sacc[i][2];
        ls1 += sacc[i][1] + sacc[i][3];
    }
    st.l[0] = st.l[0] * al0 + ls0;
    st.l[1] = st.l[1] * al1 + ls1;
#pragma unroll
    for (int mm = 0; mm < 8; ++mm) {
        st.o[mm][0] *= al0;
        st.o[mm][1] *= al1;
        st.o[mm][2] *= al0;
        st.o[mm][3] *= al1;
    }
    const int srcA = 4 * tq + (gq >> 1), srcB = 4 * (tq + 4) + (gq >> 1);
    const bool odd = (gq & 1) != 0;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
        const uint32_t H0 = pack_bf162(sacc[j][0], sacc[j][2]);
        const uint32_t H1 = pack_bf162(sacc[j][1], sacc[j][3]);
        const uint32_t x0 = __shfl_sync(0xffffffffu, H0, srcA);
        const uint32_t x1 = __shfl_sync(0xffffffffu, H1, srcA);
        const uint32_t y0 = __shfl_sync(0xffffffffu, H0, srcB);
        const uint32_t y1 = __shfl_sync(0xffffffffu, H1, srcB);
        const uint32_t bp0 = odd ? x1 : x0, bp1 = odd ? y1 : y0;
#pragma unroll
        for (int mm = 0; mm < 8; ++mm) {
            const uint4 a = V[(j * 8 + mm) * 32 + lane];
            mma16816_bf16(st.o[mm], a.x, a.y, a.z, a.w, bp0, bp1);
        }
    }
}

// Rotated (fp16) / raw (bf16 baseline) q tiles of segments [k0, k1) of this
// CTA's range (k1 - k0 <= QSEG), built cooperatively by warps 0..NCW-2 (the
// last warp issues the ring fill): item (segment k, head row j) -> warp
// item % (NCW-1); tile (k % QSEG) row j, rows j >= g zero-filled.  A warp
// first issues the loads of all its items, then rotates them (one memory
// round trip per warp, not per item).  `gate`: the first wave of a launch whose
// ring fill was not issued ahead of griddepcontrol.wait -- every warp meets at
// named barrier 1 once its q loads are in flight, and only then does the fill
// warp queue the NST bulk copies (tens of MB over the GPU), so the q loads are
// not stuck behind them in the memory system.  Each segment's rotation runs
// once per CTA instead of once per warp.
template <int BITS, int NCW>
__device__ __forceinline__ void build_q_tiles(const AttnArgs &a, __half *tiles, int64_t seg_first, int k0, int k1,
                                              int warp, int lane, bool gate) {
    constexpr int QW = NCW - 1;                  // item warps
    constexpr int MAXI = (QSEG * 8 + QW - 1) / QW;  // items per warp
    const int g = a.g;
    uint2 u[MAXI];
    int row_of[MAXI];  // tile row of item i (-1: none)
#pragma unroll
    for (int i = 0; i < MAXI; ++i) {
        const int item = k0 * 8 + warp + i * QW;
        row_of[i] = (warp < QW && item < k1 * 8) ? ((item >> 3) % QSEG) * 8 + (item & 7) : -1;
        u[i] = make_uint2(0u, 0u);
        if (row_of[i] >= 0 && (item & 7) < g) {
            const int bh = (int)seg_first + (item >> 3);
            u[i] = *(reinterpret_cast<const uint2 *>(reinterpret_cast<const __nv_bfloat16 *>(a.q) +
                                                     ((int64_t)(bh / a.Hkv) * a.Hq + (bh % a.Hkv) * g + (item & 7)) * D) +
                     lane);
        }
    }
    if (gate) named_bar(1, NCW * 32);
#pragma unroll
    for (int i = 0; i < MAXI; ++i) {
        if (row_of[i] < 0) continue;
        uint2 *row = reinterpret_cast<uint2 *>(tiles + row_of[i] * QH_STRIDE) + lane;
        if ((row_of[i] & 7) >= g || BITS == 0) {  // padding rows; the bf16 baseline attends raw q
            *row = u[i];
            continue;
        }
        float x[4];
        x[0] = __uint_as_float(u[i].x << 16);
        x[1] = __uint_as_float(u[i].x & 0xffff0000u);
        x[2] = __uint_as_float(u[i].y << 16);
        x[3] = __uint_as_float(u[i].y & 0xffff0000u);
        if (a.rotates) fht128_warp(x, lane);
        *row = make_uint2(pack_half2(x[0], x[1]), pack_half2(x[2], x[3]));
    }
}

// One 16-token tile [t0, t0+16) of the residual window (+ the current token at
// index r) for one (b, kv head), merged into the warp's partial slot.
//   QK^T: D[token, head] = sum_c K[token, c] q[head, c]    A = K rows (ring, row-major)
//   P.V : D[chan, head]  = sum_t V^T[chan, t] P[head, t]   A = V^T rows (ring, tile-major)
// Invalid tokens (>= ntok) get -inf logits and zero V; the ring is read
// through L2 (written by the previous steps).
struct ResidualRefs {
    const uint16_t *ringk, *ringv;  // this (b, kv head)'s rings
    const uint16_t *kc, *vc;        // current token or null
    int g, r, rotate_v;
    int f16;  // rings hold fp16 (fp64-form caches; no current token): fp16 MMAs, q converted
};

// The tile's partial in registers: o in the packed partial's fragment layout
// (rows gq / gq+8 of m-tile mm = channels 16mm+gq / +8, cols 2tq / 2tq+1 =
// heads), m / l per head column in log2 units.
struct ResPartial {
    float o[8][4];
    float m0, m1, l0, l1;
};

__device__ __forceinline__ void residual_compute(const ResidualRefs rr, const __nv_bfloat16 *qbase, int t0,
                                                 int ntok, int lane, float c0, ResPartial &rp) {
    const int gq = lane >> 2, tq = lane & 3;
    const int g = rr.g, r = rr.r;
    const uint16_t *ringk = rr.ringk, *ringv = rr.ringv, *kc = rr.kc, *vc = rr.vc;
    // token rows of this lane's A fragments: t0 + gq, t0 + gq + 8
    const int tA = t0 + gq, tB = tA + 8;
    auto krow = [&](int t) -> const uint16_t * {
        if (t < r) return ringk + (int64_t)t * D;
        if (t < ntok) return kc;  // t == r: the current token
        return nullptr;
    };
    const uint16_t *kA = krow(tA), *kB = krow(tB);
    auto ld32 = [](const uint16_t *p, int c) -> uint32_t {
        return p ? *reinterpret_cast<const uint32_t *>(p + c) : 0u;
    };
    const int u0 = t0 + 2 * tq, u1 = u0 + 8;  // token pairs (u0, u0+1), (u1, u1+1) of this lane
    auto vpair = [&](int c, int u) -> uint32_t {
        uint32_t w = (u + 1 < r) ? *reinterpret_cast<const uint32_t *>(ringv + vring_index(c, u)) : 0u;
        if (u + 1 >= r && u < ntok) {  // tail of the window: per-token select ring / current / zero
            const uint32_t lo = u < r ? ringv[vring_index(c, u)] : (u < ntok ? vc[c] : 0u);
            const uint32_t hi = u + 1 < r ? ringv[vring_index(c, u + 1)] : (u + 1 < ntok ? vc[c] : 0u);
            w = lo | (hi << 16);
        }
        return w;
    };
    // ---- every global load of the tile up front (one L2 round trip): K rows, raw q
    //      (B: lane holds q[head gq][16s + 2tq (+1), +8 (+9)]) and the V^T pairs ----
    const uint16_t *qrow = gq < g ? reinterpret_cast<const uint16_t *>(qbase) + gq * D : nullptr;
    uint32_t kf[8][4], qb[8][2], vf[8][4];
#pragma unroll
    for (int s = 0; s < 8; ++s) {
        const int c = 16 * s + 2 * tq;
        kf[s][0] = ld32(kA, c);
        kf[s][1] = ld32(kB, c);
        kf[s][2] = ld32(kA, c + 8);
        kf[s][3] = ld32(kB, c + 8);
        qb[s][0] = ld32(qrow, c);
        qb[s][1] = ld32(qrow, c + 8);
    }
    if (rr.f16) {  // the bf16 query pairs as fp16 (exact within fp16's range)
#pragma unroll
        for (int s = 0; s < 8; ++s)
#pragma unroll
            for (int e = 0; e < 2; ++e)
                qb[s][e] = pack_half2(__uint_as_float(qb[s][e] << 16), __uint_as_float(qb[s][e] & 0xffff0000u));
    }
#pragma unroll
    for (int mm = 0; mm < 8; ++mm) {
        const int cA = 16 * mm + gq, cB = cA + 8;
        vf[mm][0] = vpair(cA, u0);
        vf[mm][1] = vpair(cB, u0);
        vf[mm][2] = vpair(cA, u1);
        vf[mm][3] = vpair(cB, u1);
    }
    // ---- QK^T ----
    float sacc[4] = {0.f, 0.f, 0.f, 0.f};
    if (rr.f16) {
#pragma unroll
        for (int s = 0; s < 8; ++s) mma16816(sacc, kf[s][0], kf[s][1], kf[s][2], kf[s][3], qb[s][0], qb[s][1]);
    } else {
#pragma unroll
        for (int s = 0; s < 8; ++s) mma16816_bf16(sacc, kf[s][0], kf[s][1], kf[s][2], kf[s][3], qb[s][0], qb[s][1]);
    }
    // logits in log2 units; rows gq / gq+8 = tokens tA / tB; cols 2tq, 2tq+1 = heads
    const bool vA = tA < ntok, vB = tB < ntok;
    sacc[0] = vA ? sacc[0] * c0 : -CUDART_INF_F;
    sacc[1] = vA ? sacc[1] * c0 : -CUDART_INF_F;
    sacc[2] = vB ? sacc[2] * c0 : -CUDART_INF_F;
    sacc[3] = vB ? sacc[3] * c0 : -CUDART_INF_F;
    float m0 = fmaxf(sacc[0], sacc[2]), m1 = fmaxf(sacc[1], sacc[3]);
#pragma unroll
    for (int o = 4; o < 32; o <<= 1) {
        m0 = fmaxf(m0, __shfl_xor_sync(0xffffffffu, m0, o));
        m1 = fmaxf(m1, __shfl_xor_sync(0xffffffffu, m1, o));
    }
    sacc[0] = fast_exp2(sacc[0] - m0);
    sacc[1] = fast_exp2(sacc[1] - m1);
    sacc[2] = fast_exp2(sacc[2] - m0);
    sacc[3] = fast_exp2(sacc[3] - m1);
    float l0 = sacc[0] + sacc[2], l1 = sacc[1] + sacc[3];
#pragma unroll
    for (int o = 4; o < 32; o <<= 1) {
        l0 += __shfl_xor_sync(0xffffffffu, l0, o);
        l1 += __shfl_xor_sync(0xffffffffu, l1, o);
    }
    // ---- P as the B operand: lane (gq, tq) needs P[head gq][tokens 2tq, 2tq+1, 2tq+8, 2tq+9],
    //      held by lanes (2tq, gq/2) and (2tq+1, gq/2) in accumulator layout ----
    const uint32_t X = rr.f16 ? pack_half2(sacc[0], sacc[1]) : pack_bf162(sacc[0], sacc[1]);
    const uint32_t Y = rr.f16 ? pack_half2(sacc[2], sacc[3]) : pack_bf162(sacc[2], sacc[3]);
    const int sa = (2 * tq) * 4 + (gq >> 1), sbl = (2 * tq + 1) * 4 + (gq >> 1);
    const uint32_t xa = __shfl_sync(0xffffffffu, X, sa), ya = __shfl_sync(0xffffffffu, Y, sa);
    const uint32_t xb = __shfl_sync(0xffffffffu, X, sbl), yb = __shfl_sync(0xffffffffu, Y, sbl);
    const uint32_t sel = (gq & 1) ? 0x7632u : 0x5410u;
    const uint32_t b0 = __byte_perm(xa, xb, sel), b1 = __byte_perm(ya, yb, sel);
    // ---- P.V: A = V^T [16 channels x 16 tokens] ----
#pragma unroll
    for (int mm = 0; mm < 8; ++mm) {
        rp.o[mm][0] = rp.o[mm][1] = rp.o[mm][2] = rp.o[mm][3] = 0.f;
        if (rr.f16) mma16816(rp.o[mm], vf[mm][0], vf[mm][1], vf[mm][2], vf[mm][3], b0, b1);
        else mma16816_bf16(rp.o[mm], vf[mm][0], vf[mm][1], vf[mm][2], vf[mm][3], b0, b1);
    }
    rp.m0 = m0;
    rp.m1 = m1;
    rp.l0 = l0;
    rp.l1 = l1;
}

// merge a tile partial into the warp's slot (read-modify-write); in explicit-V
// mode the packed partial lives in the rotated space, so the raw-V tile
// partial is rotated head by head first
__device__ __forceinline__ void residual_merge(const ResPartial &rp, float *slot, int g, int rotate_v, int lane) {
    const int gq = lane >> 2, tq = lane & 3;
    const float m0 = rp.m0, m1 = rp.m1, l0 = rp.l0, l1 = rp.l1;
    __syncwarp();
    const int h0 = 2 * tq, h1 = h0 + 1;
    const float ms0 = slot[8 * D + h0], ms1 = slot[8 * D + h1];
    const float ls0 = slot[8 * D + 8 + h0], ls1 = slot[8 * D + 8 + h1];
    const float M0 = fmaxf(ms0, m0), M1 = fmaxf(ms1, m1);
    const float fs0 = (ms0 == -CUDART_INF_F) ? 0.f : fast_exp2(ms0 - M0);
    const float fs1 = (ms1 == -CUDART_INF_F) ? 0.f : fast_exp2(ms1 - M1);
    const float fr0 = fast_exp2(m0 - M0), fr1 = fast_exp2(m1 - M1);
    // (rows of padding heads, h >= g, are neither written by the warp partial nor read)
    if (!rotate_v && h0 < g) {
#pragma unroll
        for (int mm = 0; mm < 8; ++mm) {
            const int cA = 16 * mm + gq, cB = cA + 8;
            slot[h0 * D + cA] = slot[h0 * D + cA] * fs0 + rp.o[mm][0] * fr0;
            slot[h1 * D + cA] = slot[h1 * D + cA] * fs1 + rp.o[mm][1] * fr1;
            slot[h0 * D + cB] = slot[h0 * D + cB] * fs0 + rp.o[mm][2] * fr0;
            slot[h1 * D + cB] = slot[h1 * D + cB] * fs1 + rp.o[mm][3] * fr1;
        }
    }
    // rotate_v: rescale the packed partial, then add the rotated residual partial head by head
    float *part = slot + 8 * D + 16;  // 128 floats of scratch reserved after m/l
#pragma unroll
    for (int mm = 0; mm < 8 && rotate_v && h0 < g; ++mm) {
        const int cA = 16 * mm + gq, cB = cA + 8;
        slot[h0 * D + cA] *= fs0;
        slot[h1 * D + cA] *= fs1;
        slot[h0 * D + cB] *= fs0;
        slot[h1 * D + cB] *= fs1;
    }
    for (int h = 0; h < g && rotate_v; ++h) {
        __syncwarp();
        if ((h >> 1) == tq) {
            const bool e = (h & 1) != 0;
            const float f = e ? fr1 : fr0;
#pragma unroll
            for (int mm = 0; mm < 8; ++mm) {
                part[16 * mm + gq] = (e ? rp.o[mm][1] : rp.o[mm][0]) * f;
                part[16 * mm + gq + 8] = (e ? rp.o[mm][3] : rp.o[mm][2]) * f;
            }
        }
        __syncwarp();
        float x[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) x[e] = part[4 * lane + e];
        fht128_warp(x, lane);
#pragma unroll
        for (int e = 0; e < 4; ++e) slot[h * D + 4 * lane + e] += x[e];
    }
    __syncwarp();
    if (gq == 0) {
        slot[8 * D + h0] = M0;
        slot[8 * D + h1] = M1;
        slot[8 * D + 8 + h0] = ls0 * fs0 + l0 * fr0;
        slot[8 * D + 8 + h1] = ls1 * fs1 + l1 * fr1;
    }
    __syncwarp();
}

// One 16-token tile [t0, t0+16) of the residual window (+ the current token at
// index r), merged into the warp's partial slot.
// one normalised output row (b, kv head bh's query head h): out / lse, or the
// peer receive areas of a sequence-shard exchange
__device__ __forceinline__ void write_row(const AttnArgs &a, int b, int kvh, int h, const float (&x)[4],
                                          float lse_row, int lane) {
    const int64_t row = (int64_t)b * a.Hq + kvh * a.g + h;
    if (a.pub.world > 0) {
        peer_publish_row(a.pub, a.pub_epoch, row, make_float4(x[0], x[1], x[2], x[3]), lse_row, lane);
    } else {
        *reinterpret_cast<float4 *>(a.out + row * D + lane * 4) = make_float4(x[0], x[1], x[2], x[3]);
        if (a.lse && lane == 0) a.lse[row] = lse_row;
    }
}

constexpr int LL_FB = 8;  // flag-in-word partials merged per batch (the poll path: one batch)

// Poll-mode split-KV final merge of one (b, kv head) head row h: the
// flag-in-word partials in slots [s_begin, expected) are polled until written,
// then cleared to zero for the next launch, and merged on top of a running
// (M, x, Lw) (the merging CTA's own partial; Lw is this lane's share of the
// denominator).  Writes the normalised row (out / lse, or the peer receive areas).
__device__ __forceinline__ void final_merge_ll(const AttnArgs &a, int64_t bh, int h, int s_begin, int expected, float M,
                                            float Lw, float (&x)[4], int lane) {
    uint64_t *pmb = a.part_ml + bh * a.maxp * 16;
    uint64_t *pob = a.part_o + bh * a.maxp * 8 * D;
    constexpr int FB = LL_FB;  // partials per batch: every lane's loads of a batch in flight at once
    uint64_t t0 = 0;
    bool ok = true;
    for (int s0 = s_begin; s0 < expected && ok; s0 += FB) {
        const bool mine = lane < FB && s0 + lane < expected;  // lane u < FB: (m, l) of partial s0 + u
        uint64_t wm = 0, wl = 0;
        uint64_t w[FB][4];
        for (;;) {
            if (mine) ld_volatile_v2_u64(pmb + (s0 + lane) * 16 + 2 * h, wm, wl);
#pragma unroll
            for (int u = 0; u < FB; ++u) {
                if (s0 + u < expected) {
                    const uint64_t *r = pob + (int64_t)(s0 + u) * 8 * D + h * D + lane * 4;
                    ld_volatile_v2_u64(r, w[u][0], w[u][1]);
                    ld_volatile_v2_u64(r + 2, w[u][2], w[u][3]);
                }
            }
            uint32_t f = mine ? (uint32_t)(wm >> 32) & (uint32_t)(wl >> 32) : 1u;
#pragma unroll
            for (int u = 0; u < FB; ++u)
                if (s0 + u < expected)
                    f &= (uint32_t)(w[u][0] >> 32) & (uint32_t)(w[u][1] >> 32) & (uint32_t)(w[u][2] >> 32) &
                         (uint32_t)(w[u][3] >> 32);
            if (__all_sync(0xffffffffu, f == 1u)) break;
            if (t0 == 0) t0 = gtime();
            __nanosleep(64);
            if (gtime() - t0 > 2000000000ull) {  // a partial never arrived: fail loudly, don't hang
                ok = false;
                break;
            }
        }
        if (!ok) break;
        // consumed: back to zero ("not written") for the next launch
        if (mine) st_volatile_v2_u64(pmb + (s0 + lane) * 16 + 2 * h, 0ull, 0ull);
#pragma unroll
        for (int u = 0; u < FB; ++u) {
            if (s0 + u < expected) {
                uint64_t *r = pob + (int64_t)(s0 + u) * 8 * D + h * D + lane * 4;
                st_volatile_v2_u64(r, 0ull, 0ull);
                st_volatile_v2_u64(r + 2, 0ull, 0ull);
            }
        }
        const float ml = mine ? __uint_as_float((uint32_t)wm) : -CUDART_INF_F;
        const float ll = mine ? __uint_as_float((uint32_t)wl) : 0.f;
        float bm = fmaxf(M, ml);
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) bm = fmaxf(bm, __shfl_xor_sync(0xffffffffu, bm, o));
        const float sc = (M == -CUDART_INF_F) ? 0.f : fast_exp2(M - bm);
        const float fl = (ml == -CUDART_INF_F) ? 0.f : fast_exp2(ml - bm);
        Lw = Lw * sc + ll * fl;
#pragma unroll
        for (int e = 0; e < 4; ++e) x[e] *= sc;
#pragma unroll
        for (int u = 0; u < FB; ++u) {
            const float fu = __shfl_sync(0xffffffffu, fl, u);
            if (s0 + u < expected) {
#pragma unroll
                for (int e = 0; e < 4; ++e) x[e] += __uint_as_float((uint32_t)w[u][e]) * fu;
            }
        }
        M = bm;
    }
    const int b = (int)(bh / a.Hkv), kvh = (int)(bh % a.Hkv);
    if (!ok) {
        if (lane == 0 && a.status) atomicOr(a.status, STATUS_MERGE_TIMEOUT);
        float nanrow[4] = {CUDART_NAN_F, CUDART_NAN_F, CUDART_NAN_F, CUDART_NAN_F};
        write_row(a, b, kvh, h, nanrow, CUDART_NAN_F, lane);
        return;
    }
    const float L = warp_sum(Lw);
    const float inv = (L > 0.f) ? 1.f / L : 0.f;
#pragma unroll
    for (int e = 0; e < 4; ++e) x[e] *= inv;
    if (a.rotate_v) fht128_warp(x, lane);  // explicit-V mode: rotate the output back
    write_row(a, b, kvh, h, x, (L > 0.f) ? (M + __log2f(L)) * LN2 : -CUDART_INF_F, lane);
}

// ---- residual-window tiles as pipeline units (the TILES kernel, small launches) ------
// A tile's bytes ride the ring 17 units ahead like the records instead of a dependent
// round trip of their own.  Stage layout of a tile (tokens t0..t0+15 of one (b, kv head)):
//   [0, 4096)      K rows [16][128] bf16 (ring rows t0..r-1; row r = the current token)
//   [4096, 8192)   the ring's V tile [128][16] bf16 (tile-major ring: one 4 KB span)
//   [8192, 8448)   the current token's V row [128] bf16 (when t0 <= r < t0 + 16)
//   [8448, ...)    the raw q rows of the (b, kv head) [g][128] bf16
constexpr int TILE_V_OFF = 4096, TILE_VCUR_OFF = 8192, TILE_Q_OFF = 8448;

__device__ __noinline__ void tile_compute_smem(const uint8_t *__restrict__ sb, int t0, int r, int ntok, int g,
                                               int lane, float c0, ResPartial *out) {
    ResPartial &rp = *out;
    const int gq = lane >> 2, tq = lane & 3;
    const uint16_t *K = reinterpret_cast<const uint16_t *>(sb);
    const uint16_t *V = reinterpret_cast<const uint16_t *>(sb + TILE_V_OFF);
    const uint16_t *VC = reinterpret_cast<const uint16_t *>(sb + TILE_VCUR_OFF);
    const uint16_t *Q = reinterpret_cast<const uint16_t *>(sb + TILE_Q_OFF);
    const int tA = t0 + gq, tB = tA + 8;
    const bool vA = tA < ntok, vB = tB < ntok;
    uint32_t kf[8][4], qb[8][2], vf[8][4];
#pragma unroll
    for (int s = 0; s < 8; ++s) {
        const int c = 16 * s + 2 * tq;
        kf[s][0] = vA ? *reinterpret_cast<const uint32_t *>(K + gq * D + c) : 0u;
        kf[s][1] = vB ? *reinterpret_cast<const uint32_t *>(K + (gq + 8) * D + c) : 0u;
        kf[s][2] = vA ? *reinterpret_cast<const uint32_t *>(K + gq * D + c + 8) : 0u;
        kf[s][3] = vB ? *reinterpret_cast<const uint32_t *>(K + (gq + 8) * D + c + 8) : 0u;
        qb[s][0] = gq < g ? *reinterpret_cast<const uint32_t *>(Q + gq * D + c) : 0u;
        qb[s][1] = gq < g ? *reinterpret_cast<const uint32_t *>(Q + gq * D + c + 8) : 0u;
    }
    const int u0 = 2 * tq, u1 = u0 + 8;  // tile-local token pairs of this lane
    auto vpair = [&](int c, int ul) -> uint32_t {
        const int u = t0 + ul;
        if (u + 1 < r) return *reinterpret_cast<const uint32_t *>(V + c * 16 + ul);
        const uint32_t lo = u < r ? V[c * 16 + ul] : (u < ntok ? VC[c] : 0u);
        const uint32_t hi = u + 1 < r ? V[c * 16 + ul + 1] : (u + 1 < ntok ? VC[c] : 0u);
        return lo | (hi << 16);
    };
#pragma unroll
    for (int mm = 0; mm < 8; ++mm) {
        const int cA = 16 * mm + gq, cB = cA + 8;
        vf[mm][0] = vpair(cA, u0);
        vf[mm][1] = vpair(cB, u0);
        vf[mm][2] = vpair(cA, u1);
        vf[mm][3] = vpair(cB, u1);
    }
    float sacc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int s = 0; s < 8; ++s) mma16816_bf16(sacc, kf[s][0], kf[s][1], kf[s][2], kf[s][3], qb[s][0], qb[s][1]);
    sacc[0] = vA ? sacc[0] * c0 : -CUDART_INF_F;
    sacc[1] = vA ? sacc[1] * c0 : -CUDART_INF_F;
    sacc[2] = vB ? sacc[2] * c0 : -CUDART_INF_F;
    sacc[3] = vB ? sacc[3] * c0 : -CUDART_INF_F;
    float m0 = fmaxf(sacc[0], sacc[2]), m1 = fmaxf(sacc[1], sacc[3]);
#pragma unroll
    for (int o = 4; o < 32; o <<= 1) {
        m0 = fmaxf(m0, __shfl_xor_sync(0xffffffffu, m0, o));
        m1 = fmaxf(m1, __shfl_xor_sync(0xffffffffu, m1, o));
    }
    sacc[0] = fast_exp2(sacc[0] - m0);  // (a tile holds >= 1 valid token: m0, m1 finite)
    sacc[1] = fast_exp2(sacc[1] - m1);
    sacc[2] = fast_exp2(sacc[2] - m0);
    sacc[3] = fast_exp2(sacc[3] - m1);
    float l0 = sacc[0] + sacc[2], l1 = sacc[1] + sacc[3];
#pragma unroll
    for (int o = 4; o < 32; o <<= 1) {
        l0 += __shfl_xor_sync(0xffffffffu, l0, o);
        l1 += __shfl_xor_sync(0xffffffffu, l1, o);
    }
    const uint32_t X = pack_bf162(sacc[0], sacc[1]);
    const uint32_t Y = pack_bf162(sacc[2], sacc[3]);
    const int sa = (2 * tq) * 4 + (gq >> 1), sbl = (2 * tq + 1) * 4 + (gq >> 1);
    const uint32_t xa = __shfl_sync(0xffffffffu, X, sa), ya = __shfl_sync(0xffffffffu, Y, sa);
    const uint32_t xb = __shfl_sync(0xffffffffu, X, sbl), yb = __shfl_sync(0xffffffffu, Y, sbl);
    const uint32_t sel = (gq & 1) ? 0x7632u : 0x5410u;
    const uint32_t b0 = __byte_perm(xa, xb, sel), b1 = __byte_perm(ya, yb, sel);
#pragma unroll
    for (int mm = 0; mm < 8; ++mm) {
        rp.o[mm][0] = rp.o[mm][1] = rp.o[mm][2] = rp.o[mm][3] = 0.f;
        mma16816_bf16(rp.o[mm], vf[mm][0], vf[mm][1], vf[mm][2], vf[mm][3], b0, b1);
    }
    rp.m0 = m0;
    rp.m1 = m1;
    rp.l0 = l0;
    rp.l1 = l1;
}

// online-softmax merge of a tile partial (natural units) into the warp's running
// packed-domain state: o per m-tile in code-field scale units, the denominator in
// the value-offset MMA's ones row (lanes gq == 4)
template <int BITS>
__device__ __forceinline__ void merge_tile(const ResPartial &rp, WarpState &st, int lane) {
    const int gq = lane >> 2;
    constexpr int TPW = 16 / BITS;
    constexpr int HALFT = TPW / 2;
    const float M0 = fmaxf(st.m[0], rp.m0), M1 = fmaxf(st.m[1], rp.m1);
    const float as0 = st.m[0] == -CUDART_INF_F ? 0.f : fast_exp2(st.m[0] - M0);
    const float as1 = st.m[1] == -CUDART_INF_F ? 0.f : fast_exp2(st.m[1] - M1);
    const float ar0 = fast_exp2(rp.m0 - M0), ar1 = fast_exp2(rp.m1 - M1);
#pragma unroll
    for (int mm = 0; mm < 8; ++mm) {
        const int fs = (mm % TPW) % HALFT;
        const float isc = __int_as_float((127 - 24 + BITS * fs) << 23);
        st.o[mm][0] = st.o[mm][0] * as0 + rp.o[mm][0] * (isc * ar0);
        st.o[mm][1] = st.o[mm][1] * as1 + rp.o[mm][1] * (isc * ar1);
        st.o[mm][2] = st.o[mm][2] * as0 + rp.o[mm][2] * (isc * ar0);
        st.o[mm][3] = st.o[mm][3] * as1 + rp.o[mm][3] * (isc * ar1);
    }
    st.ob[0] *= as0;
    st.ob[1] *= as1;
    st.ob2[2] *= as0;
    st.ob2[3] *= as1;
    if (gq == 4) {
        st.ob[0] += rp.l0 * ar0;
        st.ob[1] += rp.l1 * ar1;
    }
    st.m[0] = M0;
    st.m[1] = M1;
}

__device__ __noinline__ void residual_tile(const ResidualRefs rr, float *slot, const __nv_bfloat16 *qbase, int t0,
                                           int ntok, int lane, float c0, uint16_t *ring_k_w, uint16_t *ring_v_w) {
    ResPartial rp;
    residual_compute(rr, qbase, t0, ntok, lane, c0, rp);
    residual_merge(rp, slot, rr.g, rr.rotate_v, lane);
    // the tile holding the current token (index r) also appends it to the rings at
    // slot r: nothing in this launch reads that slot (tiles take it from kcur)
    if (ring_k_w && rr.kc && t0 <= rr.r && rr.r < t0 + 16) {
        reinterpret_cast<uint2 *>(ring_k_w + rr.r * D)[lane] = reinterpret_cast<const uint2 *>(rr.kc)[lane];
        const uint2 vv = reinterpret_cast<const uint2 *>(rr.vc)[lane];  // V ring is tile-major (vring_index)
        ring_v_w[vring_index(4 * lane + 0, rr.r)] = (uint16_t)(vv.x & 0xffffu);
        ring_v_w[vring_index(4 * lane + 1, rr.r)] = (uint16_t)(vv.x >> 16);
        ring_v_w[vring_index(4 * lane + 2, rr.r)] = (uint16_t)(vv.y & 0xffffu);
        ring_v_w[vring_index(4 * lane + 3, rr.r)] = (uint16_t)(vv.y >> 16);
    }
}

// The tile as the warp's INITIAL partial of its segment (computed before the
// packed units, while the CTA's ring fills -- its L2 round trip then costs no
// streaming time): the partial is returned, the current token written to the rings.
__device__ __noinline__ void residual_tile_first(const ResidualRefs rr, const __nv_bfloat16 *qbase, int t0, int ntok,
                                                 int lane, float c0, uint16_t *ring_k_w, uint16_t *ring_v_w,
                                                 ResPartial *out) {
    ResPartial rp;
    residual_compute(rr, qbase, t0, ntok, lane, c0, rp);
    *out = rp;
    if (ring_k_w && rr.kc && t0 <= rr.r && rr.r < t0 + 16) {
        reinterpret_cast<uint2 *>(ring_k_w + rr.r * D)[lane] = reinterpret_cast<const uint2 *>(rr.kc)[lane];
        const uint2 vv = reinterpret_cast<const uint2 *>(rr.vc)[lane];  // V ring is tile-major (vring_index)
        ring_v_w[vring_index(4 * lane + 0, rr.r)] = (uint16_t)(vv.x & 0xffffu);
        ring_v_w[vring_index(4 * lane + 1, rr.r)] = (uint16_t)(vv.x >> 16);
        ring_v_w[vring_index(4 * lane + 2, rr.r)] = (uint16_t)(vv.y & 0xffffu);
        ring_v_w[vring_index(4 * lane + 3, rr.r)] = (uint16_t)(vv.y >> 16);
    }
}

// DEFER: the tiles of a CTA's tail segments after its first run once the packed
// units are done (launches where a CTA spans many (b, kv head) segments)
template <int BITS, int NCW_, bool DEFER, bool TILES = false>
__global__ void __launch_bounds__(NCW_ * 32, 1) decode_attn_kernel(const AttnArgs a) {
    using C = AttnCfg<BITS, NCW_, TILES>;
    constexpr int NCW = C::NCW;
    constexpr int SUB = C::SUB;
    extern __shared__ __align__(1024) uint8_t smem[];
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + C::BAR_OFF);
    int *consumed = reinterpret_cast<int *>(smem + C::CNT_OFF);
    uint8_t *ring = smem + C::RING_OFF;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int gq = lane >> 2, tq = lane & 3;
    // (cta_perm: experiments -- which stream-K range a block takes; the scratch and
    //  partial indexing follow the range, so any permutation is consistent)
    const int cta = a.cta_perm ? (int)((blockIdx.x * (unsigned)a.cta_perm) % (unsigned)a.ncta) : (int)blockIdx.x;
    const int g = a.g;
    const int64_t nb = a.nb * SUB;  // pipeline units per (b, kv head)
    const int64_t total = (int64_t)a.BH * nb;
    int64_t start = 0, end = 0;
    const Split sp{nb, a.BH, a.ncta, a.seg_cost, a.tail_cost};
    if (total > 0) {
        start = sp.begin(cta);
        end = sp.end(cta);
    }
    const int64_t nunits = end - start;
    const uint64_t pol = l2_evict_first_policy();
    // Shared ring, any number of warps: unit p of this CTA's range lives in
    // stage p % NST, round p / NST.  Its consumer (warp p % NCW) first waits
    // until the stage's previous round is consumed (software counter) -- which
    // also means the TMA for unit p was issued, so the full-barrier wait is on
    // the right phase -- and after consuming refills the stage with unit p+NST.
    const int nb32 = (int)nb;  // units per (b, kv head) fit 32 bits
    const uint32_t consumed_s = smem_u32(consumed), full_s = smem_u32(full);
    auto issue_stage = [&](int stg, int64_t bh, int uidx) {  // uidx: unit index within bh
        mbar_arrive_expect_tx(&full[stg], C::STAGE);
        bulk_g2s(ring + stg * C::STAGE,
                 a.blocks + (bh * a.max_blocks + uidx / SUB) * (int64_t)C::BYTES + (uidx % SUB) * C::STAGE, C::STAGE,
                 &full[stg], pol);
    };
    auto issue = [&](int64_t p, int64_t bh, int uidx) { issue_stage((int)p % C::NST, bh, uidx); };
    // ---- TILES kernel: the pipeline positions are the range's packed units and, after
    //      the last unit of every (b, kv head) whose tail this CTA owns, its window tiles ----
    const bool tmode = TILES && total > 0;
    const int ntu = tmode ? ((a.r + (a.kcur ? 1 : 0) + 15) >> 4) : 0;  // tiles per owned tail
    int P32 = (int)nunits;
    if (TILES && ntu > 0 && nunits > 0) {
        const int64_t sf = start / nb, sl = (end - 1) / nb;
        P32 += (int)((sl - sf) + (end == (sl + 1) * nb ? 1 : 0)) * ntu;
    }
    auto seg_np = [&](int64_t bh) -> int {  // packed units of bh in this CTA's range
        const int64_t l0 = bh * nb > start ? bh * nb : start, h0 = (bh + 1) * nb < end ? (bh + 1) * nb : end;
        return (int)(h0 - l0);
    };
    auto seg_len = [&](int64_t bh, int np) -> int { return np + ((bh + 1) * nb <= end ? ntu : 0); };
    // a window tile (tokens 16j..16j+15 of bh): K rows, the V tile, the current token
    // (K row into its slot, V row apart), the raw q rows -- all bulk copies
    auto issue_tile = [&](int stg, int64_t bh, int j) {
        const int t0 = 16 * j, r = a.r;
        const int64_t b = bh / a.Hkv, kvh = bh % a.Hkv;
        const bool cur = a.kcur != nullptr && r >= t0 && r < t0 + 16;
        const int nk = r - t0 < 0 ? 0 : (r - t0 > 16 ? 16 : r - t0);
        uint8_t *dst = ring + stg * C::STAGE;
        mbar_arrive_expect_tx(&full[stg], (uint32_t)(nk * 256 + 4096 + (cur ? 512 : 0) + g * 256));
        const uint8_t *rk = reinterpret_cast<const uint8_t *>(a.ring_k) + (bh * R + t0) * (int64_t)(D * 2);
        const uint8_t *rv = reinterpret_cast<const uint8_t *>(a.ring_v) + (bh * R + t0) * (int64_t)(D * 2);
        if (nk > 0) bulk_g2s(dst, rk, (uint32_t)(nk * 256), &full[stg], pol);
        bulk_g2s(dst + TILE_V_OFF, rv, 4096u, &full[stg], pol);
        if (cur) {
            const int64_t cb = (b * a.Hkv + kvh) * (int64_t)(D * 2);
            bulk_g2s(dst + (r - t0) * 256, reinterpret_cast<const uint8_t *>(a.kcur) + cb, 256u, &full[stg], pol);
            bulk_g2s(dst + TILE_VCUR_OFF, reinterpret_cast<const uint8_t *>(a.vcur) + cb, 256u, &full[stg], pol);
        }
        bulk_g2s(dst + TILE_Q_OFF, reinterpret_cast<const uint8_t *>(a.q) + (b * a.Hq + kvh * g) * (int64_t)(D * 2),
                 (uint32_t)(g * 256), &full[stg], pol);
    };
    // position pos of a walked segment (bh, ps = its first position, np packed units):
    // pass 0: packed units only (may run ahead of griddepcontrol.wait), 1: tiles only, 2: both
    auto issue_at = [&](int stg, int64_t bh, int ps, int np, int pos, int pass) {
        const int off = pos - ps;
        if (off < np) {
            if (pass != 1) issue_stage(stg, bh, (int)((bh * nb > start ? bh * nb : start) - bh * nb) + off);
        } else if (pass != 0) {
            issue_tile(stg, bh, off - np);
        }
    };

    // Programmatic dependent launch: the next decode step's CTAs may start as
    // this grid's CTAs retire; each new CTA streams its first NST packed
    // records into shared memory BEFORE waiting on this grid (the packed
    // blocks are written only by the quantize kernel, and the host clears
    // pdl_prefetch after a flush), then waits for the previous grid's
    // completion + memory flush before touching q, the current token, the
    // residual ring or any scratch the previous grid wrote.
    const unsigned long long g_entry = kProf ? gtime() : 0;
    unsigned long long g_t0 = 0, g_t1 = 0, g_dep = 0, g_qb = 0;  // profiling: TMA issue start/end, dep wait, q built
    griddep_launch_dependents();
    // the ring fill: the first NST units of the range, issued by lane 0 of the last warp
    const bool fill_thread = threadIdx.x == (NCW - 1) * 32;
    auto fill = [&](int pass) {
        if constexpr (TILES) {
            if (nunits > 0) {
                int64_t bh = start / nb;
                int ps = 0, np = seg_np(bh), len = seg_len(bh, np);
                for (int p = 0; p < P32 && p < C::NST; ++p) {
                    while (p >= ps + len) {
                        ps += len;
                        ++bh;
                        np = seg_np(bh);
                        len = seg_len(bh, np);
                    }
                    issue_at(p, bh, ps, np, p, pass);
                }
            }
        } else {
            (void)pass;
            if (nunits > 0) {
                int64_t bh = start / nb, uidx = start % nb;
                for (int64_t p = 0; p < nunits && p < C::NST; ++p) {
                    issue(p, bh, uidx);
                    if (++uidx == nb) {
                        uidx = 0;
                        ++bh;
                    }
                }
            }
        }
        if (kProf) g_t1 = gtime();
    };
    if (fill_thread) {
        for (int i = 0; i < C::NST; ++i) {
            mbar_init(&full[i], 1);
            st_volatile_shared(&consumed[i], 0);
        }
        fence_mbar_init();
        if (kProf) g_t0 = gtime();
        if (a.pdl_prefetch) fill(0);  // (packed records: independent of the previous grid)
    }
    griddep_wait();
    if (kProf) g_dep = gtime();
    if constexpr (TILES) {
        if (fill_thread && a.pdl_prefetch && ntu > 0) fill(1);  // the tiles read the ring, q, the current token
    }
    // segments: residual-only mode (nb == 0): CTA c <-> bh c
    const bool active = total > 0 ? nunits > 0 : cta < a.BH;
    const int64_t seg_first = !active ? 0 : (total > 0 ? start / nb : cta);
    const int64_t seg_last = !active ? -1 : (total > 0 ? (end - 1) / nb : cta);
    const int nseg_all = (int)(seg_last - seg_first + 1);
    __half *qtiles = reinterpret_cast<__half *>(smem + C::QH_OFF);  // QSEG segment tiles of 8 x QH_STRIDE
    const bool gate = !a.pdl_prefetch;
    build_q_tiles<BITS, NCW>(a, qtiles, seg_first, 0, nseg_all < QSEG ? nseg_all : QSEG, warp, lane, gate);
    if (kProf) g_qb = gtime();
    if (fill_thread && !a.pdl_prefetch) fill(2);  // after every warp's q loads are in flight
    __syncthreads();  // barrier init + first wave of q tiles visible
    if (!active) return;
    const unsigned long long g_ready = kProf ? gtime() : 0;
    const float c0 = LOG2E * 0.08838834764831845f;  // log2(e)/sqrt(128)
    long long tmr[12] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
    const long long tk0 = (kProf && a.prof) ? clk() : 0;

    // the stage of warp w's final unit (positions p = w, w + NCW, ... < nunits), free
    // after it is consumed: p + NST >= nunits (NST > NCW), so it is never refilled;
    // a warp with no unit at all (nunits < NCW) takes stage w, which no unit uses
    const bool smem_last = total > 0 && C::NST > NCW;
    const int nu32 = TILES ? P32 : (int)nunits;  // pipeline positions
    auto last_seg_slot = [&](int w) -> float * {
        if (smem_last) {
            const int pw = w < nu32 ? nu32 - 1 - ((nu32 - 1 - w) % NCW) : w;
            return reinterpret_cast<float *>(ring + (pw % C::NST) * C::STAGE);
        }
        return a.warp_part + (((int64_t)cta * a.maxseg + (seg_last - seg_first)) * NCW_MAX + w) * MERGE_FLOATS;
    };
    // residual tiles handed out so far (round-robin over warps), starting at the
    // first warp with one unit fewer than warp 0 (units go round-robin from warp 0)
    int rtile_base = (int)(nunits % NCW);
    bool seen_tail = false;
    (void)seen_tail;
    int seg_ps = 0;  // (TILES) first pipeline position of the segment
    int *wk = reinterpret_cast<int *>(smem + C::WALK_OFF) + warp * 4;  // (TILES) refill walker: bh, ps, np, len
    if constexpr (TILES) {
        if (tmode && lane == 0) {
            const int np0 = seg_np(start / nb);
            wk[0] = (int)(start / nb);
            wk[1] = 0;
            wk[2] = np0;
            wk[3] = seg_len(start / nb, np0);
        }
    }
    for (int64_t bh = seg_first; bh <= seg_last; ++bh) {
        const int k = (int)(bh - seg_first);
        const int b = (int)(bh / a.Hkv), kvh = (int)(bh % a.Hkv);
        const int64_t lo = total > 0 ? (bh * nb > start ? bh * nb : start) : 0;
        const int64_t hi = total > 0 ? ((bh + 1) * nb < end ? (bh + 1) * nb : end) : 0;
        const bool owns_tail = total == 0 || hi == (bh + 1) * nb;
        const __nv_bfloat16 *qbase = reinterpret_cast<const __nv_bfloat16 *>(a.q) + ((int64_t)b * a.Hq + kvh * g) * D;

        const long long tq0 = (kProf && a.prof) ? clk() : 0;
        // ---- q fragments from this segment's CTA-shared tile; every QSEG segments
        //      the next wave of tiles is built (all warps walk the same segments) ----
        if (k > 0 && k % QSEG == 0) {
            __syncthreads();
            build_q_tiles<BITS, NCW>(a, qtiles, seg_first, k, (k + QSEG < nseg_all ? k + QSEG : nseg_all), warp, lane,
                                     false);
            __syncthreads();
        }
        const __half *qh = qtiles + (k % QSEG) * 8 * QH_STRIDE;
        uint32_t qf[8][2];
#pragma unroll
        for (int s = 0; s < 8; ++s) {
            qf[s][0] = *reinterpret_cast<const uint32_t *>(qh + gq * QH_STRIDE + 16 * s + 2 * tq);
            qf[s][1] = *reinterpret_cast<const uint32_t *>(qh + gq * QH_STRIDE + 16 * s + 2 * tq + 8);
        }

        WarpState st;
#pragma unroll
        for (int mm = 0; mm < 8; ++mm) st.o[mm][0] = st.o[mm][1] = st.o[mm][2] = st.o[mm][3] = 0.f;
        st.ob[0] = st.ob[1] = st.ob[2] = st.ob[3] = 0.f;
        st.ob2[0] = st.ob2[1] = st.ob2[2] = st.ob2[3] = 0.f;
        st.m[0] = st.m[1] = -CUDART_INF_F;
        st.l[0] = st.l[1] = 0.f;
        if (kProf && a.prof) tmr[6] += clk() - tq0;

        // ---- residual window + current token on the tensor cores (bf16 mma, raw q . raw k:
        //      the key transform is orthonormal up to the stored norm, so attending the raw
        //      bf16 rows IS attend_one over the full-precision residual, pipeline.cpp:152-180):
        //      one 16-token tile per warp of the tail owner (all its loads in one round trip).
        //      The tile runs FIRST and seeds the warp's partial (its latency overlaps the ring
        //      fill); in explicit-V mode (its partial is rotated head by head) and for the
        //      deferred tails it is merged into the slot after the packed units instead ----
        const int ntok_t = a.r + (a.kcur ? 1 : 0);
        const int ntiles_t = (ntok_t + 15) >> 4;
        int tile_j = -1;     // this warp's tile of this segment
        bool tile_late = false;
        if (owns_tail && !tmode) {
            const int j = (warp - rtile_base % NCW + NCW) % NCW;
            rtile_base += ntiles_t;
            bool now = true;
            if constexpr (DEFER) {
                now = !seen_tail;
                seen_tail = true;
            }
            if (now && j < ntiles_t) {
                tile_j = j;
                tile_late = a.rotate_v != 0;
            }
        }
        auto tile_refs = [&]() {
            ResidualRefs rr;
            rr.ringk = reinterpret_cast<const uint16_t *>(a.ring_k) + bh * R * D;
            rr.ringv = reinterpret_cast<const uint16_t *>(a.ring_v) + bh * R * D;
            rr.kc = a.kcur ? reinterpret_cast<const uint16_t *>(a.kcur) + ((int64_t)b * a.Hkv + kvh) * D : nullptr;
            rr.vc = a.vcur ? reinterpret_cast<const uint16_t *>(a.vcur) + ((int64_t)b * a.Hkv + kvh) * D : nullptr;
            rr.g = g;
            rr.r = a.r;
            rr.rotate_v = a.rotate_v;
            rr.f16 = a.ring_f16;
            return rr;
        };
        if (tile_j >= 0 && !tile_late && !OSK_SKIP_TILES) {
            ResPartial rp;
            residual_tile_first(tile_refs(), qbase, tile_j * 16, ntok_t, lane, c0,
                                a.write_ring ? reinterpret_cast<uint16_t *>(a.ring_k) + bh * R * D : nullptr,
                                reinterpret_cast<uint16_t *>(a.ring_v) + bh * R * D, &rp);
            // the tile's partial in the packed accumulators' domain: o per m-tile in units of
            // the code-field scale (exact powers of two), the denominator in the value-offset
            // MMA's ones row (lanes gq == 4) -- or, for the bf16 baseline, st.l on one lane row
            constexpr int TPW_ = BITS == 0 ? 8 : 16 / (BITS == 0 ? 2 : BITS);
            constexpr int HALFT_ = TPW_ / 2;
#pragma unroll
            for (int mm = 0; mm < 8; ++mm) {
                const int fs = (mm % TPW_) % HALFT_;
                const float isc = (BITS == 0) ? 1.f : __int_as_float((127 - 24 + (BITS == 0 ? 0 : BITS) * fs) << 23);
#pragma unroll
                for (int e = 0; e < 4; ++e) st.o[mm][e] = rp.o[mm][e] * isc;
            }
            st.m[0] = rp.m0;
            st.m[1] = rp.m1;
            if constexpr (BITS == 0) {
                if (gq == 0) {
                    st.l[0] = rp.l0;
                    st.l[1] = rp.l1;
                }
            } else {
                if (gq == 4) {
                    st.ob[0] = rp.l0;
                    st.ob[1] = rp.l1;
                }
            }
        }

        // ---- packed units of this segment: positions p = gidx - start, p % NCW == warp ----
        const int plen = (int)(hi - lo) + (tmode && owns_tail ? ntu : 0);  // (TILES) positions of bh
        if (total > 0) {
            // positions are CTA-local (32-bit); stage and round advance incrementally
            const int p0 = TILES ? seg_ps : (int)(lo - start);
            const int u_seg0 = (int)(lo - bh * nb);  // unit index within bh of position p0
            const int first = p0 + ((warp - p0 % NCW) + NCW) % NCW;
            const int pend = p0 + (int)(hi - lo);
            int stg = first % C::NST, round = first / C::NST;
            int p = first;
            for (; p < pend; p += NCW) {
                const long long ts0 = (kProf && a.prof) ? clk() : 0;
                // every lane polls the same word (a broadcast): no divergent region
                while (ld_volatile_shared_u32(consumed_s + 4 * stg) < round) {
                }
                const long long ts1 = (kProf && a.prof) ? clk() : 0;
                mbar_wait_s(full_s + 8 * stg, (uint32_t)(round & 1));
                if (kProf && a.prof) {
                    const long long ts2 = clk();
                    tmr[5] += ts1 - ts0;
                    tmr[0] += ts2 - ts1;
                }
                const uint8_t *sb = ring + stg * C::STAGE;
                if constexpr (BITS == 0) {
                    process_quarter_bf16(sb, st, qf, lane, c0);
                } else {
                    process_block<BITS>(sb, st, qh + gq * QH_STRIDE + 2 * tq, lane, c0, (kProf && a.prof) ? tmr : nullptr);
                }
                // stage consumed: refill it with unit p + NST, then publish the round.
                // No proxy fence: this warp's generic-proxy reads of the stage have all
                // returned (their registers fed the MMAs above) before the bulk copy is
                // issued -- the same consumer-release ordering TMA pipelines rely on.
                __syncwarp();
                if (lane == 0) {
                    if (TILES && p + C::NST < nu32) {
                        // (TILES) position p + NST: a packed unit of bh, or beyond bh the walker
                        const int tp = p + C::NST;
                        if (tp < pend) {
                            issue_stage(stg, bh, u_seg0 + (tp - p0));
                        } else {
                            int wbh = wk[0], wps = wk[1], wnp = wk[2], wlen = wk[3];
                            while (tp >= wps + wlen) {
                                wps += wlen;
                                ++wbh;
                                wnp = seg_np(wbh);
                                wlen = seg_len(wbh, wnp);
                            }
                            wk[0] = wbh;
                            wk[1] = wps;
                            wk[2] = wnp;
                            wk[3] = wlen;
                            issue_at(stg, wbh, wps, wnp, tp, 2);
                        }
                    } else if (p + C::NST < nu32) {
                        int64_t bh2 = bh;
                        int u2 = u_seg0 + (p - p0) + C::NST;  // unit index within bh (32-bit)
                        while (u2 >= nb32) {
                            u2 -= nb32;
                            ++bh2;
                        }
                        issue_stage(stg, bh2, u2);  // unit p + NST lands in the same stage
                    }
                    // no fence needed: a waiter only relies on phase `round` of this
                    // stage being complete, which held before this warp consumed it
                    st_volatile_shared_u32(consumed_s + 4 * stg, round + 1);
                }
                stg += NCW;
                if (stg >= C::NST) {
                    stg -= C::NST;
                    ++round;
                }
            }
            if constexpr (TILES && BITS != 0) {
                // ---- (TILES) the segment's window tiles: positions pend + j, streamed like
                //      the records, computed from shared memory, merged into the partial ----
                for (; p < p0 + plen; p += NCW) {
                    while (ld_volatile_shared_u32(consumed_s + 4 * stg) < round) {
                    }
                    mbar_wait_s(full_s + 8 * stg, (uint32_t)(round & 1));
                    const uint8_t *sb = ring + stg * C::STAGE;
                    const int t0 = 16 * (p - pend), r = a.r;
                    ResPartial rp;
                    tile_compute_smem(sb, t0, r, r + (a.kcur ? 1 : 0), g, lane, c0, &rp);
                    merge_tile<BITS>(rp, st, lane);
                    if (a.write_ring && a.kcur && r >= t0 && r < t0 + 16) {  // append the current token
                        uint16_t *rkw = reinterpret_cast<uint16_t *>(a.ring_k) + (bh * R + r) * D;
                        uint16_t *rvw = reinterpret_cast<uint16_t *>(a.ring_v) + bh * R * D;
                        reinterpret_cast<uint2 *>(rkw)[lane] = reinterpret_cast<const uint2 *>(sb + (r - t0) * 256)[lane];
                        const uint2 vv = reinterpret_cast<const uint2 *>(sb + TILE_VCUR_OFF)[lane];
                        rvw[vring_index(4 * lane + 0, r)] = (uint16_t)(vv.x & 0xffffu);
                        rvw[vring_index(4 * lane + 1, r)] = (uint16_t)(vv.x >> 16);
                        rvw[vring_index(4 * lane + 2, r)] = (uint16_t)(vv.y & 0xffffu);
                        rvw[vring_index(4 * lane + 3, r)] = (uint16_t)(vv.y >> 16);
                    }
                    __syncwarp();
                    if (lane == 0) {
                        const int tp = p + C::NST;
                        if (tp < nu32) {
                            int wbh = wk[0], wps = wk[1], wnp = wk[2], wlen = wk[3];
                            while (tp >= wps + wlen) {
                                wps += wlen;
                                ++wbh;
                                wnp = seg_np(wbh);
                                wlen = seg_len(wbh, wnp);
                            }
                            wk[0] = wbh;
                            wk[1] = wps;
                            wk[2] = wnp;
                            wk[3] = wlen;
                            issue_at(stg, wbh, wps, wnp, tp, 2);
                        }
                        st_volatile_shared_u32(consumed_s + 4 * stg, round + 1);
                    }
                    stg += NCW;
                    if (stg >= C::NST) {
                        stg -= C::NST;
                        ++round;
                    }
                }
            }
        }
        if constexpr (TILES) seg_ps += plen;

        const long long te0 = (kProf && a.prof) ? clk() : 0;
        // ---- warp partial -> slot (unnormalized O[h][c], m[h], l[h]).  For the CTA's
        //      last segment the slot is the warp's last ring stage (shared memory: no
        //      stage is refilled or re-read once its final round is consumed), else
        //      global scratch ----
        float *slot = bh == seg_last ? last_seg_slot(warp)
                                     : a.warp_part + (((int64_t)cta * a.maxseg + k) * NCW_MAX + warp) * MERGE_FLOATS;
        {
            float l0, l1;
            if constexpr (BITS == 0) {
                l0 = st.l[0];
                l1 = st.l[1];
#pragma unroll
                for (int o = 4; o < 32; o <<= 1) {
                    l0 += __shfl_xor_sync(0xffffffffu, l0, o);
                    l1 += __shfl_xor_sync(0xffffffffu, l1, o);
                }
            } else {  // sum_t P: row 4 (even token tiles) + row 12 (odd) of the value-offset MMAs
                l0 = __shfl_sync(0xffffffffu, st.ob[0] + st.ob2[2], 16 + tq);
                l1 = __shfl_sync(0xffffffffu, st.ob[1] + st.ob2[3], 16 + tq);
            }
            float vb0[4], vb1[4];
#pragma unroll
            for (int gc = 0; gc < 4; ++gc) {
                vb0[gc] = __shfl_sync(0xffffffffu, st.ob[0] + st.ob2[2], gc * 4 + tq);
                vb1[gc] = __shfl_sync(0xffffffffu, st.ob[1] + st.ob2[3], gc * 4 + tq);
            }
            constexpr int TPW = BITS == 0 ? 8 : 16 / (BITS == 0 ? 2 : BITS);
            constexpr int HALFT = TPW / 2;
#pragma unroll
            for (int mm = 0; mm < 8; ++mm) {
                const int fs = (mm % TPW) % HALFT;
                const float sc = (BITS == 0) ? 1.f : __int_as_float((127 + 24 - (BITS == 0 ? 0 : BITS) * fs) << 23);
                const int cA = 16 * mm + gq, cB = cA + 8;
                const int h0 = 2 * tq, h1 = 2 * tq + 1;
                const float bb0 = BITS == 0 ? 0.f : vb0[mm >> 1], bb1 = BITS == 0 ? 0.f : vb1[mm >> 1];
                if (h0 < g) {  // rows of padding heads (g < 8) are never read
                    slot[h0 * D + cA] = st.o[mm][0] * sc + bb0;
                    slot[h1 * D + cA] = st.o[mm][1] * sc + bb1;
                    slot[h0 * D + cB] = st.o[mm][2] * sc + bb0;
                    slot[h1 * D + cB] = st.o[mm][3] * sc + bb1;
                }
            }
            if (gq == 0) {
                slot[8 * D + 2 * tq] = st.m[0];
                slot[8 * D + 2 * tq + 1] = st.m[1];
                slot[8 * D + 8 + 2 * tq] = l0;
                slot[8 * D + 8 + 2 * tq + 1] = l1;
            }
            __syncwarp();
        }

        // explicit-V mode: the tile's raw-V partial is rotated into the slot after the units
        if (tile_j >= 0 && tile_late)
            residual_tile(tile_refs(), slot, qbase, tile_j * 16, ntok_t, lane, c0,
                          a.write_ring ? reinterpret_cast<uint16_t *>(a.ring_k) + bh * R * D : nullptr,
                          reinterpret_cast<uint16_t *>(a.ring_v) + bh * R * D);

        if (kProf && a.prof) tmr[7] += clk() - te0;
    }

    if (DEFER && !TILES && !OSK_SKIP_TILES) {  // tiles of the tail segments after the first, after the packed units
        const int ntok = a.r + (a.kcur ? 1 : 0);
        const int ntiles = (ntok + 15) >> 4;
        int rbase = (int)(nunits % NCW);
        bool first_tail = true;
        for (int64_t bh = seg_first; ntiles > 0 && bh <= seg_last; ++bh) {
            const int64_t hi = total > 0 ? ((bh + 1) * nb < end ? (bh + 1) * nb : end) : 0;
            if (!(total == 0 || hi == (bh + 1) * nb)) continue;  // not this CTA's tail
            const int j = (warp - rbase % NCW + NCW) % NCW;
            rbase += ntiles;
            const bool ran = first_tail;
            first_tail = false;
            if (ran || j >= ntiles) continue;
            const int k = (int)(bh - seg_first);
            const int b = (int)(bh / a.Hkv), kvh = (int)(bh % a.Hkv);
            float *slot = bh == seg_last ? last_seg_slot(warp)
                                         : a.warp_part + (((int64_t)cta * a.maxseg + k) * NCW_MAX + warp) * MERGE_FLOATS;
            ResidualRefs rr;
            rr.ringk = reinterpret_cast<const uint16_t *>(a.ring_k) + bh * R * D;
            rr.ringv = reinterpret_cast<const uint16_t *>(a.ring_v) + bh * R * D;
            rr.kc = a.kcur ? reinterpret_cast<const uint16_t *>(a.kcur) + ((int64_t)b * a.Hkv + kvh) * D : nullptr;
            rr.vc = a.vcur ? reinterpret_cast<const uint16_t *>(a.vcur) + ((int64_t)b * a.Hkv + kvh) * D : nullptr;
            rr.g = g;
            rr.r = a.r;
            rr.rotate_v = a.rotate_v;
            rr.f16 = a.ring_f16;
            residual_tile(rr, slot, reinterpret_cast<const __nv_bfloat16 *>(a.q) + ((int64_t)b * a.Hq + kvh * g) * D,
                          j * 16, ntok, lane, c0,
                          a.write_ring ? reinterpret_cast<uint16_t *>(a.ring_k) + bh * R * D : nullptr,
                          reinterpret_cast<uint16_t *>(a.ring_v) + bh * R * D);
        }
    }

    // ======== end of the CTA's work: cooperative merges (all warps finish within
    //          ~one unit of each other under the static round-robin schedule) ========
    const long long tm0 = (kProf && a.prof) ? clk() : 0;
    const unsigned long long g_stream = kProf ? gtime() : 0;
    if (lane == 0) reinterpret_cast<float **>(smem + C::TAB_OFF)[warp] = last_seg_slot(warp);
    __syncthreads();
    const unsigned long long g_sync1 = kProf ? gtime() : 0;
    int *lastflag = reinterpret_cast<int *>(smem + C::SEG_OFF);  // [nseg] (segcnt area reused)
    const int nseg = (int)(seg_last - seg_first + 1);
    const bool poll = a.poll_merge != 0;
    // (1) CTA partial per segment: warp-per-(segment, head), lane = 4-channel chunk.
    //     A split segment is merged one of two ways:
    //     * poll (every CTA resident, <= LL_FB + 1 partials): its FIRST CTA -- which
    //       reaches the segment at the end of its range, the others at the start of
    //       theirs -- merges right here, polling the others' flag-in-word partials
    //       (no fence, no atomic, no second barrier); the others publish and are done;
    //     * ticket: fp32 partials, one acq_rel ticket per CTA and segment, the
    //       last-arriving CTA merges (many partials: 32 loads in flight per batch)
    bool any_ticket = false;
    for (int item = warp; item < nseg * g; item += NCW) {
        const int kk = item / g, h = item % g;
        const int64_t bh = seg_first + kk;
        const float *wp = a.warp_part + ((int64_t)cta * a.maxseg + kk) * NCW_MAX * MERGE_FLOATS;
        const bool lastk = kk == nseg - 1;
        const float *const *tab = reinterpret_cast<const float *const *>(smem + C::TAB_OFF);
        auto src = [&](int w) -> const float * { return lastk ? tab[w] : wp + w * MERGE_FLOATS; };
        // a segment entirely inside this CTA's range: its CTA partial IS the result
        // (no split-KV partial, ticket or final merge)
        const bool single = total == 0 || (bh * nb >= start && (bh + 1) * nb <= end);
        int first_cta = 0, expected = 1;
        if (!single) {
            first_cta = (int)sp.cta_of(bh * nb);
            expected = (int)sp.cta_of((bh + 1) * nb - 1) - first_cta + 1;
        }
        const bool pollseg = poll && expected - 1 <= LL_FB;
        const int pslot = cta - first_cta;
        uint64_t *po = a.part_o + ((int64_t)bh * a.maxp + pslot) * 8 * D;
        uint64_t *pml = a.part_ml + ((int64_t)bh * a.maxp + pslot) * 16;
        // lane w < NCW holds warp w's (m, l) of head h
        const float mwv = lane < NCW ? src(lane)[8 * D + h] : -CUDART_INF_F;
        const float lwv = lane < NCW ? src(lane)[8 * D + 8 + h] : 0.f;
        float4 v[NCW];
#pragma unroll
        for (int w = 0; w < NCW; ++w)  // all loads in flight at once
            v[w] = *reinterpret_cast<const float4 *>(src(w) + h * D + lane * 4);
        float M = mwv;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
        const float fw = (mwv == -CUDART_INF_F) ? 0.f : fast_exp2(mwv - M);
        const float L = warp_sum(lwv * fw);
        float4 O = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int w = 0; w < NCW; ++w) {
            const float f = __shfl_sync(0xffffffffu, fw, w);
            if (f != 0.f) {
                O.x += v[w].x * f;
                O.y += v[w].y * f;
                O.z += v[w].z * f;
                O.w += v[w].w * f;
            }
        }
        if (single) {
            const float inv = (L > 0.f) ? 1.f / L : 0.f;
            float x[4] = {O.x * inv, O.y * inv, O.z * inv, O.w * inv};
            if (a.rotate_v) fht128_warp(x, lane);  // explicit-V mode: rotate the output back
            write_row(a, (int)(bh / a.Hkv), (int)(bh % a.Hkv), h, x, (L > 0.f) ? (M + __log2f(L)) * LN2 : -CUDART_INF_F,
                      lane);
        } else if (pollseg && pslot == 0) {
            float x[4] = {O.x, O.y, O.z, O.w};
            final_merge_ll(a, bh, h, 1, expected, M, lane == 0 ? L : 0.f, x, lane);
        } else if (pollseg) {
            st_volatile_v2_u64(po + h * D + lane * 4, ll_word(O.x, 1u), ll_word(O.y, 1u));
            st_volatile_v2_u64(po + h * D + lane * 4 + 2, ll_word(O.z, 1u), ll_word(O.w, 1u));
            if (lane == 0) st_volatile_v2_u64(pml + 2 * h, ll_word(M, 1u), ll_word(L, 1u));
        } else {  // ticket segment: fp32 partial in the first half of the slot's words
            any_ticket = true;
            reinterpret_cast<float4 *>(po)[h * D / 4 + lane] = O;
            if (lane == 0) {
                reinterpret_cast<float *>(pml)[2 * h] = M;
                reinterpret_cast<float *>(pml)[2 * h + 1] = L;
            }
        }
    }
    const unsigned long long g_phase1 = kProf ? gtime() : 0;
    const bool ticket_phase = __syncthreads_or(any_ticket) != 0;
    const unsigned long long g_sync2 = kProf ? gtime() : 0;
    unsigned long long g_ticket = g_sync2;
    const long long tp0 = (kProf && a.prof) ? clk() : 0;
    const long long tf0 = tp0;
    if (ticket_phase) {
        // (2) publish: one acq_rel ticket per ticket segment (cumulative over the barrier)
        if (threadIdx.x < nseg) {
            const int64_t bh = seg_first + threadIdx.x;
            int flag = 0;
            if (!(total == 0 || (bh * nb >= start && (bh + 1) * nb <= end))) {
                const int expected = (int)(sp.cta_of((bh + 1) * nb - 1) - sp.cta_of(bh * nb) + 1);
                if (!(poll && expected - 1 <= LL_FB)) {
                    const int prev = atomic_add_acq_rel_gpu(&a.counters[bh], 1);
                    flag = (prev == expected - 1) ? expected : 0;
                }
            }
            lastflag[threadIdx.x] = flag;
        }
        __syncthreads();
        if (kProf) g_ticket = gtime();
        // (3) final merge for the ticket segments this CTA completed last: warp-per-(segment, head)
        for (int item = warp; item < nseg * g; item += NCW) {
            const int kk = item / g, h = item % g;
            const int expected = lastflag[kk];
            if (expected == 0) continue;
            const int64_t bh = seg_first + kk;
            const int b = (int)(bh / a.Hkv), kvh = (int)(bh % a.Hkv);
            // one pass, online over batches of FB partials: lane u loads the (m, l) of
            // partial s0 + u, every lane its 4 channels of all FB partials' O rows (all
            // loads in flight at once; registers are free at this point of the kernel).
            // A segment keeps its merge form for the whole launch plan (the host clears
            // the partial words when the plan changes), so fp32 partials left here are
            // never read as flag-in-word ones
            float M = -CUDART_INF_F, Lw = 0.f;  // Lw: this lane's share of the denominator
            float x[4] = {0.f, 0.f, 0.f, 0.f};
            constexpr int FB = OSK_TICKET_FB;
            for (int s0 = 0; s0 < expected; s0 += FB) {
                const bool mine = s0 + lane < expected;
                const float *pm =
                    reinterpret_cast<const float *>(a.part_ml + ((int64_t)bh * a.maxp + s0 + lane) * 16) + 2 * h;
                const float ml = mine ? __ldcg(pm) : -CUDART_INF_F;
                const float ll = mine ? __ldcg(pm + 1) : 0.f;
                float4 v[FB];
#pragma unroll
                for (int u = 0; u < FB; ++u)
                    v[u] = (s0 + u < expected)
                               ? __ldcg(reinterpret_cast<const float4 *>(a.part_o + ((int64_t)bh * a.maxp + s0 + u) * 8 * D) +
                                        h * D / 4 + lane)
                               : make_float4(0.f, 0.f, 0.f, 0.f);
                float bm = fmaxf(M, ml);
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) bm = fmaxf(bm, __shfl_xor_sync(0xffffffffu, bm, o));
                const float sc = (M == -CUDART_INF_F) ? 0.f : fast_exp2(M - bm);
                const float fl = (ml == -CUDART_INF_F) ? 0.f : fast_exp2(ml - bm);
                Lw = Lw * sc + ll * fl;
#pragma unroll
                for (int e = 0; e < 4; ++e) x[e] *= sc;
#pragma unroll
                for (int u = 0; u < FB; ++u) {
                    const float f = __shfl_sync(0xffffffffu, fl, u);
                    x[0] += v[u].x * f;
                    x[1] += v[u].y * f;
                    x[2] += v[u].z * f;
                    x[3] += v[u].w * f;
                }
                M = bm;
            }
            const float L = warp_sum(Lw);
            const float inv = (L > 0.f) ? 1.f / L : 0.f;
#pragma unroll
            for (int e = 0; e < 4; ++e) x[e] *= inv;
            if (a.rotate_v) fht128_warp(x, lane);  // explicit-V mode: rotate the output back
            write_row(a, b, kvh, h, x, (L > 0.f) ? (M + __log2f(L)) * LN2 : -CUDART_INF_F, lane);
            if (h == 0 && lane == 0) a.counters[bh] = 0;  // the ticket is complete: reset for the next launch
        }
    }
    if (kProf && a.prof) {
        tmr[8] += clk() - tm0;
        tmr[9] += clk() - tp0;  // the ticket (atomic) part
    }
    if (kProf && a.prof) tmr[10] += clk() - tf0;
    if (kProf && a.prof) tmr[4] += clk() - tm0;
    if (kProf && a.prof && lane == 0) {
        // per-warp phase cycles: [wait, qk, softmax, pv, merge, spin, qprologue, segtail]; total in slot 4 of the
        // host view is replaced below by the whole-kernel cycles
        // [0..7] wait qk softmax pv merge spin qprologue segtail, [8] total, [9] cta merge,
        // [10] ticket, [11] smid, [12] final merge
        unsigned long long *pp = a.prof + ((int64_t)cta * NCW_MAX + warp) * kProfStride;
        for (int i = 0; i < 8; ++i) pp[i] = (unsigned long long)tmr[i];
        pp[8] = (unsigned long long)(clk() - tk0);
        pp[9] = (unsigned long long)tmr[8];
        pp[10] = (unsigned long long)tmr[9];
        pp[12] = (unsigned long long)tmr[10];
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        pp[11] = smid;
        pp[13] = g_entry;  // globaltimer (ns): kernel entry, end of this warp's streaming, exit
        pp[14] = g_stream;
        pp[15] = gtime();
        pp[16] = g_sync1;  // after the first end-of-work barrier
        pp[17] = g_phase1;  // CTA partials done (this warp)
        pp[18] = g_sync2;
        pp[19] = g_ticket;  // tickets + barrier
        pp[20] = g_ready;   // q tiles built (after the first barrier)
        pp[21] = g_t0;      // thread 0: barriers initialised (0 on other warps)
        pp[22] = g_t1;      // thread 0: first NST bulk copies issued
        pp[23] = g_dep;     // after griddepcontrol.wait
        pp[24] = g_qb;      // this warp's q-tile items done
    }
}

__global__ void lse_merge_kernel(const float *outs, const float *lses, int64_t parts, int64_t rows, int64_t d,
                                 float *out, float *lse_out) {
    const int64_t row = blockIdx.x;
    float M = -CUDART_INF_F;
    for (int64_t p = 0; p < parts; ++p) M = fmaxf(M, lses[p * rows + row]);
    for (int64_t c = threadIdx.x; c < d; c += blockDim.x) {
        float O = 0.f, L = 0.f;
        for (int64_t p = 0; p < parts; ++p) {
            const float l = lses[p * rows + row];
            const float w = (l == -CUDART_INF_F) ? 0.f : __expf(l - M);
            O += outs[(p * rows + row) * d + c] * w;
            L += w;
        }
        out[row * d + c] = L > 0.f ? O / L : 0.f;
        if (lse_out && c == 0) lse_out[row] = L > 0.f ? M + __logf(L) : -CUDART_INF_F;
    }
}

template <int BITS, int NCW, bool DEFER, bool TILES = false>
cudaError_t launch_d(const AttnArgs &a, cudaStream_t st) {
    using C = AttnCfg<BITS, NCW, TILES>;
    static std::atomic<uint64_t> attr_done{0};
    if (cudaError_t e = ensure_smem_attr(decode_attn_kernel<BITS, NCW, DEFER, TILES>, C::SMEM, attr_done);
        e != cudaSuccess)
        return e;
    // programmatic stream serialization: may overlap the previous kernel's tail
    // (the kernel orders its dependent accesses with griddepcontrol.wait)
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)a.ncta);
    cfg.blockDim = dim3(C::NTHREADS);
    cfg.dynamicSmemBytes = C::SMEM;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, decode_attn_kernel<BITS, NCW, DEFER, TILES>, a);
}

// DEFER pays off when CTAs span several (b, kv head) segments (each with its own
// tail): more than two segments per CTA on average
template <int BITS, int NCW>
cudaError_t launch_t(const AttnArgs &a, cudaStream_t st) {
    static const long force = env_knob("OSCAR_DEFER", -1);  // OSCAR_DEFER=0|1 overrides the choice (experiments)
    const bool defer = force >= 0 ? force == 1 : (a.nb > 0 && (int64_t)a.BH > 2 * (int64_t)a.ncta);
    if constexpr (BITS != 0 && NCW == 12)
        if (a.tile_units) return launch_d<BITS, NCW, false, true>(a, st);  // (supersedes DEFER)
    return defer ? launch_d<BITS, NCW, true>(a, st) : launch_d<BITS, NCW, false>(a, st);
}

}  // namespace

static int ncw_choice(int bits);

// persistent grid: one CTA per SM, but never fewer than ~one pipeline unit per
// warp per CTA -- small workloads (few sequences x short contexts) then use
// fewer CTAs and every (b, kv head) has fewer split-KV partials to merge
int attention_grid(int bits, int num_sms, int64_t nb, int BH) {
    const int64_t units = nb * BH * (bits == 0 ? 4 : 1);
    if (units == 0) return BH;
    // small launches: ~2/3 of the warps stream packed units, the rest take the
    // residual-window tiles concurrently
    static const long per_env = env_knob("OSCAR_CTA_UNITS", 0);  // experiments: packed units per CTA
    const int64_t per = per_env > 0 ? per_env : (ncw_choice(bits) * 2) / 3;
    const int64_t want = (units + per - 1) / per;
    int64_t n = want < num_sms ? want : num_sms;
    // small launches (<= 24 units per CTA) over fewer segments than CTAs: a grid of a
    // multiple of the segment count gives every segment the same CTAs and no CTA two
    // segments (one CTA merge, fewer split partials); taken when it costs <= 15 % of the
    // grid (C3 B=8 layer: 148 -> 128 CTAs, 18.6 -> 17.7 us; profiles/r02/ab_cta_grid.txt)
    if (units <= 24 * n && BH < n) {
        const int64_t al = (int64_t)BH * (n / BH);
        if (al * 100 >= n * 85) n = al;
    }
    return (int)n;
}

int64_t attention_scratch_floats(int64_t slots) {
    return slots * NCW_MAX * MERGE_FLOATS;  // per (CTA, segment) slot: one partial per warp
}

// warps per CTA: OSCAR_NCW=8|12 overrides the default (tuning knob)
static int ncw_choice(int bits) {
    static const long env = env_knob("OSCAR_NCW", 0);
    if (env == 8 || env == 12 || env == 16) return env;
    return bits == 4 ? 8 : 12;
}

cudaError_t launch_attention(int bits, const AttnArgs &a, cudaStream_t st) {
    const int ncw = ncw_choice(bits);
    switch (bits) {
        case 2: return ncw == 8 ? launch_t<2, 8>(a, st) : ncw == 16 ? launch_t<2, 16>(a, st) : launch_t<2, 12>(a, st);
        case 4: return ncw == 8 ? launch_t<4, 8>(a, st) : launch_t<4, 12>(a, st);
        case 0: return ncw == 8 ? launch_t<0, 8>(a, st) : launch_t<0, 12>(a, st);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_lse_merge(const float *outs, const float *lses, int64_t parts, int64_t rows, int64_t d, float *out,
                             float *lse_out, cudaStream_t st) {
    if (rows == 0) return cudaSuccess;
    lse_merge_kernel<<<(unsigned)rows, 128, 0, st>>>(outs, lses, parts, rows, d, out, lse_out);
    return cudaGetLastError();
}

}  // namespace osk
