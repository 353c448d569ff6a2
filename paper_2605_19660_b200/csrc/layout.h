// layout.h -- the device cache layout (shared by the quantize kernel, the
// decode-attention kernel and the host-side export).
//
// One R-block (R = 128 tokens) of one (sequence, KV head) is ONE contiguous
// record in HBM, fetched by a single cp.async.bulk into shared memory:
//
//   INT2 record (12800 B)                       INT4 record (20992 B)
//   K part (6656 B):                             K part (10752 B):
//   [K codes  4096 B]  mma A-fragment order      [K codes  8192 B]
//   [K a      1024 B]  fp16 step  per (ch,grp)   ... same params/norms ...
//   [K b      1024 B]  fp16 offset -delta*zp per (ch,grp)
//   [norms     512 B]  fp32 per token
//   V part (6144 B):                             V part (10240 B):
//   [V codes  4096 B]  mma A-fragment order      [V codes  8192 B]
//   [V a      1024 B]  fp16 step  per (tok,gc)
//   [V b      1024 B]  fp16 offset per (tok,gc)
//
// Everything the QK^T half of the attention reads is the contiguous K part,
// everything P.V reads the V part: the kernel streams them into separate
// shared-memory slots and hands each back to the TMA as soon as its half of
// the work is done (more bytes in flight per SM than whole-record stages).
//
// Keys and values both dequantise as x = a*code + b with a = delta and
// b = -delta*zp (a constant group stores a = 0, b = constant; its codes are 0)
// -- the reference's dequantize_one (quant.cpp:65-68) with step and offset
// narrowed to fp16.  The attention kernel folds a into the MMA B operand and
// b into one small MMA per k-step (keys) / token tile (values).
//
// The codes are the reference's codes (bit-identical values) permuted inside
// the block so that every 32-bit word a lane loads IS an mma.m16n8k16 A
// register after one AND: the low half-word carries 8 codes of one (row, k)
// element pair for 8 different m-tiles, the high half the partner k element.
// Masking a 2-bit field at position 2i leaves the fp16 SUBNORMAL code*2^(2i-24)
// (exact; tensor cores keep fp16 subnormals -- measured, scratch/mma_probe.cu),
// whose power-of-two scale is removed per m-tile in the fp32 epilogue.
//
// QK^T:  D[token, head] = sum_c codeK[token, c] * (Qrot[head, c] * aK[c, grp])
//   m-tile i (0..7) = tokens 16i..16i+15 (one quantisation group: grp = i/2),
//   row r -> token 16i + r; k-step s (0..7) = channels 16s..16s+15, k-col kc
//   -> channel 16s + kc.
// P.V:   D[channel, head] = sum_t codeV[t, channel] * (P[head, t] * aV[t, gc])
//   m-tile m (0..7) = channels 16m..16m+15 (gc = m/2), row r -> channel 16m+r;
//   k-step j (0..7) = tokens of QK m-tile j with k-col -> token
//   16j + {tq, tq+8, tq+4, tq+12} for k = {2tq, 2tq+1, 2tq+8, 2tq+9} -- the
//   order that turns the QK accumulator into the PV B operand with two
//   shuffles per register.
//
// export (oscar_kv_export) inverts the permutation back to the reference's
// channel-major K / token-major V code order (kv_cache.cpp:116, 146) and
// pack_2bit words (quant.cpp:162-175).
#pragma once
#include <stdint.h>

#ifdef __CUDACC__
#define OSK_HD __host__ __device__ __forceinline__
#else
#define OSK_HD inline
#endif

namespace osk {

constexpr int D = 128;        // head_dim
constexpr int R = 128;        // residual_len (block)
constexpr int G = 32;         // group_size
constexpr int NGRP = R / G;   // K groups per channel per block (4)
constexpr int NGC = D / G;    // V groups per token (4)

// Residual-window V ring of one (sequence, KV head): tile-major [R/16][D][16] bf16 --
// the 16 tokens of a 16-token tile are contiguous per channel (a token pair is one
// 32-bit word, the P.V A operand), and a whole tile is one contiguous 4 KB span that a
// single bulk copy moves into shared memory.  (The K ring is token-major [R][D].)
OSK_HD int64_t vring_index(int channel, int token) {
    return (int64_t)(token >> 4) * (D * 16) + channel * 16 + (token & 15);
}

template <int BITS>
struct Block {
    static constexpr int CODE_BYTES = R * D * BITS / 8;      // per K or V
    static constexpr int K_OFF = 0;
    static constexpr int KA_OFF = CODE_BYTES;
    static constexpr int KB_OFF = KA_OFF + D * NGRP * 2;
    static constexpr int NORM_OFF = KB_OFF + D * NGRP * 2;
    static constexpr int K_PART = NORM_OFF + R * 4;           // [K codes][K a][K b][norms]
    static constexpr int V_OFF = K_PART;
    static constexpr int VA_OFF = V_OFF + CODE_BYTES;
    static constexpr int VB_OFF = VA_OFF + R * NGC * 2;
    static constexpr int BYTES = VB_OFF + R * NGC * 2;
    static constexpr int V_PART = BYTES - K_PART;              // [V codes][V a][V b]
    // words per lane per k-step (each word = 8/BITS*... m-tiles)
    static constexpr int TILES_PER_WORD = 16 / BITS;          // 8 (int2) / 4 (int4)
    static constexpr int WORDS_PER_LANE_STEP = 4 * 8 / TILES_PER_WORD;  // 4 / 8
};
static_assert(Block<2>::BYTES == 12800, "int2 block size");
static_assert(Block<4>::BYTES == 20992, "int4 block size");
static_assert(Block<2>::K_PART % 128 == 0 && Block<4>::K_PART % 128 == 0, "16-byte aligned parts for bulk copies");
// bits == 0 (exact bf16 cache, the unquantized baseline): an R-block is four
// 32-token quarters, each [K 8 KB][V 8 KB] of raw bf16 in A-fragment order so
// a lane's four A registers are one 16-byte load.
constexpr int BF16_BLOCK_BYTES = 2 * R * D * 2;
constexpr int BF16_QUARTER_BYTES = BF16_BLOCK_BYTES / 4;
// K word w (32-bit = 2 bf16) of a quarter: w = ((i*8 + s)*32 + lane)*4 + reg,
//   reg 0:(row g, k 2tq) 1:(row g+8, k 2tq) 2:(row g, k 2tq+8) 3:(row g+8, k 2tq+8)
//   row -> token 16i + row (within the quarter), k -> channel 16s + k (+0/+1 halves)
OSK_HD void bf16_k_coords(int w, int hi, int &token, int &channel) {
    const int reg = w & 3, lane = (w >> 2) & 31, s = (w >> 7) & 7, i = w >> 10;
    const int g = lane >> 2, tq = lane & 3;
    token = 16 * i + g + ((reg & 1) ? 8 : 0);
    channel = 16 * s + 2 * tq + ((reg & 2) ? 8 : 0) + hi;
}
// V word w of a quarter: w = ((j*8 + m)*32 + lane)*4 + reg,
//   reg 0:(row g; t1,t2) 1:(row g+8; t1,t2) 2:(row g; t3,t4) 3:(row g+8; t3,t4)
//   row -> channel 16m + row; t1 = 16j+tq, t2 = t1+8, t3 = t1+4, t4 = t1+12 (hi = 2nd)
OSK_HD void bf16_v_coords(int w, int hi, int &token, int &channel) {
    const int reg = w & 3, lane = (w >> 2) & 31, m = (w >> 7) & 7, j = w >> 10;
    const int g = lane >> 2, tq = lane & 3;
    channel = 16 * m + g + ((reg & 1) ? 8 : 0);
    token = 16 * j + tq + ((reg & 2) ? 4 : 0) + (hi ? 8 : 0);
}

// ---- K code words --------------------------------------------------------
// word index w = ((s*32 + lane)*4 + fam)*WPF + half, WPF = 8/TILES_PER_WORD
//   fam: 0 (pair0,row g) 1 (pair0,row g+8) 2 (pair1,row g) 3 (pair1,row g+8)
//   pair0 = channels (16s+2tq, 16s+2tq+1), pair1 = (16s+2tq+8, 16s+2tq+9)
// field f (0..TILES_PER_WORD-1) of the low/high half -> m-tile i = half*TPW+f
OSK_HD void k_word_coords(int BITS, int w, int f, int hi, int &token, int &channel) {
    const int tpw = 16 / BITS, wpf = 8 / tpw;
    const int half = w % wpf;
    const int fam = (w / wpf) % 4;
    const int lane = (w / wpf / 4) % 32;
    const int s = w / wpf / 4 / 32;
    const int g = lane >> 2, tq = lane & 3;
    const int i = half * tpw + f;
    const int row = g + ((fam & 1) ? 8 : 0);
    token = 16 * i + row;
    channel = 16 * s + 2 * tq + ((fam & 2) ? 8 : 0) + hi;
}

// ---- V code words ----------------------------------------------------------
// word index w = ((j*32 + lane)*4 + fam)*WPF + half
//   fam: 0 (row g; k 2tq,2tq+1) 1 (row g+8; same k) 2 (row g; k 2tq+8,2tq+9) 3 (row g+8; same k)
//   k = token within the 16-token tile j in natural order (the P.V B operand is the
//   movmatrix transpose of the QK accumulator, whose rows are tokens 16j..16j+15)
//   low half -> the even k of the pair, high half -> the odd one
// field f -> PV m-tile m = half*TPW + f -> channel 16m + row
OSK_HD void v_word_coords(int BITS, int w, int f, int hi, int &token, int &channel) {
    const int tpw = 16 / BITS, wpf = 8 / tpw;
    const int half = w % wpf;
    const int fam = (w / wpf) % 4;
    const int lane = (w / wpf / 4) % 32;
    const int j = w / wpf / 4 / 32;
    const int g = lane >> 2, tq = lane & 3;
    const int m = half * tpw + f;
    const int row = g + ((fam & 1) ? 8 : 0);
    channel = 16 * m + row;
    token = 16 * j + 2 * tq + (hi ? 1 : 0) + ((fam & 2) ? 8 : 0);
}

// ---- inverse maps (element -> word, bit shift), for per-element readers --------
// K code of (token t, channel c): inverse of k_word_coords
OSK_HD void k_code_loc(int BITS, int t, int c, int &word, int &shift) {
    const int tpw = 16 / BITS, wpf = 8 / tpw;
    const int i = t >> 4, row = t & 15, s = c >> 4, kc = c & 15;
    const int tq = (kc & 7) >> 1, hi = kc & 1;
    const int fam = (row >= 8 ? 1 : 0) + (kc >= 8 ? 2 : 0);
    const int lane = (row & 7) * 4 + tq;
    const int half = i / tpw, f = i % tpw;
    word = ((s * 32 + lane) * 4 + fam) * wpf + half;
    shift = hi * 16 + f * BITS;
}
// V code of (token t, channel c): inverse of v_word_coords
OSK_HD void v_code_loc(int BITS, int t, int c, int &word, int &shift) {
    const int tpw = 16 / BITS, wpf = 8 / tpw;
    const int m = c >> 4, row = c & 15, j = t >> 4, r = t & 15;
    const int tq = (r & 7) >> 1, hi = r & 1;
    const int fam = (row >= 8 ? 1 : 0) + (r >= 8 ? 2 : 0);
    const int lane = (row & 7) * 4 + tq;
    const int half = m / tpw, f = m % tpw;
    word = ((j * 32 + lane) * 4 + fam) * wpf + half;
    shift = hi * 16 + f * BITS;
}
// raw bf16 K of (token t in 0..R-1, channel c) in a bf16 record: byte offset of
// the 16-bit value (inverse of bf16_k_coords over the four quarters)
OSK_HD int bf16_k_byte(int t, int c) {
    const int qu = t >> 5, tt = t & 31;
    const int i = tt >> 4, row = tt & 15, s = c >> 4, kc = c & 15;
    const int tq = (kc & 7) >> 1, hi = kc & 1;
    const int reg = (row >= 8 ? 1 : 0) + (kc >= 8 ? 2 : 0);
    const int lane = (row & 7) * 4 + tq;
    const int w = ((i * 8 + s) * 32 + lane) * 4 + reg;
    return qu * BF16_QUARTER_BYTES + w * 4 + hi * 2;
}

// ---- params ----------------------------------------------------------------
// channel c = 16s + kc; slot of kc within the lane's 4 B-fragment channels
OSK_HD void k_chan_split(int c, int &s, int &tq, int &slot) {
    s = c >> 4;
    const int kc = c & 15;
    tq = (kc & 7) >> 1;
    slot = (kc & 1) + ((kc >> 3) << 1);
}
// K a-params: [s][tq][grp][slot]  (lane reads 32 B per k-step: all 4 groups)
OSK_HD int ka_index(int c, int grp) {
    int s, tq, slot;
    k_chan_split(c, s, tq, slot);
    return ((s * 4 + tq) * 4 + grp) * 4 + slot;
}
// K b-params: [s/2][grp][tq][word][half], word = (slot/2)*2 + s%2: one 16-byte
// load per k-step PAIR is an A quad (x_s, x_s+1, y_s, y_s+1) whose rows g hold
// k-step s and rows g+8 k-step s+1, so the bias MMAs read it without moves
// (lane (g, tq) reads chunk (s/2)*16 + (g&3)*4 + tq: k-step-pair major, so the
// 8 lanes of each quarter-warp phase read 8 consecutive 16-byte chunks --
// conflict-free; a [grp][tq][s/2] order put them 64 B apart, 4-way conflicts)
OSK_HD int kb_index(int c, int grp) {
    int s, tq, slot;
    k_chan_split(c, s, tq, slot);
    return (((s >> 1) * 16 + grp * 4 + tq)) * 8 + ((slot >> 1) * 2 + (s & 1)) * 2 + (slot & 1);
}
// token t = 16j + r; B-fragment k = r (natural order): lane pair tq = (r mod 8) / 2,
// slot = (r & 1) + 2 (r >= 8)  (slots 0,1 -> b0 = k 2tq,2tq+1; 2,3 -> b1 = k 2tq+8,2tq+9)
OSK_HD void v_tok_split(int t, int &j, int &tq, int &slot) {
    j = t >> 4;
    const int r = t & 15;
    tq = (r & 7) >> 1;
    slot = (r & 1) + ((r >> 3) << 1);
}
// V a-params: [j][tq][gc][slot]
OSK_HD int va_index(int t, int gc) {
    int j, tq, slot;
    v_tok_split(t, j, tq, slot);
    return ((j * 4 + tq) * 4 + gc) * 4 + slot;
}
// V b-params: [j/2][gc][tq][word][half], paired (and conflict-free) like the K b-params
OSK_HD int vb_index(int t, int gc) {
    int j, tq, slot;
    v_tok_split(t, j, tq, slot);
    return (((j >> 1) * 16 + gc * 4 + tq)) * 8 + ((slot >> 1) * 2 + (j & 1)) * 2 + (slot & 1);
}
// norms: [g][i][2] -> token 16i + g (+8 for slot 1)
OSK_HD int norm_index(int t) {
    const int i = t >> 4, r = t & 15;
    return ((r & 7) * 8 + i) * 2 + (r >> 3);
}

// exact shadow (keep_exact): per block K lohi [ch][grp][2], V lohi [tok][gc][2],
// norms fp64 [tok]
constexpr int SHADOW_K_DOUBLES = D * NGRP * 2;
constexpr int SHADOW_V_DOUBLES = R * NGC * 2;
constexpr int SHADOW_N_DOUBLES = R;
constexpr int SHADOW_DOUBLES = SHADOW_K_DOUBLES + SHADOW_V_DOUBLES + SHADOW_N_DOUBLES;

}  // namespace osk
