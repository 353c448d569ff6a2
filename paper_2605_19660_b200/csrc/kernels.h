// kernels.h -- host-side launchers of the device kernels (internal to the
// library; the public boundary is include/oscar_kv.h).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include <atomic>

namespace osk {

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device):
// function attributes live in the device's context, so a process driving
// several GPUs (one handle per device) must set them on each.  `done` is a
// per-kernel bit set of devices; concurrent first calls both set the
// attribute, which is idempotent.
template <typename Kernel>
inline cudaError_t ensure_smem_attr(Kernel kernel, int bytes, std::atomic<uint64_t> &done) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    const uint64_t bit = dev < 64 ? (uint64_t{1} << dev) : 0;
    if (bit && (done.load(std::memory_order_acquire) & bit)) return cudaSuccess;
    e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e == cudaSuccess && bit) done.fetch_or(bit, std::memory_order_acq_rel);
    return e;
}

// integer tuning knob from the environment, read once (thread-safe static init
// at the call site: `static const long v = env_knob("X", dflt);`)
inline long env_knob(const char *name, long dflt) {
    const char *e = getenv(name);
    return e ? atol(e) : dflt;
}

struct TransformCfg {
    int bits;       // 0, 2, 4 (0 => raw bf16 block, no transform)
    int rotates;    // K (and Q) Hadamard rotation
    int scales;     // Omni-Token Scaling of K
    int scaling;    // 0 l2, 1 rsqrt, 2 max, 3 mean-abs
    int rotate_v;   // explicit V rotation
};

// Quantise n_blocks R-blocks per (sequence, head) from a bf16 source.
// Key element (b, h, token t, channel c) lives at
//   k + b*sb + (tok0 + t)*st + h*sh + c,
// value element at v + b*sb + (tok0 + t)*vst + h*sh + c*vsc (vsc = 1 for a
// token-major source); vsc = 0: v is a residual V ring (tile-major, layout.h vring_index).
// Block k of (b,h) is written to blocks[((b*H+h)*max_blocks + blk0 + k)*bytes].
struct QuantizeArgs {
    const void *k, *v;
    int64_t sb, st, sh, tok0;
    int64_t vst, vsc;
    int B, H;
    int64_t n_blocks;
    uint8_t *blocks;
    int64_t max_blocks, blk0;
    double *shadow;  // nullable: [bh][max_blocks][SHADOW_DOUBLES]
    TransformCfg tc;
    // optional residual-window prefix of block 0: its first rtok tokens come from
    // the rings (K [bh][R][D], V [bh][D][R]), the rest from the source above
    const void *rk = nullptr, *rv = nullptr;
    int64_t rtok = 0;
    // device status word (nullable): bit 0 = an fp16 step/offset of the record
    // overflowed (the exact fp64 params are still exported), bit 1 = a group
    // had non-finite input (the reference's params are then non-finite too)
    int *status = nullptr;
};
constexpr int STATUS_FP16_OVERFLOW = 1, STATUS_NONFINITE_INPUT = 2, STATUS_MERGE_TIMEOUT = 4;
cudaError_t launch_quantize(const QuantizeArgs &a, cudaStream_t st);

// Copy n tokens of raw bf16 K/V into the residual ring at slot0: K ring
// [bh][R][D] token-major, V ring [bh][R/16][D][16] tile-major (layout.h
// vring_index: the attention kernel's P.V A fragments are contiguous token
// pairs, and one 16-token tile is one contiguous 4 KB span).
struct RingCopyArgs {
    const void *k, *v;
    int64_t sb, st, sh, tok0;
    int B, H;
    int64_t n;
    void *ring_k, *ring_v;  // K [bh][R][D], V [bh][D][R]
    int64_t slot0;
};
cudaError_t launch_ring_copy(const RingCopyArgs &a, cudaStream_t st);

// ---- reference-form fp64 appends (f64_path.cu) ----------------------------------
// strided fp64 rows: element (b, h, t, c) at p[b*sb + h*sh + t*st + c] (norms: c = 0)
struct F64Src {
    const double *p;
    int64_t sb, sh, st;
};
// one R-block per (block, b*H + h): the K part (part 0: K_u rows + norms) or the
// V part (part 1) of records blk0 + i from source tokens tok0 + i*R ...
struct QuantizeF64Args {
    F64Src src, norms;
    int part, bits;
    int B, H;
    int64_t tok0, n_blocks;
    uint8_t *blocks;
    int64_t max_blocks, blk0;
    double *shadow;  // [bh][max_blocks][SHADOW_DOUBLES]
    int *status;
};
cudaError_t launch_quantize_f64(const QuantizeF64Args &a, cudaStream_t st);
// n tokens (source tokens tok0 ...) into window slots slot0 ...: the exact fp64
// residual (res_k / res_n or res_v, [bh][R][D] / [bh][R]) and the bf16 image the
// decode kernel attends (rings)
struct WindowF64Args {
    F64Src src, norms;
    int part;
    int B, H;
    int64_t tok0, n, slot0;
    int rotates, scales;
    double *res_k, *res_n, *res_v;  // (the rings take fp16 images)
    void *ring_k, *ring_v;
};
cudaError_t launch_window_f64(const WindowF64Args &a, cudaStream_t st);

// Sequence-shard exchange plan (C5): rank r's receive area recv[r] holds
// [2 parities][world][rows][PEER_STRIDE] 8-byte words (epoch << 32 | fp32 bits:
// O[0..127], LSE at 128); it lives on rank r's GPU and is mapped into every
// peer (CUDA IPC).  Same layout as oscar_peer_plan.
constexpr int PEER_MAX = 8;
constexpr int PEER_STRIDE = 132;  // words per row: 128 + LSE, padded to 32 B
struct PeerPlan {
    int32_t world, rank;
    int64_t rows;
    uint64_t *recv[PEER_MAX];
};

// profiling build: 64-bit slots per warp in AttnArgs::prof
constexpr int kProfStride = 32;

struct AttnArgs {
    const uint8_t *blocks;
    int64_t max_blocks;
    int64_t nb;        // packed blocks per (b,h)
    int BH, Hkv, g, Hq;
    const void *q;     // bf16 [B][Hq][D]
    const void *kcur, *vcur;  // bf16 [B][Hkv][D] or null
    void *ring_k, *ring_v;    // K [bh][R][D], V [bh][D][R]
    int r;             // residual rows in ring
    int write_ring;    // store kcur/vcur at ring slot r
    int tile_units;    // small launches: the residual window's 16-token tiles are pipeline units of
                       // the tail owner, bulk-copied into the shared-memory ring like the records
                       // (K rows, the tile-major V tile, the current token, the raw q rows)
    int ring_f16;      // rings hold fp16 images (fp64-form caches: the exact rows are in the
                       // residual shadow; fp16 keeps the window's rounding 8x below bf16's)
    int rotates;       // rotate q for the packed part
    int scales;        // unused on device (norms are stored), kept for clarity
    int rotate_v;      // un-rotate output
    float *out;        // fp32 [B][Hq][D]
    float *lse;        // fp32 [B][Hq] or null
    // split-KV partials of the CTAs sharing a (b, kv head), as flag-in-word
    // 8-byte words (1 << 32 | fp32 bits; zero = not written): the merging CTA
    // polls them and clears them again, so they are zero between launches
    uint64_t *part_o;  // [BH][maxp][8][D]
    uint64_t *part_ml; // [BH][maxp][8][2]
    int *counters;     // [BH], zero between launches (ticket mode)
    int poll_merge;    // 1: every CTA is resident (ncta <= SMs): the first CTA of a (b, kv head)
                       // polls the others' partials; 0: last-arriving CTA by atomic ticket
    int *status;       // device status word (STATUS_*) or null
    float *warp_part;  // [ncta][maxseg][12][8*D+16] per-warp partial scratch
    int maxseg;        // segment slots per CTA in warp_part
    int maxp;
    int ncta;
    int64_t seg_cost;  // virtual units per (b, kv head) segment in the stream-K split (split.h)
    int64_t tail_cost; // virtual units charged to a segment's residual-window tiles (split.h)
    int cta_perm;      // 0, or a multiplier coprime with ncta: block i takes range (i * cta_perm) % ncta
    int pdl_prefetch;  // packed records unchanged since the previous launch on this stream:
                       // the ring fill may start before griddepcontrol.wait
    unsigned long long *prof;  // debug: per-warp phase cycles [ncta][NCW][5] or null
    // fused sequence-shard exchange (peer.cu): when pub_world > 0 the final merge
    // stores each normalised row (O, LSE) straight into every rank's receive area
    // over peer memory and raises its flag, instead of writing out / lse
    PeerPlan pub;
    uint32_t pub_epoch;
};
// bits: 2, 4 or 0 (bf16 baseline)
cudaError_t launch_attention(int bits, const AttnArgs &a, cudaStream_t st);
int64_t attention_scratch_floats(int64_t slots);  // floats of `slots` (CTA, segment) warp-partial slots
int attention_grid(int bits, int num_sms, int64_t nb, int BH);

// logits.cu: StepOutput.logits (pipeline.hpp:54-58) from the device records:
// fp32 [B][Hq][s_total], natural units, packed tokens then window then current
struct LogitsArgs {
    const uint8_t *blocks;
    int64_t max_blocks, block_bytes;
    int64_t nb;               // packed blocks per (b, kv head)
    int BH, Hkv, g, Hq;
    const void *q;            // bf16 [B][Hq][D]
    const void *kcur;         // bf16 [B][Hkv][D] or null
    const void *ring_k;       // K ring [bh][R][D]
    int ring_f16;             // ring K holds fp16 (fp64-form caches) instead of bf16
    int r;                    // window tokens
    int rotates;              // rotate q for the packed tokens
    float *logits;
    int64_t s_total;          // nb*R + r + (kcur ? 1 : 0)
};
cudaError_t launch_logits(int bits, const LogitsArgs &a, cudaStream_t st);

// peer.cu: wait for every rank's row of this epoch in recv[rank], merge -> out/lse;
// status (optional, device int) is set to 1 if a peer did not publish within ~5 s
cudaError_t launch_peer_merge(const PeerPlan &p, uint32_t epoch, float *out, float *lse, int *status,
                              cudaStream_t st);
// an empty shard publishes LSE = -inf rows (it contributes nothing to the softmax)
cudaError_t launch_peer_publish_empty(const PeerPlan &p, uint32_t epoch, cudaStream_t st);

cudaError_t launch_lse_merge(const float *outs, const float *lses, int64_t parts, int64_t rows, int64_t d,
                             float *out, float *lse_out, cudaStream_t st);

}  // namespace osk
