/* oscar_kv.h -- C-ABI of the B200-native OScaR KV-cache path.
 *
 * Drop-in boundary for the reference's C++ cache API
 * (/root/reference/proj/include/oscar/kv_cache.hpp, pipeline.hpp).  Plain
 * pointers and sizes only; device pointers are CUDA device addresses, streams
 * are cudaStream_t passed as void*.  Every entry point returns 0 on success,
 * 1 invalid argument (reference std::invalid_argument), 2 logic/state error
 * (std::logic_error, e.g. residual overflow kv_cache.cpp:225-227), 3 CUDA /
 * runtime error; oscar_last_error() holds the thread-local message.
 *
 * One handle = one writer (kv_cache.hpp:58-60 single-writer contract) holding
 * `batch` sequences of identical length, each with `heads` KV heads.  All
 * work is enqueued on the caller's stream; no internal host synchronisation
 * except the *_host and export entry points, which synchronise their stream.
 */
#ifndef OSCAR_KV_H
#define OSCAR_KV_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Method / Scaling enums, same values as the reference (kv_cache.hpp:11-12). */
enum oscar_method { OSCAR_FP = 0, OSCAR_KIVI = 1, OSCAR_ROTATE_ONLY = 2, OSCAR_SCALE_ONLY = 3, OSCAR_OSCAR = 4 };
enum oscar_scaling { OSCAR_L2 = 0, OSCAR_RSQRT = 1, OSCAR_MAX = 2, OSCAR_MEAN_ABS = 3 };

/* PipelineConfig (kv_cache.hpp:19-32) plus the value-rotation mode.
 * rotate_v = 0: V arrives already rotated (W_V folded by preprocess,
 *               pipeline.cpp:38-78) and attention outputs stay in that space;
 * rotate_v = 1: the append kernel applies the Hadamard rotation to V and the
 *               attention output is rotated back (explicit mode). */
typedef struct oscar_kv_config {
    int32_t method;
    int32_t bits;          /* 0 (exact bf16 cache), 2, 4 on device */
    int64_t group_size;    /* G; device kernels: 32 */
    int64_t residual_len;  /* R; device kernels: 128 */
    int32_t scaling;
    int32_t rotate_v;
    int64_t head_dim;      /* d_h; device kernels: 128 */
    int64_t heads;         /* H = KV heads */
} oscar_kv_config;

/* MemoryReport (kv_cache.hpp:45-56): the reference's accounting (fp64 params
 * and norms) plus the device's actual resident bytes. */
typedef struct oscar_kv_memory_report {
    int64_t packed_tokens, residual_tokens;
    int64_t packed_k_payload_bits, packed_v_payload_bits;
    int64_t residual_k_payload_bits, residual_v_payload_bits;
    int64_t k_norm_bits, param_bits;
    double effective_bits_per_value;
    int64_t device_hot_bytes;    /* bytes the decode kernel streams per sequence */
    int64_t device_total_bytes;  /* all device allocations of the handle */
} oscar_kv_memory_report_t;

typedef struct oscar_kv_handle oscar_kv_handle;

const char *oscar_last_error(void);

/* PipelineConfig::validate (kv_cache.cpp:51-67) + device shape limits. */
int oscar_kv_config_validate(const oscar_kv_config *cfg);

/* KvCache(const PipelineConfig&) (kv_cache.cpp:80-85).  q_heads = GQA query
 * heads (q_heads % heads == 0, q_heads/heads <= 8); max_tokens = capacity per
 * sequence; keep_exact = keep fp64 (lo, hi) per group and fp64 norms on
 * device so oscar_kv_export can return bit-exact reference params. */
int oscar_kv_create(const oscar_kv_config *cfg, int64_t batch, int64_t q_heads, int64_t max_tokens,
                    int device, int keep_exact, oscar_kv_handle **out);
int oscar_kv_destroy(oscar_kv_handle *h);

/* buffer_quant_k + buffer_quant_v fused (kv_cache.cpp:194-292), taking RAW
 * keys: the kernel applies apply_method's key transform (fht_tensor +
 * omni_token_scale, pipeline.cpp:224-236) in fp64 first.
 * k, v: bf16 [batch, n_tokens, heads, head_dim] device pointers.  The first
 * call is the prefill branch (S - S mod R packed, the rest residual); later
 * calls append token by token and flush at exactly R. */
int oscar_kv_append(oscar_kv_handle *h, const void *k, const void *v, int64_t n_tokens, void *stream);

/* The reference's own call shapes, fp64 rows as KvCache receives them
 * (kv_cache.hpp:80-84):
 *   oscar_kv_append_k = buffer_quant_k(new_k, norms) (kv_cache.cpp:194-249):
 *     k_t: fp64 [batch, n_tokens, heads, head_dim], the ALREADY transformed
 *     keys K_u (apply_method's output), norms: fp64 [batch, n_tokens, heads];
 *   oscar_kv_append_v = buffer_quant_v(new_v) (kv_cache.cpp:251-292):
 *     v: fp64 [batch, n_tokens, heads, head_dim], stored as given.
 * Device pointers (host pointers are accepted too and staged through the
 * device, synchronously).  K and V advance separately (first call = prefill branch,
 * then token by token with a flush at exactly R), packed codes, params and
 * norms bit-exact vs the reference; the residual window is kept exactly in
 * fp64 (export / dump / flush) with a bf16 image for the decode kernel.  A
 * cache takes one input form: these calls and oscar_kv_append /
 * oscar_kv_decode_step (raw bf16 rows) cannot be mixed on one handle (status
 * 2).  Needs bits 2 or 4 and rotate_v = 0.  Attention requires both streams
 * to hold the same number of tokens. */
int oscar_kv_append_k(oscar_kv_handle *h, const double *k_t, const double *norms, int64_t n_tokens, void *stream);
int oscar_kv_append_v(oscar_kv_handle *h, const double *v, int64_t n_tokens, void *stream);
/* decode_step (pipeline.cpp:292-323) with the current token in that form:
 * k_t fp64 [batch, heads, d] (K_u of the token), norms fp64 [batch, heads],
 * v fp64 [batch, heads, d]; q bf16 [batch, q_heads, d] (raw, rotated by the
 * kernel).  Attends history + current token at full precision, then the
 * flush at R, like oscar_kv_decode_step. */
int oscar_kv_decode_step_f64(oscar_kv_handle *h, const void *q, const double *k_t, const double *norms,
                             const double *v, float *out, float *lse, void *stream);
/* Value-stream counters of the fp64 form (the reference's v_packed_tokens_ /
 * v_residual_; oscar_kv_stats counts keys). */
int oscar_kv_stats_v(const oscar_kv_handle *h, int64_t *v_packed, int64_t *v_residual);

/* decode_step body (pipeline.cpp:292-323) without projections:
 * attention of q over (cache history + the current token at full precision),
 * then the current token is appended (a flush, if the window fills, runs
 * after the attention kernel -- the reference's ordering contract).
 * q: bf16 [batch, q_heads, d]; k, v: bf16 [batch, heads, d] (current token);
 * out: fp32 [batch, q_heads, d]; lse: optional fp32 [batch, q_heads] (natural
 * log of the softmax denominator of logits q.k/sqrt(d)). */
int oscar_kv_decode_step(oscar_kv_handle *h, const void *q, const void *k, const void *v, float *out,
                         float *lse, void *stream);

/* decode_step that also returns StepOutput.logits (pipeline.hpp:54-58,
 * pipeline.cpp:314-318): logits fp32 [batch, q_heads, S_total] with
 * S_total = total tokens before the step + 1 (history then the current
 * token), natural units q.k/sqrt(d) as attend_one writes them
 * (pipeline.cpp:158-165), computed from the device cache's records.  A
 * debug/fidelity output: one extra kernel before the attention kernel.
 * logits may be NULL (== oscar_kv_decode_step). */
int oscar_kv_decode_step_logits(oscar_kv_handle *h, const void *q, const void *k, const void *v, float *out,
                                float *lse, float *logits, void *stream);

/* The same logits without attending or appending: over the cache contents,
 * plus the current token's key k (bf16 [batch, heads, d]) when k is non-NULL.
 * logits: fp32 [batch, q_heads, total_tokens (+1)]. */
int oscar_kv_logits(oscar_kv_handle *h, const void *q, const void *k, float *logits, void *stream);

/* decode_step for n independent caches (e.g. the layers of one model step)
 * in ONE host call: element i of every array belongs to handles[i]; lse may
 * be NULL (or contain NULLs).  Same semantics as n oscar_kv_decode_step
 * calls in order on one stream, without the per-call host round trip. */
int oscar_kv_decode_step_many(int32_t n, oscar_kv_handle *const *handles, const void *const *q,
                              const void *const *k, const void *const *v, float *const *out, float *const *lse,
                              void *stream);

/* Attention over the cache contents only (no current token, no append).
 * Used for sequence sharding: each rank attends its R-aligned shard and the
 * (out, lse) partials are merged with oscar_lse_merge. */
int oscar_kv_attend(oscar_kv_handle *h, const void *q, float *out, float *lse, void *stream);

/* decode_step with HOST buffers (pinned or pageable): copies q/k/v in and
 * out/lse back inside the call; synchronises the stream. */
int oscar_kv_decode_step_host(oscar_kv_handle *h, const void *q_host, const void *k_host,
                              const void *v_host, float *out_host, float *lse_host, void *stream);

/* Device-side status accumulated by the quantize/append kernels since the
 * last clear (synchronises the handle's last stream):
 *   OSCAR_STATUS_FP16_OVERFLOW  a group's step or offset exceeds the fp16 range
 *                               of the attention record (attention over that
 *                               group is not finite; export/dump stay exact),
 *   OSCAR_STATUS_NONFINITE      a group had non-finite input values.
 * The reference has no such condition for finite inputs (it keeps fp64). */
#define OSCAR_STATUS_FP16_OVERFLOW 1
#define OSCAR_STATUS_NONFINITE 2
/*   OSCAR_STATUS_MERGE_TIMEOUT  a split-KV merge waited > 2 s for another CTA's partial
 *                               (cannot happen while every CTA is resident; its rows are NaN) */
#define OSCAR_STATUS_MERGE_TIMEOUT 4
int oscar_kv_status(oscar_kv_handle *h, int32_t *flags, int32_t clear);

/* packed_tokens / residual_tokens / flush_count (kv_cache.hpp:67-71). */
int oscar_kv_stats(const oscar_kv_handle *h, int64_t *packed, int64_t *residual, int64_t *flushes);
int oscar_kv_memory_report(const oscar_kv_handle *h, oscar_kv_memory_report_t *out);

/* Export sequence b in the reference's own layout (PackedBlock,
 * kv_cache.hpp:38-43 / KvCache members 104-122).  Counts per head:
 *   nblk = packed/R; K params per block d*(R/G) at [j*(R/G)+g];
 *   V params per block R*(d/G) at [t*(d/G)+g];
 *   bits==2 payload: R*d/8 uint16 words per block (pack_2bit, quant.cpp:162-175)
 *   bits==4 payload: R*d uint16 codes per block; bits==0: raw fp64 rows.
 * Any pointer may be NULL to skip that section.  Requires keep_exact for
 * the params and norms.  Synchronises the handle's last stream. */
typedef struct oscar_kv_export_t {
    uint16_t *k_payload, *v_payload;  /* [H][nblk][...] */
    double *k_delta, *k_constant, *v_delta, *v_constant;
    int64_t *k_zp, *v_zp;
    double *k_raw, *v_raw;           /* bits==0: [H][nblk][R*d] */
    double *k_norms;                 /* [H][packed] */
    double *k_residual;              /* [r][H][d] transformed K_u rows */
    double *k_norms_residual;        /* [r*H] */
    double *v_residual;              /* [r][H][d] */
} oscar_kv_export_t;
int oscar_kv_export(oscar_kv_handle *h, int64_t b, oscar_kv_export_t *out);

/* KvCache::dump (kv_cache.cpp:469-507): KVC1 file for sequence b, readable by
 * the reference's KvCache::load. */
int oscar_kv_dump(oscar_kv_handle *h, int64_t b, const char *path);

/* KvCache::load (kv_cache.cpp:509-549): sequence b of the handle from a KVC1
 * file (written by the reference's KvCache::dump or oscar_kv_dump).  The
 * config (method, bits, G, R, scaling, H, d_h) must match; a fresh handle
 * adopts the file's token counts, a filled one must already hold the same
 * counts (one handle = sequences of equal length).  Residual rows that are
 * the transform of bf16 inputs (verified bit for bit) go to the raw form's
 * bf16 rings; any other fp64 residual rows put the handle in the fp64 form
 * (see oscar_kv_append_k; bits 2/4, rotate_v = 0).  The bits-0 raw rows must
 * be bf16 transforms; quantized blocks need keep_exact.  Synchronous. */
int oscar_kv_load(oscar_kv_handle *h, int64_t b, const char *path);

/* The config and token count of a KVC1 file (its manifest), for creating a
 * handle to load it into (static KvCache::load, kv_cache.hpp:95).  rotate_v
 * is 0; tokens = packed + residual. */
int oscar_kvc1_read_config(const char *path, oscar_kv_config *cfg, int64_t *tokens);

/* materialize_k / materialize_v (kv_cache.cpp:327-381) of sequence b into
 * host fp64 [total, H, d] buffers (a debug/parity path, not the hot path). */
int oscar_kv_materialize(oscar_kv_handle *h, int64_t b, double *k_out, double *v_out);

/* Log-sum-exp merge of P partial attention results (sequence sharding):
 * outs: fp32 [P, rows, d], lses: fp32 [P, rows] -> out fp32 [rows, d],
 * lse_out optional.  Device pointers. */
int oscar_lse_merge(const float *outs, const float *lses, int64_t parts, int64_t rows, int64_t d,
                    float *out, float *lse_out, void *stream);

/* ---- fused sequence-shard exchange over peer memory (C5) ----
 * Replaces "attend -> all-gather (O, LSE) -> oscar_lse_merge" by: the
 * attention kernel's final merge stores each normalised row straight into
 * every rank's receive area (NVLink peer stores); oscar_peer_merge on each
 * rank waits for the rows and merges.  No fences or separate flags: every
 * 8-byte word of a row is (epoch << 32 | fp32 bits) and the reader polls the
 * words until their epoch matches.
 * Rank r's receive area (oscar_peer_area_bytes, on rank r's GPU, mapped into
 * every peer with oscar_ipc_*): uint64 recv[2][world][rows][OSCAR_PEER_STRIDE]
 * (O[0..127], LSE at 128), zeroed before the first epoch.
 * Epochs start at 1 and increase by one per step on every rank. */
#define OSCAR_PEER_MAX 8
#define OSCAR_PEER_STRIDE 132
typedef struct oscar_peer_plan {
    int32_t world, rank;              /* this handle's shard; world <= OSCAR_PEER_MAX */
    int64_t rows;                     /* batch * q_heads */
    uint64_t *recv[OSCAR_PEER_MAX];   /* rank p's receive area, as mapped here */
} oscar_peer_plan;
int64_t oscar_peer_area_bytes(int32_t world, int64_t rows);
/* attend (k = v = NULL) or decode_step (current token attended and appended)
 * whose result is published to every rank of the plan instead of returned. */
int oscar_kv_attend_publish(oscar_kv_handle *h, const void *q, const void *k, const void *v,
                            const oscar_peer_plan *plan, uint32_t epoch, void *stream);
/* an empty shard's contribution (LSE = -inf rows) */
int oscar_peer_publish_empty(const oscar_peer_plan *plan, uint32_t epoch, void *stream);
/* wait for all ranks' rows of `epoch` in this rank's area, merge -> out
 * fp32 [rows, 128], lse optional; status (device int32, optional) becomes 1
 * and out / lse NaN if a peer does not publish within ~5 s. */
int oscar_peer_merge(const oscar_peer_plan *plan, uint32_t epoch, float *out, float *lse, int32_t *status,
                     void *stream);
/* CUDA IPC plumbing for the receive areas (64-byte handles). */
int oscar_ipc_alloc(int64_t bytes, int32_t device, void **dptr, void *handle_out);
int oscar_ipc_open(const void *handle, int32_t device, void **dptr);
int oscar_ipc_close(void *dptr);
int oscar_ipc_free(void *dptr);

/* Number of kernels the last decode/attend call launched (instrumentation). */
int oscar_kv_last_launch_count(const oscar_kv_handle *h);

#ifdef __cplusplus
}
#endif
#endif
