/* ORACLE / TEST INFRASTRUCTURE ONLY -- a plain-C restatement of the reference
 * OScaR KV-cache path (/root/reference/proj), used as the parity checker for
 * the CUDA path.  Pinned against the compiled reference (oracle/_ref) and the
 * reference's known answers in tests/test_oracle.py.  Never linked into the
 * product library. */
#ifndef OSCAR_ORACLE_H
#define OSCAR_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* enums mirror kv_cache.hpp:11-12 */
enum { OO_FP = 0, OO_KIVI = 1, OO_ROTATE_ONLY = 2, OO_SCALE_ONLY = 3, OO_OSCAR = 4 };
enum { OO_L2 = 0, OO_RSQRT = 1, OO_MAX = 2, OO_MEAN_ABS = 3 };

void oo_fht(double *v, int64_t d);
double oo_fast_rsqrt(double x);
int64_t oo_token_scale(const double *x, int64_t S, int64_t H, int64_t d, int strategy,
                       double *scaled, double *norms);
void oo_quant_params(const double *v, int64_t n, int bits, double *delta, int64_t *zp,
                     double *constant);
uint16_t oo_quantize_one(double x, double delta, int64_t zp, int bits);
double oo_dequantize_one(uint16_t code, double delta, int64_t zp, double constant);
void oo_pack_2bit(const uint16_t *codes, int64_t n, uint16_t *words);
void oo_unpack_2bit(const uint16_t *words, int64_t n, uint16_t *codes);
void oo_attention(const double *q, int64_t Tq, const double *k, const double *v, int64_t S,
                  int64_t H, int64_t d, double *out);

typedef struct oo_cache oo_cache;
/* returns NULL on an invalid config (PipelineConfig::validate, kv_cache.cpp:51-67) */
oo_cache *oo_cache_create(int method, int bits, int64_t G, int64_t R, int scaling, int64_t d,
                          int64_t H, int rotate_v);
void oo_cache_destroy(oo_cache *c);
/* raw keys/values [S,H,d]; transform (apply_method) + buffer_quant_k/v.
 * returns 0 ok, 2 residual overflow (logic_error) */
int oo_cache_append(oo_cache *c, const double *xk, const double *xv, int64_t S);
void oo_cache_stats(const oo_cache *c, int64_t *out4);
/* export accessors in the reference's own per-head/per-block layout */
int64_t oo_cache_num_blocks(const oo_cache *c, int is_v, int64_t head);
/* codes: d*R uint16 (K channel-major j*R+t; V token-major t*d+c); params: n
 * entries of delta/zp/constant; returns number of params (0 for raw blocks) */
int64_t oo_cache_block(const oo_cache *c, int is_v, int64_t head, int64_t blk, uint16_t *codes,
                       double *delta, int64_t *zp, double *constant, double *raw);
void oo_cache_k_norms(const oo_cache *c, int64_t head, double *norms);
/* residual: k_u rows [r,H,d], norms [r*H], v rows [r,H,d] */
void oo_cache_residual(const oo_cache *c, double *k_rows, double *k_norms, double *v_rows);
void oo_cache_materialize(const oo_cache *c, double *k_out, double *v_out);
/* decode_step body without projections; GQA g query heads per KV head;
 * q head h*g+j served by KV head h */
int oo_decode_step(oo_cache *c, const double *q_raw, const double *k_raw, const double *v_raw,
                   int64_t g, double *out, int do_append);

#ifdef __cplusplus
}
#endif
#endif
