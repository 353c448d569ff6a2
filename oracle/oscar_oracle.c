/* ORACLE / TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference OScaR KV-cache path, written from the
 * reference's documented behaviour; each function cites the reference
 * file:line it restates (paths relative to /root/reference/proj).  Compiled
 * with -O2 -ffp-contract=off so fp64 rounding follows the reference's
 * (FMA-free, sequential) operation order.  Used only by tests/, smoke() and
 * bench.py's CPU legs as the checker; pinned against the compiled reference
 * (oracle/_ref) by tests/test_oracle.py.
 */
#include "oscar_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ---- hadamard.cpp:10-26 : Sylvester butterfly, half = 1,2,4,.., then
 * multiply by scale = 1/sqrt(d) ------------------------------------------ */
void oo_fht(double *v, int64_t d) {
    for (int64_t half = 1; half < d; half <<= 1) {
        for (int64_t base = 0; base < d; base += half << 1) {
            for (int64_t i = base; i < base + half; ++i) {
                const double a = v[i];
                const double b = v[i + half];
                v[i] = a + b;
                v[i + half] = a - b;
            }
        }
    }
    const double scale = 1.0 / sqrt((double)d);
    for (int64_t i = 0; i < d; ++i) v[i] *= scale;
}

/* ---- pipeline.cpp:80-88 ------------------------------------------------- */
double oo_fast_rsqrt(double x) {
    const float xf = (float)x;
    if (xf <= 0.0f || !isfinite(xf)) return 1.0 / sqrt(x);
    double y = (double)(1.0f / sqrtf(xf));
    y = y * (1.5 - 0.5 * x * y * y);
    return y;
}

/* ---- pipeline.cpp:90-148 : per-(token, head) scaling ------------------- */
int64_t oo_token_scale(const double *x, int64_t S, int64_t H, int64_t d, int strategy,
                       double *scaled, double *norms) {
    const double eps = 1e-12;
    int64_t degenerate = 0;
    for (int64_t t = 0; t < S; ++t) {
        for (int64_t h = 0; h < H; ++h) {
            const double *src = x + (t * H + h) * d;
            double s = 0.0, inv = 0.0;
            int zero = 1;
            for (int64_t c = 0; c < d; ++c)
                if (src[c] != 0.0) zero = 0; /* -0.0 counts as zero (line 101) */
            if (zero) {
                s = eps;
                inv = 1.0 / eps;
                ++degenerate;
            } else if (strategy == OO_L2) {
                double ss = 0.0;
                for (int64_t c = 0; c < d; ++c) ss += src[c] * src[c];
                s = sqrt(ss);
                inv = 1.0 / s;
            } else if (strategy == OO_RSQRT) {
                double ss = 0.0;
                for (int64_t c = 0; c < d; ++c) ss += src[c] * src[c];
                inv = oo_fast_rsqrt(ss);
                s = 1.0 / inv;
            } else if (strategy == OO_MAX) {
                double m = 0.0;
                for (int64_t c = 0; c < d; ++c) {
                    const double a = fabs(src[c]);
                    m = (m < a) ? a : m; /* std::max(m, a) */
                }
                s = m;
                inv = 1.0 / s;
            } else {
                double m = 0.0;
                for (int64_t c = 0; c < d; ++c) m += fabs(src[c]);
                s = m / (double)d;
                inv = 1.0 / s;
            }
            norms[t * H + h] = s;
            double *dst = scaled + (t * H + h) * d;
            for (int64_t c = 0; c < d; ++c) dst[c] = src[c] * inv;
        }
    }
    return degenerate;
}

/* ---- quant.cpp:21-47 : asymmetric params; zero point NOT clamped -------- */
void oo_quant_params(const double *v, int64_t n, int bits, double *delta, int64_t *zp,
                     double *constant) {
    double lo = v[0], hi = v[0];
    for (int64_t i = 0; i < n; ++i) {
        const double x = v[i];
        lo = (x < lo) ? x : lo; /* std::min(lo, x) keeps lo on ties */
        hi = (hi < x) ? x : hi; /* std::max(hi, x) keeps hi on ties */
    }
    if (hi == lo) {
        *delta = 0.0;
        *zp = 0;
        *constant = lo;
        return;
    }
    *delta = (hi - lo) / (double)((1LL << bits) - 1);
    *zp = llround(-lo / *delta);
    *constant = lo;
}

/* ---- quant.cpp:53-57 ---------------------------------------------------- */
uint16_t oo_quantize_one(double x, double delta, int64_t zp, int bits) {
    if (delta == 0.0) return 0;
    int64_t q = llround(x / delta) + zp;
    const int64_t mx = (1LL << bits) - 1;
    if (q < 0) q = 0;
    if (q > mx) q = mx;
    return (uint16_t)q;
}

/* ---- quant.cpp:65-68 ---------------------------------------------------- */
double oo_dequantize_one(uint16_t code, double delta, int64_t zp, double constant) {
    if (delta == 0.0) return constant;
    return delta * ((double)code - (double)zp);
}

/* ---- quant.cpp:162-183 : 8 codes per uint16, LSB first ----------------- */
void oo_pack_2bit(const uint16_t *codes, int64_t n, uint16_t *words) {
    memset(words, 0, sizeof(uint16_t) * (size_t)((n + 7) / 8));
    for (int64_t i = 0; i < n; ++i)
        words[i / 8] = (uint16_t)(words[i / 8] | (codes[i] << (2 * (i % 8))));
}

void oo_unpack_2bit(const uint16_t *words, int64_t n, uint16_t *codes) {
    for (int64_t i = 0; i < n; ++i) codes[i] = (uint16_t)((words[i / 8] >> (2 * (i % 8))) & 0x3);
}

/* ---- pipeline.cpp:152-180 (attend_one) + 184-198 (attention) ------------ */
static void attend_one(const double *q, const double *k, const double *v, int64_t S, int64_t H,
                       int64_t d, int64_t head, double *out) {
    const double temp = 1.0 / sqrt((double)d);
    double *logits = (double *)malloc(sizeof(double) * (size_t)(S > 0 ? S : 1));
    double mx = -HUGE_VAL;
    for (int64_t s = 0; s < S; ++s) {
        const double *kr = k + (s * H + head) * d;
        double dot = 0.0;
        for (int64_t c = 0; c < d; ++c) dot += q[c] * kr[c];
        logits[s] = dot * temp;
        mx = (mx < dot * temp) ? dot * temp : mx;
    }
    double z = 0.0;
    for (int64_t s = 0; s < S; ++s) {
        logits[s] = exp(logits[s] - mx);
        z += logits[s];
    }
    for (int64_t c = 0; c < d; ++c) out[c] = 0.0;
    for (int64_t s = 0; s < S; ++s) {
        const double w = logits[s] / z;
        const double *vr = v + (s * H + head) * d;
        for (int64_t c = 0; c < d; ++c) out[c] += w * vr[c];
    }
    free(logits);
}

void oo_attention(const double *q, int64_t Tq, const double *k, const double *v, int64_t S,
                  int64_t H, int64_t d, double *out) {
    for (int64_t i = 0; i < Tq * H; ++i) {
        const int64_t t = i / H, h = i % H;
        attend_one(q + (t * H + h) * d, k, v, S, H, d, h, out + (t * H + h) * d);
    }
}

/* ---- kv_cache.hpp:38-43 / 61-123 : the cache state machine -------------- */
typedef struct {
    int64_t nparams;
    double *delta, *constant;
    int64_t *zp;
    uint16_t *codes; /* d*R, reference order; NULL for raw blocks */
    double *raw;     /* R*d token-major when not quantizing */
} oo_block;

typedef struct {
    oo_block *b;
    int64_t n, cap;
} oo_blocks;

struct oo_cache {
    int method, bits, scaling, rotate_v;
    int64_t G, R, d, H;
    int k_prefilled, v_prefilled;
    int64_t packed_tokens, v_packed_tokens, flush_count;
    oo_blocks *kb, *vb; /* [H] */
    double **k_norms;   /* [H][packed] */
    int64_t *k_norms_n, *k_norms_cap;
    double *k_res, *k_norms_res, *v_res; /* capacity R rows */
    int64_t k_res_rows, v_res_rows;
};

static int rotates(const oo_cache *c) { return c->method == OO_ROTATE_ONLY || c->method == OO_OSCAR; }
static int scales(const oo_cache *c) { return c->method == OO_SCALE_ONLY || c->method == OO_OSCAR; }
static int quantizes(const oo_cache *c) { return c->method != OO_FP && c->bits != 0; }

oo_cache *oo_cache_create(int method, int bits, int64_t G, int64_t R, int scaling, int64_t d,
                          int64_t H, int rotate_v) {
    /* PipelineConfig::validate (kv_cache.cpp:51-67) */
    if (H <= 0 || d <= 0) return NULL;
    if (bits != 0 && bits != 2 && bits != 3 && bits != 4 && bits != 8 && bits != 16) return NULL;
    if (R <= 0 || G <= 0 || R % G != 0) return NULL;
    oo_cache *c = (oo_cache *)calloc(1, sizeof(oo_cache));
    c->method = method;
    c->bits = bits;
    c->scaling = scaling;
    c->rotate_v = rotate_v;
    c->G = G;
    c->R = R;
    c->d = d;
    c->H = H;
    if (quantizes(c) && d % G != 0) { free(c); return NULL; }
    if (rotates(c) && (d & (d - 1)) != 0) { free(c); return NULL; }
    c->kb = (oo_blocks *)calloc((size_t)H, sizeof(oo_blocks));
    c->vb = (oo_blocks *)calloc((size_t)H, sizeof(oo_blocks));
    c->k_norms = (double **)calloc((size_t)H, sizeof(double *));
    c->k_norms_n = (int64_t *)calloc((size_t)H, sizeof(int64_t));
    c->k_norms_cap = (int64_t *)calloc((size_t)H, sizeof(int64_t));
    c->k_res = (double *)malloc(sizeof(double) * (size_t)(R * H * d));
    c->k_norms_res = (double *)malloc(sizeof(double) * (size_t)(R * H));
    c->v_res = (double *)malloc(sizeof(double) * (size_t)(R * H * d));
    return c;
}

static void free_block(oo_block *b) {
    free(b->delta); free(b->constant); free(b->zp); free(b->codes); free(b->raw);
}

void oo_cache_destroy(oo_cache *c) {
    if (!c) return;
    for (int64_t h = 0; h < c->H; ++h) {
        for (int64_t i = 0; i < c->kb[h].n; ++i) free_block(&c->kb[h].b[i]);
        for (int64_t i = 0; i < c->vb[h].n; ++i) free_block(&c->vb[h].b[i]);
        free(c->kb[h].b); free(c->vb[h].b); free(c->k_norms[h]);
    }
    free(c->kb); free(c->vb); free(c->k_norms); free(c->k_norms_n); free(c->k_norms_cap);
    free(c->k_res); free(c->k_norms_res); free(c->v_res);
    free(c);
}

static oo_block *push_block(oo_blocks *bs) {
    if (bs->n == bs->cap) {
        bs->cap = bs->cap ? bs->cap * 2 : 16;
        bs->b = (oo_block *)realloc(bs->b, sizeof(oo_block) * (size_t)bs->cap);
    }
    oo_block *b = &bs->b[bs->n++];
    memset(b, 0, sizeof(*b));
    return b;
}

static void alloc_params(oo_block *b, int64_t n) {
    b->nparams = n;
    b->delta = (double *)malloc(sizeof(double) * (size_t)n);
    b->constant = (double *)malloc(sizeof(double) * (size_t)n);
    b->zp = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
}

/* kv_cache.cpp:101-129 + quant.cpp:76-101 : per-channel groups of G tokens;
 * params at [j*(R/G)+g], codes channel-major [j*R+t] */
static void flush_k_block(oo_cache *c, int64_t head, const double *rows, const double *norms) {
    const int64_t R = c->R, d = c->d, G = c->G;
    oo_block *blk = push_block(&c->kb[head]);
    if (!quantizes(c)) {
        blk->raw = (double *)malloc(sizeof(double) * (size_t)(R * d));
        memcpy(blk->raw, rows, sizeof(double) * (size_t)(R * d));
    } else {
        const int64_t groups = R / G;
        alloc_params(blk, d * groups);
        blk->codes = (uint16_t *)malloc(sizeof(uint16_t) * (size_t)(d * R));
        double *vals = (double *)malloc(sizeof(double) * (size_t)G);
        for (int64_t j = 0; j < d; ++j) {
            for (int64_t g = 0; g < groups; ++g) {
                for (int64_t i = 0; i < G; ++i) vals[i] = rows[(g * G + i) * d + j];
                const int64_t p = j * groups + g;
                oo_quant_params(vals, G, c->bits, &blk->delta[p], &blk->zp[p], &blk->constant[p]);
                for (int64_t i = 0; i < G; ++i)
                    blk->codes[j * R + g * G + i] =
                        oo_quantize_one(vals[i], blk->delta[p], blk->zp[p], c->bits);
            }
        }
        free(vals);
    }
    /* k_norms_grouped_ (kv_cache.cpp:127-128) */
    if (c->k_norms_n[head] + R > c->k_norms_cap[head]) {
        c->k_norms_cap[head] = 2 * (c->k_norms_n[head] + R);
        c->k_norms[head] = (double *)realloc(c->k_norms[head], sizeof(double) * (size_t)c->k_norms_cap[head]);
    }
    memcpy(c->k_norms[head] + c->k_norms_n[head], norms, sizeof(double) * (size_t)R);
    c->k_norms_n[head] += R;
}

/* kv_cache.cpp:131-157 + quant.cpp:103-128 : per-token groups of G channels;
 * params at [t*(d/G)+g], codes token-major [t*d+c] */
static void flush_v_block(oo_cache *c, int64_t head, const double *rows) {
    const int64_t R = c->R, d = c->d, G = c->G;
    oo_block *blk = push_block(&c->vb[head]);
    if (!quantizes(c)) {
        blk->raw = (double *)malloc(sizeof(double) * (size_t)(R * d));
        memcpy(blk->raw, rows, sizeof(double) * (size_t)(R * d));
        return;
    }
    const int64_t groups = d / G;
    alloc_params(blk, R * groups);
    blk->codes = (uint16_t *)malloc(sizeof(uint16_t) * (size_t)(R * d));
    for (int64_t t = 0; t < R; ++t) {
        for (int64_t g = 0; g < groups; ++g) {
            const double *vals = rows + t * d + g * G;
            const int64_t p = t * groups + g;
            oo_quant_params(vals, G, c->bits, &blk->delta[p], &blk->zp[p], &blk->constant[p]);
            for (int64_t i = 0; i < G; ++i)
                blk->codes[t * d + g * G + i] =
                    oo_quantize_one(vals[i], blk->delta[p], blk->zp[p], c->bits);
        }
    }
}

/* apply_method, key half (pipeline.cpp:224-236) */
static void transform_k(const oo_cache *c, const double *xk, int64_t S, double *k_out,
                        double *norms) {
    const int64_t H = c->H, d = c->d;
    double *tmp = (double *)malloc(sizeof(double) * (size_t)(S * H * d + 1));
    memcpy(tmp, xk, sizeof(double) * (size_t)(S * H * d));
    if (rotates(c))
        for (int64_t i = 0; i < S * H; ++i) oo_fht(tmp + i * d, d);
    if (scales(c)) {
        oo_token_scale(tmp, S, H, d, c->scaling, k_out, norms);
    } else {
        memcpy(k_out, tmp, sizeof(double) * (size_t)(S * H * d));
        for (int64_t i = 0; i < S * H; ++i) norms[i] = 1.0;
    }
    free(tmp);
}

/* KvCache::buffer_quant_k (kv_cache.cpp:194-250) */
static int buffer_quant_k(oo_cache *c, const double *k, const double *norms, int64_t S) {
    const int64_t R = c->R, d = c->d, H = c->H;
    double *rows = (double *)malloc(sizeof(double) * (size_t)(R * d));
    double *bn = (double *)malloc(sizeof(double) * (size_t)R);
    int rc = 0;
    if (!c->k_prefilled) {
        c->k_prefilled = 1;
        const int64_t r = S % R;
        /* pack_k_tokens (kv_cache.cpp:159-177): block-major, head-minor */
        for (int64_t b = 0; b < (S - r) / R; ++b) {
            for (int64_t h = 0; h < H; ++h) {
                for (int64_t t = 0; t < R; ++t) {
                    const int64_t tok = b * R + t;
                    memcpy(rows + t * d, k + (tok * H + h) * d, sizeof(double) * (size_t)d);
                    bn[t] = norms[tok * H + h];
                }
                flush_k_block(c, h, rows, bn);
            }
        }
        c->packed_tokens += S - r;
        for (int64_t t = S - r; t < S; ++t) {
            memcpy(c->k_res + c->k_res_rows * H * d, k + t * H * d, sizeof(double) * (size_t)(H * d));
            for (int64_t h = 0; h < H; ++h) c->k_norms_res[c->k_res_rows * H + h] = norms[t * H + h];
            ++c->k_res_rows;
        }
        goto done;
    }
    for (int64_t t = 0; t < S; ++t) {
        if (c->k_res_rows + 1 > R) { rc = 2; goto done; } /* logic_error, line 225-227 */
        memcpy(c->k_res + c->k_res_rows * H * d, k + t * H * d, sizeof(double) * (size_t)(H * d));
        for (int64_t h = 0; h < H; ++h) c->k_norms_res[c->k_res_rows * H + h] = norms[t * H + h];
        ++c->k_res_rows;
        if (c->k_res_rows == R) {
            for (int64_t h = 0; h < H; ++h) {
                for (int64_t i = 0; i < R; ++i) {
                    memcpy(rows + i * d, c->k_res + (i * H + h) * d, sizeof(double) * (size_t)d);
                    bn[i] = c->k_norms_res[i * H + h];
                }
                flush_k_block(c, h, rows, bn);
            }
            c->packed_tokens += R;
            ++c->flush_count;
            c->k_res_rows = 0;
        }
    }
done:
    free(rows);
    free(bn);
    return rc;
}

/* KvCache::buffer_quant_v (kv_cache.cpp:252-292) */
static int buffer_quant_v(oo_cache *c, const double *v, int64_t S) {
    const int64_t R = c->R, d = c->d, H = c->H;
    double *rows = (double *)malloc(sizeof(double) * (size_t)(R * d));
    int rc = 0;
    if (!c->v_prefilled) {
        c->v_prefilled = 1;
        const int64_t r = S % R;
        for (int64_t b = 0; b < (S - r) / R; ++b) {
            for (int64_t h = 0; h < H; ++h) {
                for (int64_t t = 0; t < R; ++t)
                    memcpy(rows + t * d, v + ((b * R + t) * H + h) * d, sizeof(double) * (size_t)d);
                flush_v_block(c, h, rows);
            }
        }
        c->v_packed_tokens += S - r;
        for (int64_t t = S - r; t < S; ++t) {
            memcpy(c->v_res + c->v_res_rows * H * d, v + t * H * d, sizeof(double) * (size_t)(H * d));
            ++c->v_res_rows;
        }
        goto done;
    }
    for (int64_t t = 0; t < S; ++t) {
        if (c->v_res_rows + 1 > R) { rc = 2; goto done; }
        memcpy(c->v_res + c->v_res_rows * H * d, v + t * H * d, sizeof(double) * (size_t)(H * d));
        ++c->v_res_rows;
        if (c->v_res_rows == R) {
            for (int64_t h = 0; h < H; ++h) {
                for (int64_t i = 0; i < R; ++i)
                    memcpy(rows + i * d, c->v_res + (i * H + h) * d, sizeof(double) * (size_t)d);
                flush_v_block(c, h, rows);
            }
            c->v_packed_tokens += R;
            c->v_res_rows = 0;
        }
    }
done:
    free(rows);
    return rc;
}

int oo_cache_append(oo_cache *c, const double *xk, const double *xv, int64_t S) {
    const int64_t H = c->H, d = c->d;
    double *k = (double *)malloc(sizeof(double) * (size_t)(S * H * d + 1));
    double *n = (double *)malloc(sizeof(double) * (size_t)(S * H + 1));
    transform_k(c, xk, S, k, n);
    int rc = buffer_quant_k(c, k, n, S);
    free(k);
    free(n);
    if (rc) return rc;
    double *v = (double *)malloc(sizeof(double) * (size_t)(S * H * d + 1));
    memcpy(v, xv, sizeof(double) * (size_t)(S * H * d));
    if (c->rotate_v)
        for (int64_t i = 0; i < S * H; ++i) oo_fht(v + i * d, d);
    rc = buffer_quant_v(c, v, S);
    free(v);
    return rc;
}

void oo_cache_stats(const oo_cache *c, int64_t *out4) {
    out4[0] = c->packed_tokens;
    out4[1] = c->k_res_rows;
    out4[2] = c->packed_tokens + c->k_res_rows;
    out4[3] = c->flush_count;
}

int64_t oo_cache_num_blocks(const oo_cache *c, int is_v, int64_t head) {
    return is_v ? c->vb[head].n : c->kb[head].n;
}

int64_t oo_cache_block(const oo_cache *c, int is_v, int64_t head, int64_t blk, uint16_t *codes,
                       double *delta, int64_t *zp, double *constant, double *raw) {
    const oo_block *b = is_v ? &c->vb[head].b[blk] : &c->kb[head].b[blk];
    const int64_t n = c->R * c->d;
    if (b->codes) {
        if (codes) memcpy(codes, b->codes, sizeof(uint16_t) * (size_t)n);
        if (delta) memcpy(delta, b->delta, sizeof(double) * (size_t)b->nparams);
        if (zp) memcpy(zp, b->zp, sizeof(int64_t) * (size_t)b->nparams);
        if (constant) memcpy(constant, b->constant, sizeof(double) * (size_t)b->nparams);
        return b->nparams;
    }
    if (raw) memcpy(raw, b->raw, sizeof(double) * (size_t)n);
    return 0;
}

void oo_cache_k_norms(const oo_cache *c, int64_t head, double *norms) {
    memcpy(norms, c->k_norms[head], sizeof(double) * (size_t)c->k_norms_n[head]);
}

void oo_cache_residual(const oo_cache *c, double *k_rows, double *k_norms, double *v_rows) {
    const int64_t H = c->H, d = c->d;
    if (k_rows) memcpy(k_rows, c->k_res, sizeof(double) * (size_t)(c->k_res_rows * H * d));
    if (k_norms) memcpy(k_norms, c->k_norms_res, sizeof(double) * (size_t)(c->k_res_rows * H));
    if (v_rows) memcpy(v_rows, c->v_res, sizeof(double) * (size_t)(c->v_res_rows * H * d));
}

/* unpack_block + materialize_k/v (kv_cache.cpp:297-381) */
void oo_cache_materialize(const oo_cache *c, double *k_out, double *v_out) {
    const int64_t R = c->R, d = c->d, H = c->H, G = c->G;
    const int64_t totk = c->packed_tokens + c->k_res_rows;
    (void)totk;
    for (int64_t h = 0; h < H; ++h) {
        for (int64_t b = 0; b < c->kb[h].n; ++b) {
            const oo_block *blk = &c->kb[h].b[b];
            for (int64_t t = 0; t < R; ++t) {
                const int64_t tok = b * R + t;
                const double s = c->k_norms[h][tok];
                for (int64_t j = 0; j < d; ++j) {
                    double x;
                    if (blk->raw) {
                        x = blk->raw[t * d + j];
                    } else {
                        const int64_t p = j * (R / G) + t / G;
                        x = oo_dequantize_one(blk->codes[j * R + t], blk->delta[p], blk->zp[p], blk->constant[p]);
                    }
                    k_out[(tok * H + h) * d + j] = x * s;
                }
            }
        }
        for (int64_t b = 0; b < c->vb[h].n; ++b) {
            const oo_block *blk = &c->vb[h].b[b];
            for (int64_t t = 0; t < R; ++t) {
                for (int64_t j = 0; j < d; ++j) {
                    double x;
                    if (blk->raw) {
                        x = blk->raw[t * d + j];
                    } else {
                        const int64_t p = t * (d / G) + j / G;
                        x = oo_dequantize_one(blk->codes[t * d + j], blk->delta[p], blk->zp[p], blk->constant[p]);
                    }
                    v_out[((b * R + t) * H + h) * d + j] = x;
                }
            }
        }
    }
    for (int64_t t = 0; t < c->k_res_rows; ++t)
        for (int64_t h = 0; h < H; ++h) {
            const double s = c->k_norms_res[t * H + h];
            for (int64_t j = 0; j < d; ++j)
                k_out[((c->packed_tokens + t) * H + h) * d + j] = c->k_res[(t * H + h) * d + j] * s;
        }
    for (int64_t t = 0; t < c->v_res_rows; ++t)
        memcpy(v_out + (c->v_packed_tokens + t) * H * d, c->v_res + t * H * d, sizeof(double) * (size_t)(H * d));
}

/* decode_step body (pipeline.cpp:292-323) without projections */
int oo_decode_step(oo_cache *c, const double *q_raw, const double *k_raw, const double *v_raw,
                   int64_t g, double *out, int do_append) {
    const int64_t H = c->H, d = c->d;
    const int64_t hist = c->packed_tokens + c->k_res_rows, total = hist + 1;
    double *kall = (double *)malloc(sizeof(double) * (size_t)(total * H * d));
    double *vall = (double *)malloc(sizeof(double) * (size_t)(total * H * d));
    oo_cache_materialize(c, kall, vall);
    double *kt = (double *)malloc(sizeof(double) * (size_t)(H * d));
    double *nt = (double *)malloc(sizeof(double) * (size_t)H);
    transform_k(c, k_raw, 1, kt, nt);
    double *vt = (double *)malloc(sizeof(double) * (size_t)(H * d));
    memcpy(vt, v_raw, sizeof(double) * (size_t)(H * d));
    if (c->rotate_v)
        for (int64_t h = 0; h < H; ++h) oo_fht(vt + h * d, d);
    for (int64_t h = 0; h < H; ++h) {
        for (int64_t j = 0; j < d; ++j) kall[(hist * H + h) * d + j] = kt[h * d + j] * nt[h];
        memcpy(vall + (hist * H + h) * d, vt + h * d, sizeof(double) * (size_t)d);
    }
    double *q = (double *)malloc(sizeof(double) * (size_t)(g * H * d));
    for (int64_t h = 0; h < H; ++h)
        for (int64_t j = 0; j < g; ++j) {
            memcpy(q + (j * H + h) * d, q_raw + (h * g + j) * d, sizeof(double) * (size_t)d);
            if (rotates(c)) oo_fht(q + (j * H + h) * d, d);
        }
    double *o = (double *)malloc(sizeof(double) * (size_t)(g * H * d));
    oo_attention(q, g, kall, vall, total, H, d, o);
    for (int64_t h = 0; h < H; ++h)
        for (int64_t j = 0; j < g; ++j)
            memcpy(out + (h * g + j) * d, o + (j * H + h) * d, sizeof(double) * (size_t)d);
    int rc = 0;
    if (do_append) {
        rc = buffer_quant_k(c, kt, nt, 1);
        if (!rc) rc = buffer_quant_v(c, vt, 1);
    }
    free(kall); free(vall); free(kt); free(nt); free(vt); free(q); free(o);
    return rc;
}
