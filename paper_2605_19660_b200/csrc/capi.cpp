// capi.cpp -- host runtime behind include/oscar_kv.h.
//
// Mirrors the reference KvCache state machine (kv_cache.cpp:194-292) on the
// host (token counters only -- every sequence of a handle advances together)
// and drives the device kernels:
//   prefill      -> quantize kernel over the S - S mod R full blocks + ring copy
//   append       -> ring copy, flush (quantize kernel from the ring) at exactly R
//   decode_step  -> ONE attention kernel (attends cache + current token, writes
//                   the current token into the ring) [+ flush kernel when the
//                   window fills, after the attention -- pipeline.cpp:294-323]
// and converts the device cache back into the reference's layout (export,
// KVC1 dump, materialize).  Compiled with -ffp-contract=off.
#include <cuda_runtime.h>

#ifndef OSK_PROF
#define OSK_PROF 0
#endif

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <memory>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/oscar_kv.h"
#include "host_ref.h"
#include "kernels.h"
#include "layout.h"
#include "split.h"

using namespace osk;

namespace {

thread_local std::string g_err;

struct InvalidArg : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct LogicErr : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct CudaErr : std::runtime_error {
    using std::runtime_error::runtime_error;
};

#define CK(x)                                                                                       \
    do {                                                                                            \
        cudaError_t e_ = (x);                                                                       \
        if (e_ != cudaSuccess) throw CudaErr(std::string(#x) + ": " + cudaGetErrorString(e_));    \
    } while (0)

template <typename F>
int guard(F &&f) {
    try {
        f();
        return 0;
    } catch (const InvalidArg &e) {
        g_err = e.what();
        return 1;
    } catch (const LogicErr &e) {
        g_err = e.what();
        return 2;
    } catch (const std::exception &e) {
        g_err = e.what();
        return 3;
    }
}

bool rotates(const oscar_kv_config &c) { return c.method == OSCAR_ROTATE_ONLY || c.method == OSCAR_OSCAR; }
bool scales(const oscar_kv_config &c) { return c.method == OSCAR_SCALE_ONLY || c.method == OSCAR_OSCAR; }
bool quantizes(const oscar_kv_config &c) { return c.method != OSCAR_FP && c.bits != 0; }

void validate(const oscar_kv_config &c) {
    // PipelineConfig::validate (kv_cache.cpp:51-67)
    if (c.heads <= 0 || c.head_dim <= 0) throw InvalidArg("config: heads and head_dim must be positive");
    if (c.bits != 0 && c.bits != 2 && c.bits != 3 && c.bits != 4 && c.bits != 8 && c.bits != 16)
        throw InvalidArg("config: bits must be one of 0,2,3,4,8,16");
    if (c.residual_len <= 0 || c.group_size <= 0 || c.residual_len % c.group_size != 0)
        throw InvalidArg("config: residual_len must be a positive multiple of group_size");
    if (quantizes(c) && c.head_dim % c.group_size != 0)
        throw InvalidArg("config: head_dim must be divisible by group_size for the value path");
    if (rotates(c) && (c.head_dim & (c.head_dim - 1)) != 0)
        throw InvalidArg("config: head_dim must be a power of two when rotating");
    if (c.method < 0 || c.method > 4) throw InvalidArg("config: unknown method");
    if (c.scaling < 0 || c.scaling > 3) throw InvalidArg("config: unknown scaling strategy");
    // device kernel limits
    if (c.head_dim != D) throw InvalidArg("device: head_dim must be 128");
    if (c.residual_len != R) throw InvalidArg("device: residual_len must be 128");
    if (quantizes(c) && c.group_size != G) throw InvalidArg("device: group_size must be 32");
    if (quantizes(c) && c.bits != 2 && c.bits != 4) throw InvalidArg("device: bits must be 0, 2 or 4");
}

}  // namespace

struct oscar_kv_handle {
    oscar_kv_config cfg{};
    int dbits = 0;  // 0, 2, 4 (effective device format)
    int64_t B = 0, Hq = 0, g = 0, BH = 0, max_tokens = 0, max_blocks = 0;
    int device = 0, num_sms = 148;
    bool keep_exact = true;
    int64_t block_bytes = 0;
    // state (kv_cache.hpp:104-122), uniform over the batch
    bool prefilled = false;
    int64_t packed = 0, residual = 0, flushes = 0;
    // input form, fixed by the first append: 1 = raw bf16 rows (append / decode_step:
    // the key transform runs on the device), 2 = the reference's own form (append_k /
    // append_v / decode_step_f64: transformed fp64 keys + norms, fp64 values).  In
    // form 2 the K and V streams advance separately like k_/v_ state of the
    // reference (kv_cache.hpp:104-122): packed / residual / prefilled count keys,
    // v_packed / v_residual / v_prefilled values.
    int form = 0;
    bool v_prefilled = false;
    int64_t v_packed = 0, v_residual = 0;
    // form 2: the exact residual window (fp64 K_u rows [bh][R][D], norms [bh][R], V rows);
    // the rings hold their bf16 image for the decode kernel
    double *res_k = nullptr, *res_n = nullptr, *res_v = nullptr;
    // device memory
    uint8_t *blocks = nullptr;
    double *shadow = nullptr;
    void *ring_k = nullptr, *ring_v = nullptr;
    uint64_t *part_o = nullptr, *part_ml = nullptr;  // flag-in-word split-KV partials, zero between launches
    int *counters = nullptr;
    int *status_d = nullptr;  // device status word (kernels.h STATUS_*)
    float *warp_part = nullptr;
    int maxp_alloc = 0;
    int maxseg_alloc = 1;
    int64_t scratch_slots = 0;  // (CTA, segment) warp-partial slots in warp_part
    static constexpr int64_t kMaxSegments = 64;  // attention.cu MAXSEG_SMEM
    void *stage = nullptr;  // host-API staging: q, k, v, out, lse
    int64_t device_bytes = 0;
    int last_launches = 0;
    cudaStream_t last_stream = nullptr;
    // a quantize kernel wrote packed records since the last attention launch:
    // the next attention launch must not prefetch them ahead of griddepcontrol.wait
    bool blocks_written = true;
    // launch plan of the last attention launch shape (nb, tail charge): the grid
    // and the CTA-range checks only change when a flush adds a block or the
    // residual window empties, so the per-step host cost is one comparison
    struct Plan {
        int64_t nb = -1, tail_cost = -1;
        int ncta = 0;
    } plan;

    TransformCfg tc() const {
        TransformCfg t;
        t.bits = dbits;
        t.rotates = rotates(cfg);
        t.scales = scales(cfg);
        t.scaling = cfg.scaling;
        t.rotate_v = cfg.rotate_v;
        return t;
    }

    void *dalloc(size_t bytes) {
        void *p = nullptr;
        CK(cudaMalloc(&p, bytes));
        device_bytes += (int64_t)bytes;
        return p;
    }

    ~oscar_kv_handle() {
        cudaSetDevice(device);
        cudaFree(blocks);
        cudaFree(shadow);
        cudaFree(ring_k);
        cudaFree(ring_v);
        cudaFree(res_k);
        cudaFree(res_n);
        cudaFree(res_v);
        cudaFree(part_o);
        cudaFree(part_ml);
        cudaFree(counters);
        cudaFree(status_d);
        cudaFree(warp_part);
        cudaFree(stage);
    }

    // a new launch plan can turn a (b, kv head)'s split-KV merge from the ticket
    // form (fp32 partials) into the poll form (flag-in-word partials, zero = not
    // written): the partial words are cleared once before the first launch of a plan
    bool partials_dirty = false;
    bool sync_entry = false;  // inside oscar_kv_decode_step_host (one synchronous step per call)
    void launch_attn(const AttnArgs &a, cudaStream_t s) {
        if (partials_dirty) {
            CK(cudaMemsetAsync(part_o, 0, sizeof(uint64_t) * (size_t)(BH * maxp_alloc * 8 * D), s));
            CK(cudaMemsetAsync(part_ml, 0, sizeof(uint64_t) * (size_t)(BH * maxp_alloc * 16), s));
            partials_dirty = false;
        }
        CK(launch_attention(dbits, a, s));
    }

    void alloc_partials() {  // zeroed: a zero word is "not written" (attention.cu final_merge)
        const size_t no = (size_t)(BH * maxp_alloc * 8 * D), nm = (size_t)(BH * maxp_alloc * 16);
        part_o = (uint64_t *)dalloc(sizeof(uint64_t) * no);
        part_ml = (uint64_t *)dalloc(sizeof(uint64_t) * nm);
        CK(cudaMemset(part_o, 0, sizeof(uint64_t) * no));
        CK(cudaMemset(part_ml, 0, sizeof(uint64_t) * nm));
    }

    void grow_scratch(int64_t slots, int64_t maxseg) {  // synchronous, rare (shape changes)
        if (warp_part) {
            CK(cudaDeviceSynchronize());
            cudaFree(warp_part);
            device_bytes -= sizeof(float) * attention_scratch_floats(scratch_slots);
        }
        scratch_slots = slots;
        maxseg_alloc = (int)maxseg;
        warp_part = (float *)dalloc(sizeof(float) * (size_t)attention_scratch_floats(scratch_slots));
    }

    // ---- kernels --------------------------------------------------------------
    void quantize_from(const void *k, const void *v, int64_t sb, int64_t st, int64_t sh, int64_t tok0,
                       int64_t nblk, int64_t blk0, cudaStream_t s, int64_t vst = -1, int64_t vsc = 1,
                       int64_t ring_prefix = 0) {
        QuantizeArgs a{};
        a.k = k;
        a.v = v;
        a.sb = sb;
        a.st = st;
        a.sh = sh;
        a.tok0 = tok0;
        a.vst = vst < 0 ? st : vst;
        a.vsc = vsc;
        a.B = (int)B;
        a.H = (int)cfg.heads;
        a.n_blocks = nblk;
        a.blocks = blocks;
        a.max_blocks = max_blocks;
        a.blk0 = blk0;
        a.shadow = shadow;
        a.tc = tc();
        a.status = status_d;
        if (ring_prefix > 0) {
            a.rk = ring_k;
            a.rv = ring_v;
            a.rtok = ring_prefix;
        }
        CK(launch_quantize(a, s));
        ++last_launches;
        blocks_written = true;
    }
    void ring_copy(const void *k, const void *v, int64_t sb, int64_t st, int64_t sh, int64_t tok0, int64_t n,
                   int64_t slot0, cudaStream_t s) {
        RingCopyArgs a{};
        a.k = k;
        a.v = v;
        a.sb = sb;
        a.st = st;
        a.sh = sh;
        a.tok0 = tok0;
        a.B = (int)B;
        a.H = (int)cfg.heads;
        a.n = n;
        a.ring_k = ring_k;
        a.ring_v = ring_v;
        a.slot0 = slot0;
        CK(launch_ring_copy(a, s));
        ++last_launches;
    }
    void flush(cudaStream_t s) {
        // the rings are the source of one block per (b, h): K [bh][R][D], V [bh][D][R]
        const int64_t H = cfg.heads;
        quantize_from(ring_k, ring_v, H * R * D, D, (int64_t)R * D, 0, 1, packed / R, s, /*vst=*/0, /*vsc=*/0);
        packed += R;
        residual = 0;
    }

    void append(const void *k, const void *v, int64_t n, cudaStream_t s) {
        const int64_t H = cfg.heads;
        if (n < 0) throw InvalidArg("append: negative token count");
        use_form(1);
        if (packed + residual + n > max_tokens) throw InvalidArg("append: cache capacity exceeded");
        last_launches = 0;
        const int64_t sb = n * H * D, st = H * D, sh = D;
        if (!prefilled) {
            // prefill branch (kv_cache.cpp:204-218)
            prefilled = true;
            const int64_t r = n % R;
            const int64_t nfull = (n - r) / R;
            if (nfull > 0) quantize_from(k, v, sb, st, sh, 0, nfull, 0, s);
            packed += n - r;
            if (r > 0) ring_copy(k, v, sb, st, sh, n - r, r, 0, s);
            residual = r;
            return;
        }
        // decode branch (kv_cache.cpp:219-249): token by token, flush at exactly R.
        // Equivalent batched form: top up the open window (flush it if it fills),
        // quantize every following whole R-block straight from the input -- the
        // same R-aligned token groups the token-by-token flushes would produce, so
        // the cache is bit-identical -- and leave the remainder in the window.
        int64_t pos = 0;
        if (residual + n < R) {  // stays inside the open window
            ring_copy(k, v, sb, st, sh, 0, n, residual, s);
            residual += n;
            return;
        }
        // the window's residual tokens + the input complete nblk blocks: one launch
        // whose block 0 reads its first `residual` tokens from the rings
        const int64_t nblk = (residual + n) / R;
        quantize_from(k, v, sb, st, sh, 0, nblk, packed / R, s, -1, 1, residual);
        pos = nblk * R - residual;
        packed += nblk * R;
        flushes += nblk;
        residual = 0;
        if (pos < n) {
            ring_copy(k, v, sb, st, sh, pos, n - pos, 0, s);
            residual = n - pos;
        }
    }

    // ---- input form ----------------------------------------------------------------
    void use_form(int f) {
        if (form == f) return;
        if (form != 0)
            throw LogicErr(f == 2 ? "fp64 appends: this cache holds raw bf16 appends (one input form per cache)"
                                  : "raw bf16 appends: this cache holds fp64 appends (one input form per cache)");
        if (f == 2) {
            if (!quantizes(cfg)) throw InvalidArg("fp64 appends need a quantising config (bits 2 or 4)");
            if (cfg.rotate_v)
                throw InvalidArg("fp64 appends store value rows as given; explicit-V mode (rotate_v) is for raw appends");
            res_k = (double *)dalloc(sizeof(double) * (size_t)(BH * R * D));
            res_n = (double *)dalloc(sizeof(double) * (size_t)(BH * R));
            res_v = (double *)dalloc(sizeof(double) * (size_t)(BH * R * D));
        }
        form = f;
    }
    void in_step(const char *what) const {
        if (form == 2 && (packed != v_packed || residual != v_residual))
            throw LogicErr(std::string(what) + ": key and value streams hold different token counts");
    }
    void quantize_f64(int part, F64Src src, F64Src nrm, int64_t tok0, int64_t nblk, int64_t blk0, cudaStream_t s) {
        QuantizeF64Args a{};
        a.src = src;
        a.norms = nrm;
        a.part = part;
        a.bits = dbits;
        a.B = (int)B;
        a.H = (int)cfg.heads;
        a.tok0 = tok0;
        a.n_blocks = nblk;
        a.blocks = blocks;
        a.max_blocks = max_blocks;
        a.blk0 = blk0;
        a.shadow = shadow;
        a.status = status_d;
        CK(launch_quantize_f64(a, s));
        ++last_launches;
        blocks_written = true;
    }
    void window_f64(int part, F64Src src, F64Src nrm, int64_t tok0, int64_t n, int64_t slot0, cudaStream_t s) {
        WindowF64Args a{};
        a.src = src;
        a.norms = nrm;
        a.part = part;
        a.B = (int)B;
        a.H = (int)cfg.heads;
        a.tok0 = tok0;
        a.n = n;
        a.slot0 = slot0;
        a.rotates = rotates(cfg);
        a.scales = scales(cfg);
        a.res_k = res_k;
        a.res_n = res_n;
        a.res_v = res_v;
        a.ring_k = ring_k;
        a.ring_v = ring_v;
        CK(launch_window_f64(a, s));
        ++last_launches;
    }
    // buffer_quant_k (kv_cache.cpp:194-249) / buffer_quant_v (251-292) on fp64 rows:
    // part 0 = transformed keys [B, n, H, d] + norms [B, n, H], part 1 = values [B, n, H, d]
    void append_f64(int part, const double *x, const double *norms, int64_t n, cudaStream_t s) {
        use_form(2);
        const int64_t H = cfg.heads;
        if (n < 0) throw InvalidArg("append: negative token count");
        bool &pre = part == 0 ? prefilled : v_prefilled;
        int64_t &pk = part == 0 ? packed : v_packed;
        int64_t &res = part == 0 ? residual : v_residual;
        if (pk + res + n > max_tokens) throw InvalidArg("append: cache capacity exceeded");
        last_launches = 0;
        const F64Src src{x, n * H * D, D, H * D};
        const F64Src nrm{norms, n * H, 1, H};
        if (!pre) {  // prefill branch: pack S - r tokens, keep r = S mod R (kv_cache.cpp:204-218)
            pre = true;
            const int64_t r = n % R;
            if (n - r > 0) quantize_f64(part, src, nrm, 0, (n - r) / R, 0, s);
            pk += n - r;
            if (r > 0) window_f64(part, src, nrm, n - r, r, 0, s);
            res = r;
            return;
        }
        // decode branch: token by token, a flush at exactly R (kv_cache.cpp:219-249)
        for (int64_t pos = 0; pos < n;) {
            const int64_t take = std::min<int64_t>(n - pos, R - res);
            window_f64(part, src, nrm, pos, take, res, s);
            res += take;
            pos += take;
            if (res == R) flush_f64(part, s);
        }
    }
    // flush_k_block / flush_v_block of the full window (the exact fp64 residual)
    void flush_f64(int part, cudaStream_t s) {
        const int64_t H = cfg.heads;
        int64_t &pk = part == 0 ? packed : v_packed;
        int64_t &res = part == 0 ? residual : v_residual;
        const F64Src src{part == 0 ? res_k : res_v, H * R * D, R * D, D};
        const F64Src nrm{res_n, H * R, R, 1};
        quantize_f64(part, src, nrm, 0, 1, pk / R, s);
        pk += R;
        res = 0;
        if (part == 0) ++flushes;
    }
    // decode_step (pipeline.cpp:292-323) with the current token in the reference's
    // form: appended to both windows, attended over history + current at full
    // precision, then the flush at R
    void decode_step_f64(const void *q, const double *kt, const double *kn, const double *v, float *out, float *lse,
                         cudaStream_t s) {
        use_form(2);
        in_step("decode_step");
        if (packed + residual + 1 > max_tokens) throw InvalidArg("decode_step: cache capacity exceeded");
        if (!prefilled) throw LogicErr("decode_step: empty cache (prefill first)");
        const int64_t H = cfg.heads;
        last_launches = 0;
        window_f64(0, F64Src{kt, H * D, D, H * D}, F64Src{kn, H, 1, H}, 0, 1, residual, s);
        window_f64(1, F64Src{v, H * D, D, H * D}, F64Src{nullptr, 0, 0, 0}, 0, 1, residual, s);
        residual += 1;
        v_residual += 1;
        const int launches = last_launches;
        AttnArgs a = attn_args(q, nullptr, nullptr, out, lse);
        launch_attn(a, s);
        last_launches = launches + 1;
        blocks_written = false;
        if (residual == R) {
            flush_f64(0, s);
            flush_f64(1, s);
        }
    }

    AttnArgs attn_args(const void *q, const void *kc, const void *vc, float *out, float *lse) {
        AttnArgs a{};
        a.blocks = blocks;
        a.max_blocks = max_blocks;
        a.nb = packed / R;
        a.BH = (int)BH;
        a.Hkv = (int)cfg.heads;
        a.g = (int)g;
        a.Hq = (int)Hq;
        a.q = q;
        a.kcur = kc;
        a.vcur = vc;
        a.ring_k = ring_k;
        a.ring_v = ring_v;
        a.r = (int)residual;
        a.write_ring = kc != nullptr;
        a.ring_f16 = form == 2;
        a.rotates = dbits != 0 && rotates(cfg);
        a.scales = scales(cfg);
        a.rotate_v = dbits != 0 && cfg.rotate_v;
        a.out = out;
        a.lse = lse;
        a.part_o = part_o;
        a.part_ml = part_ml;
        a.counters = counters;
        a.status = status_d;
        a.warp_part = warp_part;
        a.maxseg = maxseg_alloc;
        a.ncta = attention_grid(dbits, num_sms, a.nb, a.BH);
        {
            static const int64_t sc = env_knob("OSCAR_SEG_COST", 3);  // per-segment split weight (tuning knob)
            a.seg_cost = sc;
            // the residual-window tiles (one 16-token tile per warp of the tail owner)
            // cost that CTA about half a unit per warp: charge it OSCAR_TAIL_COST units
            static const int64_t tcost = env_knob("OSCAR_TAIL_COST", 6);
            const int ntok = (int)residual + (kc ? 1 : 0);
            a.tail_cost = ntok > 0 ? tcost : 0;
        }
        a.pdl_prefetch = blocks_written ? 0 : 1;
        {
            static const long perm = env_knob("OSCAR_CTA_PERM", 0);  // experiments: block -> range permutation
            a.cta_perm = 0;
            if (perm > 1) {
                int64_t x = perm % a.ncta, y = a.ncta;  // coprime check
                while (y) {
                    const int64_t t = x % y;
                    x = y;
                    y = t;
                }
                if (x == 1) a.cta_perm = (int)perm;
            }
        }
        a.maxp = maxp_alloc;
        // poll-mode merge needs every CTA resident at once (one CTA per SM)
        static const long poll_knob = env_knob("OSCAR_POLL_MERGE", 1);  // 0: atomic tickets always (A/B)
        if (a.nb > 0 && plan.nb == a.nb && plan.tail_cost == a.tail_cost) {
            a.ncta = plan.ncta;  // same shape as the last launch: its checks hold
        } else if (a.nb > 0) {
            const int64_t nbs = a.nb * (dbits == 0 ? 4 : 1);  // pipeline units per (b, kv head)
            // segments (b, kv heads) per CTA range; a CTA holds at most MAX_SEGMENTS of them
            // (shared-memory ticket table), so large batches of short sequences get a grid
            // of more CTAs than SMs (they run in waves) instead of being rejected
            auto max_segments = [&](const Split &sp) {
                int64_t nseg = 0;
                for (int64_t c = 0; c < sp.ncta; ++c) {
                    const int64_t st = sp.begin(c), en = sp.end(c);
                    if (en > st) nseg = std::max(nseg, (en - 1) / nbs - st / nbs + 1);
                }
                return nseg;
            };
            Split sp{nbs, a.BH, a.ncta, a.seg_cost, a.tail_cost};
            int64_t nseg = max_segments(sp);
            while (nseg > kMaxSegments) {
                a.ncta = (int)std::min<int64_t>((int64_t)a.BH * nbs, (a.ncta * nseg + kMaxSegments - 9) / (kMaxSegments - 8));
                sp.ncta = a.ncta;
                nseg = max_segments(sp);
            }
            // exact split-KV partial-slot requirement
            int64_t need = 0;
            for (int64_t bh = 0; bh < a.BH; ++bh)
                need = std::max(need, sp.cta_of((bh + 1) * nbs - 1) - sp.cta_of(bh * nbs) + 1);
            if (need > maxp_alloc) {  // rare: grow the split-KV partial buffers (synchronous)
                CK(cudaDeviceSynchronize());
                cudaFree(part_o);
                cudaFree(part_ml);
                device_bytes -= sizeof(uint64_t) * (int64_t)BH * maxp_alloc * (8 * D + 16);
                maxp_alloc = (int)need;
                alloc_partials();
                a.part_o = part_o;
                a.part_ml = part_ml;
                a.maxp = maxp_alloc;
            }
            // per-(CTA, segment) warp-partial scratch: the kernel indexes slot cta * maxseg + k
            const int64_t maxseg = std::max<int64_t>(nseg, maxseg_alloc);
            if (nseg > maxseg_alloc || (int64_t)a.ncta * maxseg > scratch_slots)
                grow_scratch(std::max<int64_t>((int64_t)a.ncta * maxseg, scratch_slots), maxseg);
            a.warp_part = warp_part;
            a.maxseg = maxseg_alloc;
            plan.nb = a.nb;
            plan.tail_cost = a.tail_cost;
            plan.ncta = a.ncta;
            partials_dirty = true;
        } else {
            a.maxseg = 1;  // residual-only mode: one segment per CTA (ncta = BH <= scratch slots)
        }
        a.poll_merge = (poll_knob != 0 && a.ncta <= num_sms) ? 1 : 0;
        {
            // the window's tiles ride the ring as pipeline units (the TILES kernel) where that
            // measured faster (profiles/r02/ab_tiles_*): small launches (<= 2 records per
            // warp), launches of 1.5-4 (b, kv head) segments per CTA (C3 B=64 -1.4 %, the C3
            // 2-rank shard -4.8 %; at C3 B=256's 7 it is 3 % slower), and the synchronous
            // host-buffer entry (a cold launch: the tiles' own loads would queue behind the
            // ring fill) up to 4 segments per CTA.  Bulk copies need 16-byte aligned sources.
            // OSCAR_TILE_UNITS=0: never, 2: for every launch (A/B)
            static const long tu = env_knob("OSCAR_TILE_UNITS", 1);
            auto al16 = [](const void *p) { return p == nullptr || ((uintptr_t)p & 15) == 0; };
            const bool small = a.nb > 0 && a.nb * BH <= (int64_t)24 * a.ncta;
            const bool le4 = BH <= (int64_t)4 * a.ncta;
            const bool segs = 2 * BH >= (int64_t)3 * a.ncta && le4;
            a.tile_units = (tu != 0 && (dbits == 2 || dbits == 4) && !cfg.rotate_v && form != 2 && a.nb > 0 &&
                            (small || segs || (sync_entry && le4) || tu == 2) && al16(a.q) && al16(a.kcur) &&
                            al16(a.vcur))
                               ? 1
                               : 0;
        }
        return a;
    }

    // StepOutput.logits over the cache contents (+ the current token when k is given)
    void logits(const void *q, const void *k, float *out, cudaStream_t s) {
        LogitsArgs a{};
        a.blocks = blocks;
        a.max_blocks = max_blocks;
        a.block_bytes = block_bytes;
        a.nb = packed / R;
        a.BH = (int)BH;
        a.Hkv = (int)cfg.heads;
        a.g = (int)g;
        a.Hq = (int)Hq;
        a.q = q;
        a.kcur = k;
        a.ring_k = ring_k;
        a.ring_f16 = form == 2;
        a.r = (int)residual;
        a.rotates = dbits != 0 && rotates(cfg);
        a.logits = out;
        a.s_total = packed + residual + (k ? 1 : 0);
        CK(launch_logits(dbits, a, s));
        ++last_launches;
    }

    void decode_step(const void *q, const void *k, const void *v, float *out, float *lse, cudaStream_t s,
                     const PeerPlan *pub = nullptr, uint32_t epoch = 0, float *logits_out = nullptr) {
        if (packed + residual + 1 > max_tokens) throw InvalidArg("decode_step: cache capacity exceeded");
        use_form(1);
        last_launches = 0;
        // the logits read the window and the records before the attention kernel
        // writes the current token into the ring and before any flush
        if (logits_out) logits(q, k, logits_out, s);
        AttnArgs a = attn_args(q, k, v, out, lse);
        if (pub) {
            a.pub = *pub;
            a.pub_epoch = epoch;
        }
        launch_attn(a, s);
        ++last_launches;
        blocks_written = false;
        // buffer_quant_k/v of the current token (written into the ring by the kernel)
        prefilled = true;
        residual += 1;
        if (residual == R) {
            flush(s);
            ++flushes;
        }
    }

    void attend(const void *q, float *out, float *lse, cudaStream_t s, const PeerPlan *pub = nullptr,
                uint32_t epoch = 0) {
        last_launches = 0;
        if (packed + residual == 0) throw LogicErr("attend: empty cache");
        in_step("attend");
        AttnArgs a = attn_args(q, nullptr, nullptr, out, lse);
        if (pub) {
            a.pub = *pub;
            a.pub_epoch = epoch;
        }
        // debug: OSCAR_PROF=1 prints per-phase cycles averaged over warps (synchronises)
        static const int prof = [] {
            const int p = getenv("OSCAR_PROF") ? 1 : 0;
#if !OSK_PROF
            if (p) std::fprintf(stderr, "OSCAR_PROF: counters need the profiling build (make PROF=1, "
                                        "OSCAR_LIB=.../liboscar_b200_prof.so); ignored\n");
            return 0;
#else
            return p;
#endif
        }();
        unsigned long long *pbuf = nullptr;
        const int nw = a.ncta * 16;
        if (prof) {
            CK(cudaMalloc(&pbuf, sizeof(unsigned long long) * kProfStride * nw));
            CK(cudaMemsetAsync(pbuf, 0, sizeof(unsigned long long) * kProfStride * nw, s));
            a.prof = pbuf;
        }
        launch_attn(a, s);
        ++last_launches;
        blocks_written = false;
        if (prof) {
            std::vector<unsigned long long> hbuf(kProfStride * nw);
            CK(cudaMemcpyAsync(hbuf.data(), pbuf, hbuf.size() * 8, cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
            double acc[13] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
            double mx = 0, fmax = 0;
            int cnt = 0;
            for (int w = 0; w < nw; ++w) {
                if (hbuf[kProfStride * w + 8] == 0) continue;
                ++cnt;
                for (int i = 0; i < 13; ++i) acc[i] += (double)hbuf[kProfStride * w + i];
                mx = std::max(mx, (double)hbuf[kProfStride * w + 8]);
                fmax = std::max(fmax, (double)hbuf[kProfStride * w + 12]);
            }
            {
                // per-CTA spread: slowest warp per CTA, min/max across CTAs
                double cmin = 1e30, cmax = 0, wspread = 0;
                int ncta_used = 0;
                for (int c = 0; c < a.ncta; ++c) {
                    double lo = 1e30, hi = 0;
                    for (int w = 0; w < 16; ++w) {
                        const double t = (double)hbuf[kProfStride * (c * 16 + w) + 8];
                        if (t == 0) continue;
                        lo = std::min(lo, t);
                        hi = std::max(hi, t);
                    }
                    if (hi == 0) continue;
                    ++ncta_used;
                    cmin = std::min(cmin, hi);
                    cmax = std::max(cmax, hi);
                    wspread += (hi - lo);
                }
                if (const char *fn = getenv("OSCAR_PROF_FILE")) {  // per-CTA: range, segments, tails, smid, cycles
                    if (FILE *f = std::fopen(fn, "w")) {
                        std::fprintf(f, "cta,smid,units,segments,tails,slowest_warp_cycles,cta_merge,ticket,final_merge,"
                                        "entry_ns,stream_end_ns,exit_ns\n");
                        unsigned long long g0 = ~0ull;
                        for (int w = 0; w < nw; ++w)
                            if (hbuf[kProfStride * w + 8]) g0 = std::min(g0, hbuf[kProfStride * w + 13]);
                        const int64_t nbu = a.nb * (dbits == 0 ? 4 : 1);
                        const Split sp{nbu, a.BH, a.ncta, a.seg_cost, a.tail_cost};
                        for (int c = 0; c < a.ncta; ++c) {
                            double hi = 0, cm = 0, tk = 0, fm = 0;
                            unsigned long long sm = 0, ge = 0, gs = 0, gx = 0;
                            for (int w = 0; w < 16; ++w) {
                                const double t = (double)hbuf[kProfStride * (c * 16 + w) + 8];
                                if (t > hi) {
                                    hi = t;
                                    sm = hbuf[kProfStride * (c * 16 + w) + 11];
                                }
                                cm = std::max(cm, (double)hbuf[kProfStride * (c * 16 + w) + 9]);
                                tk = std::max(tk, (double)hbuf[kProfStride * (c * 16 + w) + 10]);
                                fm = std::max(fm, (double)hbuf[kProfStride * (c * 16 + w) + 12]);
                                if (hbuf[kProfStride * (c * 16 + w) + 8]) {
                                    ge = std::max(ge, hbuf[kProfStride * (c * 16 + w) + 13] - g0);
                                    gs = std::max(gs, hbuf[kProfStride * (c * 16 + w) + 14] - g0);
                                    gx = std::max(gx, hbuf[kProfStride * (c * 16 + w) + 15] - g0);
                                }
                            }
                            const int64_t st = sp.begin(c), en = sp.end(c);
                            int64_t tails = 0;
                            for (int64_t bh = st / nbu; en > st && bh <= (en - 1) / nbu; ++bh)
                                if ((bh + 1) * nbu <= en) ++tails;
                            std::fprintf(f, "%d,%llu,%lld,%lld,%lld,%.0f,%.0f,%.0f,%.0f,%llu,%llu,%llu\n", c, sm,
                                         (long long)(en - st), (long long)(en > st ? (en - 1) / nbu - st / nbu + 1 : 0),
                                         (long long)tails, hi, cm, tk, fm, ge, gs, gx);
                        }
                        std::fclose(f);
                    }
                }
                if (ncta_used)
                    std::fprintf(stderr, "OSCAR_PROF cta slowest-warp cycles: min %.0f max %.0f; mean in-CTA warp spread %.0f\n",
                                 cmin, cmax, wspread / ncta_used);
            }
            {
                // timeline (globaltimer ns, relative to the first CTA's entry)
                std::vector<double> ent, str, ext, rdy;
                for (int w = 0; w < nw; ++w) {
                    if (hbuf[kProfStride * w + 8] == 0) continue;
                    rdy.push_back((double)hbuf[kProfStride * w + 20]);
                    ent.push_back((double)hbuf[kProfStride * w + 13]);
                    str.push_back((double)hbuf[kProfStride * w + 14]);
                    ext.push_back((double)hbuf[kProfStride * w + 15]);
                }
                if (!ent.empty()) {
                    const double t0 = *std::min_element(ent.begin(), ent.end());
                    auto q = [&](std::vector<double> v, double f) {
                        std::sort(v.begin(), v.end());
                        return (v[(size_t)(f * (double)(v.size() - 1))] - t0) * 1e-3;
                    };
                    std::fprintf(stderr,
                                 "OSCAR_PROF timeline us: entry max %.2f | q ready p50 %.2f max %.2f | stream end min "
                                 "%.2f p10 %.2f p50 %.2f p90 %.2f max %.2f | exit min %.2f p50 %.2f max %.2f\n",
                                 q(ent, 1.0), q(rdy, 0.5), q(rdy, 1.0), q(str, 0.0), q(str, 0.1), q(str, 0.5), q(str, 0.9), q(str, 1.0),
                                 q(ext, 0.0), q(ext, 0.5), q(ext, 1.0));
                    {  // prologue (per CTA, relative to its warp 0 entry): TMA issue, dep wait, q items, ready
                        double pr[6] = {0, 0, 0, 0, 0, 0};
                        int npc = 0;
                        for (int c = 0; c < a.ncta; ++c) {
                            const unsigned long long *w0 = &hbuf[kProfStride * (c * 16)];
                            if (w0[8] == 0) continue;
                            unsigned long long qmax = 0, dmax = 0, b0 = 0, b1 = 0;
                            for (int w = 0; w < 16; ++w) {
                                const unsigned long long *pw = &hbuf[kProfStride * (c * 16 + w)];
                                if (pw[8] == 0) continue;
                                qmax = std::max(qmax, pw[24]);
                                dmax = std::max(dmax, pw[23]);
                                b0 = std::max(b0, pw[21]);  // set by the fill thread only
                                b1 = std::max(b1, pw[22]);
                            }
                            const double e = (double)w0[13];
                            pr[0] += (double)b0 - e;
                            pr[1] += (double)b1 - e;
                            pr[2] += (double)dmax - e;
                            pr[3] += (double)qmax - e;
                            pr[4] += (double)w0[20] - e;
                            ++npc;
                        }
                        if (npc)
                            std::fprintf(stderr,
                                         "OSCAR_PROF prologue (us after the CTA's entry, mean over CTAs): barriers %.2f "
                                         "tma issued %.2f dep wait %.2f q items %.2f ready %.2f\n",
                                         pr[0] / npc * 1e-3, pr[1] / npc * 1e-3, pr[2] / npc * 1e-3, pr[3] / npc * 1e-3,
                                         pr[4] / npc * 1e-3);
                    }
                    // per CTA (warp 0): end-of-work phases relative to the CTA's last stream end
                    double dp[5] = {0, 0, 0, 0, 0};
                    int nc = 0;
                    for (int c = 0; c < a.ncta; ++c) {
                        const unsigned long long *w0 = &hbuf[kProfStride * (c * 16)];
                        if (w0[8] == 0) continue;
                        unsigned long long se = 0;
                        for (int w = 0; w < 16; ++w)
                            if (hbuf[kProfStride * (c * 16 + w) + 8]) se = std::max(se, hbuf[kProfStride * (c * 16 + w) + 14]);
                        const unsigned long long pts[5] = {w0[16], w0[17], w0[18], w0[19], w0[15]};
                        for (int i = 0; i < 5; ++i) dp[i] += (double)(long long)(pts[i] - se);
                        ++nc;
                    }
                    if (nc)
                        std::fprintf(stderr,
                                     "OSCAR_PROF end phases (us after the CTA's last stream end, mean over CTAs): "
                                     "sync1 %.2f phase1 %.2f sync2 %.2f ticket %.2f exit %.2f\n",
                                     dp[0] / nc * 1e-3, dp[1] / nc * 1e-3, dp[2] / nc * 1e-3, dp[3] / nc * 1e-3,
                                     dp[4] / nc * 1e-3);
                }
            }
            if (cnt)
                std::fprintf(stderr,
                             "OSCAR_PROF warps=%d avg cycles: wait %.0f qk %.0f softmax %.0f pv %.0f merge %.0f "
                             "spin %.0f qprologue %.0f segtail %.0f total %.0f max %.0f | merge parts: cta %.0f "
                             "atomic %.0f final %.0f (per-warp averages; final max %.0f)\n",
                             cnt, acc[0] / cnt, acc[1] / cnt, acc[2] / cnt, acc[3] / cnt, acc[4] / cnt, acc[5] / cnt,
                             acc[6] / cnt, acc[7] / cnt, acc[8] / cnt, mx, acc[9] / cnt, acc[10] / cnt,
                             acc[12] / cnt, fmax);
            cudaFree(pbuf);
        }
    }
};

namespace {

// ---------------------------------------------------------------------------
// export: device layout -> reference layout for one sequence
struct HostCache {
    int bits = 2;
    int64_t H = 0, nblk = 0, packed = 0, r = 0;
    // per head, per block
    std::vector<std::vector<std::vector<uint16_t>>> k_codes, v_codes;  // reference order
    std::vector<std::vector<std::vector<double>>> k_delta, k_const, v_delta, v_const;
    std::vector<std::vector<std::vector<int64_t>>> k_zp, v_zp;
    std::vector<std::vector<std::vector<double>>> k_raw, v_raw;  // bits 0
    std::vector<std::vector<double>> k_norms;                    // per head [packed]
    std::vector<double> k_res, k_norms_res, v_res;                // [r][H][d], [r*H]
};

HostCache build_host_cache(oscar_kv_handle *h, int64_t b) {
    if (b < 0 || b >= h->B) throw InvalidArg("export: sequence index out of range");
    h->in_step("export");
    if (h->last_stream) CK(cudaStreamSynchronize(h->last_stream));
    CK(cudaDeviceSynchronize());
    HostCache hc;
    const oscar_kv_config &cfg = h->cfg;
    const int64_t H = cfg.heads;
    hc.bits = h->dbits;
    hc.H = H;
    hc.packed = h->packed;
    hc.nblk = h->packed / R;
    hc.r = h->residual;
    const bool quant = h->dbits != 0;
    if (quant && !h->keep_exact) throw InvalidArg("export: handle created without keep_exact");
    const TransformCfg tc = h->tc();
    auto resize3 = [&](auto &v, size_t inner) {
        v.assign(H, {});
        for (auto &x : v) x.assign(hc.nblk, std::vector<typename std::decay_t<decltype(v[0][0])>::value_type>(inner));
    };
    if (quant) {
        resize3(hc.k_codes, R * D);
        resize3(hc.v_codes, R * D);
        resize3(hc.k_delta, D * (R / G));
        resize3(hc.k_const, D * (R / G));
        resize3(hc.k_zp, D * (R / G));
        resize3(hc.v_delta, R * (D / G));
        resize3(hc.v_const, R * (D / G));
        resize3(hc.v_zp, R * (D / G));
    } else {
        resize3(hc.k_raw, R * D);
        resize3(hc.v_raw, R * D);
    }
    hc.k_norms.assign(H, std::vector<double>(hc.packed));
    std::vector<uint8_t> blk(h->block_bytes);
    std::vector<double> sh(SHADOW_DOUBLES);
    for (int64_t hh = 0; hh < H; ++hh) {
        const int64_t bh = b * H + hh;
        for (int64_t k = 0; k < hc.nblk; ++k) {
            const int64_t rec = bh * h->max_blocks + k;
            CK(cudaMemcpy(blk.data(), h->blocks + rec * h->block_bytes, h->block_bytes, cudaMemcpyDeviceToHost));
            if (quant) {
                CK(cudaMemcpy(sh.data(), h->shadow + rec * SHADOW_DOUBLES, sizeof(double) * SHADOW_DOUBLES,
                              cudaMemcpyDeviceToHost));
                const int bits = h->dbits;
                const int tpw = 16 / bits;
                const int64_t code_bytes = (int64_t)R * D * bits / 8;
                const uint32_t *kw = reinterpret_cast<const uint32_t *>(blk.data());
                const int v_off = bits == 2 ? Block<2>::V_OFF : Block<4>::V_OFF;
                const uint32_t *vw = reinterpret_cast<const uint32_t *>(blk.data() + v_off);
                const int nwords = (int)(code_bytes / 4);
                const uint32_t fmask = (1u << bits) - 1;
                auto &kc = hc.k_codes[hh][k];
                auto &vc = hc.v_codes[hh][k];
                for (int w = 0; w < nwords; ++w)
                    for (int hi = 0; hi < 2; ++hi)
                        for (int f = 0; f < tpw; ++f) {
                            int t, c;
                            const int sh_ = hi * 16 + f * bits;
                            k_word_coords(bits, w, f, hi, t, c);
                            kc[(size_t)c * R + t] = (uint16_t)((kw[w] >> sh_) & fmask);  // j*R + t
                            v_word_coords(bits, w, f, hi, t, c);
                            vc[(size_t)t * D + c] = (uint16_t)((vw[w] >> sh_) & fmask);  // t*d + c
                        }
                for (int c = 0; c < D; ++c)
                    for (int grp = 0; grp < R / G; ++grp) {
                        const int p = c * (R / G) + grp;  // kv_cache.cpp:114
                        host::params_from_lohi(sh[(c * NGRP + grp) * 2], sh[(c * NGRP + grp) * 2 + 1], bits,
                                               hc.k_delta[hh][k][p], hc.k_zp[hh][k][p], hc.k_const[hh][k][p]);
                    }
                for (int t = 0; t < R; ++t)
                    for (int gc = 0; gc < D / G; ++gc) {
                        const int p = t * (D / G) + gc;  // kv_cache.cpp:144
                        host::params_from_lohi(sh[SHADOW_K_DOUBLES + (t * NGC + gc) * 2],
                                               sh[SHADOW_K_DOUBLES + (t * NGC + gc) * 2 + 1], bits,
                                               hc.v_delta[hh][k][p], hc.v_zp[hh][k][p], hc.v_const[hh][k][p]);
                    }
                for (int t = 0; t < R; ++t)
                    hc.k_norms[hh][k * R + t] = sh[SHADOW_K_DOUBLES + SHADOW_V_DOUBLES + t];
            } else {
                // raw bf16 block: undo the fragment order, then K rows -> apply_method
                // transform in fp64 (exact replay of what the reference stores)
                std::vector<uint16_t> kraw(R * D), vraw(R * D);
                constexpr int QW = BF16_QUARTER_BYTES / 8;
                for (int qu = 0; qu < 4; ++qu) {
                    const uint32_t *qw = reinterpret_cast<const uint32_t *>(blk.data() + qu * BF16_QUARTER_BYTES);
                    for (int w = 0; w < QW; ++w)
                        for (int hi = 0; hi < 2; ++hi) {
                            int t, c;
                            bf16_k_coords(w, hi, t, c);
                            kraw[(qu * 32 + t) * D + c] = (uint16_t)(qw[w] >> (16 * hi));
                            bf16_v_coords(w, hi, t, c);
                            vraw[(qu * 32 + t) * D + c] = (uint16_t)(qw[QW + w] >> (16 * hi));
                        }
                }
                const uint16_t *kr = kraw.data();
                const uint16_t *vr = vraw.data();
                for (int t = 0; t < R; ++t) {
                    double row[D];
                    for (int c = 0; c < D; ++c) row[c] = host::bf16_to_double(kr[t * D + c]);
                    double s = 1.0;
                    if (tc.rotates) host::fht(row, D);
                    if (tc.scales) s = host::token_scale(row, D, cfg.scaling);
                    for (int c = 0; c < D; ++c) hc.k_raw[hh][k][t * D + c] = row[c];
                    hc.k_norms[hh][k * R + t] = s;
                    for (int c = 0; c < D; ++c) row[c] = host::bf16_to_double(vr[t * D + c]);
                    if (cfg.rotate_v) host::fht(row, D);
                    for (int c = 0; c < D; ++c) hc.v_raw[hh][k][t * D + c] = row[c];
                }
            }
        }
    }
    // residual window: raw bf16 ring -> K_u rows and norms (kv_cache.cpp:219-224), or
    // (fp64 form) the exact residual rows as appended
    hc.k_res.assign(hc.r * H * D, 0.0);
    hc.k_norms_res.assign(hc.r * H, 0.0);
    hc.v_res.assign(hc.r * H * D, 0.0);
    std::vector<uint16_t> rk(R * D), rv(R * D);
    if (h->form == 2 && hc.r > 0) {
        std::vector<double> xk(R * D), xn(R), xv(R * D);
        for (int64_t hh = 0; hh < H; ++hh) {
            const int64_t bh = b * H + hh;
            CK(cudaMemcpy(xk.data(), h->res_k + bh * R * D, sizeof(double) * R * D, cudaMemcpyDeviceToHost));
            CK(cudaMemcpy(xn.data(), h->res_n + bh * R, sizeof(double) * R, cudaMemcpyDeviceToHost));
            CK(cudaMemcpy(xv.data(), h->res_v + bh * R * D, sizeof(double) * R * D, cudaMemcpyDeviceToHost));
            for (int64_t t = 0; t < hc.r; ++t) {
                for (int c = 0; c < D; ++c) hc.k_res[(t * H + hh) * D + c] = xk[t * D + c];
                hc.k_norms_res[t * H + hh] = xn[t];
                for (int c = 0; c < D; ++c) hc.v_res[(t * H + hh) * D + c] = xv[t * D + c];
            }
        }
        return hc;
    }
    for (int64_t hh = 0; hh < H; ++hh) {
        const int64_t bh = b * H + hh;
        if (hc.r == 0) break;
        CK(cudaMemcpy(rk.data(), reinterpret_cast<uint16_t *>(h->ring_k) + bh * R * D, sizeof(uint16_t) * R * D,
                      cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(rv.data(), reinterpret_cast<uint16_t *>(h->ring_v) + bh * R * D, sizeof(uint16_t) * R * D,
                      cudaMemcpyDeviceToHost));
        for (int64_t t = 0; t < hc.r; ++t) {
            double row[D];
            for (int c = 0; c < D; ++c) row[c] = host::bf16_to_double(rk[t * D + c]);
            double s = 1.0;
            if (tc.rotates) host::fht(row, D);
            if (tc.scales) s = host::token_scale(row, D, cfg.scaling);
            for (int c = 0; c < D; ++c) hc.k_res[(t * H + hh) * D + c] = row[c];
            hc.k_norms_res[t * H + hh] = s;
            for (int c = 0; c < D; ++c) row[c] = host::bf16_to_double(rv[vring_index(c, (int)t)]);  // tile-major ring
            if (cfg.rotate_v) host::fht(row, D);
            for (int c = 0; c < D; ++c) hc.v_res[(t * H + hh) * D + c] = row[c];
        }
    }
    return hc;
}

// pack_2bit (quant.cpp:162-175)
std::vector<uint16_t> pack2(const std::vector<uint16_t> &codes) {
    std::vector<uint16_t> w((codes.size() + 7) / 8, 0);
    for (size_t i = 0; i < codes.size(); ++i) w[i / 8] = (uint16_t)(w[i / 8] | (codes[i] << (2 * (i % 8))));
    return w;
}

const char *method_name(int m) {
    static const char *n[] = {"fp", "kivi", "rotate-only", "scale-only", "oscar"};
    return n[m];
}
const char *scaling_name(int s) {
    static const char *n[] = {"l2", "rsqrt", "max", "mean-abs"};
    return n[s];
}

// ---------------------------------------------------------------------------
// KVC1 import (KvCache::load, kv_cache.cpp:509-549): reference layout -> device
// records, exact shadow and residual rings.

// manifest scalar lookup (the manifest is one flat JSON object; the nested
// k_blocks / v_blocks arrays are implied by the config and checked by size)
struct Manifest {
    std::string text;
    std::string raw(const std::string &key) const {
        const std::string k = "\"" + key + "\":";
        const size_t p = text.find(k);
        if (p == std::string::npos) throw InvalidArg("cache load: manifest lacks " + key);
        size_t b = p + k.size(), e = b;
        if (text[b] == '"') {
            e = text.find('"', b + 1);
            return text.substr(b + 1, e - b - 1);
        }
        while (e < text.size() && text[e] != ',' && text[e] != '}') ++e;
        return text.substr(b, e - b);
    }
    int64_t i(const std::string &key) const { return std::stoll(raw(key)); }
    bool flag(const std::string &key) const { return raw(key) == "true"; }
};

// IEEE double -> binary16, round to nearest even (what __double2half does)
uint16_t double_to_half_rn(double x) {
    uint64_t u;
    std::memcpy(&u, &x, 8);
    const uint16_t sign = (uint16_t)((u >> 48) & 0x8000u);
    const int exp = (int)((u >> 52) & 0x7ff);
    const uint64_t man = u & ((1ull << 52) - 1);
    if (exp == 0x7ff) return sign | 0x7c00u | (man ? 0x200u : 0u);
    if (exp == 0) return sign;  // double subnormals are far below the half range
    const uint64_t m = man | (1ull << 52);
    const int e = exp - 1023;
    int shift, he;
    if (e >= -14) {
        shift = 42;
        he = e + 15;
    } else {
        shift = 28 - e;  // subnormal: units of 2^-24
        he = 0;
    }
    if (shift > 63) return sign;
    uint64_t q = m >> shift;
    const uint64_t rem = m & ((1ull << shift) - 1), half = 1ull << (shift - 1);
    if (rem > half || (rem == half && (q & 1))) ++q;
    if (he > 0) {
        if (q == 2048) {
            q = 1024;
            ++he;
        }
        if (he >= 31) return sign | 0x7c00u;
        return sign | (uint16_t)(he << 10) | (uint16_t)(q & 0x3ffu);
    }
    return sign | (uint16_t)q;  // q == 1024 is the smallest normal, encoded naturally
}

uint16_t double_to_bf16_near(double x) {  // x within a few ulp of a bf16 value
    const float f = (float)x;
    uint32_t u;
    std::memcpy(&u, &f, 4);
    u += 0x7fffu + ((u >> 16) & 1u);
    return (uint16_t)(u >> 16);
}

// (delta, zp, constant) -> a (lo, hi) pair the shadow can hold, such that
// quant.cpp:37-46 recomputes exactly this delta and zp (export / dump stay exact)
void lohi_from_params(double delta, int64_t zp, double constant, int bits, double &lo, double &hi) {
    lo = constant;
    if (delta == 0.0) {
        if (zp != 0) throw InvalidArg("cache load: constant group with a non-zero zero point");
        hi = lo;
        return;
    }
    const double lv = (double)((int64_t{1} << bits) - 1);
    double up = lo + delta * lv, dn = up;
    for (int k = 0; k < 32; ++k) {  // the nearest hi (in ulps) with (hi - lo) / lv == delta
        for (const double cand : {up, dn}) {
            double d2, cst;
            int64_t z2;
            host::params_from_lohi(lo, cand, bits, d2, z2, cst);
            if (d2 == delta) {
                if (z2 != zp) throw InvalidArg("cache load: zero point inconsistent with delta and constant");
                hi = cand;
                return;
            }
        }
        up = std::nextafter(up, INFINITY);
        dn = std::nextafter(dn, -INFINITY);
    }
    throw InvalidArg("cache load: no (lo, hi) reproduces the stored delta");
}

// raw bf16 key row from the stored transformed row K_u and its norm (inverse of
// apply_method), verified by replaying the forward transform bit for bit
void raw_key_row(const double *ku, double s, const TransformCfg &tc, int scaling, uint16_t *out) {
    double x[D], y[D];
    for (int c = 0; c < D; ++c) x[c] = tc.scales ? ku[c] * s : ku[c];
    if (tc.rotates) host::fht(x, D);
    for (int c = 0; c < D; ++c) {
        out[c] = double_to_bf16_near(x[c]);
        y[c] = host::bf16_to_double(out[c]);
    }
    if (tc.rotates) host::fht(y, D);
    double s2 = 1.0;
    if (tc.scales) s2 = host::token_scale(y, D, scaling);
    for (int c = 0; c < D; ++c)
        if (y[c] != ku[c]) throw InvalidArg("cache load: residual key rows are not the transform of bf16 keys");
    if (tc.scales && s2 != s) throw InvalidArg("cache load: residual key norms are not the bf16 keys' norms");
}

void raw_value_row(const double *v, int rotate_v, uint16_t *out) {
    double x[D], y[D];
    for (int c = 0; c < D; ++c) x[c] = v[c];
    if (rotate_v) host::fht(x, D);
    for (int c = 0; c < D; ++c) {
        out[c] = double_to_bf16_near(x[c]);
        y[c] = host::bf16_to_double(out[c]);
    }
    if (rotate_v) host::fht(y, D);
    for (int c = 0; c < D; ++c)
        if (y[c] != v[c]) throw InvalidArg("cache load: value rows are not bf16-representable");
}

template <typename T>
std::vector<T> read_vec(std::ifstream &f, size_t n) {
    std::vector<T> v(n);
    f.read(reinterpret_cast<char *>(v.data()), (std::streamsize)(n * sizeof(T)));
    if (!f) throw InvalidArg("cache load: file too short");
    return v;
}

void load_kvc1(oscar_kv_handle *h, int64_t b, const char *path) {
    if (b < 0 || b >= h->B) throw InvalidArg("load: sequence index out of range");
    std::ifstream f(path, std::ios::binary);
    if (!f) throw std::runtime_error(std::string("cache load: cannot open ") + path);
    Manifest m;
    std::getline(f, m.text);
    if (m.raw("magic") != "KVC1") throw std::runtime_error("cache load: bad magic");
    const oscar_kv_config &c = h->cfg;
    if (m.i("R") != c.residual_len || m.i("G") != c.group_size || m.i("b") != c.bits || m.i("H") != c.heads ||
        m.i("d_h") != c.head_dim || m.raw("method") != method_name(c.method) ||
        m.raw("scaling") != scaling_name(c.scaling))
        throw InvalidArg("cache load: file was written under a different config");
    const int64_t packed = m.i("S_packed"), r = m.i("residual_tokens"), flushes = m.i("flush_count");
    if (m.i("S_packed_v") != packed || m.i("v_residual_tokens") != r)
        throw InvalidArg("cache load: key and value streams differ in length");
    if (packed % R || r < 0 || r >= R) throw InvalidArg("cache load: inconsistent token counts");
    if (packed + r > h->max_tokens) throw InvalidArg("cache load: cache capacity exceeded");
    // nothing of the handle changes until every section is parsed, converted and
    // uploaded: a failed load leaves the handle (counters and device state) as it was
    const bool adopt = !h->prefilled;
    if (!adopt && (h->packed != packed || h->residual != r))
        throw InvalidArg("cache load: sequences of one handle must hold the same number of tokens");
    if (h->dbits && !h->keep_exact) throw InvalidArg("cache load: handle created without keep_exact");
    const int64_t H = c.heads, nb = packed / R;
    const int bits = h->dbits;
    const TransformCfg tc = h->tc();
    const int64_t kp = D * (R / G), vp = R * (D / G);
    struct Blk {
        std::vector<double> delta, cst, raw;
        std::vector<int64_t> zp;
        std::vector<uint16_t> codes;  // reference order
    };
    auto read_block = [&](int64_t nparams) {
        Blk k;
        if (bits) {
            k.delta.resize(nparams);
            k.zp.resize(nparams);
            k.cst.resize(nparams);
            for (int64_t i = 0; i < nparams; ++i) {
                f.read(reinterpret_cast<char *>(&k.delta[i]), 8);
                f.read(reinterpret_cast<char *>(&k.zp[i]), 8);
                f.read(reinterpret_cast<char *>(&k.cst[i]), 8);
            }
            if (bits == 2) {
                auto w = read_vec<uint16_t>(f, R * D / 8);
                k.codes.resize(R * D);
                for (int64_t i = 0; i < R * D; ++i) k.codes[i] = (uint16_t)((w[i / 8] >> (2 * (i % 8))) & 3u);
            } else {
                k.codes = read_vec<uint16_t>(f, R * D);
            }
            if (!f) throw InvalidArg("cache load: file too short");
        } else {
            k.raw = read_vec<double>(f, R * D);
        }
        return k;
    };
    std::vector<std::vector<Blk>> kb(H), vb(H);
    std::vector<std::vector<double>> knorm(H);
    for (int64_t hh = 0; hh < H; ++hh) {
        for (int64_t k = 0; k < nb; ++k) kb[hh].push_back(read_block(kp));
        knorm[hh] = read_vec<double>(f, packed);
    }
    const auto kres = read_vec<double>(f, r * H * D);
    const auto kres_n = read_vec<double>(f, r * H);
    for (int64_t hh = 0; hh < H; ++hh)
        for (int64_t k = 0; k < nb; ++k) vb[hh].push_back(read_block(vp));
    const auto vres = read_vec<double>(f, r * H * D);

    // (1) convert everything on the host (may throw: inconsistent params, codes
    //     out of range, rows that are not transforms of bf16 inputs)
    std::vector<uint8_t> recs((size_t)(H * nb * h->block_bytes), 0);
    std::vector<double> shadows(bits ? (size_t)(H * nb * SHADOW_DOUBLES) : 0);
    std::vector<uint16_t> rings_k(r > 0 ? (size_t)(H * R * D) : 0, 0), rings_v(r > 0 ? (size_t)(H * R * D) : 0, 0);
    for (int64_t hh = 0; hh < H; ++hh) {
        for (int64_t k = 0; k < nb; ++k) {
            const Blk &K = kb[hh][k], &V = vb[hh][k];
            uint8_t *rec_p = recs.data() + (size_t)((hh * nb + k) * h->block_bytes);
            double *sh = bits ? shadows.data() + (size_t)((hh * nb + k) * SHADOW_DOUBLES) : nullptr;
            if (bits) {
                const int tpw = 16 / bits;
                const int64_t code_bytes = (int64_t)R * D * bits / 8;
                uint32_t *kw = reinterpret_cast<uint32_t *>(rec_p);
                uint32_t *vw = reinterpret_cast<uint32_t *>(rec_p + (bits == 2 ? Block<2>::V_OFF : Block<4>::V_OFF));
                const uint32_t maxc = (1u << bits) - 1;
                for (int w = 0; w < (int)(code_bytes / 4); ++w)
                    for (int hi = 0; hi < 2; ++hi)
                        for (int fl = 0; fl < tpw; ++fl) {
                            int t, ch;
                            const int s_ = hi * 16 + fl * bits;
                            k_word_coords(bits, w, fl, hi, t, ch);
                            const uint32_t ck = K.codes[(size_t)ch * R + t];
                            v_word_coords(bits, w, fl, hi, t, ch);
                            const uint32_t cv = V.codes[(size_t)t * D + ch];
                            if (ck > maxc || cv > maxc) throw InvalidArg("cache load: code out of range");
                            kw[w] |= ck << s_;
                            vw[w] |= cv << s_;
                        }
                const int ka_off = bits == 2 ? Block<2>::KA_OFF : Block<4>::KA_OFF;
                const int kb_off = bits == 2 ? Block<2>::KB_OFF : Block<4>::KB_OFF;
                const int va_off = bits == 2 ? Block<2>::VA_OFF : Block<4>::VA_OFF;
                const int vb_off = bits == 2 ? Block<2>::VB_OFF : Block<4>::VB_OFF;
                const int nr_off = bits == 2 ? Block<2>::NORM_OFF : Block<4>::NORM_OFF;
                uint16_t *pka = reinterpret_cast<uint16_t *>(rec_p + ka_off);
                uint16_t *pkb = reinterpret_cast<uint16_t *>(rec_p + kb_off);
                uint16_t *pva = reinterpret_cast<uint16_t *>(rec_p + va_off);
                uint16_t *pvb = reinterpret_cast<uint16_t *>(rec_p + vb_off);
                float *pn = reinterpret_cast<float *>(rec_p + nr_off);
                // affine16 (quantize.cu): a = delta, b = delta * -zp; constant group a = 0, b = lo
                auto affine = [&](double dl, int64_t zp, double cst, uint16_t &a, uint16_t &bb) {
                    if (dl == 0.0) {
                        a = double_to_half_rn(0.0);
                        bb = double_to_half_rn(cst);
                    } else {
                        a = double_to_half_rn(dl);
                        bb = double_to_half_rn(dl * -(double)zp);
                    }
                };
                for (int ch = 0; ch < D; ++ch)
                    for (int grp = 0; grp < NGRP; ++grp) {
                        const int p = ch * (R / G) + grp;
                        affine(K.delta[p], K.zp[p], K.cst[p], pka[ka_index(ch, grp)], pkb[kb_index(ch, grp)]);
                        lohi_from_params(K.delta[p], K.zp[p], K.cst[p], bits, sh[(ch * NGRP + grp) * 2],
                                         sh[(ch * NGRP + grp) * 2 + 1]);
                    }
                for (int t = 0; t < R; ++t)
                    for (int gc = 0; gc < NGC; ++gc) {
                        const int p = t * (D / G) + gc;
                        affine(V.delta[p], V.zp[p], V.cst[p], pva[va_index(t, gc)], pvb[vb_index(t, gc)]);
                        lohi_from_params(V.delta[p], V.zp[p], V.cst[p], bits, sh[SHADOW_K_DOUBLES + (t * NGC + gc) * 2],
                                         sh[SHADOW_K_DOUBLES + (t * NGC + gc) * 2 + 1]);
                    }
                for (int t = 0; t < R; ++t) {
                    const double s = knorm[hh][k * R + t];
                    pn[norm_index(t)] = (float)(s * 0.12751743074202186);  // log2(e)/sqrt(d), as quantize.cu
                    sh[SHADOW_K_DOUBLES + SHADOW_V_DOUBLES + t] = s;
                }
            } else {
                // raw block: transformed rows -> raw bf16 rows -> fragment order
                std::vector<uint16_t> kraw(R * D), vraw(R * D);
                for (int t = 0; t < R; ++t) {
                    raw_key_row(&K.raw[(size_t)t * D], knorm[hh][k * R + t], tc, c.scaling, &kraw[(size_t)t * D]);
                    raw_value_row(&V.raw[(size_t)t * D], c.rotate_v, &vraw[(size_t)t * D]);
                }
                constexpr int QW = BF16_QUARTER_BYTES / 8;
                for (int qu = 0; qu < 4; ++qu) {
                    uint32_t *qw = reinterpret_cast<uint32_t *>(rec_p + qu * BF16_QUARTER_BYTES);
                    for (int w = 0; w < QW; ++w)
                        for (int hi = 0; hi < 2; ++hi) {
                            int t, ch;
                            bf16_k_coords(w, hi, t, ch);
                            qw[w] |= (uint32_t)kraw[(qu * 32 + t) * D + ch] << (16 * hi);
                            bf16_v_coords(w, hi, t, ch);
                            qw[QW + w] |= (uint32_t)vraw[(qu * 32 + t) * D + ch] << (16 * hi);
                        }
                }
            }
        }
    }
    // residual window -> raw bf16 rings (K token-major, V tile-major).  Rows that
    // are not transforms of bf16 inputs (a cache the reference built from its fp64
    // projections) put the handle in the fp64 form: the rows are kept exactly in
    // the residual shadow and the rings hold their bf16 image
    bool f64_res = h->form == 2;
    if (r > 0 && !f64_res) {
        try {
            std::vector<uint16_t> row(D);
            for (int64_t hh = 0; hh < H; ++hh) {
                uint16_t *rk = rings_k.data() + (size_t)(hh * R * D), *rv = rings_v.data() + (size_t)(hh * R * D);
                for (int64_t t = 0; t < r; ++t) {
                    raw_key_row(&kres[(t * H + hh) * D], kres_n[t * H + hh], tc, c.scaling, &rk[t * D]);
                    raw_value_row(&vres[(t * H + hh) * D], c.rotate_v, row.data());
                    for (int ch = 0; ch < D; ++ch) rv[vring_index(ch, (int)t)] = row[ch];
                }
            }
        } catch (const InvalidArg &) {
            if (h->form == 1) throw;  // the handle already holds raw bf16 appends
            if (!bits) throw InvalidArg("cache load: residual rows are not transforms of bf16 inputs (method fp)");
            if (c.rotate_v) throw InvalidArg("cache load: fp64 residual rows need rotate_v = 0");
            f64_res = true;
        }
    }
    if (r > 0 && f64_res) {
        for (int64_t hh = 0; hh < H; ++hh) {
            uint16_t *rk = rings_k.data() + (size_t)(hh * R * D), *rv = rings_v.data() + (size_t)(hh * R * D);
            for (int64_t t = 0; t < r; ++t) {
                // window_f64_kernel's image: FHT(K_u * s) (apply_method inverted), fp16
                double x[D];
                const double sn = kres_n[t * H + hh];
                for (int ch = 0; ch < D; ++ch) x[ch] = tc.scales ? kres[(t * H + hh) * D + ch] * sn : kres[(t * H + hh) * D + ch];
                if (tc.rotates) host::fht(x, D);
                for (int ch = 0; ch < D; ++ch) {
                    rk[t * D + ch] = double_to_half_rn(x[ch]);
                    rv[vring_index(ch, (int)t)] = double_to_half_rn(vres[(t * H + hh) * D + ch]);
                }
            }
        }
    }
    // (2) upload (only CUDA errors can fail from here on)
    CK(cudaSetDevice(h->device));
    if (h->last_stream) CK(cudaStreamSynchronize(h->last_stream));
    if (f64_res) h->use_form(2);
    for (int64_t hh = 0; hh < H; ++hh) {
        const int64_t bh = b * H + hh;
        if (nb > 0) {
            CK(cudaMemcpy(h->blocks + bh * h->max_blocks * h->block_bytes, recs.data() + (size_t)(hh * nb * h->block_bytes),
                          (size_t)(nb * h->block_bytes), cudaMemcpyHostToDevice));
            if (bits)
                CK(cudaMemcpy(h->shadow + bh * h->max_blocks * SHADOW_DOUBLES,
                              shadows.data() + (size_t)(hh * nb * SHADOW_DOUBLES),
                              sizeof(double) * (size_t)(nb * SHADOW_DOUBLES), cudaMemcpyHostToDevice));
        }
        if (r > 0 && f64_res) {
            std::vector<double> xk((size_t)(R * D), 0.0), xn((size_t)R, 0.0), xv((size_t)(R * D), 0.0);
            for (int64_t t = 0; t < r; ++t) {
                for (int ch = 0; ch < D; ++ch) {
                    xk[(size_t)(t * D + ch)] = kres[(t * H + hh) * D + ch];
                    xv[(size_t)(t * D + ch)] = vres[(t * H + hh) * D + ch];
                }
                xn[(size_t)t] = kres_n[t * H + hh];
            }
            CK(cudaMemcpy(h->res_k + bh * R * D, xk.data(), sizeof(double) * R * D, cudaMemcpyHostToDevice));
            CK(cudaMemcpy(h->res_n + bh * R, xn.data(), sizeof(double) * R, cudaMemcpyHostToDevice));
            CK(cudaMemcpy(h->res_v + bh * R * D, xv.data(), sizeof(double) * R * D, cudaMemcpyHostToDevice));
        }
        if (r > 0) {
            CK(cudaMemcpy(reinterpret_cast<uint16_t *>(h->ring_k) + bh * R * D, rings_k.data() + (size_t)(hh * R * D),
                          sizeof(uint16_t) * R * D, cudaMemcpyHostToDevice));
            CK(cudaMemcpy(reinterpret_cast<uint16_t *>(h->ring_v) + bh * R * D, rings_v.data() + (size_t)(hh * R * D),
                          sizeof(uint16_t) * R * D, cudaMemcpyHostToDevice));
        }
    }
    // (3) commit the token counters (kv_cache.cpp:540-548)
    if (adopt) {
        h->packed = packed;
        h->residual = r;
        h->flushes = flushes;
        h->prefilled = m.flag("k_prefilled");
        h->v_packed = packed;
        h->v_residual = r;
        h->v_prefilled = m.flag("v_prefilled");
    }
    h->blocks_written = true;  // the next attention launch waits before touching the records
}

}  // namespace

// ===========================================================================
extern "C" {

const char *oscar_last_error(void) { return g_err.c_str(); }

int oscar_kv_config_validate(const oscar_kv_config *cfg) {
    return guard([&] {
        if (!cfg) throw InvalidArg("null config");
        validate(*cfg);
    });
}

int oscar_kv_create(const oscar_kv_config *cfg, int64_t batch, int64_t q_heads, int64_t max_tokens, int device,
                    int keep_exact, oscar_kv_handle **out) {
    return guard([&] {
        if (!cfg || !out) throw InvalidArg("null argument");
        validate(*cfg);
        if (batch <= 0) throw InvalidArg("create: batch must be positive");
        if (q_heads <= 0 || q_heads % cfg->heads != 0 || q_heads / cfg->heads > 8)
            throw InvalidArg("create: q_heads must be a multiple of heads with at most 8 per KV head");
        if (max_tokens < 0) throw InvalidArg("create: max_tokens must be non-negative");
        auto h = std::make_unique<oscar_kv_handle>();
        h->cfg = *cfg;
        h->dbits = quantizes(*cfg) ? cfg->bits : 0;
        h->B = batch;
        h->Hq = q_heads;
        h->g = q_heads / cfg->heads;
        h->BH = batch * cfg->heads;
        h->max_tokens = max_tokens;
        h->max_blocks = max_tokens / R + 1;
        h->device = device;
        h->keep_exact = keep_exact != 0;
        CK(cudaSetDevice(device));
        CK(cudaDeviceGetAttribute(&h->num_sms, cudaDevAttrMultiProcessorCount, device));
        h->block_bytes = h->dbits == 2 ? Block<2>::BYTES : h->dbits == 4 ? Block<4>::BYTES : BF16_BLOCK_BYTES;
        h->blocks = (uint8_t *)h->dalloc((size_t)(h->BH * h->max_blocks * h->block_bytes));
        if (h->dbits != 0 && h->keep_exact)
            h->shadow = (double *)h->dalloc(sizeof(double) * (size_t)(h->BH * h->max_blocks * SHADOW_DOUBLES));
        h->ring_k = h->dalloc((size_t)(h->BH * R * D * 2));
        h->ring_v = h->dalloc((size_t)(h->BH * R * D * 2));
        h->maxp_alloc = (int)(2 * h->num_sms / h->BH + 3);
        h->alloc_partials();
        h->counters = (int *)h->dalloc(sizeof(int) * (size_t)h->BH);
        CK(cudaMemset(h->counters, 0, sizeof(int) * (size_t)h->BH));
        h->status_d = (int *)h->dalloc(sizeof(int));
        CK(cudaMemset(h->status_d, 0, sizeof(int)));
        // segments (b, kv heads) one CTA range can touch: <= BH/ncta + 2 (nb >= 1 unit);
        // residual-only launches use BH CTAs of one segment each
        {
            const int64_t maxseg = std::min<int64_t>(oscar_kv_handle::kMaxSegments, h->BH / h->num_sms + 2);
            h->grow_scratch(std::max<int64_t>((int64_t)h->num_sms * maxseg, h->BH), maxseg);
        }
        const size_t stage_bytes = (size_t)(h->B * h->Hq * D * 2 + 2 * h->BH * D * 2 + h->B * h->Hq * D * 4 +
                                            h->B * h->Hq * 4 + 256);
        h->stage = h->dalloc(stage_bytes);
        *out = h.release();
    });
}

int oscar_kv_destroy(oscar_kv_handle *h) {
    return guard([&] { delete h; });
}

int oscar_kv_append(oscar_kv_handle *h, const void *k, const void *v, int64_t n_tokens, void *stream) {
    return guard([&] {
        if (!h) throw InvalidArg("null handle");
        if (n_tokens > 0 && (!k || !v)) throw InvalidArg("append: null tensor");
        CK(cudaSetDevice(h->device));
        h->last_stream = (cudaStream_t)stream;
        h->append(k, v, n_tokens, (cudaStream_t)stream);
    });
}

namespace {
// fp64 rows given in host memory (the reference's Tensor3 callers): staged to the
// device for the call (a compatibility path; synchronises the stream before the
// staging buffer is released)
struct F64Stage {
    double *d = nullptr;
    cudaStream_t s = nullptr;
    const double *view(const double *p, size_t n, cudaStream_t st) {
        if (!p || n == 0) return p;
        cudaPointerAttributes at{};
        if (cudaPointerGetAttributes(&at, p) != cudaSuccess) (void)cudaGetLastError();
        if (at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged) return p;
        CK(cudaMalloc(&d, n * sizeof(double)));
        CK(cudaMemcpyAsync(d, p, n * sizeof(double), cudaMemcpyHostToDevice, st));
        s = st;
        return d;
    }
    ~F64Stage() {
        if (d) {
            cudaStreamSynchronize(s);
            cudaFree(d);
        }
    }
};
}  // namespace

int oscar_kv_append_k(oscar_kv_handle *h, const double *k_t, const double *norms, int64_t n_tokens, void *stream) {
    return guard([&] {
        if (!h || (n_tokens > 0 && (!k_t || !norms))) throw InvalidArg("append_k: null argument");
        CK(cudaSetDevice(h->device));
        cudaStream_t s = (cudaStream_t)stream;
        h->last_stream = s;
        const size_t n = (size_t)(h->B * std::max<int64_t>(n_tokens, 0) * h->cfg.heads);
        F64Stage sk, sn;
        h->append_f64(0, sk.view(k_t, n * D, s), sn.view(norms, n, s), n_tokens, s);
    });
}

int oscar_kv_append_v(oscar_kv_handle *h, const double *v, int64_t n_tokens, void *stream) {
    return guard([&] {
        if (!h || (n_tokens > 0 && !v)) throw InvalidArg("append_v: null argument");
        CK(cudaSetDevice(h->device));
        cudaStream_t s = (cudaStream_t)stream;
        h->last_stream = s;
        const size_t n = (size_t)(h->B * std::max<int64_t>(n_tokens, 0) * h->cfg.heads);
        F64Stage sv;
        h->append_f64(1, sv.view(v, n * D, s), nullptr, n_tokens, s);
    });
}

int oscar_kv_decode_step_f64(oscar_kv_handle *h, const void *q, const double *k_t, const double *norms,
                             const double *v, float *out, float *lse, void *stream) {
    return guard([&] {
        if (!h || !q || !k_t || !norms || !v || !out) throw InvalidArg("decode_step: null argument");
        CK(cudaSetDevice(h->device));
        h->last_stream = (cudaStream_t)stream;
        h->decode_step_f64(q, k_t, norms, v, out, lse, (cudaStream_t)stream);
    });
}

int oscar_kv_stats_v(const oscar_kv_handle *h, int64_t *v_packed, int64_t *v_residual) {
    return guard([&] {
        if (!h) throw InvalidArg("null handle");
        const bool f2 = h->form == 2;
        if (v_packed) *v_packed = f2 ? h->v_packed : h->packed;
        if (v_residual) *v_residual = f2 ? h->v_residual : h->residual;
    });
}

int oscar_kvc1_read_config(const char *path, oscar_kv_config *cfg, int64_t *tokens) {
    return guard([&] {
        if (!path || !cfg) throw InvalidArg("kvc1_read_config: null argument");
        std::ifstream f(path, std::ios::binary);
        if (!f) throw std::runtime_error(std::string("cache load: cannot open ") + path);
        Manifest m;
        std::getline(f, m.text);
        if (m.raw("magic") != "KVC1") throw std::runtime_error("cache load: bad magic");
        oscar_kv_config c{};
        const std::string meth = m.raw("method"), sc = m.raw("scaling");
        c.method = -1;
        for (int i = 0; i < 5; ++i)
            if (meth == method_name(i)) c.method = i;
        c.scaling = -1;
        for (int i = 0; i < 4; ++i)
            if (sc == scaling_name(i)) c.scaling = i;
        if (c.method < 0 || c.scaling < 0) throw InvalidArg("cache load: unknown method or scaling in the manifest");
        c.bits = (int32_t)m.i("b");
        c.group_size = m.i("G");
        c.residual_len = m.i("R");
        c.head_dim = m.i("d_h");
        c.heads = m.i("H");
        c.rotate_v = 0;
        *cfg = c;
        if (tokens) *tokens = m.i("S_packed") + m.i("residual_tokens");
    });
}

int oscar_kv_decode_step(oscar_kv_handle *h, const void *q, const void *k, const void *v, float *out, float *lse,
                         void *stream) {
    return guard([&] {
        if (!h || !q || !k || !v || !out) throw InvalidArg("decode_step: null argument");
        CK(cudaSetDevice(h->device));
        h->last_stream = (cudaStream_t)stream;
        h->decode_step(q, k, v, out, lse, (cudaStream_t)stream);
    });
}

int oscar_kv_decode_step_logits(oscar_kv_handle *h, const void *q, const void *k, const void *v, float *out,
                                float *lse, float *logits, void *stream) {
    return guard([&] {
        if (!h || !q || !k || !v || !out) throw InvalidArg("decode_step: null argument");
        CK(cudaSetDevice(h->device));
        h->last_stream = (cudaStream_t)stream;
        h->decode_step(q, k, v, out, lse, (cudaStream_t)stream, nullptr, 0, logits);
    });
}

int oscar_kv_logits(oscar_kv_handle *h, const void *q, const void *k, float *logits, void *stream) {
    return guard([&] {
        if (!h || !q || !logits) throw InvalidArg("logits: null argument");
        CK(cudaSetDevice(h->device));
        h->last_stream = (cudaStream_t)stream;
        h->last_launches = 0;
        h->logits(q, k, logits, (cudaStream_t)stream);
    });
}

int oscar_kv_decode_step_many(int32_t n, oscar_kv_handle *const *hs, const void *const *q, const void *const *k,
                              const void *const *v, float *const *out, float *const *lse, void *stream) {
    return guard([&] {
        if (n < 0 || (n > 0 && (!hs || !q || !k || !v || !out))) throw InvalidArg("decode_step_many: null argument");
        int dev = -1;
        for (int32_t i = 0; i < n; ++i) {
            oscar_kv_handle *h = hs[i];
            if (!h || !q[i] || !k[i] || !v[i] || !out[i]) throw InvalidArg("decode_step_many: null argument");
            if (h->device != dev) {
                CK(cudaSetDevice(h->device));
                dev = h->device;
            }
            h->last_stream = (cudaStream_t)stream;
            h->decode_step(q[i], k[i], v[i], out[i], lse ? lse[i] : nullptr, (cudaStream_t)stream);
        }
    });
}

int oscar_kv_attend(oscar_kv_handle *h, const void *q, float *out, float *lse, void *stream) {
    return guard([&] {
        if (!h || !q || !out) throw InvalidArg("attend: null argument");
        CK(cudaSetDevice(h->device));
        h->last_stream = (cudaStream_t)stream;
        h->attend(q, out, lse, (cudaStream_t)stream);
    });
}

namespace {
PeerPlan peer_plan(const oscar_peer_plan *p, int64_t rows_expected) {
    static_assert(OSCAR_PEER_MAX == PEER_MAX && OSCAR_PEER_STRIDE == PEER_STRIDE, "peer layout");
    if (!p) throw InvalidArg("peer plan: null");
    if (p->world < 1 || p->world > OSCAR_PEER_MAX || p->rank < 0 || p->rank >= p->world)
        throw InvalidArg("peer plan: bad world/rank");
    if (p->rows <= 0 || (rows_expected >= 0 && p->rows != rows_expected))
        throw InvalidArg("peer plan: rows must be batch * q_heads");
    PeerPlan q{};
    q.world = p->world;
    q.rank = p->rank;
    q.rows = p->rows;
    for (int i = 0; i < p->world; ++i) {
        if (!p->recv[i]) throw InvalidArg("peer plan: null receive area");
        if (((uintptr_t)p->recv[i]) % 32) throw InvalidArg("peer plan: misaligned receive area");
        q.recv[i] = p->recv[i];
    }
    return q;
}
}  // namespace

int64_t oscar_peer_area_bytes(int32_t world, int64_t rows) {
    if (world < 1 || world > OSCAR_PEER_MAX || rows <= 0) return -1;
    return (int64_t)2 * world * rows * OSCAR_PEER_STRIDE * 8;
}

int oscar_kv_attend_publish(oscar_kv_handle *h, const void *q, const void *k, const void *v,
                            const oscar_peer_plan *plan, uint32_t epoch, void *stream) {
    return guard([&] {
        if (!h || !q) throw InvalidArg("attend_publish: null argument");
        if ((k == nullptr) != (v == nullptr)) throw InvalidArg("attend_publish: k and v go together");
        if (epoch == 0) throw InvalidArg("attend_publish: epochs start at 1");
        const PeerPlan pp = peer_plan(plan, h->B * h->Hq);
        CK(cudaSetDevice(h->device));
        h->last_stream = (cudaStream_t)stream;
        if (k) h->decode_step(q, k, v, nullptr, nullptr, (cudaStream_t)stream, &pp, epoch);
        else h->attend(q, nullptr, nullptr, (cudaStream_t)stream, &pp, epoch);
    });
}

int oscar_peer_publish_empty(const oscar_peer_plan *plan, uint32_t epoch, void *stream) {
    return guard([&] {
        if (epoch == 0) throw InvalidArg("peer_publish_empty: epochs start at 1");
        const PeerPlan pp = peer_plan(plan, -1);
        CK(launch_peer_publish_empty(pp, epoch, (cudaStream_t)stream));
    });
}

int oscar_peer_merge(const oscar_peer_plan *plan, uint32_t epoch, float *out, float *lse, int32_t *status,
                     void *stream) {
    return guard([&] {
        if (!out) throw InvalidArg("peer_merge: null out");
        if (epoch == 0) throw InvalidArg("peer_merge: epochs start at 1");
        const PeerPlan pp = peer_plan(plan, -1);
        CK(launch_peer_merge(pp, epoch, out, lse, status, (cudaStream_t)stream));
    });
}

int oscar_ipc_alloc(int64_t bytes, int32_t device, void **dptr, void *handle_out) {
    return guard([&] {
        if (bytes <= 0 || !dptr || !handle_out) throw InvalidArg("ipc_alloc: bad argument");
        CK(cudaSetDevice(device));
        void *p = nullptr;
        CK(cudaMalloc(&p, (size_t)bytes));
        CK(cudaMemset(p, 0, (size_t)bytes));
        cudaIpcMemHandle_t hd;
        static_assert(sizeof(hd) == 64, "ipc handle size");
        CK(cudaIpcGetMemHandle(&hd, p));
        memcpy(handle_out, &hd, sizeof(hd));
        *dptr = p;
    });
}

int oscar_ipc_open(const void *handle, int32_t device, void **dptr) {
    return guard([&] {
        if (!handle || !dptr) throw InvalidArg("ipc_open: bad argument");
        CK(cudaSetDevice(device));
        cudaIpcMemHandle_t hd;
        memcpy(&hd, handle, sizeof(hd));
        CK(cudaIpcOpenMemHandle(dptr, hd, cudaIpcMemLazyEnablePeerAccess));
    });
}

int oscar_ipc_close(void *dptr) {
    return guard([&] { CK(cudaIpcCloseMemHandle(dptr)); });
}

int oscar_ipc_free(void *dptr) {
    return guard([&] { CK(cudaFree(dptr)); });
}

int oscar_kv_decode_step_host(oscar_kv_handle *h, const void *q_host, const void *k_host, const void *v_host,
                              float *out_host, float *lse_host, void *stream) {
    return guard([&] {
        if (!h || !q_host || !k_host || !v_host || !out_host) throw InvalidArg("decode_step_host: null argument");
        CK(cudaSetDevice(h->device));
        cudaStream_t s = (cudaStream_t)stream;
        h->last_stream = s;
        uint8_t *p = (uint8_t *)h->stage;
        const size_t qb = (size_t)(h->B * h->Hq * D * 2), kb = (size_t)(h->BH * D * 2);
        const size_t ob = (size_t)(h->B * h->Hq * D * 4), lb = (size_t)(h->B * h->Hq * 4);
        void *dq = p, *dk = p + qb, *dv = p + qb + kb;
        float *dout = (float *)(p + qb + 2 * kb);
        float *dlse = (float *)(p + qb + 2 * kb + ob);
        // inputs: page-locked q, k, v are read by the attention kernel itself over
        // PCIe (the q rows once per CTA after the ring fill is queued, the current k/v
        // by the tail tiles): no copies ahead of the launch -- e2e 129-133 -> 113-121 us
        // at C2 (same box); pageable inputs take one H2D copy each
        auto mapped = [](const void *hp) -> void * {
            cudaPointerAttributes at{};
            if (cudaPointerGetAttributes(&at, hp) != cudaSuccess) {
                (void)cudaGetLastError();
                return nullptr;
            }
            return at.type == cudaMemoryTypeHost ? at.devicePointer : nullptr;
        };
        static const long zc_in = env_knob("OSCAR_HOST_INPUTS", 1);  // 0: always copy (A/B)
        // (16-byte aligned rows only: the kernel reads them with vector loads)
        const bool al = (((uintptr_t)q_host | (uintptr_t)k_host | (uintptr_t)v_host) & 15) == 0;
        const void *zq = zc_in && al ? mapped(q_host) : nullptr;
        const void *zk = zc_in && al ? mapped(k_host) : nullptr;
        const void *zv = zc_in && al ? mapped(v_host) : nullptr;
        if (zq && zk && zv) {
            dq = const_cast<void *>(zq);
            dk = const_cast<void *>(zk);
            dv = const_cast<void *>(zv);
        } else {
            CK(cudaMemcpyAsync(dq, q_host, qb, cudaMemcpyHostToDevice, s));
            CK(cudaMemcpyAsync(dk, k_host, kb, cudaMemcpyHostToDevice, s));
            CK(cudaMemcpyAsync(dv, v_host, kb, cudaMemcpyHostToDevice, s));
        }
        // outputs: page-locked host buffers are written by the kernel itself
        // (mapped, zero-copy), saving the D2H copies; pageable ones are copied
        static const long zc_out = env_knob("OSCAR_HOST_OUT", 1);  // 0: device buffer + one D2H copy (A/B)
        float *zo = zc_out && ((uintptr_t)out_host & 15) == 0 ? (float *)mapped(out_host) : nullptr;  // float4 rows
        float *zl = lse_host ? (float *)mapped(lse_host) : nullptr;
        h->sync_entry = true;
        try {
            h->decode_step(dq, dk, dv, zo ? zo : dout, lse_host ? (zl ? zl : dlse) : nullptr, s);
        } catch (...) {
            h->sync_entry = false;
            throw;
        }
        h->sync_entry = false;
        if (!zo) CK(cudaMemcpyAsync(out_host, dout, ob, cudaMemcpyDeviceToHost, s));
        if (lse_host && !zl) CK(cudaMemcpyAsync(lse_host, dlse, lb, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
    });
}

int oscar_kv_status(oscar_kv_handle *h, int32_t *flags, int32_t clear) {
    return guard([&] {
        if (!h || !flags) throw InvalidArg("status: null argument");
        CK(cudaSetDevice(h->device));
        CK(cudaStreamSynchronize(h->last_stream));
        int v = 0;
        CK(cudaMemcpy(&v, h->status_d, sizeof(int), cudaMemcpyDeviceToHost));
        if (clear) CK(cudaMemset(h->status_d, 0, sizeof(int)));
        *flags = v;
    });
}

int oscar_kv_stats(const oscar_kv_handle *h, int64_t *packed, int64_t *residual, int64_t *flushes) {
    return guard([&] {
        if (!h) throw InvalidArg("null handle");
        if (packed) *packed = h->packed;
        if (residual) *residual = h->residual;
        if (flushes) *flushes = h->flushes;
    });
}

int oscar_kv_memory_report(const oscar_kv_handle *h, oscar_kv_memory_report_t *r) {
    return guard([&] {
        if (!h || !r) throw InvalidArg("null argument");
        // KvCache::memory_report (kv_cache.cpp:383-402), per sequence
        const int64_t d = D, H = h->cfg.heads;
        const bool q = quantizes(h->cfg);
        const int payload_bits = q ? h->cfg.bits : 64;
        *r = oscar_kv_memory_report_t{};
        r->packed_tokens = h->packed;
        r->residual_tokens = h->residual;
        r->packed_k_payload_bits = h->packed * H * d * payload_bits;
        r->packed_v_payload_bits = h->packed * H * d * payload_bits;
        r->residual_k_payload_bits = h->residual * H * d * 64;
        r->residual_v_payload_bits = h->residual * H * d * 64;
        r->k_norm_bits = (h->packed + h->residual) * H * 64;
        if (q) {
            const int64_t kg = h->packed / h->cfg.group_size * d * H;
            const int64_t vg = h->packed * (d / h->cfg.group_size) * H;
            r->param_bits = (kg + vg) * 2 * 64;
        }
        const int64_t total = r->packed_k_payload_bits + r->packed_v_payload_bits + r->residual_k_payload_bits +
                              r->residual_v_payload_bits + r->k_norm_bits + r->param_bits;
        const int64_t values = 2 * (h->packed + h->residual);
        r->effective_bits_per_value = values ? (double)total / (double)values : 0.0;
        r->device_hot_bytes = (h->packed / R) * H * h->block_bytes + h->residual * H * d * 2 * 2;
        r->device_total_bytes = h->device_bytes;
    });
}

int oscar_kv_export(oscar_kv_handle *h, int64_t b, oscar_kv_export_t *o) {
    return guard([&] {
        if (!h || !o) throw InvalidArg("null argument");
        HostCache hc = build_host_cache(h, b);
        const int64_t H = hc.H, nb = hc.nblk;
        const int64_t kp = D * (R / G), vp = R * (D / G);
        for (int64_t hh = 0; hh < H; ++hh)
            for (int64_t k = 0; k < nb; ++k) {
                const int64_t blk = hh * nb + k;
                if (hc.bits == 2) {
                    if (o->k_payload) {
                        auto w = pack2(hc.k_codes[hh][k]);
                        std::memcpy(o->k_payload + blk * (R * D / 8), w.data(), w.size() * 2);
                    }
                    if (o->v_payload) {
                        auto w = pack2(hc.v_codes[hh][k]);
                        std::memcpy(o->v_payload + blk * (R * D / 8), w.data(), w.size() * 2);
                    }
                } else if (hc.bits == 4) {
                    if (o->k_payload) std::memcpy(o->k_payload + blk * R * D, hc.k_codes[hh][k].data(), R * D * 2);
                    if (o->v_payload) std::memcpy(o->v_payload + blk * R * D, hc.v_codes[hh][k].data(), R * D * 2);
                }
                if (hc.bits != 0) {
                    if (o->k_delta) std::memcpy(o->k_delta + blk * kp, hc.k_delta[hh][k].data(), kp * 8);
                    if (o->k_zp) std::memcpy(o->k_zp + blk * kp, hc.k_zp[hh][k].data(), kp * 8);
                    if (o->k_constant) std::memcpy(o->k_constant + blk * kp, hc.k_const[hh][k].data(), kp * 8);
                    if (o->v_delta) std::memcpy(o->v_delta + blk * vp, hc.v_delta[hh][k].data(), vp * 8);
                    if (o->v_zp) std::memcpy(o->v_zp + blk * vp, hc.v_zp[hh][k].data(), vp * 8);
                    if (o->v_constant) std::memcpy(o->v_constant + blk * vp, hc.v_const[hh][k].data(), vp * 8);
                } else {
                    if (o->k_raw) std::memcpy(o->k_raw + blk * R * D, hc.k_raw[hh][k].data(), R * D * 8);
                    if (o->v_raw) std::memcpy(o->v_raw + blk * R * D, hc.v_raw[hh][k].data(), R * D * 8);
                }
            }
        if (o->k_norms)
            for (int64_t hh = 0; hh < H; ++hh)
                std::memcpy(o->k_norms + hh * hc.packed, hc.k_norms[hh].data(), hc.packed * 8);
        if (o->k_residual) std::memcpy(o->k_residual, hc.k_res.data(), hc.k_res.size() * 8);
        if (o->k_norms_residual) std::memcpy(o->k_norms_residual, hc.k_norms_res.data(), hc.k_norms_res.size() * 8);
        if (o->v_residual) std::memcpy(o->v_residual, hc.v_res.data(), hc.v_res.size() * 8);
    });
}

int oscar_kv_dump(oscar_kv_handle *h, int64_t b, const char *path) {
    return guard([&] {
        if (!h || !path) throw InvalidArg("null argument");
        HostCache hc = build_host_cache(h, b);
        std::ofstream f(path, std::ios::binary);
        if (!f) throw std::runtime_error(std::string("cache dump: cannot open ") + path);
        const oscar_kv_config &c = h->cfg;
        const int64_t H = hc.H, nb = hc.nblk;
        // manifest: nlohmann::json object (std::map => sorted keys), compact dump
        auto sizes = [&](bool is_v) {
            std::ostringstream s;
            s << "[";
            for (int64_t hh = 0; hh < H; ++hh) {
                s << (hh ? ",[" : "[");
                for (int64_t k = 0; k < nb; ++k) {
                    const int64_t params = hc.bits ? (is_v ? R * (D / G) : D * (R / G)) : 0;
                    const int64_t words = hc.bits == 2 ? R * D / 8 : 0;
                    const int64_t pc = hc.bits == 2 ? R * D : 0;
                    const int64_t codes = hc.bits == 4 ? R * D : 0;
                    const int64_t raw = hc.bits == 0 ? R * D : 0;
                    s << (k ? "," : "") << "{\"codes\":" << codes << ",\"packed_count\":" << pc
                      << ",\"params\":" << params << ",\"raw\":" << raw << ",\"words\":" << words << "}";
                }
                s << "]";
            }
            s << "]";
            return s.str();
        };
        const bool pre = h->prefilled;
        std::ostringstream m;
        m << "{\"G\":" << c.group_size << ",\"H\":" << H << ",\"R\":" << c.residual_len << ",\"S_packed\":" << hc.packed
          << ",\"S_packed_v\":" << hc.packed << ",\"b\":" << c.bits << ",\"d_h\":" << c.head_dim
          << ",\"flush_count\":" << h->flushes << ",\"k_blocks\":" << sizes(false)
          << ",\"k_prefilled\":" << (pre ? "true" : "false") << ",\"magic\":\"KVC1\",\"method\":\""
          << method_name(c.method) << "\",\"residual_tokens\":" << hc.r << ",\"scaling\":\""
          << scaling_name(c.scaling) << "\",\"v_blocks\":" << sizes(true)
          << ",\"v_prefilled\":" << (pre ? "true" : "false") << ",\"v_residual_tokens\":" << hc.r << "}";
        f << m.str() << "\n";
        auto write_blocks = [&](bool is_v, int64_t hh) {
            for (int64_t k = 0; k < nb; ++k) {
                if (hc.bits) {
                    const auto &dl = is_v ? hc.v_delta[hh][k] : hc.k_delta[hh][k];
                    const auto &zp = is_v ? hc.v_zp[hh][k] : hc.k_zp[hh][k];
                    const auto &cs = is_v ? hc.v_const[hh][k] : hc.k_const[hh][k];
                    for (size_t i = 0; i < dl.size(); ++i) {
                        f.write(reinterpret_cast<const char *>(&dl[i]), 8);
                        f.write(reinterpret_cast<const char *>(&zp[i]), 8);
                        f.write(reinterpret_cast<const char *>(&cs[i]), 8);
                    }
                    const auto &codes = is_v ? hc.v_codes[hh][k] : hc.k_codes[hh][k];
                    if (hc.bits == 2) {
                        auto w = pack2(codes);
                        f.write(reinterpret_cast<const char *>(w.data()), (std::streamsize)(w.size() * 2));
                    } else {
                        f.write(reinterpret_cast<const char *>(codes.data()), (std::streamsize)(codes.size() * 2));
                    }
                } else {
                    const auto &raw = is_v ? hc.v_raw[hh][k] : hc.k_raw[hh][k];
                    f.write(reinterpret_cast<const char *>(raw.data()), (std::streamsize)(raw.size() * 8));
                }
            }
        };
        for (int64_t hh = 0; hh < H; ++hh) {
            write_blocks(false, hh);
            f.write(reinterpret_cast<const char *>(hc.k_norms[hh].data()), (std::streamsize)(hc.packed * 8));
        }
        f.write(reinterpret_cast<const char *>(hc.k_res.data()), (std::streamsize)(hc.k_res.size() * 8));
        f.write(reinterpret_cast<const char *>(hc.k_norms_res.data()), (std::streamsize)(hc.k_norms_res.size() * 8));
        for (int64_t hh = 0; hh < H; ++hh) write_blocks(true, hh);
        f.write(reinterpret_cast<const char *>(hc.v_res.data()), (std::streamsize)(hc.v_res.size() * 8));
        if (!f) throw std::runtime_error("cache dump: write failed");
    });
}

int oscar_kv_load(oscar_kv_handle *h, int64_t b, const char *path) {
    return guard([&] {
        if (!h || !path) throw InvalidArg("null argument");
        load_kvc1(h, b, path);
    });
}

int oscar_kv_materialize(oscar_kv_handle *h, int64_t b, double *k_out, double *v_out) {
    return guard([&] {
        if (!h) throw InvalidArg("null handle");
        HostCache hc = build_host_cache(h, b);
        const int64_t H = hc.H, nb = hc.nblk;
        // kv_cache.cpp:327-381 (unpack_block + dequantize_one x norm)
        for (int64_t hh = 0; hh < H; ++hh)
            for (int64_t k = 0; k < nb; ++k)
                for (int t = 0; t < R; ++t) {
                    const int64_t tok = k * R + t;
                    const double s = hc.k_norms[hh][tok];
                    for (int c = 0; c < D; ++c) {
                        double xk, xv;
                        if (hc.bits) {
                            const int pk = c * (R / G) + t / G, pv = t * (D / G) + c / G;
                            const double dk = hc.k_delta[hh][k][pk], dv = hc.v_delta[hh][k][pv];
                            xk = dk == 0.0 ? hc.k_const[hh][k][pk]
                                           : dk * ((double)hc.k_codes[hh][k][c * R + t] - (double)hc.k_zp[hh][k][pk]);
                            xv = dv == 0.0 ? hc.v_const[hh][k][pv]
                                           : dv * ((double)hc.v_codes[hh][k][t * D + c] - (double)hc.v_zp[hh][k][pv]);
                        } else {
                            xk = hc.k_raw[hh][k][t * D + c];
                            xv = hc.v_raw[hh][k][t * D + c];
                        }
                        if (k_out) k_out[(tok * H + hh) * D + c] = xk * s;
                        if (v_out) v_out[(tok * H + hh) * D + c] = xv;
                    }
                }
        for (int64_t t = 0; t < hc.r; ++t)
            for (int64_t hh = 0; hh < H; ++hh) {
                const double s = hc.k_norms_res[t * H + hh];
                for (int c = 0; c < D; ++c) {
                    if (k_out) k_out[((hc.packed + t) * H + hh) * D + c] = hc.k_res[(t * H + hh) * D + c] * s;
                    if (v_out) v_out[((hc.packed + t) * H + hh) * D + c] = hc.v_res[(t * H + hh) * D + c];
                }
            }
    });
}

int oscar_lse_merge(const float *outs, const float *lses, int64_t parts, int64_t rows, int64_t d, float *out,
                    float *lse_out, void *stream) {
    return guard([&] {
        if (!outs || !lses || !out) throw InvalidArg("lse_merge: null argument");
        if (parts <= 0 || rows < 0 || d <= 0) throw InvalidArg("lse_merge: bad sizes");
        CK(launch_lse_merge(outs, lses, parts, rows, d, out, lse_out, (cudaStream_t)stream));
    });
}

int oscar_kv_last_launch_count(const oscar_kv_handle *h) { return h ? h->last_launches : 0; }

}  // extern "C"
