"""Numpy model of the decode kernel's fp16 operand roundings (test tooling).

process_block (paper_2605_19660_b200/csrc/attention.cu) computes, per packed
block, with fp16 tensor-core operands and fp32 accumulation:

  logit_t = norm_t * c0 * ( sum_c code[t,c] * f16(q16[c] * a16[c,grp(t)])
                            + sum_c b16[c,grp(t)] * q16[c] )
  P_t     = exp2(logit_t - m)             (fp32; the sum l uses this value)
  o[c]    = sum_t code[t,c] * f16(f16(P_t) * av16[t,grp(c)]) + sum_t f16(P_t) * bv16[t,grp(c)]
  out     = o / l

with q16 = f16(FHT(q)), a16/b16 = f16(delta), f16(-delta*zp) (a constant group:
a = 0, b = lo) as stored in the 12.8 KB record.  The oracle computes the same
sums in fp64 on the dequantized cache (pipeline.cpp:152-180).  `emulate` with
every rounding on reproduces the kernel to fp32 accumulation noise; with every
rounding off it IS the oracle.  Each rounding is ~2^-12 relative and enters the
logit, so the kernel's deviation from the oracle grows with the logit spread.
"""
from __future__ import annotations

import numpy as np

ROUNDINGS = ("q", "ka", "kb", "foldk", "p", "va", "vb", "foldv")
C0 = np.log2(np.e) / np.sqrt(128.0)


def f16(x):
    return np.asarray(x, np.float64).astype(np.float16).astype(np.float64)


def head_arrays(ec, h: int):
    """Per-token views of one head of an ExportedCache (packed blocks only):
    K codes/a/b [T, d], V codes/a/b [T, d], key norms [T]."""
    R, G, d = ec.R, ec.G, ec.d
    kc, ka, kb, vc, va, vb = [], [], [], [], [], []
    pk = np.arange(d)[None, :] * (R // G) + (np.arange(R) // G)[:, None]  # kv_cache.cpp:194-250 layout
    pv = np.arange(R)[:, None] * (d // G) + (np.arange(d) // G)[None, :]
    for blk in ec.k_blocks[h]:
        dl, zp, cst = blk["delta"][pk], blk["zp"][pk], blk["constant"][pk]
        kc.append(blk["codes"].reshape(d, R).T.astype(np.float64))
        ka.append(dl)
        kb.append(np.where(dl == 0, cst, -dl * zp))
    for blk in ec.v_blocks[h]:
        dl, zp, cst = blk["delta"][pv], blk["zp"][pv], blk["constant"][pv]
        vc.append(blk["codes"].reshape(R, d).astype(np.float64))
        va.append(dl)
        vb.append(np.where(dl == 0, cst, -dl * zp))
    cat = np.concatenate
    T = len(ec.k_blocks[h]) * R
    return (cat(kc), cat(ka), cat(kb)), (cat(vc), cat(va), cat(vb)), np.asarray(ec.k_norms[h][:T], np.float64)


def emulate(q_rot: np.ndarray, K, V, norms, on=ROUNDINGS):
    """Attention of one rotated query row over one head's packed tokens."""
    kc, ka, kb = K
    vc, va, vb = V

    def r(name):
        return f16 if name in on else (lambda x: np.asarray(x, np.float64))

    q16 = r("q")(q_rot)
    bq = r("foldk")(q16[None, :] * r("ka")(ka))
    logit = ((kc * bq).sum(1) + (r("kb")(kb) * q16[None, :]).sum(1)) * norms * C0
    P = np.exp2(logit - logit.max())
    l = P.sum()
    P16 = r("p")(P)
    bv = r("foldv")(P16[:, None] * r("va")(va))
    o = (vc * bv).sum(0) + (P16[:, None] * r("vb")(vb)).sum(0)
    return o / l
