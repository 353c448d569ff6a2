"""Synthetic K/V/Q inputs for the OScaR KV-cache path (no datasets, no network).

Keys follow the reference's pipeline-evaluation TNI recipe
(tools/oscar_cli.cpp:364-384, generator datagen.cpp:69-134): i.i.d. N(0,1)
base, four offset channels {0..3} at +-18 with width 0.3, eight variance-scaled
channels {4..11} x8, and eight flat "sink" tokens at 0.01 x the typical token
norm.  Values and queries are N(0,1).  Everything is rounded to bf16 (round to
nearest even) so the CPU oracle and the device path see identical inputs
(SURVEY.md §8(d)).  numpy's PCG64 is used for the stream; the reference's
mt19937_64 stream is not needed because inputs are passed explicitly.
"""
from __future__ import annotations

import numpy as np


def to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """fp32/fp64 -> bf16 bit patterns (uint16), round to nearest even."""
    f = np.ascontiguousarray(x, dtype=np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    rounding = ((u >> 16) & 1) + 0x7FFF
    return ((u + rounding) >> 16).astype(np.uint16)


def bf16_bits_to_f64(b: np.ndarray) -> np.ndarray:
    return (np.asarray(b, dtype=np.uint16).astype(np.uint32) << 16).view(np.float32).astype(np.float64)


def round_bf16(x: np.ndarray) -> np.ndarray:
    return bf16_bits_to_f64(to_bf16_bits(x))


def tni_keys(rng: np.random.Generator, S: int, H: int, d: int = 128, sinks: int = 8) -> np.ndarray:
    x = rng.standard_normal((S, H, d))
    offset = [c for c in (0, 1, 2, 3) if c < d]
    scaled = [c for c in range(4, 12) if c < d]
    signs = np.where(rng.random((H, len(offset))) < 0.5, -1.0, 1.0)
    for ci, c in enumerate(offset):
        x[:, :, c] = signs[None, :, ci] * 18.0 + 0.3 * x[:, :, c]
    for c in scaled:
        x[:, :, c] *= 8.0
    tn2 = (d - len(offset) - len(scaled)) + len(offset) * (18.0**2 + 0.3**2) + len(scaled) * 64.0
    sink_scale = 0.01 * np.sqrt(tn2 / d)
    if S > 0 and sinks > 0:
        for t in rng.choice(S, size=min(sinks, S), replace=False):
            x[t] = sink_scale * rng.standard_normal((H, d))
    return x


def make_inputs(seed: int, S: int, H: int, d: int = 128, tni: bool = True):
    """bf16-representable fp64 arrays: keys [S,H,d], values [S,H,d]."""
    rng = np.random.default_rng(seed)
    k = tni_keys(rng, S, H, d) if tni else rng.standard_normal((S, H, d))
    v = rng.standard_normal((S, H, d))
    return round_bf16(k), round_bf16(v)


def make_queries(seed: int, n: int, Hq: int, d: int = 128, gain: float = 1.0):
    rng = np.random.default_rng(seed + 7919)
    return round_bf16(gain * rng.standard_normal((n, Hq, d)))
