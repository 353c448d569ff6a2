"""Accuracy side of the fp16-operand trade-off: the decode
kernel's deviation from the fp64 oracle with each design variant's roundings
removed, from the numpy model of the kernel (tests/fp16_model.py, pinned to
the device by tests/test_gpu_numerics.py).  The speed side of each variant is
measured on the B200 by cost builds of the library (OSK_COST_* in
csrc/attention.cu, scripts/gpu_accuracy_cost.sh).  CPU only; test tooling.

    python scripts/accuracy_cost.py --bits 2 --trials 8
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
from fp16_model import ROUNDINGS, emulate, f16, head_arrays  # noqa: E402
from oracle import bindings as ob  # noqa: E402

# variant -> the roundings it removes (fp16_model.ROUNDINGS: q, ka, kb, foldk, p, va, vb, foldv)
VARIANTS = {
    "shipped (all fp16 operands)": (),
    "K offset b as hi+lo fp16 (+1 KB/record, +8 HMMA)": ("kb",),
    "K side exact: b hi+lo, q*a hi+lo (+2 KB, +72 HMMA, +64 HMUL2)": ("kb", "ka", "foldk"),
    "K side + q exact": ("kb", "ka", "foldk", "q"),
    "everything exact (the oracle)": ROUNDINGS,
}


def keys(kind, rng, S, d):
    k = rng.standard_normal((S, 1, d))
    if kind == "outliers":  # tests/test_gpu_scale.py distribution
        k[..., 0:4] = 18.0 * np.sign(rng.standard_normal((1, 1, 4))) + 0.3 * k[..., 0:4]
        k[..., 4:12] *= 8.0
    elif kind == "tni":  # bench.py synth_kv (oscar_cli.cpp:364-384 recipe)
        k[..., 0:4] = np.sign(rng.standard_normal((1, 1, 4))) * 18.0 + 0.3 * k[..., 0:4]
        k[..., 4:12] *= 8.0
        sinks = rng.integers(0, S, 8)
        k[sinks] = 0.01 * 44.0 * rng.standard_normal((8, 1, d)) / 11.3
    return k


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--bits", type=int, default=2)
    ap.add_argument("--S", type=int, default=16384)
    ap.add_argument("--trials", type=int, default=8)
    args = ap.parse_args()
    d = 128
    out = {"bits": args.bits, "S": args.S, "trials": args.trials, "metric": "max|o - o_oracle| / max|o_oracle|"}
    for kind in ("normal", "tni", "outliers"):
        rng = np.random.default_rng(11)
        k = keys(kind, rng, args.S, d)
        v = rng.standard_normal((args.S, 1, d))
        o = ob.PortCache(H=1, bits=args.bits)
        o.append(f16(k), f16(v))
        K, V, norms = head_arrays(o.export(), 0)
        res = {name: [] for name in VARIANTS}
        for _ in range(args.trials):
            qr = ob.port_fht(f16(rng.standard_normal(d)))
            exact = emulate(qr, K, V, norms, on=())
            scale = np.abs(exact).max()
            for name, off in VARIANTS.items():
                on = tuple(r for r in ROUNDINGS if r not in off)
                res[name].append(float(np.abs(emulate(qr, K, V, norms, on=on) - exact).max() / scale))
        out[kind] = {name: {"mean": float(np.mean(e)), "max": float(np.max(e))} for name, e in res.items()}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
