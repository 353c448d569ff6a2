"""Attribute the decode kernel's deviation from the fp64 oracle to its fp16
operand roundings (tests/fp16_model.py), one rounding at a time, on the
test_gpu_scale.py key distribution.  CPU only; test tooling.

    python scripts/numerics_emul.py --bits 4 --trials 8
"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
from fp16_model import ROUNDINGS, emulate, f16, head_arrays  # noqa: E402
from oracle import bindings as ob  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--bits", type=int, default=4)
    ap.add_argument("--S", type=int, default=16384)
    ap.add_argument("--trials", type=int, default=8)
    args = ap.parse_args()
    rng = np.random.default_rng(5)
    S, d = args.S, 128
    k = rng.standard_normal((S, 1, d))
    k[..., 0:4] = 18.0 * np.sign(rng.standard_normal((1, 1, 4))) + 0.3 * k[..., 0:4]
    k[..., 4:12] *= 8.0
    v = rng.standard_normal((S, 1, d))
    o = ob.PortCache(H=1, bits=args.bits)
    o.append(f16(k), f16(v))
    K, V, norms = head_arrays(o.export(), 0)
    res = {}
    for _ in range(args.trials):
        qr = ob.port_fht(f16(rng.standard_normal(d)))
        exact = emulate(qr, K, V, norms, on=())
        scale = np.abs(exact).max()
        for on in [(n,) for n in ROUNDINGS] + [ROUNDINGS]:
            e = np.abs(emulate(qr, K, V, norms, on=on) - exact).max() / scale
            res.setdefault("+".join(on) if len(on) == 1 else "all", []).append(e)
    print(f"bits={args.bits} S={S} trials={args.trials}: error / max|out| vs the fp64 oracle")
    for name, v in res.items():
        print(f"  {name:6s} mean {np.mean(v):.2e} max {np.max(v):.2e}")


if __name__ == "__main__":
    main()
