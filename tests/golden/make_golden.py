"""Generate golden fixtures from the COMPILED REFERENCE (oracle/_ref).

Run in the build container (needs /root/reference to build oracle/_ref):
    python tests/golden/make_golden.py
Each fixture stores bf16 inputs, the reference cache exported through its own
KVC1 dump (kv_cache.cpp:469-507) and one decode-step output
(ref_decode_step = pipeline.cpp:292-323 body without projections).
"""
import os
import sys
import tempfile

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from oracle import bindings as ob  # noqa: E402
from paper_2605_19660_b200.synthetic import make_inputs, make_queries  # noqa: E402
from test_oracle import export_to_flat  # noqa: E402

FIXTURES = [
    # name, method, bits, scaling, S, prefill, H, d, R, rotate_v, gqa, seed
    ("oscar_int2_l2", "oscar", 2, "l2", 300, 290, 2, 128, 128, False, 4, 11),
    ("oscar_int4_l2", "oscar", 4, "l2", 260, 255, 2, 128, 128, False, 4, 12),
    ("oscar_int2_rsqrt_rotv", "oscar", 2, "rsqrt", 200, 120, 1, 128, 128, True, 7, 13),
    ("kivi_int2", "kivi", 2, "l2", 140, 139, 1, 128, 128, False, 1, 14),
]


def main():
    ob.build()
    out_dir = os.path.dirname(os.path.abspath(__file__))
    for name, method, bits, scaling, S, cut, H, d, R, rotv, g, seed in FIXTURES:
        k, v = make_inputs(seed, S + 1, H, d)
        q = make_queries(seed, 1, H * g, d)[0]
        ref = ob.RefCache(method=method, bits=bits, scaling=scaling, d=d, H=H, R=R, rotate_v=rotv)
        ref.append(k[:cut], v[:cut])
        for t in range(cut, S):
            ref.append(k[t : t + 1], v[t : t + 1])
        with tempfile.TemporaryDirectory() as td:
            flat = export_to_flat(ref.export(td))
        o = ref.decode_step(q, k[S], v[S], g, append=False)
        arrays = {"x_" + n: a for n, a in flat.items()}
        for n in ("k_codes", "v_codes"):
            arrays["x_" + n] = arrays["x_" + n].astype(np.uint16)
        np.savez_compressed(
            os.path.join(out_dir, f"cache_{name}.npz"),
            method=np.array(method), scaling=np.array(scaling),
            meta_bits=np.array(bits), meta_d=np.array(d), meta_H=np.array(H), meta_R=np.array(R),
            meta_rotate_v=np.array(int(rotv)), meta_prefill=np.array(cut), meta_gqa=np.array(g),
            k_in=k[:S], v_in=v[:S], q_in=q, k_cur=k[S], v_cur=v[S], x_decode_out=o, **arrays,
        )
        print("wrote", name)


if __name__ == "__main__":
    main()
