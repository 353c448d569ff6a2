"""Helpers shared by the GPU parity tests (device tensors, export conversion)."""
from __future__ import annotations

import numpy as np

from oracle import bindings as ob
from paper_2605_19660_b200.synthetic import to_bf16_bits

R, D, G = 128, 128, 32


def dev_bf16(x: np.ndarray):
    import torch

    bits = to_bf16_bits(np.ascontiguousarray(x))
    return torch.from_numpy(bits.view(np.int16)).view(torch.bfloat16).cuda()


def export_to_oracle(ex: dict, H: int, R_: int = R, G_: int = G) -> ob.ExportedCache:
    """Device export (oscar_kv_export) -> the oracle's ExportedCache."""
    bits = ex["bits"]
    ec = ob.ExportedCache(bits, H, D, R_, G_, ex["packed"], ex["residual"], ex["flushes"])
    nb = ex["packed"] // R_
    for kind in ("k", "v"):
        heads = []
        for h in range(H):
            blocks = []
            for b in range(nb):
                if bits:
                    pay = ex[f"{kind}_payload"][h, b]
                    codes = ob.unpack_2bit_np(pay, R_ * D) if bits == 2 else pay.astype(np.uint16)
                    blocks.append(dict(codes=codes, delta=ex[f"{kind}_delta"][h, b], zp=ex[f"{kind}_zp"][h, b],
                                       constant=ex[f"{kind}_constant"][h, b], raw=np.zeros(0)))
                else:
                    blocks.append(dict(codes=np.zeros(0, np.uint16), delta=np.zeros(0), zp=np.zeros(0, np.int64),
                                       constant=np.zeros(0), raw=ex[f"{kind}_raw"][h, b]))
            heads.append(blocks)
        if kind == "k":
            ec.k_blocks = heads
        else:
            ec.v_blocks = heads
    ec.k_norms = [ex["k_norms"][h] for h in range(H)]
    ec.k_residual = ex["k_residual"]
    ec.k_norms_residual = ex["k_norms_residual"]
    ec.v_residual = ex["v_residual"]
    return ec


def rel_err(a: np.ndarray, ref: np.ndarray) -> float:
    return float(np.max(np.abs(a - ref)) / max(np.max(np.abs(ref)), 1e-30))


def log_err(tag: str, err: float) -> None:
    """Append a measured parity error to gpurun_out/parity_errors.jsonl (evidence)."""
    import json
    import os

    d = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "gpurun_out")
    if os.path.isdir(d):
        with open(os.path.join(d, "parity_errors.jsonl"), "a") as f:
            f.write(json.dumps({"test": tag, "max_abs_err_rel_to_max_abs_out": err}) + "\n")
