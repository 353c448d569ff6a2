"""bf16 decode baseline through FlashInfer (library) at the C2 shape:
BatchDecodeWithPagedKVCacheWrapper, 16 sequences x 32K tokens, 32 q / 8 kv heads."""
import json
import sys
import time

import torch


def run(B=16, S=32768, Hq=32, Hkv=8, D=128, page=16, iters=20):
    import flashinfer

    dev = torch.device("cuda")
    npages = S // page
    kv = torch.randn((B * npages, 2, page, Hkv, D), device=dev, dtype=torch.bfloat16)  # NHD
    indptr = torch.arange(0, B + 1, device=dev, dtype=torch.int32) * npages
    indices = torch.arange(0, B * npages, device=dev, dtype=torch.int32)
    last = torch.full((B,), page, device=dev, dtype=torch.int32)
    ws = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
    w = flashinfer.BatchDecodeWithPagedKVCacheWrapper(ws, "NHD")
    t0 = time.time()
    w.plan(indptr, indices, last, Hq, Hkv, D, page, q_data_type=torch.bfloat16, kv_data_type=torch.bfloat16)
    q = torch.randn((B, Hq, D), device=dev, dtype=torch.bfloat16)
    o = w.run(q, kv)
    torch.cuda.synchronize()
    setup_s = time.time() - t0
    for _ in range(3):
        w.run(q, kv)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        w.run(q, kv)
    e1.record()
    torch.cuda.synchronize()
    us = 1e3 * e0.elapsed_time(e1) / iters
    byt = 2 * B * Hkv * S * D * 2
    return {"us": us, "achieved_gbs": byt / (us * 1e-6) / 1e9, "setup_s": setup_s, "version": flashinfer.__version__,
            "out_finite": bool(torch.isfinite(o).all())}


if __name__ == "__main__":
    pages = [int(x) for x in sys.argv[1:]] or [16]
    print(json.dumps({p: run(page=p) for p in pages}))
