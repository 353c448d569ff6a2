"""Boundary robustness of the CUDA path: argument checks in the Python mirror,
atomic KVC1 import, and launch shapes with more (sequence, kv head) segments
per CTA than the kernel's shared-memory ticket table (the grid grows beyond
one CTA per SM instead of rejecting the shape)."""
import os

import numpy as np
import pytest

from oracle import bindings as ob
from paper_2605_19660_b200.synthetic import make_inputs, make_queries

from gpu_util import dev_bf16, log_err, rel_err

pytestmark = pytest.mark.gpu


def _cache(B=2, H=2, g=4, S=300, bits=2):
    from paper_2605_19660_b200 import KvCache, PipelineConfig

    data = [make_inputs(300 + b, S + 1, H) for b in range(B)]
    k = np.stack([d[0] for d in data])
    v = np.stack([d[1] for d in data])
    c = KvCache(PipelineConfig(heads=H, bits=bits), batch=B, q_heads=H * g, max_tokens=S + 64)
    c.buffer_quant(dev_bf16(k[:, :S]), dev_bf16(v[:, :S]))
    return c, k, v


def test_wrapper_rejects_bad_tensors():
    import torch

    c, k, v = _cache()
    B, H, g = 2, 2, 4
    q = dev_bf16(make_queries(5, B, H * g))  # [B, Hq, d]
    kc, vc = dev_bf16(k[:, 300]), dev_bf16(v[:, 300])
    with pytest.raises(ValueError, match="contiguous"):
        c.decode_step(q.transpose(0, 1).contiguous().transpose(0, 1), kc, vc)
    with pytest.raises(ValueError, match="bfloat16"):
        c.decode_step(q.float(), kc, vc)
    with pytest.raises(ValueError, match="shape"):
        c.decode_step(q[:1].contiguous(), kc, vc)  # fewer sequences than the handle
    with pytest.raises(ValueError, match="elements"):
        c.decode_step(q, kc, vc, out=torch.empty((1, H * g, 128), device="cuda"))
    with pytest.raises(ValueError, match="contiguous"):  # a strided sequence slice (sliced prefill)
        big = dev_bf16(np.concatenate([k[:, :10], k[:, :10]], axis=2))  # [B, 10, 2H, d]
        c.buffer_quant(big[:, :, :H], big[:, :, H:])
    with pytest.raises(ValueError, match="CUDA"):
        c.decode_step(q.cpu(), kc, vc)
    # a good call still works after the rejected ones (nothing was launched)
    out = c.decode_step(q, kc, vc)
    assert torch.isfinite(out).all()


def test_failed_load_leaves_handle_unchanged(tmp_path):
    """A truncated KVC1 file must not leave token counters pointing at records
    that were never uploaded (load is all-or-nothing)."""
    from paper_2605_19660_b200 import KvCache, PipelineConfig

    src, k, v = _cache(B=1, S=300)
    good = str(tmp_path / "good.kvc1")
    src.dump(0, good)
    raw = open(good, "rb").read()
    bad = str(tmp_path / "bad.kvc1")
    open(bad, "wb").write(raw[:-4096])  # drops the tail of the value section
    dst = KvCache(PipelineConfig(heads=2, bits=2), batch=1, q_heads=8, max_tokens=400)
    with pytest.raises(ValueError, match="too short"):
        dst.load(0, bad)
    assert (dst.packed_tokens, dst.residual_tokens, dst.flush_count) == (0, 0, 0)
    dst.load(0, good)
    assert (dst.packed_tokens, dst.residual_tokens) == (256, 44)
    a, b = src.export(0), dst.export(0)
    for key in ("k_payload", "v_payload", "k_delta", "k_zp", "v_delta", "v_zp", "k_norms", "k_residual"):
        assert np.array_equal(a[key], b[key]), key


def test_more_segments_than_the_ticket_table():
    """B=1200 x 8 KV heads x 200 tokens (1 packed block + a 72-token window):
    9600 (b, kv head) segments over 148 SMs is ~65 per CTA, beyond the 64-entry
    shared-memory table; the launch uses more CTAs than SMs instead of failing.
    Sampled sequences are checked against the CPU oracle."""
    import torch

    from paper_2605_19660_b200 import KvCache, PipelineConfig

    B, H, g, S = 1200, 8, 4, 200
    gen = torch.Generator(device="cuda")
    gen.manual_seed(5)
    k = torch.randn((B, S + 1, H, 128), generator=gen, device="cuda").to(torch.bfloat16)
    v = torch.randn((B, S + 1, H, 128), generator=gen, device="cuda").to(torch.bfloat16)
    q = torch.randn((B, H * g, 128), generator=gen, device="cuda").to(torch.bfloat16)
    c = KvCache(PipelineConfig(heads=H, bits=2), batch=B, q_heads=H * g, max_tokens=S + 8, keep_exact=False)
    c.buffer_quant(k[:, :S].contiguous(), v[:, :S].contiguous())
    out = c.decode_step(q, k[:, S].contiguous(), v[:, S].contiguous()).cpu().numpy()
    for b in (0, 611, B - 1):
        o = ob.PortCache(H=H, bits=2)
        kb = k[b].float().cpu().numpy().astype(np.float64)
        vb = v[b].float().cpu().numpy().astype(np.float64)
        o.append(kb[:S], vb[:S])
        ref = o.decode_step(q[b].float().cpu().numpy().astype(np.float64), kb[S], vb[S], g, append=False)
        err = rel_err(out[b].astype(np.float64), ref)
        log_err(f"many_segments_grid_growth[B=1200,S=200,H=8][b={b}]", err)
        assert err <= 5e-3, (b, err)


_MERGE_FORMS_SCRIPT = r"""
import sys, numpy as np, torch
sys.path[:0] = sys.argv[1:2]
from paper_2605_19660_b200 import KvCache, PipelineConfig
gen = torch.Generator(device="cuda"); gen.manual_seed(11)
outs = []
# ~2 CTA partials per segment; 9 (the largest poll-form merge); 20 (ticket form in both runs)
for B, H, g, S in ((16, 8, 4, 4 * 1024 + 77), (1, 1, 4, 72 * 128 + 5), (2, 1, 4, 160 * 128 + 5)):
    k = torch.randn((B, S + 3, H, 128), generator=gen, device="cuda").to(torch.bfloat16)
    v = torch.randn((B, S + 3, H, 128), generator=gen, device="cuda").to(torch.bfloat16)
    q = torch.randn((B, H * g, 128), generator=gen, device="cuda").to(torch.bfloat16)
    c = KvCache(PipelineConfig(heads=H, bits=2), batch=B, q_heads=H * g, max_tokens=S + 64, keep_exact=False)
    c.buffer_quant(k[:, :S].contiguous(), v[:, :S].contiguous())
    for t in range(S, S + 3):
        outs.append(c.decode_step(q, k[:, t].contiguous(), v[:, t].contiguous()).cpu().numpy().ravel())
    assert c.status()["raw"] == 0
np.save(sys.argv[2], np.concatenate(outs))
"""


def test_poll_and_ticket_merge_forms_agree(tmp_path):
    """The split-KV merge has two forms (attention.cu: the segment's first CTA polls
    flag-in-word partials, or the last-arriving CTA merges after an atomic ticket).
    The same decode steps with the poll form allowed (default) and with tickets only
    (OSCAR_POLL_MERGE=0, read once per process) agree to fp32 rounding, at shapes
    whose segments have ~2, 9 and 20 partials."""
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script = tmp_path / "forms.py"
    script.write_text(_MERGE_FORMS_SCRIPT)
    res = {}
    for mode in ("1", "0"):
        env = dict(os.environ, OSCAR_POLL_MERGE=mode)
        out = tmp_path / f"out{mode}.npy"
        subprocess.run([sys.executable, str(script), root, str(out)], env=env, check=True, timeout=300)
        res[mode] = np.load(out)
    scale = np.abs(res["0"]).max()
    err = np.abs(res["1"] - res["0"]).max() / scale
    log_err("merge_forms_poll_vs_ticket", float(err))
    assert err < 1e-5, err
