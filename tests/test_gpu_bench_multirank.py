"""bench.py's multi-rank contract under torchrun (one process per GPU on the
driver's boxes): barrier + max-over-ranks timing, rank 0 prints ONE JSON line
with the whole-job value, other ranks print nothing; `--impl reference` runs on
rank 0 only.  The GPU boxes here have one B200, so both ranks share cuda:0 over
gloo (the OSCAR_BENCH_ONE_DEVICE test hook; never set for measurements)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _torchrun(args, port, timeout=600):
    env = dict(os.environ, OSCAR_BENCH_ONE_DEVICE="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"),
           "--gpus", "2"] + args
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    return lines


def test_bench_two_ranks_one_json_line():
    lines = _torchrun(["--steps", "8", "--warmup", "3", "--no-compare", "--no-cpu"], 29561)
    assert len(lines) == 1, lines
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["steps"] == 8 and d["warmup"] == 3
    assert d["scaling"] == "weak" and d["value"] > 0 and d["ms_per_step"] > 0
    assert d["e2e"]["value"] > 0 and d["gpu_launches"] > 0


def test_bench_reference_arm_rank0_only():
    lines = _torchrun(["--impl", "reference", "--steps", "1", "--warmup", "1"], 29562)
    assert len(lines) == 1, lines
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["cores"] >= 1


@pytest.mark.parametrize("extra,port", [(["--config", "c3", "--batch", "16", "--layers", "2"], 29563),
                                        (["--config", "c4"], 29564),
                                        (["--config", "c5", "--exchange", "nccl"], 29565),
                                        (["--config", "c5", "--exchange", "p2p"], 29566)])
def test_bench_sharded_configs_two_ranks(extra, port):
    """batch (C3), head (C4) and sequence (C5; NCCL-path and peer-memory exchange)
    sharding through bench.py on two ranks."""
    lines = _torchrun(extra + ["--steps", "4", "--warmup", "3"], port)
    assert len(lines) == 1, lines
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0
