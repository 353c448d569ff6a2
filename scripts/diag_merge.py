"""Per-launch time of the sequence-shard merge kernels (p2p peer_merge vs NCCL-path lse_merge)."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2605_19660_b200 import kv_cache as kc  # noqa: E402
from paper_2605_19660_b200.sharding import local_peer_plans  # noqa: E402


def timed(fn, n=300):
    for _ in range(20):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) * 1e3 / n


rows, world = 28, 8
plans, areas = local_peer_plans(world, rows)
torch.cuda.synchronize()
for p in plans:
    kc.peer_publish_empty(p, 1)
out = torch.empty((rows, 128), device="cuda")
outs = torch.randn((world, rows, 128), device="cuda")
lses = torch.randn((world, rows), device="cuda")
res = {
    "peer_merge_us": timed(lambda: kc.peer_merge(plans[0], 1, out)),
    "peer_publish_empty_us": timed(lambda: kc.peer_publish_empty(plans[0], 1)),
    "lse_merge_us": timed(lambda: kc.lse_merge(outs, lses, out=out)),
    "empty_torch_kernel_us": timed(lambda: out.zero_()),
}
print(json.dumps(res))
