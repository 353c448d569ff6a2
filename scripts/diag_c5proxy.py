"""C5 tail-rank proxy (64K shard of 512K over 8): which part of the step costs what.
Device time of K queued steps (host submission hidden behind a sleep kernel)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from bench import step_inputs, synth_kv
from paper_2605_19660_b200 import KvCache, PipelineConfig
from paper_2605_19660_b200 import kv_cache as kcm
from paper_2605_19660_b200 import sharding as shd
W = int(sys.argv[1]) if len(sys.argv) > 1 else 8
S, Hq, Hkv = 524288 // W, 28, 4
dev = torch.device("cuda")
st = torch.cuda.Stream(); torch.cuda.set_stream(st); sh = st.cuda_stream
cache = KvCache(PipelineConfig(heads=Hkv, bits=2), batch=1, q_heads=Hq, max_tokens=S + 1024, keep_exact=False)
k, v = synth_kv(1, S, Hkv, 7, dev); cache.buffer_quant(k, v, stream=sh); del k, v
q, kn, vn = step_inputs(400, 1, Hq, Hkv, 11, dev)
plans, areas = shd.local_peer_plans(W, Hq, dev)
out = torch.empty((Hq, 128), device=dev); o3 = torch.empty((1, Hq, 128), device=dev); lse = torch.empty((1, Hq), device=dev)
status = torch.zeros(1, dtype=torch.int32, device=dev)
torch.cuda.synchronize()
ep = [0]; pos = [0]
def timeit(fn, n=32):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    torch.cuda._sleep(int(2e6 * n))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(n): fn()
    e1.record(st); torch.cuda.synchronize()
    return round(1e3 * e0.elapsed_time(e1) / n, 2)
res = {"world": W, "shard_tokens": S}
res["attend_us"] = timeit(lambda: cache.attend(q[0], o3, lse, stream=sh))
def dec():
    cache.decode_step(q[pos[0]], kn[pos[0]], vn[pos[0]], out=o3, stream=sh); pos[0] += 1
res["decode_us"] = timeit(dec)
def pub_only():
    ep[0] += 1
    cache.attend_publish(q[0], plans[W - 1], ep[0], stream=sh)
res["attend_publish_us"] = timeit(pub_only)
def empties():
    ep[0] += 1
    for r in range(W - 1): kcm.peer_publish_empty(plans[r], ep[0], stream=sh)
res["publish_empty_x%d_us" % (W - 1)] = timeit(empties)
def full():
    ep[0] += 1
    for r in range(W - 1): kcm.peer_publish_empty(plans[r], ep[0], stream=sh)
    cache.attend_publish(q[0], plans[W - 1], ep[0], stream=sh)
    kcm.peer_merge(plans[W - 1], ep[0], out, status=status, stream=sh)
res["empties+attend_publish+merge_us"] = timeit(full)
res["status"] = int(status.item())
print(json.dumps(res))
