"""Kernel timeline of the e2e training step (api.TrainStepGraph replays at
config 2; MODE=step: the benched api.StepGraph) from torch.profiler: per-stream busy time, the critical-path gaps
and the order of the kernels of one replay."""
import json
import os
import sys
import tempfile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

from paper_2502_01826_b200 import api, parallel, raster
from paper_2502_01826_b200.scene import bench_scene, default_txs, round_to_f32

B = 64
s = round_to_f32(bench_scene(np.random.default_rng(0), 100_000, 360, 180))
ds = raster.DeviceScene.from_host(s, "cuda")
txs = default_txs(B, seed=1)
tx = torch.as_tensor(txs, dtype=torch.float32, device="cuda")
geo = raster.build_geometry(ds, psi_tx=tx, forward=True)
gt = (geo.S.abs() ** 2 * 1.3 + 0.05).float()
txh = torch.as_tensor(txs, dtype=torch.float32).pin_memory()
gth = gt.cpu().pin_memory()
reph = torch.empty((B, 4), dtype=torch.float64).pin_memory()
gb = parallel.GradBuffer(ds.n, ds.fle_degree, "cuda")
if os.environ.get("MODE", "train") == "step":  # the benched `value` step (api.StepGraph)
    lamT = raster.transpose_upstream((geo.S * 1e-3).to(torch.complex64).contiguous())
    tg = api.StepGraph(ds, tx, lamT, gb)
else:
    tg = api.TrainStepGraph(ds, txh, gth, reph, gb)
for _ in range(5):
    tg.replay()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    for _ in range(3):
        tg.replay()
    torch.cuda.synchronize()
path = os.path.join(tempfile.gettempdir(), "e2e_trace.json")
prof.export_chrome_trace(path)
ev = json.load(open(path))["traceEvents"]
gpu = [e for e in ev if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset") and "dur" in e]
gpu.sort(key=lambda e: e["ts"])
# one replay: the last third of the events by time
t_all0, t_all1 = gpu[0]["ts"], max(e["ts"] + e["dur"] for e in gpu)
span = (t_all1 - t_all0) / 3
t0 = t_all0 + 2 * span
one = [e for e in gpu if e["ts"] >= t0 - 5]
beg = one[0]["ts"]
end = max(e["ts"] + e["dur"] for e in one)
print(f"replay span {end - beg:.1f} us, events {len(one)}")
streams = {}
for e in one:
    streams.setdefault(e["args"].get("stream", e.get("tid")), []).append(e)
for k, v in streams.items():
    busy = sum(e["dur"] for e in v)
    print(f"stream {k}: {len(v)} events, busy {busy:.1f} us")
for e in one:
    print(f"{e['ts'] - beg:8.1f} {e['dur']:7.1f}  s{e['args'].get('stream', '?')}  {e['name'][:60]}")
