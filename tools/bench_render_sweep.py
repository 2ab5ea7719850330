"""Config 3 of BASELINE.json: render-only inference sweep -- N Gaussians
(default 500k, cli._bench_scene seed 0, 360x180) over T transmitter positions
(default 4096) from the default TX box.  The transmitter-independent geometry
(projection, binning, the 64-bit key sort, hit lists) is built once; the
spectra are then composited in TX chunks (psi + K7).  Reports the sort
throughput (keys/s), the composite throughput (spectra/s) and the whole
sweep, from CUDA events; prints one JSON line.
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2502_01826_b200 import raster
from paper_2502_01826_b200.scene import bench_scene, default_txs, round_to_f32

ap = argparse.ArgumentParser()
ap.add_argument("--gaussians", type=int, default=500_000)
ap.add_argument("--tx", type=int, default=4096)
ap.add_argument("--chunk", type=int, default=256)
ap.add_argument("--repeats", type=int, default=3)
a = ap.parse_args()

s = round_to_f32(bench_scene(np.random.default_rng(0), a.gaussians, 360, 180))
ds = raster.DeviceScene.from_host(s, "cuda")
txs = torch.as_tensor(default_txs(a.tx, seed=1), dtype=torch.float32, device="cuda")
ev = lambda: torch.cuda.Event(enable_timing=True)


def sweep(marks):
    e0 = ev(); e0.record()
    geo = raster.build_geometry(ds)
    e1 = ev(); e1.record()
    out = torch.empty((a.tx, 360, 180), dtype=torch.complex64, device="cuda")  # every spectrum kept
    for c in range(0, a.tx, a.chunk):
        psi = raster.compute_psi(ds, txs[c:c + a.chunk], geo.used)
        out[c:c + a.chunk] = raster.forward(geo, psi)
    e2 = ev(); e2.record()
    marks.append((e0, e1, e2, geo))
    return out


for _ in range(2):
    sweep([])
torch.cuda.synchronize()
marks = []
for _ in range(a.repeats):
    sweep(marks)
torch.cuda.synchronize()
geo_ms = float(np.median([m[0].elapsed_time(m[1]) for m in marks]))
comp_ms = float(np.median([m[1].elapsed_time(m[2]) for m in marks]))
g = marks[-1][3]
# the key sort alone, timed on the same incidences (K3, hand-written onesweep vs cub)
sort_ms = {}
for backend in ("hand", "cub"):
    keys = g.ckeys.clone()
    vals = g.vals.clone()
    perm = torch.randperm(keys.numel(), device="cuda")
    kk, vv = keys[perm].contiguous(), vals[perm].contiguous()
    for _ in range(2):
        raster.sort_pairs(kk.clone(), vv.clone(), raster.sort_end_bit(g.n_tiles), backend)
    torch.cuda.synchronize()
    t = []
    for _ in range(5):
        k2, v2 = kk.clone(), vv.clone()
        e0 = ev(); e0.record()
        raster.sort_pairs(k2, v2, raster.sort_end_bit(g.n_tiles), backend)
        e1 = ev(); e1.record()
        torch.cuda.synchronize()
        t.append(e0.elapsed_time(e1))
    sort_ms[backend] = float(np.median(t))
print(json.dumps({
    "config": f"config 3: {a.gaussians} Gaussians render-only sweep over {a.tx} TX (360x180), TX chunks of {a.chunk}",
    "data": "synthetic", "incidences_M": g.m, "live_hits_H": g.total_hits,
    "geometry_ms": round(geo_ms, 3), "composite_ms": round(comp_ms, 3),
    "composite_spectra_per_s": round(a.tx / (comp_ms / 1e3), 1),
    "sweep_spectra_per_s": round(a.tx / ((geo_ms + comp_ms) / 1e3), 1),
    "sort_keys_per_s": {k: round(g.m / (v / 1e3), 1) for k, v in sort_ms.items()},
    "sort_ms": {k: round(v, 3) for k, v in sort_ms.items()},
}))
