"""Distribution of the by-Gaussian hit spans (in 32-hit groups) at config 2 and
config 5: sizes K9c's straddle sums (k_geom_final)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2502_01826_b200 import raster
from paper_2502_01826_b200.scene import bench_scene, cube_init, default_txs, round_to_f32

out = {}
for name, s in (("config2", round_to_f32(bench_scene(np.random.default_rng(0), 100_000, 90, 45))),
                ("config5", round_to_f32(cube_init([-15] * 3, [15] * 3, 0.65, 360, 180)))):
    ds = raster.DeviceScene.from_host(s, "cuda")
    tx = torch.as_tensor(default_txs(16, seed=3), dtype=torch.float32, device="cuda")
    geo = raster.build_geometry(ds, psi_tx=tx, forward=True, index=True)
    torch.cuda.synchronize()
    rg = geo.gidx["g_rng"].view(-1, 2)[: ds.n].cpu().numpy().astype(np.int64)
    used = rg[:, 1] > rg[:, 0]
    w = ((rg[used, 1] - 1) >> 5) - (rg[used, 0] >> 5) + 1
    hits = rg[used, 1] - rg[used, 0]
    q = [50, 90, 99, 99.9, 100]
    out[name] = {"n": int(ds.n), "used": int(used.sum()), "H": int(hits.sum()),
                 "hits_per_used_pct": dict(zip(map(str, q), np.percentile(hits, q).round(1).tolist())),
                 "groups_pct": dict(zip(map(str, q), np.percentile(w, q).round(1).tolist())),
                 "frac_w1": round(float((w == 1).mean()), 3), "frac_w_gt4": round(float((w > 4).mean()), 3),
                 "sum_w_over_used": round(float(w.sum() / used.sum()), 2)}
print(json.dumps(out))
