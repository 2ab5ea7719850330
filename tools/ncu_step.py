"""One config-2 bench step for ncu, bracketed by cudaProfilerStart/Stop
(run under `ncu --profile-from-start off ...`), so a capture holds exactly the
kernels of one steady-state step (after warm-up steps with known capacities).

    ncu --profile-from-start off --set full -o out python tools/ncu_step.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2502_01826_b200 import api, parallel, raster
from paper_2502_01826_b200.scene import bench_scene, default_txs, round_to_f32

torch.cuda.set_device(0)
dev = torch.device("cuda", 0)
scene = round_to_f32(bench_scene(np.random.default_rng(0), int(os.environ.get("N", "100000")), 360, 180))
ds = raster.DeviceScene.from_host(scene, dev)
tx = torch.as_tensor(default_txs(64, seed=1), dtype=torch.float32, device=dev)
gb = parallel.GradBuffer(ds.n, ds.fle_degree, dev)
geo = raster.build_geometry(ds)
S0 = raster.forward(geo, raster.compute_psi(ds, tx, geo.used))
P0 = S0.abs() ** 2
lam = (2.0 * torch.sign(P0 - (1.3 * P0 + 0.05)) / P0[0].numel() * S0).to(torch.complex64).contiguous()
lamT = raster.transpose_upstream(lam)
for _ in range(4):
    api.fwd_bwd_device(ds, tx, None, True, "hand", None, lamT=lamT, grads=gb)
torch.cuda.synchronize()
torch.cuda.profiler.start()
api.fwd_bwd_device(ds, tx, None, True, "hand", None, lamT=lamT, grads=gb)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("ncu_step done")
