"""Config 5 after the second densify: where does an iteration's time go?
Trains 210 iterations (densify at 100, 200), then 6 more under torch.profiler."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2502_01826_b200 import datagen, raster, train
from paper_2502_01826_b200.scene import cube_init, round_to_f32

s0 = round_to_f32(cube_init([-15] * 3, [15] * 3, 0.65, 360, 180))
gen = {"mode": "spectrum", "n_samples": 256, "n_az": 360, "n_el": 180, "carrier_freq": 2.4e9, "rx": [0.0, 0.0, 0.0],
       "tx_box": {"lo": [-8, -8, -3], "hi": [8, 8, 3]}, "sigma_beam": 2.0,
       "paths": [{"reflector": None, "amplitude": 1.0},
                 {"reflector": [6.0, -4.0, 2.0], "amplitude": 0.6, "extra_phase": 0.7},
                 {"reflector": [-5.0, 7.0, -1.0], "amplitude": 0.4, "extra_phase": -1.1}]}
txs, frames = datagen.generate_dataset(gen, seed=7, device=True)
ds = raster.DeviceScene.from_host(s0, "cuda")
cfg = train.TrainConfig(iterations=600, densify_grad_threshold=1e-7)
cfg.iterations = int(os.environ.get("ITERS", "402"))
graph = os.environ.get("GRAPH", "0") == "1"
train.train_loop(ds, txs, frames.contiguous(), cfg, batch=16, seed=1, graph=graph)
torch.cuda.synchronize()
print("caps", {k: (v if not isinstance(v, dict) else len(v)) for k, v in raster._CAPS.items()})
g = raster.build_geometry(ds, psi_tx=txs[:16].contiguous(), forward=True)
print("stats (slow rays, hcap over, max live, H, max tile list, max pending, sphere, whitened, used)", g.stats[:9])
cfg2 = train.TrainConfig(iterations=8, densify_grad_threshold=1e-7)
tim = []
t0 = time.perf_counter()
train.train_loop(ds, txs, frames.contiguous(), cfg2, batch=16, seed=3, graph=graph, timings=tim)
torch.cuda.synchronize()
print("wall ms/it", (time.perf_counter() - t0) * 1e3 / 8, "device", [(round(t, 3), round(g, 3)) for _, t, _, _, g in tim])
from torch.profiler import ProfilerActivity, profile
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    train.train_loop(ds, txs, frames.contiguous(), cfg2, batch=16, seed=3, graph=graph)
    torch.cuda.synchronize()

print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=15))
