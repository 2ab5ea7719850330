"""Config 5 of BASELINE.json: training with density control (densify / prune
every 100 iterations during the first half), Gaussian count changing, the
geometry re-binned and re-sorted every iteration under the new count.

Scene: cube_init(Box([-15]*3, [15]*3), 0.65) at 360x180 (46^3 = 97,336
Gaussians, scene.py:355-388).  Data: a spectrum_oracle dataset (the
reference's multipath simulator, oracle.py:100-153, restated on the GPU in
datagen.py) of 256 TX positions drawn as cli.cmd_generate draws them: a
direct path and two reflectors; `--batch` TX per iteration.  Prints one JSON
line with the per-iteration times (CUDA events) of ordinary and N-changing
iterations (the re-bin / re-sort under the new Gaussian count).
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2502_01826_b200 import datagen, raster, train
from paper_2502_01826_b200.scene import cube_init, default_txs, round_to_f32

ap = argparse.ArgumentParser()
ap.add_argument("--iterations", type=int, default=600)
ap.add_argument("--batch", type=int, default=16)
ap.add_argument("--eager", action="store_true", help="no captured iterations (train_loop(graph=False), the default)")
ap.add_argument("--graph", action="store_true", help="captured iterations (train_loop(graph=True))")
ap.add_argument("--threshold", type=float, default=1e-7, help="densify_grad_threshold (lowered so it fires)")
a = ap.parse_args()

s0 = round_to_f32(cube_init([-15] * 3, [15] * 3, 0.65, 360, 180))
gen = {"mode": "spectrum", "n_samples": 256, "n_az": 360, "n_el": 180, "carrier_freq": 2.4e9, "rx": [0.0, 0.0, 0.0],
       "tx_box": {"lo": [-8, -8, -3], "hi": [8, 8, 3]}, "sigma_beam": 2.0,
       "paths": [{"reflector": None, "amplitude": 1.0},
                 {"reflector": [6.0, -4.0, 2.0], "amplitude": 0.6, "extra_phase": 0.7},
                 {"reflector": [-5.0, 7.0, -1.0], "amplitude": 0.4, "extra_phase": -1.1}]}
txs, frames = datagen.generate_dataset(gen, seed=7, device=True)
frames = frames.contiguous()
ds = raster.DeviceScene.from_host(s0, "cuda")
cfg = train.TrainConfig(iterations=a.iterations, densify_grad_threshold=a.threshold)
# warm-up of the density-control kernels and allocator sizes on a throwaway copy
_w = raster.DeviceScene.from_host(s0, "cuda")
_st = train.TrainState.zeros(_w.n, "cuda")
_st.grad_ema.fill_(1.0)
train.densify(_w, _st, 1, cfg, 0)
train.prune(_w, _st, 1, cfg)
# and of the step itself (module loading, allocator pools, capacities) on another copy
_w = raster.DeviceScene.from_host(s0, "cuda")
train.train_loop(_w, txs, frames, train.TrainConfig(iterations=3), batch=a.batch, seed=2, graph=a.graph and not a.eager)
del _w, _st
torch.cuda.synchronize()
tim = []
e_start, e_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e_start.record()
trace, dens, pr = train.train_loop(ds, txs, frames, cfg, batch=a.batch, seed=1, timings=tim, graph=a.graph and not a.eager)
e_end.record()
torch.cuda.synchronize()
total_ms = e_start.elapsed_time(e_end)
warm = 5
plain = [t for it, t, n, ev, gap in tim[warm:] if not ev]
gaps = np.array([gap for it, t, n, ev, gap in tim])
events = [{"iteration": it, "ms": round(t, 3), "n_after": n, "event": ev} for it, t, n, ev, gap in tim if ev]
print(json.dumps({
    "config": "config 5: cube_init 46^3 Gaussians, 360x180, densify/prune every 100 iterations (first half)",
    "data": "synthetic: spectrum_oracle dataset (datagen.generate_dataset, direct path + 2 reflectors, 256 TX)", "batch_tx": a.batch, "iterations": a.iterations,
    "n_start": int(s0.n), "n_end": int(ds.n), "ms_per_iteration_plain": round(float(np.median(plain)), 3),
    "spectra_per_s_plain": round(a.batch / (float(np.median(plain)) / 1e3), 1),
    "ms_per_iteration_whole_run": round(total_ms / a.iterations, 3),
    "ms_median_by_50": [round(float(np.median([t for it, t, n, ev, gap in tim if b <= it < b + 50] or [0])), 3)
                        for b in range(1, a.iterations + 1, 50)],
    "idle_between_iterations_ms": {"sum": round(float(gaps.sum()), 2), "median": round(float(np.median(gaps)), 3),
                                   "top": [[int(tim[i][0]), round(float(gaps[i]), 2)] for i in np.argsort(-gaps)[:8]]},
    "captured": a.graph and not a.eager, "loop_counts": train.train_loop.last_counts,
    "density_events": events,
    "loss_first": round(float(np.mean([r.total for r in trace[:10]])), 6),
    "loss_last": round(float(np.mean([r.total for r in trace[-10:]])), 6),
    "cloned_split_pruned": [[it, len(r.cloned), len(r.split)] for it, r in dens] + [[it, len(r.removed)] for it, r in pr],
}))
