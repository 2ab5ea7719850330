"""Config 5 of BASELINE.json: training with density control (densify / prune
every 100 iterations during the first half), Gaussian count changing, the
geometry re-binned and re-sorted every iteration under the new count.

Scene: cube_init(Box([-15]*3, [15]*3), 0.65) at 360x180 (46^3 = 97,336
Gaussians, scene.py:355-388).  Data: synthetic -- measured frames are
power spectra rendered by this framework (the reference's
spectrum_oracle multipath simulator is outside this tier; here the frames of
a perturbed copy of the initial scene) for 256 TX positions; `--batch` TX per iteration.  Prints one JSON line with the
per-iteration times (CUDA events) of ordinary and N-changing iterations.
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2502_01826_b200 import raster, train
from paper_2502_01826_b200.scene import cube_init, default_txs, round_to_f32

ap = argparse.ArgumentParser()
ap.add_argument("--iterations", type=int, default=600)
ap.add_argument("--batch", type=int, default=16)
ap.add_argument("--threshold", type=float, default=1e-7, help="densify_grad_threshold (lowered so it fires)")
a = ap.parse_args()

s0 = round_to_f32(cube_init([-15] * 3, [15] * 3, 0.65, 360, 180))
rng = np.random.default_rng(0)
tgt = s0.copy()  # measured frames: a perturbed copy of the initial scene
tgt.means = tgt.means + rng.normal(0, 0.2, tgt.means.shape)
tgt.trans_mag_raw = rng.normal(0, 1, tgt.n)
tgt.coeffs = tgt.coeffs * rng.uniform(0.5, 1.5, (tgt.n, 1)) * np.exp(1j * rng.uniform(-1, 1, (tgt.n, 1)))
tgt = round_to_f32(tgt)
txs = torch.as_tensor(default_txs(256, seed=7), dtype=torch.float32, device="cuda")
tds = raster.DeviceScene.from_host(tgt, "cuda")
frames = []
for c in range(0, 256, 64):
    g = raster.build_geometry(tds, psi_tx=txs[c:c + 64], forward=True)
    frames.append((g.S.abs() ** 2).float())
frames = torch.cat(frames).contiguous()
del tds, g

ds = raster.DeviceScene.from_host(s0, "cuda")
cfg = train.TrainConfig(iterations=a.iterations, densify_grad_threshold=a.threshold)
# warm-up of the density-control kernels and allocator sizes on a throwaway copy
_w = raster.DeviceScene.from_host(s0, "cuda")
_st = train.TrainState.zeros(_w.n, "cuda")
_st.grad_ema.fill_(1.0)
train.densify(_w, _st, 1, cfg, 0)
train.prune(_w, _st, 1, cfg)
del _w, _st
torch.cuda.synchronize()
tim = []
trace, dens, pr = train.train_loop(ds, txs, frames, cfg, batch=a.batch, seed=1, timings=tim)
warm = 5
plain = [t for it, t, n, ev in tim[warm:] if not ev]
events = [{"iteration": it, "ms": round(t, 3), "n_after": n, "event": ev} for it, t, n, ev in tim if ev]
print(json.dumps({
    "config": "config 5: cube_init 46^3 Gaussians, 360x180, densify/prune every 100 iterations (first half)",
    "data": "synthetic (frames of a perturbed copy of the initial scene)", "batch_tx": a.batch, "iterations": a.iterations,
    "n_start": int(s0.n), "n_end": int(ds.n), "ms_per_iteration_plain": round(float(np.median(plain)), 3),
    "spectra_per_s_plain": round(a.batch / (float(np.median(plain)) / 1e3), 1),
    "density_events": events,
    "loss_first": round(float(np.mean([r.total for r in trace[:10]])), 6),
    "loss_last": round(float(np.mean([r.total for r in trace[-10:]])), 6),
    "cloned_split_pruned": [[it, len(r.cloned), len(r.split)] for it, r in dens] + [[it, len(r.removed)] for it, r in pr],
}))
