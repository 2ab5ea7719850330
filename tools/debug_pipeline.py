"""Run the pipeline phase by phase with a sync after each call (debug aid)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2502_01826_b200 import raster, _native
from paper_2502_01826_b200.scene import bench_scene, round_to_f32, default_txs

orig = _native.call
def traced(name, *a):
    orig(name, *a)
    torch.cuda.synchronize()
    print("  ok", name, flush=True)
_native.call = traced
n = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
b = int(sys.argv[2]) if len(sys.argv) > 2 else 8
s = round_to_f32(bench_scene(np.random.default_rng(0), n, 360, 180))
ds = raster.DeviceScene.from_host(s)
tx = torch.as_tensor(default_txs(b), dtype=torch.float32, device="cuda")
for it in range(2):
    print("iter", it, flush=True)
    g = raster.build_geometry(ds)
    print("  stats", g.stats, "M", g.m, "hcap", g.hcap, flush=True)
    psi = raster.compute_psi(ds, tx)
    S = raster.forward(g, psi)
    lam = (S * 0.01).contiguous()
    gr = raster.backward(ds, g, tx, lam, True, psi=psi)
    torch.cuda.synchronize()
    print("  grads finite", all(bool(torch.isfinite(v.view(torch.float32) if v.is_complex() else v).all()) for v in gr.values()), flush=True)
