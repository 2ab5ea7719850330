"""Host-side cost of one bench step (cProfile), to find Python launch overhead."""
import cProfile, pstats, sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2502_01826_b200 import raster
from paper_2502_01826_b200.scene import bench_scene, default_txs, round_to_f32
s = round_to_f32(bench_scene(np.random.default_rng(0), 100_000, 360, 180))
ds = raster.DeviceScene.from_host(s, "cuda")
tx = torch.as_tensor(default_txs(64), dtype=torch.float32, device="cuda")
lam = torch.randn(64, 360, 180, dtype=torch.complex64, device="cuda") * 1e-6
def step():
    g0 = raster.build_geometry(ds, psi_tx=tx, forward=True)
    return raster.backward(ds, g0, tx, lam, True, psi=g0.psi)
for _ in range(5): step()
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(20): step()
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"host enqueue time per step {1e3*(t1-t0)/20:.3f} ms; wall per step {1e3*(t2-t0)/20:.3f} ms")
pr = cProfile.Profile(); pr.enable()
for _ in range(20): step()
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
