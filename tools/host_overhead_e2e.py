"""Host-side cost of one api.train_step_host call (cProfile): what the e2e number pays beyond the device time."""
import cProfile, pstats, sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2502_01826_b200 import api, raster
from paper_2502_01826_b200.scene import bench_scene, default_txs, round_to_f32
s = round_to_f32(bench_scene(np.random.default_rng(0), 100_000, 360, 180))
ds = raster.DeviceScene.from_host(s, "cuda")
B = 64
txh = torch.as_tensor(default_txs(B), dtype=torch.float32).pin_memory()
gth = (torch.rand(B, 360, 180, dtype=torch.float32) * 1e-3).pin_memory()
reph = torch.empty((B, 4), dtype=torch.float64).pin_memory()
step = lambda: api.train_step_host(ds, txh, gth, reph)
for _ in range(8): step()
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(20): step()
torch.cuda.synchronize()
t1 = time.perf_counter()
print(f"wall per e2e step {1e3*(t1-t0)/20:.3f} ms")
pr = cProfile.Profile(); pr.enable()
for _ in range(20): step()
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
