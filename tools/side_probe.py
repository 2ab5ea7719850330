import os, sys, time
sys.path.insert(0, "/root/repo")
import numpy as np, torch
from paper_2502_01826_b200 import raster
from paper_2502_01826_b200.scene import bench_scene, default_txs, round_to_f32
n = int(sys.argv[1])
s = round_to_f32(bench_scene(np.random.default_rng(0), n, 360, 180))
ds = raster.DeviceScene.from_host(s, "cuda")
tx = torch.as_tensor(default_txs(64, seed=1), dtype=torch.float32, device="cuda")
geo = raster.build_geometry(ds)
S0 = raster.forward(geo, raster.compute_psi(ds, tx, geo.used))
lam = (S0 * 1e-6).contiguous()
for it in range(8):
    torch.cuda.synchronize()
    st = torch.cuda.memory_stats()
    t0 = time.perf_counter()
    g0 = raster.build_geometry(ds, psi_tx=tx, forward=True, index=True, after_forward=lambda S: raster.transpose_upstream(lam))
    t1 = time.perf_counter()
    raster.backward(ds, g0, tx, lam, True, psi=g0.psi, lamT=g0.after_result)
    t2 = time.perf_counter()
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    st2 = torch.cuda.memory_stats()
    print(it, f"geo {1e3*(t1-t0):.2f} bwd-enq {1e3*(t2-t1):.2f} sync {1e3*(t3-t2):.2f} ms",
          "allocs", st2.get("num_device_alloc", -1) - st.get("num_device_alloc", -1),
          "retries", st2["num_alloc_retries"] - st["num_alloc_retries"], "early", raster._CAPS["h_cap"])
