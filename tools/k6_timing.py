"""Per-warp duration of K6 (k_hits) vs tile-list length: is the kernel set by its longest tiles?"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2502_01826_b200 import raster, _native
from paper_2502_01826_b200.scene import bench_scene, round_to_f32
n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000
s = round_to_f32(bench_scene(np.random.default_rng(0), n, 360, 180))
ds = raster.DeviceScene.from_host(s, "cuda")
raster.build_geometry(ds)
buf = torch.zeros(3 * 4096, dtype=torch.int64, device="cuda")
_native.call("rfs_debug_k6_timing", buf.data_ptr())
raster.build_geometry(ds)
torch.cuda.synchronize()
_native.call("rfs_debug_k6_timing", None)
b = buf.view(-1, 3).cpu().numpy()
b = b[b[:, 1] > 0]
t0 = b[:, 0].min()
dur = (b[:, 1] - b[:, 0]) / 1e3
end = (b[:, 1] - t0) / 1e3
start = (b[:, 0] - t0) / 1e3
L = b[:, 2]
print(f"N={n} warps {len(b)} kernel span {end.max():.1f} us; warp duration mean {dur.mean():.1f} median {np.median(dur):.1f} "
      f"max {dur.max():.1f}; start max {start.max():.1f} us")
for q in (0.5, 0.9, 0.99):
    print(f"  duration q{q}: {np.quantile(dur, q):.1f} us")
order = np.argsort(L)
for lo, hi in ((0, 0.25), (0.25, 0.5), (0.5, 0.75), (0.75, 1.0)):
    sel = order[int(lo * len(L)):int(hi * len(L))]
    print(f"  list length {L[sel].min()}-{L[sel].max()}: duration mean {dur[sel].mean():.1f} max {dur[sel].max():.1f}")
print("  corr(duration, list length)", np.corrcoef(dur, L)[0, 1])
