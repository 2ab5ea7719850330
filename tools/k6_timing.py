"""Per-warp duration of K6 (k_hits) vs its work: what sets the kernel's critical path?

usage: k6_timing.py [N] [split_min]   (rfs_debug_k6_timing records, u64[8] per warp)
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2502_01826_b200 import raster, _native
from paper_2502_01826_b200.scene import bench_scene, round_to_f32
n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000
if len(sys.argv) > 2:  # K6 split threshold (rfs_hits split_min; 0 = off)
    raster._CAPS["split_min"] = int(sys.argv[2])
s = round_to_f32(bench_scene(np.random.default_rng(0), n, 360, 180))
ds = raster.DeviceScene.from_host(s, "cuda")
raster.build_geometry(ds)
buf = torch.zeros(8 * 16384, dtype=torch.int64, device="cuda")
_native.call("rfs_debug_k6_timing", buf.data_ptr())
raster.build_geometry(ds)
torch.cuda.synchronize()
_native.call("rfs_debug_k6_timing", None)
b = buf.view(-1, 8).cpu().numpy()
b = b[b[:, 1] > 0]
t0 = b[:, 0].min()
dur = (b[:, 1] - b[:, 0]) / 1e3
end = (b[:, 1] - t0) / 1e3
start = (b[:, 0] - t0) / 1e3
L, chunks, rel, mx, nu, live = (b[:, k].astype(np.float64) for k in range(2, 8))
print(f"N={n} split_min={raster._CAPS['split_min']} warps {len(b)} kernel span {end.max():.1f} us; warp duration "
      f"mean {dur.mean():.1f} median {np.median(dur):.1f} max {dur.max():.1f}; start max {start.max():.1f} us")
for q in (0.5, 0.9, 0.99):
    print(f"  duration q{q}: {np.quantile(dur, q):.1f} us")
order = np.argsort(L)
for lo, hi in ((0, 0.25), (0.25, 0.5), (0.5, 0.75), (0.75, 1.0)):
    sel = order[int(lo * len(L)):int(hi * len(L))]
    print(f"  list length {L[sel].min():.0f}-{L[sel].max():.0f}: duration mean {dur[sel].mean():.1f} "
          f"max {dur[sel].max():.1f}")
# least squares: duration ~ a*chunks + b*cone survivors + c*max-lane exact tests + d*union + e*live
X = np.stack([chunks, rel, mx, nu, live, np.ones_like(dur)], 1)
coef, *_ = np.linalg.lstsq(X, dur, rcond=None)
pred = X @ coef
r2 = 1 - ((dur - pred) ** 2).sum() / ((dur - dur.mean()) ** 2).sum()
names = ["chunk", "cone survivor", "max-lane exact", "union rec", "live hit", "const"]
print("  fit (us per unit): " + ", ".join(f"{k} {c * 1e3:.1f} ns" if k != "const" else f"{k} {c:.1f} us"
                                           for k, c in zip(names, coef)) + f"; R^2 {r2:.3f}")
top = np.argsort(dur)[-5:]
for i in top:
    print(f"  slowest: dur {dur[i]:.1f} start {start[i]:.1f} L {L[i]:.0f} chunks {chunks[i]:.0f} rel {rel[i]:.0f} "
          f"mx {mx[i]:.0f} nu {nu[i]:.0f} live {live[i]:.0f}")
med = np.argsort(dur)[len(dur) // 2]
print(f"  median warp: dur {dur[med]:.1f} L {L[med]:.0f} chunks {chunks[med]:.0f} rel {rel[med]:.0f} mx {mx[med]:.0f} "
      f"nu {nu[med]:.0f} live {live[med]:.0f}")
