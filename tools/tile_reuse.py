"""Distinct live-hit Gaussians per 16x16 tile (ψ-row reuse available to a tile-staged composite)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2502_01826_b200 import raster
from paper_2502_01826_b200.scene import bench_scene, round_to_f32
for n in (100_000, 500_000, 1_000_000):
    s = round_to_f32(bench_scene(np.random.default_rng(0), n, 360, 180))
    ds = raster.DeviceScene.from_host(s, "cuda")
    g = raster.build_geometry(ds)
    counts, hits, _, _ = raster.hit_lists_host(g)
    R = 360 * 180
    u = np.repeat(np.arange(360), 180); v = np.tile(np.arange(180), 360)
    tile = (v // 16) * 23 + (u // 16)
    k = np.arange(g.hcap)[None, :] < counts[:, None]
    tg = (tile[:, None].astype(np.int64) << 32) | hits.astype(np.int64)
    pairs = np.unique(tg[k])
    per_tile = np.bincount((pairs >> 32).astype(np.int64), minlength=276)
    hits_per_tile = np.bincount(np.repeat(tile, counts), minlength=276)
    L = (g.ranges[:, 1] - g.ranges[:, 0]).cpu().numpy()
    print(n, "H", int(counts.sum()), "distinct per tile mean/max", per_tile.mean(), per_tile.max(),
          "hits per tile mean", hits_per_tile.mean(), "reuse", counts.sum() / per_tile.sum(), "list len max", L.max())
