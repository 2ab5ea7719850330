import sys, os, json
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2502_01826_b200 import raster
from paper_2502_01826_b200.scene import bench_scene, round_to_f32
for n in (500_000, 1_000_000):
    s = round_to_f32(bench_scene(np.random.default_rng(0), n, 360, 180))
    ds = raster.DeviceScene.from_host(s, "cuda")
    for mode in ("radix", "bucket"):
        raster._CAPS["tile_sort"] = mode
        raster._CAPS["tile_max"] = {}
        for _ in range(3):
            raster.build_geometry(ds)
        raster._CAPS["tile_max"] = {}
        torch.cuda.synchronize()
        res = []
        for _ in range(5):
            marks = []
            e0 = torch.cuda.Event(enable_timing=True); e0.record(); marks.append(("s", e0))
            raster._CAPS["tile_max"] = {}
            raster.build_geometry(ds, marks=marks)
            torch.cuda.synchronize()
            ph = {name: a.elapsed_time(b) for (_, a), (name, b) in zip(marks[:-1], marks[1:])}
            res.append(ph)
        keys = res[0].keys()
        print(n, mode, {k: round(float(np.median([r.get(k, 0) for r in res])), 4) for k in keys})
