import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2502_01826_b200 import raster
from paper_2502_01826_b200.scene import bench_scene, round_to_f32
s = round_to_f32(bench_scene(np.random.default_rng(0), 1_000_000, 360, 180))
ds = raster.DeviceScene.from_host(s, "cuda")
raster._CAPS["tile_sort"] = "bucket"
for _ in range(2):
    raster._CAPS["tile_max"] = {}
    raster.build_geometry(ds)
torch.cuda.synchronize()
torch.cuda.profiler.start()
raster._CAPS["tile_max"] = {}
raster.build_geometry(ds)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
