"""Per-class gradient errors of the GPU backward on the edge scenes (diagnostic)."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from helpers import GRAD_KEYS, class_rel, load, scene_from, l1_upstream
from paper_2502_01826_b200 import api
z = load("edge_scenes.npz")
for prefix in ("cube_", "special_", "hemi_"):
    g = api.backward_frame(scene_from(z, prefix), z[prefix + "tx"], l1_upstream(z[prefix + "frame"]))
    errs = {k: class_rel(getattr(g, k), z[prefix + k]) for k in GRAD_KEYS if prefix + k in z}
    print(prefix, {k: f"{v:.2e}" for k, v in errs.items()})
