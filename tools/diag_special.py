import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import oracle
from helpers import load, scene_from, l1_upstream, class_rel
from paper_2502_01826_b200 import api, raster
z = load("edge_scenes.npz")
for prefix in ["special_", "cube_", "hemi_"]:
    s = scene_from(z, prefix)
    ctx = api.prepare_context(s)
    live = ctx.geometry.ray_counts.cpu().numpy()
    d = np.flatnonzero(live != z[prefix + "live"])
    print(prefix, "live mismatches", d.size, d[:10], live[d[:10]], z[prefix + "live"][d[:10]])
    oc = oracle.OracleContext(s); oc.set_tx(z[prefix + "tx"])
    lam = l1_upstream(z[prefix + "frame"])
    g_gpu = api.backward_frame(s, z[prefix + "tx"], lam, ctx=ctx)
    g_orc = oc.backward(lam)
    for k in ["d_trans_phase", "d_trans_mag", "d_mean", "d_cov"]:
        a, r = getattr(g_gpu, k), z[prefix + k]
        print(" ", k, "gpu-vs-golden %.2e" % class_rel(a, r), "oracle-vs-golden %.2e" % class_rel(g_orc[k], r))
    a, r = g_gpu.d_trans_phase, z[prefix + "d_trans_phase"]
    i = int(np.argmax(np.abs(a - r)))
    print("  worst g", i, a[i], r[i], "hits of g on rays:", int(((raster.hit_lists_host(ctx.geometry)[1] == i) & (np.arange(ctx.geometry.hcap)[None, :] < live[:, None])).sum()))
