import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import oracle
from helpers import load, scene_from, l1_upstream, class_rel, GRAD_KEYS
from paper_2502_01826_b200 import api, raster
z = load("edge_scenes.npz")
for prefix in ["cube_", "special_"]:
    s = scene_from(z, prefix)
    ctx = api.prepare_context(s)
    S = api.render_complex_frame(s, z[prefix + "tx"], ctx=ctx)
    ref = z[prefix + "frame"]
    P, Pr = np.abs(S)**2, np.abs(ref)**2
    floor = 1e-3 * Pr.max()
    bad = np.abs(P - Pr) > 1e-4 * np.maximum(Pr, floor)
    print(prefix, "rel", np.linalg.norm(P-Pr)/np.linalg.norm(Pr), "bad rays", bad.sum(), "of", bad.size)
    oc = oracle.OracleContext(s); oc.set_tx(z[prefix + "tx"])
    counts, gg, ww, TT = raster.hit_lists_host(ctx.geometry)
    for r in np.flatnonzero(bad.ravel())[:4]:
        h = oc.ray_hits(r)
        print(" ray", r, "P", P.ravel()[r], Pr.ravel()[r], "gpu live", counts[r], "ref live", z[prefix+"live"][r])
        print("   ref g", h["g"][:12].tolist()); print("   gpu g", gg[r,:min(counts[r],12)].tolist())
        print("   ref t", np.round(h["t_mid"][:8], 12).tolist(), "clamped", h["clamped"][:8].astype(int).tolist())
        print("   ref w", h["w"][:6].tolist()); print("   gpu w", ww[r,:6].tolist())
    g = api.backward_frame(s, z[prefix + "tx"], l1_upstream(ref))
    for k in GRAD_KEYS:
        a = getattr(g, k); r_ = z[prefix + k]
        e = class_rel(a, r_)
        if e > 1e-4:
            aa = np.abs(a - r_).reshape(len(a), -1).max(1); i = int(np.argmax(aa))
            print(" grad", k, "class_rel %.2e" % e, "worst g", i, a[i].ravel()[:4], r_[i].ravel()[:4], "class max", np.abs(r_).max())
