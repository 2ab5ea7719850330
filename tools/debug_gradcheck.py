"""Debug: gradcheck scene i through api.backward_frame, per-field errors and index checks."""
import sys, os
import numpy as np
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch
from helpers import GRAD_KEYS, class_rel, l1_upstream, load, scene_from
from paper_2502_01826_b200 import api, raster

z = load("gradcheck_scenes.npz")
if os.environ.get("POLLUTE"):
    junk = torch.full((256 * 1024 * 1024,), 0x3f7f7f7f, dtype=torch.int32, device="cuda")
    del junk
for i in [int(a) for a in sys.argv[1:]] or [0, 1, 2]:
    p = f"s{i}_"
    s = scene_from(z, p)
    ctx = api.prepare_context(s)
    geo = ctx.geometry
    print("scene", i, "n", s.means.shape[0], "grid", s.n_az, s.n_el, "stats", geo.stats[:10], "gidx", geo.gidx is not None)
    g0 = api.backward_frame(s, z[p + "tx"], l1_upstream(z[p + "frame"]), ctx=ctx, include_direction_chain=False)
    g = api.backward_frame(s, z[p + "tx"], l1_upstream(z[p + "frame"]), ctx=ctx)
    print("  d_mean(no dir) vs full diff", np.abs(g0.d_mean - g.d_mean).max(), "dcoeffs diff", np.abs(g0.d_coeffs - g.d_coeffs).max())
    gi = geo.gidx
    H = int(gi["tot"].item())
    sg = gi["sorted_g"][:H].cpu().numpy()
    rng = gi["g_rng"].cpu().numpy().reshape(-1, 2)
    used = geo.used[: s.means.shape[0]].cpu().numpy()
    nu = int(torch.as_tensor(0).new_tensor(0).item())
    print("  H", H, "used", used.sum(), "distinct hit g", len(np.unique(sg)), "n_used_dev",
          int(torch.cuda.IntTensor(1).copy_(torch.zeros(1)).item()) if False else None)
    # contiguity
    change = np.flatnonzero(np.diff(sg) != 0)
    runs = len(change) + 1 if H else 0
    print("  runs", runs, "(== distinct?)", runs == len(np.unique(sg)))
    bad = [gg for gg in np.unique(sg) if not (rng[gg, 0] < rng[gg, 1] and (sg[rng[gg, 0]:rng[gg, 1]] == gg).all())]
    print("  bad ranges", bad[:10])
    order = gi["order"][: gi["u_cap"]].cpu().numpy()
    print("  order", order[:20], "u_cap", gi["u_cap"])
    sel = z[p + "grad_sel"]
    for k in GRAD_KEYS:
        print("  ", k, class_rel(getattr(g, k)[sel], z[p + k]))
