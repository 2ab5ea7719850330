"""Probe: how much would a spatial order of the Gaussians speed up the
by-Gaussian backward (K8c's lambda-row gathers, K9a)?  Runs the bench step on
the config-2 scene as generated (random order) and reordered by the Morton
code of the grid cell of each Gaussian's centre direction; prints per-phase
CUDA-event times of both."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2502_01826_b200 import raster
from paper_2502_01826_b200.scene import HostScene, bench_scene, default_txs, round_to_f32


def morton(u, v):
    def part(x):
        x = x.astype(np.uint64) & np.uint64(0xFFFF)
        x = (x | (x << np.uint64(8))) & np.uint64(0x00FF00FF)
        x = (x | (x << np.uint64(4))) & np.uint64(0x0F0F0F0F)
        x = (x | (x << np.uint64(2))) & np.uint64(0x33333333)
        x = (x | (x << np.uint64(1))) & np.uint64(0x55555555)
        return x
    return part(u) | (part(v) << np.uint64(1))


def reorder(s):
    d = s.means - s.rx
    az = np.degrees(np.arctan2(d[:, 1], d[:, 0])) % 360.0
    el = np.degrees(np.arcsin(np.clip(d[:, 2] / np.linalg.norm(d, axis=1), -1, 1))) + 90.0
    o = np.argsort(morton(np.floor(az).astype(np.int64), np.floor(el).astype(np.int64)), kind="stable")
    return HostScene(s.means[o], s.quats[o], s.log_scales[o], s.trans_mag_raw[o], s.trans_phase[o], s.coeffs[o],
                     s.rx, s.ress_radius, s.n_az, s.n_el, s.fle_degree)


base = round_to_f32(bench_scene(np.random.default_rng(0), 100_000, 360, 180))
tx = torch.as_tensor(default_txs(64, seed=1), dtype=torch.float32, device="cuda")
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
for name, s in (("random", base), ("morton", reorder(base))):
    ds = raster.DeviceScene.from_host(s, "cuda")
    geo = raster.build_geometry(ds)
    S0 = raster.forward(geo, raster.compute_psi(ds, tx, geo.used))
    lam = (S0 * 1e-6).contiguous()
    acc = {}
    for it in range(13):
        flush.fill_(1)
        marks = []
        e = torch.cuda.Event(enable_timing=True); e.record(); marks.append(("start", e))
        g0 = raster.build_geometry(ds, marks=marks, psi_tx=tx, forward=True, index=True,
                                   after_forward=lambda S: raster.transpose_upstream(lam))
        raster.backward(ds, g0, tx, lam, True, psi=g0.psi, marks=marks, lamT=g0.after_result)
        torch.cuda.synchronize()
        if it >= 3:
            for (_, a), (k, b) in zip(marks[:-1], marks[1:]):
                acc[k] = acc.get(k, 0.0) + a.elapsed_time(b) / 10
    tot = sum(acc.values())
    print(name, f"total {tot:.3f} ms", {k: round(v, 4) for k, v in acc.items()})
