"""Golden vectors for the optimizer and density control, produced by the
REFERENCE train.py (sgd_step, TrainState.observe, densify, prune).

    python tests/golden/make_golden_train.py      (build container only)

Inputs are float32-representable; gradient-EMA values and magnitudes are kept
away from the thresholds so decisions do not hinge on fp32 vs fp64 rounding.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/nb")

from rfsplat import train  # noqa: E402
from rfsplat.grad import GradientBuffer  # noqa: E402
from rfsplat.scene import Box, RFScene  # noqa: E402


def f32(a):
    return np.asarray(a, np.float32).astype(np.float64)


def main():
    rng = np.random.default_rng(3)
    n, K = 400, 16
    means = f32(rng.uniform(-10, 10, (n, 3)))
    q = rng.normal(size=(n, 4))
    quats = f32(q / np.linalg.norm(q, axis=1, keepdims=True))
    log_scales = f32(rng.uniform(np.log(0.2), np.log(6.0), (n, 3)))
    raw = f32(np.where(rng.random(n) < 0.15, rng.uniform(-9, -6.5, n), rng.uniform(-3, 3, n)))
    phase = f32(rng.uniform(-np.pi, np.pi, n))
    coeffs = (f32(rng.normal(0, 0.1, (n, K))) + 1j * f32(rng.normal(0, 0.1, (n, K))))
    scene = RFScene(means, quats, log_scales, raw, phase, coeffs, np.zeros(3), 1.0, 2.4e9, Box([-60] * 3, [60] * 3),
                    90, 45, 3)
    g = GradientBuffer(
        f32(rng.normal(0, 1e-3, (n, 3))), f32(rng.normal(0, 1e-2, (n, 4))), f32(rng.normal(0, 1e-2, (n, 3))),
        f32(rng.normal(0, 1e-2, n)), f32(rng.normal(0, 1e-2, n)),
        f32(rng.normal(0, 1e-2, (n, K))) + 1j * f32(rng.normal(0, 1e-2, (n, K))), np.zeros((n, 3, 3)))
    cfg = train.TrainConfig(iterations=3000)
    it = 700
    ema = f32(np.where(rng.random(n) < 0.3, rng.uniform(3e-4, 1e-3, n), rng.uniform(0, 1e-4, n)))
    last = f32(rng.normal(0, 1e-3, (n, 3)))
    out = {"means": means, "quats": quats, "log_scales": log_scales, "raw": raw, "phase": phase,
           "coeffs": coeffs.astype(np.complex64), "g_mean": g.d_mean, "g_quat": g.d_quat, "g_log_scale": g.d_log_scale,
           "g_mag": g.d_trans_mag, "g_phase": g.d_trans_phase, "g_coeffs": g.d_coeffs.astype(np.complex64),
           "ema": ema, "last": last, "it": np.array([it, cfg.iterations])}
    # sgd_step + observe (train.py:145-162, 102-105)
    s1 = scene.copy()
    train.sgd_step(s1, g, it, cfg)
    st = train.TrainState(ema.copy(), last.copy())
    st.observe(g, cfg.ema_decay)
    out.update({"sgd_means": s1.means, "sgd_quats": s1.quats, "sgd_log_scales": s1.log_scales,
                "sgd_raw": s1.trans_mag_raw, "sgd_phase": s1.trans_phase, "sgd_coeffs": s1.coeffs,
                "obs_ema": st.grad_ema, "obs_last": st.last_dmean})
    # densify (train.py:165-222)
    s2 = scene.copy()
    st2 = train.TrainState(ema.copy(), last.copy())
    rep = train.densify(s2, st2, it, cfg, np.random.default_rng(0))
    out.update({"dens_cloned": np.array(rep.cloned, np.int64), "dens_split": np.array(rep.split, np.int64),
                "dens_means": s2.means, "dens_quats": s2.quats, "dens_log_scales": s2.log_scales,
                "dens_raw": s2.trans_mag_raw, "dens_n": np.array([s2.n])})
    # prune (train.py:225-245)
    s3 = scene.copy()
    st3 = train.TrainState(ema.copy(), last.copy())
    prep = train.prune(s3, st3, it, cfg)
    out.update({"prune_removed": np.array(prep.removed, np.int64), "prune_means": s3.means,
                "prune_ema": st3.grad_ema, "prune_n": np.array([s3.n])})
    out["lr_mean"] = np.array([train.lr_mean(cfg, i) for i in (0, 1, 700, 1500, 3000, 4000)])
    np.savez_compressed(os.path.join(HERE, "train_golden.npz"), **out)
    print("wrote train_golden.npz", len(rep.cloned), "cloned", len(rep.split), "split", len(prep.removed), "pruned")


if __name__ == "__main__":
    main()
