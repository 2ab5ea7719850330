"""Golden vectors for the spectrum loss, produced by the REFERENCE loss.py.

    python tests/golden/make_golden_loss.py      (build container only)

Frames are float32-representable; cases: the config-1 frame power against a
scaled + noisy target, random 72x18 and 360x90 frames, identical frames, and a
constant target (dynamic-range floor).  Stored per case: pred, gt, weights,
the four loss values and grad_frame, plus S for the upstream chain (lam = 2 grad S, grad.py:119).
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/nb")

from rfsplat import loss  # noqa: E402


def f32(a):
    return np.asarray(a, np.float32).astype(np.float64)


def main():
    rng = np.random.default_rng(7)
    c1 = np.load(os.path.join(HERE, "config1_10k.npz"))
    S0 = c1["frame"].astype(np.complex64).astype(np.complex128)
    cases = []
    P0 = np.abs(S0) ** 2
    cases.append(("c1", S0, f32(1.3 * P0 + 0.05 + 0.01 * rng.random(P0.shape)), 0.2, 0.2))
    for name, shape in (("r72", (72, 18)), ("r360", (360, 90))):
        S = (rng.normal(size=shape) + 1j * rng.normal(size=shape)).astype(np.complex64).astype(np.complex128)
        gt = f32(np.abs(S) ** 2 * rng.uniform(0.5, 1.5, shape))
        cases.append((name, S, gt, 0.3, 0.1))
    S = (rng.normal(size=(72, 18)) + 1j * rng.normal(size=(72, 18))).astype(np.complex64).astype(np.complex128)
    cases.append(("same", S, f32(np.abs(S) ** 2), 0.2, 0.2))
    cases.append(("flat", S, np.full((72, 18), 0.25), 0.5, 0.25))
    out = {"names": np.array([c[0] for c in cases])}
    for name, S, gt, ws, wf in cases:
        pred = np.abs(S) ** 2
        rep = loss.spectrum_loss(pred, gt, ws, wf)
        out[name + "_S"] = S.astype(np.complex64)     # exact: S is complex64-representable
        out[name + "_gt"] = gt.astype(np.float32)     # exact: gt is float32-representable
        out[name + "_w"] = np.array([ws, wf])
        out[name + "_vals"] = np.array([rep.total, rep.l1, rep.ssim, rep.fourier])
        out[name + "_grad"] = rep.grad_frame
    # scalar modes (loss.py:158-180): (pred, gt, mode) -> (value, upstream)
    sc = [(0.3 + 0.4j, 0.1 - 0.2j, "complex"), (-1.5 + 2.0j, -1.0 + 2.5j, "complex"),
          (0.02 + 0.01j, -30.0, "real_power"), (3.0 - 4.0j, 20.0, "real_power"), (1e-12 + 0j, -50.0, "real_power")]
    out["scalar_pred"] = np.array([complex(np.complex64(c[0])) for c in sc])
    out["scalar_gt"] = np.array([complex(np.complex64(c[1])) for c in sc])
    out["scalar_mode"] = np.array([c[2] for c in sc])
    vals, ups = [], []
    for p, g, m in zip(out["scalar_pred"], out["scalar_gt"], out["scalar_mode"]):
        v, u = loss.scalar_loss(complex(p), complex(g) if m == "complex" else float(g.real), str(m))
        vals.append(v)
        ups.append(u)
    out["scalar_value"] = np.array(vals)
    out["scalar_up"] = np.array(ups, dtype=np.complex128)
    np.savez_compressed(os.path.join(HERE, "loss_frames.npz"), **out)
    print("wrote loss_frames.npz")


if __name__ == "__main__":
    main()
