"""Shared helpers for the parity tests (golden loading, tolerance metrics)."""

from __future__ import annotations

import hashlib
import os

import numpy as np

from paper_2502_01826_b200.scene import HostScene, bench_scene, round_to_f32

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
GRAD_KEYS = ("d_mean", "d_quat", "d_log_scale", "d_trans_mag", "d_trans_phase", "d_coeffs", "d_cov")


def load(name: str):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)


def scene_from(z, prefix: str) -> HostScene:
    cfg = z[prefix + "cfg"]
    return HostScene(
        z[prefix + "means"], z[prefix + "quats"], z[prefix + "log_scales"],
        z[prefix + "trans_mag_raw"], z[prefix + "trans_phase"], z[prefix + "coeffs"],
        z[prefix + "rx"], float(cfg[0]), int(cfg[1]), int(cfg[2]), int(cfg[3]),
    )


def config1_scene() -> HostScene:
    return round_to_f32(bench_scene(np.random.default_rng(0), 10_000, 360, 180))


def sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def scene_sha(s: HostScene) -> str:
    cfg = np.array([s.ress_radius, s.n_az, s.n_el, s.fle_degree], np.float64)
    return sha(s.means, s.quats, s.log_scales, s.trans_mag_raw, s.trans_phase, s.coeffs, s.rx, cfg)


def rel_err(a, b) -> float:
    a = np.asarray(a)
    b = np.asarray(b)
    d = np.linalg.norm((a - b).ravel())
    n = np.linalg.norm(b.ravel())
    return float(d / n) if n > 0 else float(d)


def class_rel(a, r, floor_frac: float = 1e-3, tiny: float = 1e-30) -> float:
    """Max per-entry |a-r| / max(|a|, |r|, floor_frac * class_max, tiny).

    The class-scale floor of gradcheck.py:11-17,213-215.
    """
    a = np.asarray(a)
    r = np.asarray(r)
    if np.iscomplexobj(a) or np.iscomplexobj(r):
        a = np.stack([np.real(a), np.imag(a)])
        r = np.stack([np.real(r), np.imag(r)])
    if r.size == 0:
        return 0.0
    cmax = float(np.max(np.abs(r)))
    den = np.maximum(np.maximum(np.abs(a), np.abs(r)), max(floor_frac * cmax, tiny))
    return float(np.max(np.abs(a - r) / den))


def l1_upstream(frame: np.ndarray) -> np.ndarray:
    p = np.abs(frame) ** 2
    d = np.sign(p - (1.3 * p + 0.05)) / p.size
    return 2.0 * d * frame
