"""Host-side scene container and synthetic workload generators.

`HostScene` has the attribute layout of the reference's `rfsplat.RFScene`
(struct of arrays, scene.py:205-352): means (N,3), quats (N,4) stored
(w,x,y,z) and normalized on use, log_scales (N,3), trans_mag_raw (N,),
trans_phase (N,), coeffs (N,(L+1)^2) complex, rx (3,), ress_radius, n_az,
n_el, fle_degree.  Any object exposing those attributes (including a real
`rfsplat.RFScene`) is accepted by the GPU entry points.

The generators restate the reference's synthetic scenes so the bench and the
parity tests use the same workloads:
- `bench_scene`  <- cli._bench_scene (cli.py:278-293), the perf scene;
- `random_scene` <- gradcheck.random_scene (gradcheck.py:82-110);
- `cube_init`    <- scene.cube_init (scene.py:355-388).
Each consumes the numpy Generator in the same order as the reference, so a
seeded generator reproduces the reference scene bit for bit.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .errors import ConfigError, ShapeError

__all__ = [
    "HostScene",
    "bench_scene",
    "random_scene",
    "cube_init",
    "round_to_f32",
    "default_txs",
]


@dataclass
class HostScene:
    means: np.ndarray
    quats: np.ndarray
    log_scales: np.ndarray
    trans_mag_raw: np.ndarray
    trans_phase: np.ndarray
    coeffs: np.ndarray
    rx: np.ndarray = field(default_factory=lambda: np.zeros(3))
    ress_radius: float = 1.0
    n_az: int = 360
    n_el: int = 180
    fle_degree: int = 3

    def __post_init__(self):
        n = len(self.means)
        self.means = np.asarray(self.means, dtype=np.float64).reshape(n, 3)
        self.quats = np.asarray(self.quats, dtype=np.float64).reshape(n, 4)
        self.log_scales = np.asarray(self.log_scales, dtype=np.float64).reshape(n, 3)
        self.trans_mag_raw = np.asarray(self.trans_mag_raw, dtype=np.float64).reshape(n)
        self.trans_phase = np.asarray(self.trans_phase, dtype=np.float64).reshape(n)
        k = (self.fle_degree + 1) ** 2
        self.coeffs = np.asarray(self.coeffs, dtype=np.complex128).reshape(n, k)
        self.rx = np.asarray(self.rx, dtype=np.float64).reshape(3)
        self.ress_radius = float(self.ress_radius)
        self.n_az = int(self.n_az)
        self.n_el = int(self.n_el)
        # scene.py:250-256
        if self.ress_radius <= 0.0:
            raise ConfigError("ress_radius must be positive")
        if not (1 <= self.n_az <= 360):
            raise ConfigError("n_az must lie in 1..360")
        if not (1 <= self.n_el <= 180):
            raise ConfigError("n_el must lie in 1..180")

    @property
    def n(self) -> int:
        return self.means.shape[0]

    @classmethod
    def from_any(cls, scene) -> "HostScene":
        """Copy the SoA attributes of any RFScene-like object."""
        if isinstance(scene, HostScene):
            return scene
        for name in ("means", "quats", "log_scales", "trans_mag_raw", "trans_phase", "coeffs"):
            if not hasattr(scene, name):
                raise ShapeError(f"scene object lacks attribute {name!r}")
        return cls(
            np.array(scene.means), np.array(scene.quats), np.array(scene.log_scales),
            np.array(scene.trans_mag_raw), np.array(scene.trans_phase), np.array(scene.coeffs),
            np.array(scene.rx), float(scene.ress_radius), int(scene.n_az), int(scene.n_el),
            int(getattr(scene, "fle_degree", 3)),
        )

    def copy(self) -> "HostScene":
        return HostScene(
            self.means.copy(), self.quats.copy(), self.log_scales.copy(),
            self.trans_mag_raw.copy(), self.trans_phase.copy(), self.coeffs.copy(),
            self.rx.copy(), self.ress_radius, self.n_az, self.n_el, self.fle_degree,
        )


def round_to_f32(scene) -> HostScene:
    """Round every parameter to the nearest float32 (complex64) value.

    The GPU path takes fp32 parameters; the parity protocol
    feeds the same fp32-representable values, upcast, to the fp64 oracle.
    rx stays fp64 (the boundary takes rx as f64[3]).
    """
    s = HostScene.from_any(scene).copy()
    s.means = s.means.astype(np.float32).astype(np.float64)
    s.quats = s.quats.astype(np.float32).astype(np.float64)
    s.log_scales = s.log_scales.astype(np.float32).astype(np.float64)
    s.trans_mag_raw = s.trans_mag_raw.astype(np.float32).astype(np.float64)
    s.trans_phase = s.trans_phase.astype(np.float32).astype(np.float64)
    s.coeffs = s.coeffs.astype(np.complex64).astype(np.complex128)
    return s


def bench_scene(rng: np.random.Generator, n: int, n_az: int = 360, n_el: int = 180) -> HostScene:
    """The reference perf scene, cli.py:278-293."""
    means = rng.uniform(-15.0, 15.0, (n, 3))
    d = np.linalg.norm(means, axis=1)
    tight = d < 2.0
    means[tight] *= 2.5 / np.maximum(d[tight, None], 1e-6)
    quats = rng.normal(size=(n, 4))
    quats /= np.linalg.norm(quats, axis=1, keepdims=True)
    log_scales = rng.uniform(np.log(0.05), np.log(0.3), (n, 3))
    raw = rng.normal(0.0, 1.0, n)
    phase = rng.uniform(-np.pi, np.pi, n)
    coeffs = rng.normal(0.0, 0.1, (n, 16)) + 1j * rng.normal(0.0, 0.1, (n, 16))
    return HostScene(means, quats, log_scales, raw, phase, coeffs, np.zeros(3), 1.0, n_az, n_el, 3)


def random_scene(rng: np.random.Generator, n: int, n_az: int = 16, n_el: int = 8) -> HostScene:
    """The gradient-check scene, gradcheck.py:82-110."""
    means = rng.uniform(-8.0, 8.0, (n, 3))
    d = np.linalg.norm(means, axis=1)
    tight = d < 2.5
    means[tight] = means[tight] * (2.5 / d[tight, None]) + np.sign(means[tight])
    quats = rng.normal(size=(n, 4))
    quats /= np.linalg.norm(quats, axis=1, keepdims=True)
    log_scales = rng.uniform(np.log(0.5), np.log(1.5), (n, 3))
    raw = rng.normal(0.0, 1.0, n)
    phase = rng.uniform(-np.pi, np.pi, n)
    coeffs = rng.normal(0.0, 0.08, (n, 16)) + 1j * rng.normal(0.0, 0.08, (n, 16))
    return HostScene(means, quats, log_scales, raw, phase, coeffs, np.zeros(3), 1.0, n_az, n_el, 3)


def cube_init(lo, hi, cube_edge: float, n_az: int = 360, n_el: int = 180, c00: complex = 0.1,
              rx=(0.0, 0.0, 0.0), ress_radius: float = 1.0, fle_degree: int = 3) -> HostScene:
    """One primitive per cube of the bounds, scene.py:355-388."""
    lo = np.asarray(lo, dtype=np.float64)
    hi = np.asarray(hi, dtype=np.float64)
    if cube_edge <= 0.0:
        raise ConfigError("cube_edge must be positive")
    ext = hi - lo
    counts = np.floor(ext / cube_edge + 1e-12).astype(int)
    if np.any(counts < 1):
        raise ConfigError("cube_edge exceeds the smallest bounds extent")
    axes = [lo[a] + cube_edge * (np.arange(counts[a]) + 0.5) for a in range(3)]
    gx, gy, gz = np.meshgrid(*axes, indexing="ij")
    means = np.stack([gx.ravel(), gy.ravel(), gz.ravel()], axis=1)
    n = means.shape[0]
    quats = np.tile(np.array([1.0, 0.0, 0.0, 0.0]), (n, 1))
    log_scales = np.full((n, 3), np.log(cube_edge / 2.0))
    k = (fle_degree + 1) ** 2
    coeffs = np.zeros((n, k), dtype=np.complex128)
    coeffs[:, 0] = c00
    return HostScene(means, quats, log_scales, np.zeros(n), np.zeros(n), coeffs,
                     np.asarray(rx, dtype=np.float64), ress_radius, n_az, n_el, fle_degree)


def default_txs(b: int, seed: int = 1) -> np.ndarray:
    """TX batch from the default tx box (cli.py:90), BASELINE.md §2."""
    return np.random.default_rng(seed).uniform([-8.0, -8.0, -3.0], [8.0, 8.0, 3.0], (b, 3))
