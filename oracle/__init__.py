"""CPU parity oracle for the B200 rasterizer -- TEST INFRASTRUCTURE ONLY.

A ctypes wrapper over `rfs_oracle.c`, a plain-C fp64 restatement of the
reference package `rfsplat` (pkg/src/rfsplat/{_kernels,splat,render,grad,
scene,fle}.py).  Only tests/, `__graft_entry__.smoke()` and bench.py's
cpu_baseline / `--impl reference` legs may import this module, and only as the
checker or the timed CPU baseline -- never as the thing measured or shipped.
The product package (paper_2502_01826_b200) does not import it.

Parity pinning: tests/golden/*.npz were produced by the reference itself
(tests/golden/make_golden.py); tests/test_oracle_golden.py checks this
restatement against them (bit-exact tile index, ~1e-12 floats).

Scenes are any object with the RFScene attribute layout (scene.py:205-352).
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

_dp = C.POINTER(C.c_double)
_u8p = C.POINTER(C.c_uint8)
_i64p = C.POINTER(C.c_int64)
_u64p = C.POINTER(C.c_uint64)


class _Ctx(C.Structure):
    _fields_ = [
        ("n", C.c_int64), ("n_az", C.c_int64), ("n_el", C.c_int64), ("degree", C.c_int64),
        ("n_coeffs", C.c_int64), ("tiles_u", C.c_int64), ("tiles_v", C.c_int64), ("m", C.c_int64),
        ("rx", C.c_double * 3), ("tx", C.c_double * 3), ("ress_radius", C.c_double),
        ("means", _dp), ("quats", _dp), ("log_scales", _dp), ("raw", _dp), ("phase", _dp), ("coeffs", _dp),
        ("covs", _dp), ("inv_covs", _dp), ("norm_consts", _dp), ("rho", _dp), ("unit_rho", _dp),
        ("bearing_alpha", _dp), ("bearing_beta", _dp), ("bearing_valid", _u8p),
        ("basis", _dp), ("basis_dalpha", _dp), ("basis_dbeta", _dp), ("psi", _dp),
        ("active", _u8p), ("center_u", _dp), ("center_v", _dp), ("radius_px", _dp),
        ("tile_radius", _dp), ("depth", _dp), ("splat_r2", _dp), ("ray_dirs", _dp),
        ("keys", _u64p), ("indices", _i64p), ("ranges", _i64p),
    ]


def build() -> str:
    """Compile liboracle.so with the committed Makefile (gcc, -fopenmp)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(_LIB_PATH) or (
                os.path.getmtime(_LIB_PATH) < os.path.getmtime(os.path.join(_HERE, "rfs_oracle.c"))
            ):
                build()
            L = C.CDLL(_LIB_PATH)
            P = C.POINTER(_Ctx)
            L.orc_prepare.argtypes = [P]
            L.orc_set_tx.argtypes = [P]
            L.orc_tiles_count.argtypes = [P]
            L.orc_tiles_count.restype = C.c_int64
            L.orc_tiles_fill.argtypes = [P]
            L.orc_forward.argtypes = [P, _dp, C.c_int]
            L.orc_forward_naive.argtypes = [P, _dp, C.c_int]
            L.orc_live_counts.argtypes = [P, _i64p, C.c_int]
            L.orc_backward.argtypes = [P, _dp, C.c_int] + [_dp] * 7 + [C.c_int]
            L.orc_ray_hits.argtypes = [P, C.c_int64, C.c_int64, _i64p, _dp, _dp, _dp, _dp, _u8p]
            L.orc_ray_hits.restype = C.c_int64
            _lib = L
    return _lib


def _p(a, t=_dp):
    return a.ctypes.data_as(t)


class OracleContext:
    """RenderContext analogue (render.py:191-248) holding every derived array.

    Construction runs prepare_context's TX-independent part and the tile
    index; `set_tx` runs the bearing/FLE part for one transmitter.
    """

    def __init__(self, scene, threads: int = 0):
        self.threads = int(threads)
        n = len(scene.means)
        self.n = n
        self.n_az, self.n_el = int(scene.n_az), int(scene.n_el)
        self.degree = int(getattr(scene, "fle_degree", 3))
        self.K = (self.degree + 1) ** 2
        f = lambda a, s: np.ascontiguousarray(np.asarray(a, dtype=np.float64).reshape(s))
        self.means = f(scene.means, (n, 3))
        self.quats = f(scene.quats, (n, 4))
        self.log_scales = f(scene.log_scales, (n, 3))
        self.raw = f(scene.trans_mag_raw, (n,))
        self.phase = f(scene.trans_phase, (n,))
        self.coeffs_c = np.ascontiguousarray(np.asarray(scene.coeffs, dtype=np.complex128).reshape(n, self.K))
        self.rx = f(scene.rx, (3,))
        self.ress_radius = float(scene.ress_radius)
        R = self.n_az * self.n_el
        z = lambda *s: np.zeros(s, dtype=np.float64)
        self.covs, self.inv_covs = z(n, 3, 3), z(n, 3, 3)
        self.norm_consts = z(n)
        self.rho, self.unit_rho = np.zeros(n, np.complex128), np.zeros(n, np.complex128)
        self.bearing_alpha, self.bearing_beta = z(n), z(n)
        self.bearing_valid = np.zeros(n, np.uint8)
        self.basis = np.zeros((n, self.K), np.complex128)
        self.basis_dalpha = np.zeros((n, self.K), np.complex128)
        self.basis_dbeta = np.zeros((n, self.K), np.complex128)
        self.psi = np.zeros(n, np.complex128)
        self.active = np.zeros(n, np.uint8)
        self.center_u, self.center_v, self.radius_px = z(n), z(n), z(n)
        self.tile_radius, self.depth, self.splat_r2 = z(n), z(n), z(n)
        self.ray_dirs = z(R, 3)
        self.tx = np.zeros(3)
        c = _Ctx()
        c.n, c.n_az, c.n_el, c.degree, c.n_coeffs = n, self.n_az, self.n_el, self.degree, self.K
        c.rx[:] = list(self.rx)
        c.ress_radius = self.ress_radius
        c.means, c.quats, c.log_scales = _p(self.means), _p(self.quats), _p(self.log_scales)
        c.raw, c.phase, c.coeffs = _p(self.raw), _p(self.phase), _p(self.coeffs_c.view(np.float64))
        c.covs, c.inv_covs, c.norm_consts = _p(self.covs), _p(self.inv_covs), _p(self.norm_consts)
        c.rho, c.unit_rho = _p(self.rho.view(np.float64)), _p(self.unit_rho.view(np.float64))
        c.bearing_alpha, c.bearing_beta = _p(self.bearing_alpha), _p(self.bearing_beta)
        c.bearing_valid = _p(self.bearing_valid, _u8p)
        c.basis = _p(self.basis.view(np.float64))
        c.basis_dalpha = _p(self.basis_dalpha.view(np.float64))
        c.basis_dbeta = _p(self.basis_dbeta.view(np.float64))
        c.psi = _p(self.psi.view(np.float64))
        c.active = _p(self.active, _u8p)
        c.center_u, c.center_v, c.radius_px = _p(self.center_u), _p(self.center_v), _p(self.radius_px)
        c.tile_radius, c.depth, c.splat_r2 = _p(self.tile_radius), _p(self.depth), _p(self.splat_r2)
        c.ray_dirs = _p(self.ray_dirs)
        self._c = c
        L = lib()
        if L.orc_prepare(C.byref(c)) != 0:
            raise ValueError("GeometryError: a Gaussian is centered on the receiver")
        self.tiles_u, self.tiles_v = int(c.tiles_u), int(c.tiles_v)
        m = int(L.orc_tiles_count(C.byref(c)))
        c.m = m
        self.keys = np.zeros(m, np.uint64)
        self.indices = np.zeros(m, np.int64)
        self.ranges = np.zeros((self.tiles_u * self.tiles_v, 2), np.int64)
        c.keys, c.indices, c.ranges = _p(self.keys, _u64p), _p(self.indices, _i64p), _p(self.ranges, _i64p)
        rc = L.orc_tiles_fill(C.byref(c))
        if rc != 0:
            raise RuntimeError(f"orc_tiles_fill failed ({rc})")

    @property
    def m(self) -> int:
        return int(self._c.m)

    def set_tx(self, tx) -> None:
        self.tx = np.asarray(tx, dtype=np.float64).reshape(3).copy()
        self._c.tx[:] = list(self.tx)
        lib().orc_set_tx(C.byref(self._c))

    def forward(self, tiled: bool = True) -> np.ndarray:
        out = np.zeros(self.n_az * self.n_el, np.complex128)
        fn = lib().orc_forward if tiled else lib().orc_forward_naive
        fn(C.byref(self._c), _p(out.view(np.float64)), self.threads)
        return out.reshape(self.n_az, self.n_el)

    def live_counts(self) -> np.ndarray:
        out = np.zeros(self.n_az * self.n_el, np.int64)
        lib().orc_live_counts(C.byref(self._c), _p(out, _i64p), self.threads)
        return out.reshape(self.n_az, self.n_el)

    def ray_hits(self, r: int) -> dict:
        """All hits of ray r sorted by (t_mid, g) (_collect_hits, _kernels.py:27-112)."""
        cap = max(self.m, 1)
        g = np.zeros(cap, np.int64)
        t, w, d1, d2 = (np.zeros(cap) for _ in range(4))
        cl = np.zeros(cap, np.uint8)
        n = int(lib().orc_ray_hits(C.byref(self._c), int(r), cap, _p(g, _i64p), _p(t), _p(w), _p(d1), _p(d2),
                                   _p(cl, _u8p)))
        return {"g": g[:n], "t_mid": t[:n], "w": w[:n], "d1": d1[:n], "d2": d2[:n], "clamped": cl[:n].astype(bool)}

    def backward(self, upstream, include_direction_chain: bool = True) -> dict:
        up = np.ascontiguousarray(np.asarray(upstream, dtype=np.complex128).reshape(-1))
        if up.size != self.n_az * self.n_el:
            raise ValueError("ShapeError: upstream frame shape does not match the scene grid")
        n, K = self.n, self.K
        g = {
            "d_mean": np.zeros((n, 3)), "d_quat": np.zeros((n, 4)), "d_log_scale": np.zeros((n, 3)),
            "d_trans_mag": np.zeros(n), "d_trans_phase": np.zeros(n),
            "d_coeffs": np.zeros((n, K), np.complex128), "d_cov": np.zeros((n, 3, 3)),
        }
        lib().orc_backward(
            C.byref(self._c), _p(up.view(np.float64)), int(bool(include_direction_chain)),
            _p(g["d_mean"]), _p(g["d_quat"]), _p(g["d_log_scale"]), _p(g["d_trans_mag"]),
            _p(g["d_trans_phase"]), _p(g["d_coeffs"].view(np.float64)), _p(g["d_cov"]), self.threads,
        )
        return g


def render_complex_frame(scene, tx, threads: int = 0, tiled: bool = True) -> np.ndarray:
    """render.render_complex_frame (render.py:282-289) on the oracle."""
    ctx = OracleContext(scene, threads)
    ctx.set_tx(tx)
    return ctx.forward(tiled)


def backward_frame(scene, tx, upstream, include_direction_chain: bool = True, threads: int = 0) -> dict:
    """grad.backward_frame (grad.py:192-259) on the oracle."""
    ctx = OracleContext(scene, threads)
    ctx.set_tx(tx)
    return ctx.backward(upstream, include_direction_chain)


def l1_upstream(frame: np.ndarray) -> np.ndarray:
    """Synthetic upstream of BASELINE.md §2 with the L1 term only.

    lambda = upstream_to_ray(dL/dP, S) (grad.py:104-120) for the L1 loss
    (loss.py:65-73) of P = |S|^2 against the target 1.3 P + 0.05
    (gradcheck.py:187): dL/dP = sign(P - target) / cells.
    """
    p = np.abs(frame) ** 2
    d = np.sign(p - (1.3 * p + 0.05)) / p.size
    return 2.0 * d * frame
