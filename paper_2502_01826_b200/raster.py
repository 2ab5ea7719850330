"""Host orchestration of the sm_100a rasterizer (torch tensors + the C ABI).

One step = `build_geometry` (K1-K6, transmitter independent) followed by the
TX-batched `compute_psi` (K5), `forward` (K7) and `backward` (K8a, K8b, K9).
PyTorch supplies device memory (caching allocator) and the current CUDA
stream; every kernel is launched through include/rfsplat_b200.h.

Host synchronisations per step: one 8-byte read of M (the incidence count
sizes the sort buffers) and one read of the hit-list statistics (slow-path
rays, hit-capacity overflow).  Both are the analogue of the reference
allocating its arrays from counts (_kernels.py:542-543, grad.py:224-231).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native
from .errors import GeometryError, ShapeError

__all__ = ["DeviceScene", "Geometry", "build_geometry", "compute_psi", "forward", "backward", "GRAD_FIELDS"]

TILE = 16
MAX_TX_PER_LAUNCH = 256
GRAD_FIELDS = ("d_mean", "d_quat", "d_log_scale", "d_trans_mag", "d_trans_mag_raw", "d_trans_phase", "d_coeffs", "d_cov")


def _ptr(t: torch.Tensor | None):
    return None if t is None else t.data_ptr()


def _stream():
    return torch.cuda.current_stream().cuda_stream


@dataclass
class DeviceScene:
    """fp32 device copy of a scene's SoA parameters (the boundary's inputs)."""

    means: torch.Tensor        # f32 [N,3]
    quats: torch.Tensor        # f32 [N,4]
    log_scales: torch.Tensor   # f32 [N,3]
    trans_mag_raw: torch.Tensor  # f32 [N]
    trans_phase: torch.Tensor  # f32 [N]
    coeffs: torch.Tensor       # c64 [N,K]
    rx: tuple = (0.0, 0.0, 0.0)
    ress_radius: float = 1.0
    n_az: int = 360
    n_el: int = 180
    fle_degree: int = 3

    @property
    def n(self) -> int:
        return int(self.means.shape[0])

    @classmethod
    def from_host(cls, scene, device="cuda") -> "DeviceScene":
        f = lambda a: torch.as_tensor(np.ascontiguousarray(a, dtype=np.float32), device=device)
        return cls(
            f(scene.means).reshape(-1, 3), f(scene.quats).reshape(-1, 4), f(scene.log_scales).reshape(-1, 3),
            f(scene.trans_mag_raw).reshape(-1), f(scene.trans_phase).reshape(-1),
            torch.as_tensor(np.ascontiguousarray(scene.coeffs, dtype=np.complex64), device=device),
            tuple(float(x) for x in np.asarray(scene.rx, dtype=np.float64).reshape(3)),
            float(scene.ress_radius), int(scene.n_az), int(scene.n_el), int(getattr(scene, "fle_degree", 3)),
        )

    def validate(self) -> None:
        n = self.n
        k = (self.fle_degree + 1) ** 2
        checks = [
            (self.means, (n, 3), torch.float32), (self.quats, (n, 4), torch.float32),
            (self.log_scales, (n, 3), torch.float32), (self.trans_mag_raw, (n,), torch.float32),
            (self.trans_phase, (n,), torch.float32), (self.coeffs, (n, k), torch.complex64),
        ]
        for t, shape, dt in checks:
            if tuple(t.shape) != shape or t.dtype != dt or not t.is_cuda or not t.is_contiguous():
                raise ShapeError(f"scene tensor must be contiguous CUDA {dt} of shape {shape}, got {tuple(t.shape)} {t.dtype}")
        if not (1 <= self.n_az <= 360 and 1 <= self.n_el <= 180):
            raise ShapeError("grid must satisfy 1 <= n_az <= 360, 1 <= n_el <= 180")
        if not (0 <= self.fle_degree <= 4):
            raise ShapeError("fle_degree must lie in 0..4")


@dataclass
class Geometry:
    """Transmitter-independent state of one step (TileIndex + hit lists)."""

    n: int
    n_az: int
    n_el: int
    tiles_u: int
    tiles_v: int
    m: int
    geom: torch.Tensor
    sph: torch.Tensor
    rho32: torch.Tensor
    ckeys: torch.Tensor
    vals: torch.Tensor
    ranges: torch.Tensor
    lb: torch.Tensor
    hcap: int
    slab: torch.Tensor
    ray_counts: torch.Tensor
    stats: list = field(default_factory=list)
    proj: torch.Tensor | None = None
    sort_backend: str = "hand"

    @property
    def n_tiles(self) -> int:
        return self.tiles_u * self.tiles_v

    @property
    def n_rays(self) -> int:
        return self.n_az * self.n_el

    @property
    def total_hits(self) -> int:
        return int(self.stats[3])


_HCAP = {"value": 64}


def sort_end_bit(n_tiles: int) -> int:
    return 31 + max(0, math.ceil(math.log2(max(n_tiles, 1))))


def sort_pairs(ckeys, vals, end_bit: int, backend: str = "hand"):
    """K3: stable sort of compact keys with u32 payload; returns sorted (ckeys, vals)."""
    m = int(ckeys.numel())
    dev = ckeys.device
    if m <= 1:
        return ckeys, vals
    raise_end = int(end_bit)
    kalt = torch.empty_like(ckeys)
    valt = torch.empty_like(vals)
    lib = _native.load()
    res = _native.C.c_int(0)
    if backend == "hand":
        tb = int(lib.rfs_sort_temp_bytes(m, raise_end))
        temp = torch.empty(max(tb, 16), dtype=torch.uint8, device=dev)
        _native.call("rfs_sort_pairs_u64", _ptr(ckeys), _ptr(vals), _ptr(kalt), _ptr(valt), m, raise_end,
                     _ptr(temp), tb, _native.C.byref(res), _stream())
        _native.launch_counter["kernels"] += 2 + (raise_end + 7) // 8
    elif backend == "cub":
        tb = int(lib.rfs_sort_cub_temp_bytes(m, raise_end))
        temp = torch.empty(max(tb, 16), dtype=torch.uint8, device=dev)
        _native.call("rfs_sort_pairs_u64_cub", _ptr(ckeys), _ptr(vals), _ptr(kalt), _ptr(valt), m, raise_end,
                     _ptr(temp), tb, _native.C.byref(res), _stream())
    else:
        raise ValueError(f"unknown sort backend {backend!r}")
    return (kalt, valt) if res.value else (ckeys, vals)



def _mark(marks, name):
    if marks is not None:
        ev = torch.cuda.Event(enable_timing=True)
        ev.record()
        marks.append((name, ev))


def build_geometry(scene: DeviceScene, sort_backend: str = "hand", want_proj: bool = False,
                   hcap: int | None = None, marks: list | None = None) -> Geometry:
    """K1-K6: projection, binning, sort, ranges, emission bounds, hit lists.

    `marks` (optional list) receives (phase, cuda.Event) pairs recorded after
    each phase on the current stream, for per-kernel timing in bench.py.
    """
    scene.validate()
    lib = _native.load()
    dev = scene.means.device
    n, n_az, n_el = scene.n, scene.n_az, scene.n_el
    tiles_u = (n_az + TILE - 1) // TILE
    tiles_v = (n_el + TILE - 1) // TILE
    n_tiles = tiles_u * tiles_v
    R = n_az * n_el
    st = _stream()
    rx = (_native.C.c_double * 3)(*scene.rx)

    geom = torch.empty(max(n, 1) * 128, dtype=torch.uint8, device=dev)
    sph = torch.empty((max(n, 1), 4), dtype=torch.float32, device=dev)
    code = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    rects = torch.empty(max(n, 1) * 16, dtype=torch.uint8, device=dev)
    counts = torch.zeros(max(n, 1), dtype=torch.int32, device=dev)
    rho32 = torch.empty((max(n, 1), 4), dtype=torch.float32, device=dev)
    proj = torch.empty((max(n, 1), 6), dtype=torch.float64, device=dev) if want_proj else None
    status = torch.zeros(8, dtype=torch.int32, device=dev)  # [0] error bits, [1] M
    _native.call("rfs_project", n, _ptr(scene.means), _ptr(scene.quats), _ptr(scene.log_scales),
                 _ptr(scene.trans_mag_raw), _ptr(scene.trans_phase), rx, float(scene.ress_radius), n_az, n_el,
                 _ptr(geom), _ptr(sph), _ptr(code), _ptr(rects), _ptr(counts), _ptr(rho32), _ptr(proj),
                 _ptr(status), st)
    offsets = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    temp = torch.empty(int(lib.rfs_scan_temp_elems(max(n, 1))), dtype=torch.int32, device=dev)
    _native.call("rfs_exclusive_scan_u32", _ptr(counts), n, _ptr(offsets), status.data_ptr() + 4, _ptr(temp), st)
    _mark(marks, "project+scan")
    host = status.cpu()  # sync #1: error flags and M
    if int(host[0]) & (1 << 1):
        raise GeometryError("a Gaussian is centered on the receiver")
    m = int(host[1]) & 0xFFFFFFFF
    ckeys = torch.empty(max(m, 1), dtype=torch.int64, device=dev)
    vals = torch.empty(max(m, 1), dtype=torch.int32, device=dev)
    if m > 0:
        _native.call("rfs_bin_fill", n, _ptr(rects), _ptr(code), _ptr(offsets), n_az, _ptr(ckeys), _ptr(vals), st)
        _mark(marks, "fill")
        ckeys, vals = sort_pairs(ckeys[:m], vals[:m], sort_end_bit(n_tiles), sort_backend)
        _mark(marks, "sort")
    ranges = torch.empty((n_tiles, 2), dtype=torch.int32, device=dev)
    _native.call("rfs_tile_ranges", _ptr(ckeys), m, n_tiles, _ptr(ranges), st)
    lb = torch.empty(max(m, 1), dtype=torch.float64, device=dev)
    _native.call("rfs_lower_bounds", _ptr(ranges), n_tiles, _ptr(vals), _ptr(geom), _ptr(lb), st)
    _mark(marks, "ranges+lb")

    hc = int(hcap or _HCAP["value"])
    ray_counts = torch.empty(R, dtype=torch.int32, device=dev)
    slow = torch.empty(R, dtype=torch.int32, device=dev)
    stats = torch.zeros(8, dtype=torch.int32, device=dev)
    while True:
        slab = torch.empty(R * hc * 16, dtype=torch.uint8, device=dev)
        _native.call("rfs_hits", _ptr(ranges), n_tiles, _ptr(vals), _ptr(lb), _ptr(sph), _ptr(geom), rx,
                     float(scene.ress_radius), n_az, n_el, hc, _ptr(slab), _ptr(ray_counts), _ptr(slow),
                     _ptr(stats), st)
        _mark(marks, "hits")
        s = stats.cpu().tolist()  # sync #2
        if s[0] > 0:
            # rays whose pending buffer overflowed: exact slow path
            pcap = max(int(s[4]), 1)
            nr = int(s[0])
            pt = torch.empty(nr * pcap, dtype=torch.float64, device=dev)
            pg = torch.empty(nr * pcap, dtype=torch.int32, device=dev)
            pw = torch.empty(nr * pcap, dtype=torch.float32, device=dev)
            _native.call("rfs_hits_slow", _ptr(slow), nr, _ptr(ranges), _ptr(vals), _ptr(lb), _ptr(sph),
                         _ptr(geom), rx, float(scene.ress_radius), n_az, n_el, hc, _ptr(slab), _ptr(ray_counts),
                         _ptr(pt), _ptr(pg), _ptr(pw), pcap, _ptr(stats), st)
            s2 = stats.cpu().tolist()
            s[1], s[2], s[3] = s2[1], s2[2], s2[3]
        if s[1] > 0:
            hc = 1 << max(6, math.ceil(math.log2(max(s[2], 1))))
            _HCAP["value"] = max(_HCAP["value"], hc)
            continue
        break
    return Geometry(n, n_az, n_el, tiles_u, tiles_v, m, geom, sph, rho32, ckeys[:max(m, 0)], vals[:max(m, 0)],
                    ranges, lb, hc, slab, ray_counts, s, proj, sort_backend)


def _check_tx(tx: torch.Tensor) -> torch.Tensor:
    if tx.dim() != 2 or tx.shape[1] != 3:
        raise ShapeError("tx must have shape [B, 3]")
    return tx.to(dtype=torch.float32).contiguous()


def compute_psi(scene: DeviceScene, tx: torch.Tensor) -> torch.Tensor:
    """K5: psi [N, B] complex64."""
    tx = _check_tx(tx)
    b = int(tx.shape[0])
    psi = torch.empty((scene.n, b), dtype=torch.complex64, device=scene.means.device)
    if scene.n and b:
        _native.call("rfs_psi", scene.n, b, scene.fle_degree, _ptr(scene.means), _ptr(scene.coeffs), _ptr(tx),
                     _ptr(psi), _stream())
    return psi


def forward(geo: Geometry, psi: torch.Tensor) -> torch.Tensor:
    """K7: S [B, n_az, n_el] complex64 from shared hit lists and psi [N, B]."""
    b = int(psi.shape[1])
    S = torch.empty((b, geo.n_az, geo.n_el), dtype=torch.complex64, device=psi.device)
    if b:
        _native.call("rfs_forward", _ptr(geo.slab), _ptr(geo.ray_counts), geo.hcap, _ptr(psi), b, geo.n_rays,
                     _ptr(S), _stream())
    return S


def backward(scene: DeviceScene, geo: Geometry, tx: torch.Tensor, grad_S: torch.Tensor,
             include_direction_chain: bool = True, psi: torch.Tensor | None = None,
             marks: list | None = None) -> dict:
    """K8a/K8b/K9: gradients summed over the TX batch (GradientBuffer.add, grad.py:85-92).

    grad_S is the complex-packed upstream lambda = dL/dRe S + i dL/dIm S
    (grad.py:4-8), which is also PyTorch's gradient convention for complex
    tensors.  Returns fp32 tensors with the GradientBuffer meaning plus
    d_trans_mag_raw (the logit chain of train.py:161-162).
    """
    tx = _check_tx(tx)
    b = int(tx.shape[0])
    if tuple(grad_S.shape) != (b, geo.n_az, geo.n_el):
        raise ShapeError("upstream frame shape does not match the scene grid")
    dev = scene.means.device
    n, K = scene.n, (scene.fle_degree + 1) ** 2
    grad_S = grad_S.to(torch.complex64).contiguous()
    st = _stream()
    out = {
        "d_mean": torch.zeros((n, 3), dtype=torch.float32, device=dev),
        "d_quat": torch.zeros((n, 4), dtype=torch.float32, device=dev),
        "d_log_scale": torch.zeros((n, 3), dtype=torch.float32, device=dev),
        "d_trans_mag": torch.zeros(n, dtype=torch.float32, device=dev),
        "d_trans_mag_raw": torch.zeros(n, dtype=torch.float32, device=dev),
        "d_trans_phase": torch.zeros(n, dtype=torch.float32, device=dev),
        "d_coeffs": torch.zeros((n, K), dtype=torch.complex64, device=dev),
        "d_cov": torch.zeros((n, 3, 3), dtype=torch.float32, device=dev),
    }
    if n == 0 or b == 0:
        return out
    R = geo.n_rays
    gslab = torch.zeros(R * geo.hcap * 4, dtype=torch.float32, device=dev)
    gacc = torch.zeros(n * 16, dtype=torch.float32, device=dev)
    chunks = []
    for c0 in range(0, b, MAX_TX_PER_LAUNCH):
        c1 = min(b, c0 + MAX_TX_PER_LAUNCH)
        txc = tx[c0:c1].contiguous()
        if psi is not None and c0 == 0 and c1 == b:
            psic = psi
        else:
            psic = compute_psi(scene, txc)
        P = torch.zeros((n, c1 - c0), dtype=torch.complex64, device=dev)
        lam = grad_S[c0:c1].contiguous()
        _native.call("rfs_backward_rays", _ptr(geo.slab), _ptr(geo.ray_counts), geo.hcap, _ptr(psic), _ptr(lam),
                     _ptr(geo.rho32), c1 - c0, R, _ptr(P), _ptr(gslab), st)
        chunks.append((txc, P))
    _mark(marks, "backward_rays")
    rx = (_native.C.c_double * 3)(*scene.rx)
    _native.call("rfs_backward_hits", _ptr(geo.slab), _ptr(geo.ray_counts), geo.hcap, _ptr(gslab), _ptr(geo.geom),
                 rx, float(scene.ress_radius), geo.n_az, geo.n_el, _ptr(gacc), st)
    _mark(marks, "backward_hits")
    for i, (txc, P) in enumerate(chunks):
        _native.call("rfs_grad_epilogue", n, int(txc.shape[0]), scene.fle_degree, _ptr(scene.means),
                     _ptr(scene.quats), _ptr(scene.log_scales), _ptr(scene.trans_mag_raw), _ptr(scene.coeffs),
                     _ptr(txc), _ptr(P), _ptr(gacc), int(bool(include_direction_chain)), int(i > 0),
                     _ptr(out["d_mean"]), _ptr(out["d_quat"]), _ptr(out["d_log_scale"]), _ptr(out["d_trans_mag"]),
                     _ptr(out["d_trans_mag_raw"]), _ptr(out["d_trans_phase"]), _ptr(out["d_coeffs"]),
                     _ptr(out["d_cov"]), st)
    _mark(marks, "epilogue")
    return out


def tile_index_host(geo: Geometry):
    """Reference-layout TileIndex arrays (splat.py:82-101): keys u64, indices i64, ranges i64."""
    m = geo.m
    keys = torch.empty(max(m, 1), dtype=torch.int64, device=geo.ckeys.device)
    if m:
        _native.call("rfs_expand_keys", _ptr(geo.ckeys), m, _ptr(keys), _stream())
    k = keys[:m].cpu().numpy().view(np.uint64)
    idx = geo.vals[:m].cpu().numpy().astype(np.int64)
    rg = geo.ranges.cpu().numpy().astype(np.int64)
    return k, idx, rg


def hit_lists_host(geo: Geometry):
    """(counts [R], hits [R, hcap] structured g/w/T) copied to the host, for tests."""
    counts = geo.ray_counts.cpu().numpy()
    raw = geo.slab.view(torch.int32).reshape(geo.n_rays, geo.hcap, 4).cpu().numpy()
    g = raw[..., 0].astype(np.int64)
    f = raw.view(np.float32)
    return counts, g, f[..., 1], f[..., 2] + 1j * f[..., 3]
