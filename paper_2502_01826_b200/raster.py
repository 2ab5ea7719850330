"""Host orchestration of the sm_100a rasterizer (torch tensors + the C ABI).

One step = `build_geometry` (K1-K6, transmitter independent) followed by the
TX-batched `compute_psi` (K5), `forward` (K7) and `backward` (K8a, K8i, K9).
PyTorch supplies device memory (caching allocator) and the current CUDA
stream; every kernel is launched through include/rfsplat_b200.h.

Host synchronisations per step: one 8-byte read of M (the incidence count
sizes the sort buffers) and one read of the hit-list statistics (slow-path
rays, hit-capacity overflow).  Both mirror the reference allocating its
arrays from counts (_kernels.py:542-543, grad.py:224-231).
"""

from __future__ import annotations

import math
import os
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native
from .errors import GeometryError, ShapeError

__all__ = ["DeviceScene", "Geometry", "build_geometry", "compute_psi", "forward", "backward", "transpose_upstream",
           "GRAD_FIELDS",
           "ray_directions"]

TILE = 16
MAX_TX_PER_LAUNCH = 256
GRAD_FIELDS = ("d_mean", "d_quat", "d_log_scale", "d_trans_mag", "d_trans_mag_raw", "d_trans_phase", "d_coeffs",
               "d_cov")


def _ptr(t: torch.Tensor | None):
    return None if t is None else t.data_ptr()


def _stream():
    """Raw cudaStream_t of the current stream (the cheap accessor: no Stream object)."""
    return torch._C._cuda_getCurrentRawStream(torch.cuda.current_device())


def _mark(marks, name):
    if marks is not None:
        ev = torch.cuda.Event(enable_timing=True)
        ev.record()
        marks.append((name, ev))


def _meta_carrier(scene):
    c = getattr(scene, "carrier_freq", None)
    return None if c is None else float(c)


def _meta_bounds(scene):
    b = getattr(scene, "bounds", None)  # RFScene: Box(lo, hi)
    if b is not None and hasattr(b, "lo"):
        return (tuple(float(x) for x in b.lo), tuple(float(x) for x in b.hi))
    lo, hi = getattr(scene, "bounds_lo", None), getattr(scene, "bounds_hi", None)  # io.CheckpointScene
    if lo is not None and hi is not None:
        return (tuple(float(x) for x in np.asarray(lo).reshape(3)), tuple(float(x) for x in np.asarray(hi).reshape(3)))
    return None


@dataclass
class DeviceScene:
    """fp32 device copy of a scene's SoA parameters (the boundary's inputs)."""

    means: torch.Tensor          # f32 [N,3]
    quats: torch.Tensor          # f32 [N,4]
    log_scales: torch.Tensor     # f32 [N,3]
    trans_mag_raw: torch.Tensor  # f32 [N]
    trans_phase: torch.Tensor    # f32 [N]
    coeffs: torch.Tensor         # c64 [N,K]
    rx: tuple = (0.0, 0.0, 0.0)
    ress_radius: float = 1.0
    n_az: int = 360
    n_el: int = 180
    fle_degree: int = 3
    # scene metadata the rasterizer does not use, carried for checkpoints
    # (RFScene.carrier_freq / bounds, scene.py:205-246); None when unknown
    carrier_freq: float | None = None
    bounds: tuple | None = None

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
            _meta_carrier(scene), _meta_bounds(scene),
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
                raise ShapeError(f"scene tensor must be contiguous CUDA {dt} of shape {shape}, "
                                 f"got {tuple(t.shape)} {t.dtype}")
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
    rho32: torch.Tensor
    dirs: torch.Tensor
    ckeys: torch.Tensor
    vals: torch.Tensor
    ranges: torch.Tensor
    hcap: int
    slab: torch.Tensor
    ray_counts: torch.Tensor
    stats: list = field(default_factory=list)
    proj: torch.Tensor | None = None
    sort_backend: str = "hand"
    rx: tuple = (0.0, 0.0, 0.0)
    ress_radius: float = 1.0
    gidx: dict | None = None             # by-Gaussian hit index (built on first backward)
    psi: torch.Tensor | None = None      # psi of build_geometry(psi_tx=...)
    S: torch.Tensor | None = None        # forward of build_geometry(psi_tx=..., forward=True)
    used: torch.Tensor | None = None     # u32 [N]: Gaussian has a live hit (psi rows needed)
    after_result: object = None          # return value of build_geometry(after_forward=...)

    @property
    def n_tiles(self) -> int:
        return self.tiles_u * self.tiles_v

    @property
    def n_rays(self) -> int:
        return self.n_az * self.n_el

    @property
    def total_hits(self) -> int:
        return int(self.stats[3])


# adaptive capacities, remembered across steps
# longest tile list the bucket path sorts in steady state: beyond one block's
# shared memory (12288) the radix path is faster -- bucket.cu's 4-CTA cluster
# class (DSMEM, up to 49152) and its global-memory class still serve the first
# step of a scene (tile_max unknown); measured at 500k / 1M Gaussians:
# bucket 382 / 761 us vs radix 270 / 477 us of binning
BUCKET_MAX_LIST = 12288
RFS_PCAP_EVICT = 0x10000  # include/rfsplat_b200.h
_CAPS = {"hcap": 64, "pcap": 16, "m_cap": {}, "h_cap": {}, "used_cap": {},
         # K6: a full pending ring keeps its smallest hits (RFS_PCAP_EVICT); turned
         # on the first time a scene sends more than 0.1 % of the rays to the slow path
         "ring_evict": False,
         # tile-key sort of the hand-written backend: "bucket" (per-tile buckets,
         # bucket.cu) or "radix" (global onesweep)
         "tile_sort": os.environ.get("RFS_TILE_SORT", "bucket"), "tile_max": {},
         # the early by-Gaussian index on the side stream (overlapping psi / K7 / loss)
         "index_side": os.environ.get("RFS_INDEX_SIDE", "1") == "1",
         # psi of every Gaussian on the side stream at the start of the step
         # (overlapping the geometry) for scenes up to this size; larger scenes
         # compute only the rows of Gaussians with live hits, after K6
         "psi_early_max": int(os.environ.get("RFS_PSI_EARLY_MAX", "0"))}
_DIRS: dict = {}
_SIDE: dict = {}


def _side_stream(dev) -> torch.cuda.Stream:
    """Second stream for work independent of the main chain (the by-Gaussian
    index, K9b).  High priority: the index's chain of small kernels gets SMs
    ahead of the composite's and the loss's large grids, which it runs beside
    (index wait 24 -> 8 us at config 2; value 93.3k -> 94.7k spectra/s)."""
    k = str(dev)
    if k not in _SIDE:
        _SIDE[k] = torch.cuda.Stream(device=dev, priority=int(os.environ.get("RFS_SIDE_PRIORITY", "-1")))
    return _SIDE[k]


def ray_directions(n_az: int, n_el: int) -> np.ndarray:
    """render.ray_directions (render.py:103-117) with numpy, as the reference."""
    cell = 360.0 / n_az
    u = np.repeat(np.arange(n_az), n_el)
    v = np.tile(np.arange(n_el), n_az)
    alpha = np.deg2rad((u + 0.5) * cell)
    beta = np.deg2rad((v + 0.5) * cell - 90.0)
    return np.stack([np.cos(beta) * np.cos(alpha), np.cos(beta) * np.sin(alpha), np.sin(beta)], axis=1)


def _dirs_table(n_az: int, n_el: int, dev) -> torch.Tensor:
    key = (n_az, n_el, str(dev))
    t = _DIRS.get(key)
    if t is None:
        t = torch.as_tensor(np.ascontiguousarray(ray_directions(n_az, n_el)), dtype=torch.float64, device=dev)
        _DIRS[key] = t
    return t


def sort_end_bit(n_tiles: int) -> int:
    return 31 + max(0, math.ceil(math.log2(max(n_tiles, 1))))


def _fresh(name: str, n: int, dtype, dev) -> torch.Tensor:
    return torch.empty(n, dtype=dtype, device=dev)


_PBUF: dict = {}
_INDEX_GEN = [0]  # generation of the index held in the persistent buffers


def _persistent(name: str, n: int, dtype, dev) -> torch.Tensor:
    """Buffers of the early by-Gaussian index, reused every step: it is built on
    the side stream, and per-step allocations there made the caching allocator
    grow new segments mid-step (multi-ms host stalls at 1M Gaussians).  Safe to
    reuse: step i+1's index starts behind its own K6, after step i's backward."""
    key = (name, str(dev), dtype)
    t = _PBUF.get(key)
    if t is None or t.numel() < n:
        t = torch.empty(max(n + n // 4, 1), dtype=dtype, device=dev)
        _PBUF[key] = t
    return t[:n]


def sort_pairs(ckeys, vals, end_bit: int, backend: str = "hand", m_dev_ptr: int | None = None, alloc=_fresh,
               tag: str = ""):
    """K3: stable sort of u64 keys with u32 payload; returns sorted (keys, vals).

    With `m_dev_ptr` (device address of a u32 count; hand-written sort only)
    the buffers are a capacity and the first min(count, capacity) keys are
    sorted without a host read.
    """
    m = int(ckeys.numel())
    dev = ckeys.device
    if m <= 1:
        return ckeys, vals
    end_bit = int(end_bit)
    kalt = alloc(tag + "sort_kalt", m, ckeys.dtype, dev)
    valt = alloc(tag + "sort_valt", m, vals.dtype, dev)
    lib = _native.load()
    res = _native.C.c_int(0)
    if backend == "hand":
        tb = int(lib.rfs_sort_temp_bytes(m, end_bit))
        temp = alloc(tag + "sort_temp", max(tb, 16), torch.uint8, dev)
        _native.call("rfs_sort_pairs_u64", _ptr(ckeys), _ptr(vals), _ptr(kalt), _ptr(valt), m, end_bit,
                     _ptr(temp), tb, _native.C.byref(res), m_dev_ptr, _stream())
        _native.launch_counter["kernels"] += 3 + (end_bit + 7) // 8
    elif backend == "cub":
        if m_dev_ptr is not None:
            raise ValueError("the cub backend needs a host-side count")
        tb = int(lib.rfs_sort_cub_temp_bytes(m, end_bit))
        temp = torch.empty(max(tb, 16), dtype=torch.uint8, device=dev)
        _native.call("rfs_sort_pairs_u64_cub", _ptr(ckeys), _ptr(vals), _ptr(kalt), _ptr(valt), m, end_bit,
                     _ptr(temp), tb, _native.C.byref(res), _stream())
    else:
        raise ValueError(f"unknown sort backend {backend!r}")
    return (kalt, valt) if res.value else (ckeys, vals)


_PINNED: dict = {}


def _pinned(dev, name: str, n: int) -> torch.Tensor:
    """Reusable pinned int32 host buffer (status / statistics readbacks)."""
    k = (str(dev), name)
    t = _PINNED.get(k)
    if t is None or t.numel() < n:
        t = torch.empty(n, dtype=torch.int32).pin_memory()
        _PINNED[k] = t
    return t[:n]


def _keep(t: torch.Tensor, stream) -> None:
    """record_stream, except under CUDA-graph capture (the graph's private
    memory pool keeps every buffer of the captured step alive)."""
    if not torch.cuda.is_current_stream_capturing():
        t.record_stream(stream)


def _spin(ev: torch.cuda.Event) -> None:
    """Wait for an event by polling: a blocking wait sleeps and wakes tens of
    microseconds late, time in which the device would drain its queue."""
    while not ev.query():
        pass


def build_geometry(scene: DeviceScene, sort_backend: str = "hand", want_proj: bool = False,
                   hcap: int | None = None, marks: list | None = None, psi_tx: torch.Tensor | None = None,
                   index: bool = False, forward: bool = False, after_forward=None,
                   tiles: tuple | None = None, deferred: dict | None = None) -> Geometry:
    """K1-K6: projection, binning, sort, ranges, emission bounds, hit lists.

    Two small device->host reads size the later buffers (M after the scan,
    the hit statistics after K6).  Each is an asynchronous copy into pinned
    memory followed by independent GPU work before the host waits, so the
    device never idles on the round trip: `psi_tx` (optional [B, 3]) enqueues
    K5 psi for that batch behind the M read (-> geo.psi), and `forward=True`
    (needs psi_tx) enqueues the K7 composite behind the statistics read
    (-> geo.S, recomputed in the rare case the hit lists had to be redone);
    `after_forward(S)` (optional) enqueues further work on S in the same
    window (e.g. the loss and the upstream transpose), result in
    geo.after_result.
    `tiles` (optional (lo, hi)): trace only the rays of tiles [lo, hi) --
    a rank's tile shard in the strong-scaling mode (parallel.TileSharder);
    the other rays get no hits, so their S is exactly zero.
    `index=True` builds the by-Gaussian hit index for the backward.  `marks`
    (optional list) receives (phase, cuda.Event) pairs recorded after each
    phase on the current stream, for per-kernel timing in bench.py.
    `deferred` (optional dict with pinned int32 tensors "stats" [16] and
    "status" [8]): the steady-state, host-sync-free form used under CUDA-graph
    capture (api.StepGraph) -- every capacity (M, hit slab, index, used
    Gaussians) comes from earlier steps, nothing is read back during the call,
    and the statistics / status words are copied into the given pinned buffers
    for the caller to validate afterwards (deferred_ok); requires psi_tx,
    index=True and known capacities.
    """
    scene.validate()
    lib = _native.load()
    dev = scene.means.device
    t_lo, t_hi = (0, -1) if tiles is None else (int(tiles[0]), int(tiles[1]))
    psi_ready = None
    psi_early = None
    psi_early_go = psi_tx is not None and 0 < scene.n <= _CAPS["psi_early_max"]

    def start_psi_early():
        # psi does not depend on the geometry: on the side stream, started once
        # the dense K1-K4 kernels are queued, so it fills the SMs K6 leaves idle
        nonlocal psi_early, psi_ready
        side = _side_stream(dev)
        psi_early = torch.empty((scene.n, int(psi_tx.shape[0])), dtype=torch.complex64, device=dev)
        side.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(side):
            compute_psi(scene, psi_tx, None, out=psi_early)
            psi_ready = torch.cuda.Event()
            psi_ready.record(side)
        _keep(psi_early, side)
        _keep(psi_tx, side)
        return psi_early, psi_ready
    psi = None
    n, n_az, n_el = scene.n, scene.n_az, scene.n_el
    tiles_u = (n_az + TILE - 1) // TILE
    tiles_v = (n_el + TILE - 1) // TILE
    n_tiles = tiles_u * tiles_v
    R = n_az * n_el
    st = _stream()
    rx = (_native.C.c_double * 3)(*scene.rx)
    dirs = _dirs_table(n_az, n_el, dev)
    nn = max(n, 1)

    geom = torch.empty(nn * 128, dtype=torch.uint8, device=dev)
    sph = torch.empty((nn, 4), dtype=torch.float32, device=dev)
    whit = torch.empty((nn, 16), dtype=torch.float32, device=dev)
    code = torch.empty(nn, dtype=torch.int32, device=dev)
    rects = torch.empty(nn * 16, dtype=torch.uint8, device=dev)
    counts = torch.zeros(nn, dtype=torch.int32, device=dev)
    rho32 = torch.empty((nn, 4), dtype=torch.float32, device=dev)
    proj = torch.empty((nn, 6), dtype=torch.float64, device=dev) if want_proj else None
    status = torch.zeros(8, dtype=torch.int32, device=dev)  # [0] error bits, [1] M
    _native.call("rfs_project", n, _ptr(scene.means), _ptr(scene.quats), _ptr(scene.log_scales),
                 _ptr(scene.trans_mag_raw), _ptr(scene.trans_phase), rx, float(scene.ress_radius), n_az, n_el,
                 _ptr(geom), _ptr(sph), _ptr(whit), _ptr(code), _ptr(rects), _ptr(counts), _ptr(rho32), _ptr(proj),
                 _ptr(status), st)
    offsets = torch.empty(nn, dtype=torch.int32, device=dev)
    temp = torch.empty(int(lib.rfs_scan_temp_elems(nn)), dtype=torch.int32, device=dev)
    _native.call("rfs_exclusive_scan_u32", _ptr(counts), n, _ptr(offsets), status.data_ptr() + 4, _ptr(temp), st)
    _mark(marks, "project+scan")
    status_h = _pinned(dev, "status", 8)
    m_dev_ptr = status.data_ptr() + 4

    def bin_tiles(cap: int, device_count: bool, bucket: bool):
        """K2b fill, K3 sort, K4 ranges, K4b bounds into buffers of capacity `cap`."""
        ck = torch.empty(max(cap, 1), dtype=torch.int64, device=dev)
        vl = torch.empty(max(cap, 1), dtype=torch.int32, device=dev)
        if bucket:  # bucket.cu: the same outputs without a global sort
            rg = torch.empty((n_tiles, 2), dtype=torch.int32, device=dev)
            lbv = torch.empty(max(cap, 1), dtype=torch.float64, device=dev)
            bc = torch.empty(max(cap, 1), dtype=torch.int32, device=dev)
            bv = torch.empty(max(cap, 1), dtype=torch.int32, device=dev)
            tt = torch.empty(max(int(lib.rfs_bin_bucket_temp_bytes(n, n_az, n_el, cap)), 16), dtype=torch.uint8,
                             device=dev)
            _native.call("rfs_bin_bucket", n, _ptr(rects), _ptr(code), n_az, n_el, cap, _ptr(geom), _ptr(bc),
                         _ptr(bv), _ptr(tt), _ptr(ck), _ptr(vl), _ptr(rg), _ptr(lbv), _ptr(status), st)
            _mark(marks, "bin+sort")
            return ck, vl, rg, lbv
        mp = m_dev_ptr if device_count else None
        if cap > 0:
            _native.call("rfs_bin_fill", n, _ptr(rects), _ptr(code), _ptr(offsets), n_az, cap, _ptr(ck), _ptr(vl), st)
            _mark(marks, "fill")
            ck, vl = sort_pairs(ck[:cap], vl[:cap], sort_end_bit(n_tiles), sort_backend, mp)
            _mark(marks, "sort")
        rg = torch.empty((n_tiles, 2), dtype=torch.int32, device=dev)
        _native.call("rfs_tile_ranges", _ptr(ck), cap, mp, n_tiles, _ptr(rg), st)
        lbv = torch.empty(max(cap, 1), dtype=torch.float64, device=dev)
        _native.call("rfs_lower_bounds", _ptr(rg), n_tiles, _ptr(vl), _ptr(geom), _ptr(lbv), st)
        _mark(marks, "ranges+lb")
        return ck, vl, rg, lbv

    # Read #1 (M) is skipped when a capacity from earlier steps is known: the
    # binning then runs on the device-side count and M is checked at read #2.
    m_cap = _CAPS.get("m_cap", {}).get((n, n_az, n_el)) if sort_backend == "hand" else None
    # scenes whose tile lists ran longer than BUCKET_MAX_LIST last time use the radix sort
    bucket = (sort_backend == "hand" and _CAPS["tile_sort"] == "bucket"
              and _CAPS["tile_max"].get((n, n_az, n_el), 0) <= BUCKET_MAX_LIST)
    if m_cap is None:
        status_h.copy_(status, non_blocking=True)
        ev_m = torch.cuda.Event()
        ev_m.record()
        _spin(ev_m)  # read #1: error flags and M
        host = status_h.tolist()
        if int(host[0]) & (1 << 1):
            raise GeometryError("a Gaussian is centered on the receiver")
        m = int(host[1]) & 0xFFFFFFFF
        ckeys, vals, ranges, lb = bin_tiles(m, False, bucket)
    else:
        ckeys, vals, ranges, lb = bin_tiles(m_cap, True, bucket)

    hc = 1 << max(0, math.ceil(math.log2(max(int(hcap or _CAPS["hcap"]), 1))))  # power of two: slot >> log2(hcap) = ray
    pc = _CAPS["pcap"] | (RFS_PCAP_EVICT if _CAPS["ring_evict"] else 0)
    if deferred is not None:
        return _geometry_deferred(scene, deferred, locals())
    ray_counts = torch.empty(R, dtype=torch.int32, device=dev)
    slow = torch.empty(R, dtype=torch.int32, device=dev)
    stats = torch.zeros(16, dtype=torch.int32, device=dev)
    stats_h = _pinned(dev, "stats", 16)
    S = None
    early = None
    redo_forward = False
    used = torch.empty(nn, dtype=torch.int32, device=dev)
    if psi_early_go:
        start_psi_early()
    while True:
        slab = torch.empty(R * hc * 16, dtype=torch.uint8, device=dev)
        _native.call("rfs_hits", _ptr(ranges), n_tiles, _ptr(vals), _ptr(lb), _ptr(sph), _ptr(whit), _ptr(geom),
                     _ptr(dirs), rx, float(scene.ress_radius), n_az, n_el, hc, pc, _ptr(slab), _ptr(ray_counts),
                     _ptr(slow), _ptr(stats), _ptr(used), n, t_lo, t_hi, st)
        ev_hits = torch.cuda.Event()
        ev_hits.record()
        _mark(marks, "hits")
        stats_h.copy_(stats, non_blocking=True)
        if m_cap is not None:
            status_h.copy_(status, non_blocking=True)
        ev_s = torch.cuda.Event()
        ev_s.record()
        if psi_tx is not None and psi is None:
            if psi_early is not None:
                torch.cuda.current_stream(dev).wait_event(psi_ready)
                psi = psi_early
            else:  # psi of the Gaussians with live hits only (K6 marks them)
                psi = compute_psi(scene, psi_tx, used)
                _mark(marks, "psi")
        if forward and psi is not None and S is None:  # queued behind the statistics read
            S = _forward_raw(slab, ray_counts, hc, psi, n_az, n_el)
            _mark(marks, "forward")
            after = after_forward(S) if after_forward is not None else None
        h_cap = _CAPS["h_cap"].get((n_az, n_el, hc)) if index and sort_backend == "hand" else None
        u_cap = _CAPS["used_cap"].get((n, n_az, n_el))
        early = None
        if h_cap is not None and u_cap is not None:  # the by-Gaussian index, also behind the statistics read
            early = Geometry(n, n_az, n_el, tiles_u, tiles_v, -1, geom, rho32, dirs, ckeys, vals, ranges, hc, slab,
                             ray_counts, [0] * 16, proj, sort_backend, tuple(scene.rx), float(scene.ress_radius))
            early.used = used
            if _CAPS["index_side"]:
                # on the side stream, right behind K6: overlaps psi, the forward composite and the loss
                side = _side_stream(dev)
                side.wait_event(ev_hits)
                with torch.cuda.stream(side):
                    gauss_index(early, h_cap, _persistent, u_cap)
                    ready = torch.cuda.Event()
                    ready.record(side)
                # the side stream reads these main-stream buffers: keep them alive
                # (a geometry dropped without a backward) until it is done
                _keep(slab, side)
                _keep(ray_counts, side)
                _INDEX_GEN[0] += 1
                early.gidx["ready"] = ready
                early.gidx["gen"] = _INDEX_GEN[0]
            else:
                gauss_index(early, h_cap, used_cap=u_cap)
                _mark(marks, "gauss_index")
        _spin(ev_s)  # read #2: hit-list statistics (and M when read #1 was skipped)
        s = stats_h.tolist()

        def join_early():
            # a redo rewrites ray_counts / the slab in place: not while the early index reads them
            if early is not None and "ready" in early.gidx:
                torch.cuda.current_stream(dev).wait_event(early.gidx["ready"])

        if m_cap is not None:
            host = status_h.tolist()
            if int(host[0]) & (1 << 1):
                raise GeometryError("a Gaussian is centered on the receiver")
            m = int(host[1]) & 0xFFFFFFFF
            _CAPS["m_cap"][(n, n_az, n_el)] = max(m_cap, m + m // 8 + 1024) if m <= m_cap else m + m // 4 + 1024
            if m > m_cap:  # capacity overflow: re-bin with the exact count, redo the hit lists
                join_early()
                m_cap = None
                ckeys, vals, ranges, lb = bin_tiles(m, False, bucket)
                redo_forward = True
                continue
            m_cap = None
        if s[0] > 0:
            # rays whose pending ring overflowed: exact slow path, and a larger
            # ring for the next steps if it happens often
            if s[0] > R // 1000:  # keep the smallest hits of a full ring first, then grow it
                if not _CAPS["ring_evict"]:
                    _CAPS["ring_evict"] = True
                elif _CAPS["pcap"] < 64:
                    _CAPS["pcap"] = 2 * _CAPS["pcap"]
            join_early()
            pcap = max(int(s[4]), 1)
            nr = int(s[0])
            pt = torch.empty(nr * pcap, dtype=torch.float64, device=dev)
            pg = torch.empty(nr * pcap, dtype=torch.int32, device=dev)
            pw = torch.empty(nr * pcap, dtype=torch.float32, device=dev)
            _native.call("rfs_hits_slow", _ptr(slow), nr, _ptr(ranges), _ptr(vals), _ptr(lb), _ptr(sph), _ptr(whit),
                         _ptr(geom), _ptr(dirs), rx, float(scene.ress_radius), n_az, n_el, hc, _ptr(slab),
                         _ptr(ray_counts), _ptr(pt), _ptr(pg), _ptr(pw), pcap, _ptr(stats), _ptr(used), n, st)
            s2 = stats.cpu().tolist()
            s[1], s[2], s[3], s[8] = s2[1], s2[2], s2[3], s2[8]
            redo_forward = True
        if s[1] > 0:
            join_early()
            hc = 1 << max(6, math.ceil(math.log2(max(s[2], 1))))
            _CAPS["hcap"] = max(_CAPS["hcap"], hc)
            redo_forward = True
            continue
        break
    if sort_backend == "hand":
        _CAPS.setdefault("m_cap", {}).setdefault((n, n_az, n_el), m + m // 8 + 1024)
        _CAPS["tile_max"][(n, n_az, n_el)] = int(s[4])  # longest tile list (k_max_range)
    geo = Geometry(n, n_az, n_el, tiles_u, tiles_v, m, geom, rho32, dirs, ckeys[:max(m, 0)], vals[:max(m, 0)],
                   ranges, hc, slab, ray_counts, s, proj, sort_backend, tuple(scene.rx), float(scene.ress_radius))
    if psi_tx is not None and redo_forward and psi_early is None:  # the hit lists changed: new used set
        psi = compute_psi(scene, psi_tx, used)
    geo.psi = psi
    geo.used = used
    if forward and psi is not None:
        if S is None or redo_forward:
            S = _forward_raw(slab, ray_counts, hc, psi, n_az, n_el)
            after = after_forward(S) if after_forward is not None else None
        geo.S = S
        geo.after_result = after
    if sort_backend == "hand":  # bound on the Gaussians with a live hit: the early index's key width
        nu = int(s[8])
        _CAPS["used_cap"][(n, n_az, n_el)] = min(max(n, 1), nu + nu // 4 + 256)
    if index:
        hh = int(s[3])
        if (early is not None and not redo_forward and hh <= h_cap
                and int(s[8]) <= early.gidx["u_cap"]):
            geo.gidx = early.gidx
        else:
            gauss_index(geo)
            _mark(marks, "gauss_index")
        if sort_backend == "hand":
            key = (n_az, n_el, hc)
            _CAPS["h_cap"][key] = max(_CAPS["h_cap"].get(key, 0), hh + hh // 8 + 4096)
    return geo


def _geometry_deferred(scene, deferred: dict, L: dict) -> Geometry:
    """build_geometry's steady-state tail without host reads (see its
    `deferred` argument): hit lists, psi (side stream), the forward composite
    and the by-Gaussian index (side stream) on the known capacities; the
    statistics / status words go to deferred["stats"] / ["status"]."""
    n, n_az, n_el, dev = L["n"], L["n_az"], L["n_el"], L["dev"]
    R, hc, pc, st = L["R"], L["hc"], L["pc"], L["st"]
    h_cap = _CAPS["h_cap"].get((n_az, n_el, hc))
    u_cap = _CAPS["used_cap"].get((n, n_az, n_el))
    if (L["m_cap"] is None or h_cap is None or u_cap is None or L["psi_tx"] is None or not L["index"]
            or L["sort_backend"] != "hand"):
        raise ValueError("deferred geometry needs the hand sort backend, psi_tx, index=True and capacities "
                         "from earlier steps")
    ray_counts = torch.empty(R, dtype=torch.int32, device=dev)
    slow = torch.empty(R, dtype=torch.int32, device=dev)
    stats = torch.zeros(16, dtype=torch.int32, device=dev)
    used = torch.empty(L["nn"], dtype=torch.int32, device=dev)
    psi, psi_ready = L["start_psi_early"]() if L["psi_early_go"] else (None, None)
    slab = torch.empty(R * hc * 16, dtype=torch.uint8, device=dev)
    _native.call("rfs_hits", _ptr(L["ranges"]), L["n_tiles"], _ptr(L["vals"]), _ptr(L["lb"]), _ptr(L["sph"]),
                 _ptr(L["whit"]), _ptr(L["geom"]), _ptr(L["dirs"]), L["rx"], float(scene.ress_radius), n_az, n_el, hc,
                 pc, _ptr(slab), _ptr(ray_counts), _ptr(slow), _ptr(stats), _ptr(used), n, L["t_lo"], L["t_hi"], st)
    ev_hits = torch.cuda.Event()
    ev_hits.record()
    marks = L["marks"]
    _mark(marks, "hits")
    if psi is None:
        psi = compute_psi(scene, L["psi_tx"], used)
    else:
        torch.cuda.current_stream(dev).wait_event(psi_ready)
    S = _forward_raw(slab, ray_counts, hc, psi, n_az, n_el) if L["forward"] else None
    _mark(marks, "forward")
    after = L["after_forward"](S) if (S is not None and L["after_forward"] is not None) else None
    geo = Geometry(n, n_az, n_el, L["tiles_u"], L["tiles_v"], -1, L["geom"], L["rho32"], L["dirs"], L["ckeys"],
                   L["vals"], L["ranges"], hc, slab, ray_counts, [], L["proj"], L["sort_backend"], tuple(scene.rx),
                   float(scene.ress_radius))
    geo.used = used
    side = _side_stream(dev)
    side.wait_event(ev_hits)
    with torch.cuda.stream(side):
        gauss_index(geo, h_cap, _persistent, u_cap)
        ready = torch.cuda.Event()
        ready.record(side)
        # the statistics for the validation after the step: off the main stream
        # (psi and the composite do not wait for the copies), behind the index;
        # the step joins the side stream before its last kernel
        deferred["stats"].copy_(stats, non_blocking=True)
        deferred["status"].copy_(L["status"], non_blocking=True)
    _keep(slab, side)
    _keep(stats, side)
    _keep(ray_counts, side)
    _INDEX_GEN[0] += 1
    geo.gidx["ready"] = ready
    geo.gidx["gen"] = _INDEX_GEN[0]
    geo.psi, geo.S, geo.after_result = psi, S, after
    deferred["caps"] = {"m_cap": L["m_cap"], "h_cap": h_cap, "u_cap": u_cap, "R": R}
    return geo


def deferred_ok(deferred: dict) -> bool:
    """Validate a deferred geometry after its work completed (the caller
    synchronized): no geometry error, M within the binning capacity, no ray on
    the slow path, no hit-slab overflow, H and the used Gaussians within the
    index capacities.  False means: redo the step eagerly (capacities grow)."""
    st = deferred["stats"].tolist()
    status = deferred["status"].tolist()
    c = deferred["caps"]
    m = int(status[1]) & 0xFFFFFFFF
    return (int(status[0]) & (1 << 1)) == 0 and m <= c["m_cap"] and st[0] == 0 and st[1] == 0 \
        and st[3] <= c["h_cap"] and st[8] <= c["u_cap"]


def _check_tx(tx: torch.Tensor) -> torch.Tensor:
    if tx.dim() != 2 or tx.shape[1] != 3:
        raise ShapeError("tx must have shape [B, 3]")
    return tx.to(dtype=torch.float32).contiguous()


def compute_psi(scene: DeviceScene, tx: torch.Tensor, used: torch.Tensor | None = None,
                out: torch.Tensor | None = None) -> torch.Tensor:
    """K5: psi [N, B] complex64; with `used` (u32 [N], Geometry.used) only the
    rows of Gaussians with live hits are computed -- the only rows K7 / K8c read."""
    tx = _check_tx(tx)
    b = int(tx.shape[0])
    psi = out if out is not None else torch.empty((scene.n, b), dtype=torch.complex64, device=scene.means.device)
    if scene.n and b:
        _native.call("rfs_psi", scene.n, b, scene.fle_degree, _ptr(scene.means), _ptr(scene.coeffs), _ptr(tx),
                     _ptr(used), _ptr(psi), _stream())
    return psi


def _forward_raw(slab, ray_counts, hcap: int, psi: torch.Tensor, n_az: int, n_el: int) -> torch.Tensor:
    b = int(psi.shape[1])
    S = torch.empty((b, n_az, n_el), dtype=torch.complex64, device=psi.device)
    if b:
        _native.call("rfs_forward", _ptr(slab), _ptr(ray_counts), hcap, _ptr(psi), b, n_az, n_el, _ptr(S), _stream())
    return S


def forward(geo: Geometry, psi: torch.Tensor) -> torch.Tensor:
    """K7: S [B, n_az, n_el] complex64 from shared hit lists and psi [N, B]."""
    if geo.S is not None and psi is geo.psi:
        return geo.S
    return _forward_raw(geo.slab, geo.ray_counts, geo.hcap, psi, geo.n_az, geo.n_el)


def gauss_index(geo: Geometry, h_cap: int | None = None, alloc=_fresh, used_cap: int | None = None) -> None:
    """K8i: by-Gaussian index of the live hits (TX independent, cached on geo).

    Hits sorted by the compact id of their Gaussian among the Gaussians with
    a live hit (K6's used marks) with a stable sort, so within a Gaussian
    they keep the (ray, k) order of the reference's bincount slots
    (grad.py:222-254) -- every per-Gaussian sum has the reference's order.
    Per sorted hit: ray, slab slot, w, w T; per Gaussian its run [first,
    end); the list of the Gaussians with hits (K9b walks only those).
    The hit count H stays on the device: `h_cap` (default: the exact H of the
    hit-list statistics) sizes the buffers and grids, every kernel reads
    min(H, h_cap) -- so build_geometry can enqueue this before it reads the
    statistics.  The compact id has ceil(log2(used_cap)) bits (at config 2 ~30k of
    100k Gaussians are hit: 15 bits, two radix passes); `used_cap` (default:
    the exact count of the hit-list statistics) bounds the number of used
    Gaussians; build_geometry rebuilds the index if the real count exceeded it.
    """
    if geo.gidx is not None:
        return
    lib = _native.load()
    dev = geo.slab.device
    st = _stream()
    R = geo.n_rays
    cap = int(h_cap if h_cap is not None else geo.total_hits)
    ucap = max(int(used_cap if used_cap is not None else geo.stats[8]), 1)
    ray_off = alloc("gi_ray_off", R, torch.int32, dev)
    tot = alloc("gi_tot", 1, torch.int32, dev)
    temp = alloc("gi_rtemp", int(lib.rfs_scan_temp_elems(max(R, geo.n))), torch.int32, dev)
    _native.call("rfs_exclusive_scan_u32", _ptr(geo.ray_counts), R, _ptr(ray_off), _ptr(tot), _ptr(temp), st)
    # compact ids of the Gaussians with a live hit, and their list (K9b walks it)
    cid = alloc("gi_cid", max(geo.n, 1), torch.int32, dev)
    n_used = alloc("gi_nused", 1, torch.int32, dev)
    _native.call("rfs_exclusive_scan_u32", _ptr(geo.used), geo.n, _ptr(cid), _ptr(n_used), _ptr(temp), st)
    order = alloc("gi_order", ucap, torch.int32, dev)
    _native.call("rfs_used_list", geo.n, _ptr(geo.used), _ptr(cid), ucap, _ptr(order), st)
    nu = n_used.data_ptr()
    rank = cid
    bits = max(1, math.ceil(math.log2(max(ucap, 2))))
    # hit keys land at ray_off[r] + k < H; positions >= cap are never read (H <= cap is checked)
    keys = alloc("gi_keys", max(R * geo.hcap, 1), torch.int64, dev)
    slots = alloc("gi_slots", max(R * geo.hcap, 1), torch.int32, dev)
    _native.call("rfs_hit_keys", _ptr(geo.slab), _ptr(geo.ray_counts), _ptr(ray_off), geo.hcap, R, _ptr(rank),
                 _ptr(keys), _ptr(slots), st)
    hd = tot.data_ptr()
    if cap > 1:
        if geo.sort_backend == "hand":
            keys, slots = sort_pairs(keys[:cap], slots[:cap], bits, "hand", hd, alloc)
        else:  # cub needs the exact count: only reached after the statistics read
            keys, slots = sort_pairs(keys[:cap], slots[:cap], bits, geo.sort_backend)
    s_ray = alloc("gi_s_ray", max(cap, 1), torch.int32, dev)
    s_w = alloc("gi_s_w", max(cap, 1), torch.float32, dev)
    s_wt = alloc("gi_s_wt", max(cap, 1), torch.complex64, dev)
    # (the rank keys are replaced by the Gaussian ids here, before the ranges)
    _native.call("rfs_gather_sorted", _ptr(slots), cap, hd, geo.hcap, _ptr(geo.slab), _ptr(s_ray), _ptr(s_w),
                 _ptr(s_wt), None, _ptr(keys), st)
    g_rng = alloc("gi_grng", 2 * max(geo.n, 1), torch.int32, dev)
    _native.call("rfs_gauss_ranges", _ptr(keys), cap, hd, geo.n, _ptr(g_rng), st)
    geo.gidx = {"h": cap, "h_dev": hd, "tot": tot, "sorted_g": keys, "g_rng": g_rng, "s_ray": s_ray, "s_w": s_w,
                "s_wt": s_wt, "s_slot": slots, "key_bits": bits, "order": order, "u_cap": ucap,
                "n_used": n_used, "n_used_dev": nu}  # (the tensors behind the device pointers stay referenced)


def transpose_upstream(grad_S: torch.Tensor) -> torch.Tensor:
    """K8t: lam [B, n_az, n_el] -> lamT [R, B] (a ray's TX row contiguous).

    backward() does this itself; callers that know lambda early may enqueue
    it sooner and pass the result as backward(lamT=...).  B <= 256.
    """
    b = int(grad_S.shape[0])
    R = int(grad_S.shape[1]) * int(grad_S.shape[2])
    grad_S = grad_S.to(torch.complex64).contiguous()
    lamT = torch.empty((R, b), dtype=torch.complex64, device=grad_S.device)
    _native.call("rfs_lam_transpose", _ptr(grad_S), b, R, _ptr(lamT), _stream())
    return lamT


def backward(scene: DeviceScene, geo: Geometry, tx: torch.Tensor, grad_S: torch.Tensor | None,
             include_direction_chain: bool = True, psi: torch.Tensor | None = None,
             marks: list | None = None, deterministic: bool = False, lamT: torch.Tensor | None = None,
             out: dict | None = None, on_coeffs=None) -> dict:
    """K8a/K8i/K9: gradients summed over the TX batch (GradientBuffer.add, grad.py:85-92).

    grad_S is the complex-packed upstream lambda = dL/dRe S + i dL/dIm S
    (grad.py:4-8), which is also PyTorch's gradient convention for complex
    tensors.  `lamT` (optional, complex64 [n_az*n_el, B], B <= 256) is the
    same upstream ray-major -- the layout K8 reads, written directly by the
    loss kernel (loss.spectrum_loss_frames(lam_layout="rays")); with it,
    grad_S may be None.  Returns fp32 tensors with the GradientBuffer meaning
    plus d_trans_mag_raw (the logit chain of train.py:161-162).

    `out` (optional): preallocated output tensors (e.g. the views of
    parallel.GradBuffer, so the all-reduce needs no packing); `on_coeffs`
    (optional callable) receives a CUDA event recorded when d_coeffs is final
    (after K9b, on the side stream) -- the hook for an all-reduce bucket that
    overlaps the rest of the epilogue.

    Every sum has a fixed order and there are no atomics: the buffer is
    bitwise reproducible.  `deterministic` is accepted for
    API compatibility (it was the opt-in for this before).
    """
    tx = _check_tx(tx)
    b = int(tx.shape[0])
    R = geo.n_rays
    if lamT is not None and (tuple(lamT.shape) != (R, b) or lamT.dtype != torch.complex64 or b > MAX_TX_PER_LAUNCH):
        raise ShapeError("lamT must be complex64 [n_az*n_el, B] with B <= 256")
    if grad_S is None:
        if lamT is None:
            raise ShapeError("backward needs grad_S or lamT")
    else:
        if tuple(grad_S.shape) != (b, geo.n_az, geo.n_el):
            raise ShapeError("upstream frame shape does not match the scene grid")
        grad_S = grad_S.to(torch.complex64).contiguous()
    dev = scene.means.device
    n, K = scene.n, (scene.fle_degree + 1) ** 2
    st = _stream()
    shapes = {"d_mean": ((n, 3), torch.float32), "d_quat": ((n, 4), torch.float32),
              "d_log_scale": ((n, 3), torch.float32), "d_trans_mag": ((n,), torch.float32),
              "d_trans_mag_raw": ((n,), torch.float32), "d_trans_phase": ((n,), torch.float32),
              "d_coeffs": ((n, K), torch.complex64), "d_cov": ((n, 3, 3), torch.float32)}
    if out is None:
        out = {k: torch.empty(sh, dtype=dt, device=dev) for k, (sh, dt) in shapes.items()}
    else:
        for k, (sh, dt) in shapes.items():
            t = out[k]
            if tuple(t.shape) != sh or t.dtype != dt or not t.is_contiguous() or t.device != dev:
                raise ShapeError(f"out[{k!r}] must be a contiguous {dt} tensor of shape {sh} on {dev}")
    if n == 0 or b == 0:
        for v in out.values():
            v.zero_()
        return out
    lib = _native.load()
    built = geo.gidx is None
    if geo.gidx is not None and geo.gidx.get("gen", _INDEX_GEN[0]) != _INDEX_GEN[0]:
        geo.gidx = None  # its persistent buffers were reused by a later geometry: rebuild
    gauss_index(geo)
    gi = geo.gidx
    if "ready" in gi:  # built on the side stream
        torch.cuda.current_stream(geo.slab.device).wait_event(gi["ready"])
    _mark(marks, "gauss_index" if built else "index_wait")
    h = gi["h"]
    main = torch.cuda.current_stream(dev)
    side = _side_stream(dev)
    C = torch.empty(R * geo.hcap, dtype=torch.complex64, device=dev)        # slab order, live slots written
    gs = torch.empty((R * geo.hcap, 4), dtype=torch.float32, device=dev)   # per-hit scalars of K8r, slab order
    dm_dir = torch.empty((n, 3), dtype=torch.float32, device=dev)          # bearing chain of d_mean (K9b)
    for c0 in range(0, b, MAX_TX_PER_LAUNCH):
        c1 = min(b, c0 + MAX_TX_PER_LAUNCH)
        nbc = c1 - c0
        txc = tx[c0:c1].contiguous()
        psic = psi if (psi is not None and c0 == 0 and c1 == b) else compute_psi(scene, txc, geo.used)
        if lamT is not None and c0 == 0 and c1 == b:
            lamTc = lamT
        else:
            lamTc = torch.empty((R, nbc), dtype=torch.complex64, device=dev)
            _native.call("rfs_lam_transpose", _ptr(grad_S[c0:c1]), nbc, R, _ptr(lamTc), st)
        P = torch.empty((n, nbc), dtype=torch.complex64, device=dev)
        part = torch.empty(int(lib.rfs_bwd_part_elems(h, nbc)), dtype=torch.complex64, device=dev)
        pcnt = torch.empty(n + 1, dtype=torch.int32, device=dev)  # straddle counts / list (zeroed in C)
        _native.call("rfs_bwd_gauss", n, h, gi["h_dev"], nbc, _ptr(gi["sorted_g"]), _ptr(gi["s_slot"]), geo.hcap,
                     _ptr(gi["s_wt"]), _ptr(gi["g_rng"]), _ptr(psic), _ptr(lamTc), int(c0 > 0), _ptr(C), _ptr(P),
                     _ptr(part), _ptr(pcnt), st)
        _mark(marks, "bwd_gauss")
        # K9b on a second stream: it needs only P, so it overlaps the ray
        # recursion and the geometry sums below (K9c waits for it)
        side.wait_stream(main)
        with torch.cuda.stream(side):
            _native.call("rfs_grad_tx", gi["u_cap"], gi["n_used_dev"], _ptr(gi["order"]), n, _ptr(gi["g_rng"]), nbc,
                         scene.fle_degree,
                         _ptr(scene.means), _ptr(scene.coeffs), _ptr(txc), _ptr(P), int(bool(include_direction_chain)),
                         int(c0 > 0),
                         _ptr(dm_dir), _ptr(out["d_coeffs"]), side.cuda_stream)
        for t in (txc, P, dm_dir, out["d_coeffs"]):
            _keep(t, side)
    if on_coeffs is not None:  # d_coeffs is final once the side stream gets here
        ev = torch.cuda.Event()
        ev.record(side)
        on_coeffs(ev)
    _mark(marks, "backward_tx")
    _native.call("rfs_bwd_rays", _ptr(geo.slab), _ptr(geo.ray_counts), geo.hcap, R, _ptr(geo.rho32), _ptr(geo.geom),
                 _ptr(C), _ptr(gs), st)
    _mark(marks, "backward_rays")
    rx = (_native.C.c_double * 3)(*geo.rx)
    npart = int(lib.rfs_geom_part_elems(h))
    acc64 = torch.empty((n, 14), dtype=torch.float64, device=dev)
    long_list = torch.empty(npart, dtype=torch.int32, device=dev)  # [0] count, then the long Gaussians
    part_v = torch.empty((npart, 14), dtype=torch.float64, device=dev)
    geom_args = [n, h, gi["h_dev"], _ptr(gi["sorted_g"]), _ptr(gi["s_ray"]), _ptr(gi["s_w"]), _ptr(gi["s_slot"]),
                 _ptr(gs), _ptr(gi["g_rng"]), _ptr(geo.geom), _ptr(geo.dirs), rx, float(geo.ress_radius),
                 _ptr(scene.quats), _ptr(scene.log_scales), _ptr(scene.trans_mag_raw), gi["u_cap"], gi["n_used_dev"],
                 _ptr(gi["order"]), _ptr(acc64), _ptr(long_list),
                 _ptr(part_v), _ptr(out["d_mean"]), _ptr(out["d_quat"]), _ptr(out["d_log_scale"]),
                 _ptr(out["d_trans_mag"]), _ptr(out["d_trans_mag_raw"]), _ptr(out["d_trans_phase"]),
                 _ptr(out["d_cov"]), _ptr(dm_dir)]
    _native.call("rfs_grad_geom", *geom_args, 1, st)  # K9a: per-hit sums, alongside K9b
    main.wait_stream(side)  # K9c adds K9b's bearing chain (dm_dir)
    _native.call("rfs_grad_geom", *geom_args, 2, st)  # K9c
    _native.launch_counter["kernels"] += 4  # fill, k_geom_seg, k_geom_span, k_geom_final
    _mark(marks, "grad_geom")
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
    """(counts [R], g [R,hcap], w [R,hcap], T [R,hcap]) copied to the host, for tests."""
    counts = geo.ray_counts.cpu().numpy()
    raw = geo.slab.view(torch.int32).reshape(geo.n_rays, geo.hcap, 4).cpu().numpy()
    g = raw[..., 0].astype(np.int64)
    f = raw.view(np.float32)
    return counts, g, f[..., 1], f[..., 2] + 1j * f[..., 3]
