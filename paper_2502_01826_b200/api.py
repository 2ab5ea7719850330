"""Reference-shaped entry points (drop-in for rfsplat's render / grad / splat).

These mirror the reference's plain-function API over host numpy scenes so a
caller of `rfsplat` can switch by changing the import:

    render.render_complex_frame(scene, tx, workers, tiled, ctx)  render.py:282-289
    render.render_spectrum / render_scalar                        render.py:292-307
    grad.backward_frame(scene, tx, upstream, workers, include_direction_chain, ctx)
                                                                  grad.py:192-259
    splat.build_tiles_for_render(scene, proj) -> TileIndex        splat.py:374-380
    splat.project_scene(scene) -> SceneProjection                 splat.py:212-268

`workers` and `tiled` are accepted and ignored (the GPU path is always
tiled and stream-ordered).  Batched variants take a TX batch [B, 3] and share
the transmitter-independent geometry across it.
Results come back as float64 / complex128 numpy arrays in the reference
layouts; the arithmetic is fp32 (geometry fp64).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import raster
from .errors import ContractViolationError, ShapeError
from .scene import HostScene

__all__ = [
    "GradientBuffer", "TileIndex", "SceneProjection", "SpectrumFrame", "RenderContextGPU",
    "prepare_context", "render_complex_frame", "render_complex_frames", "render_spectrum", "render_scalar",
    "backward_frame", "backward_frames", "upstream_to_ray", "build_tiles_for_render", "project_scene",
    "fwd_bwd_host", "fwd_bwd_device", "train_step_host",
]


@dataclass
class TileIndex:
    """splat.TileIndex (splat.py:82-101)."""

    n_az: int
    n_el: int
    tiles_u: int
    tiles_v: int
    keys: np.ndarray
    indices: np.ndarray
    ranges: np.ndarray

    @property
    def n_tiles(self) -> int:
        return self.tiles_u * self.tiles_v


@dataclass
class SceneProjection:
    """splat.SceneProjection (splat.py:104-118)."""

    active: np.ndarray
    center_u: np.ndarray
    center_v: np.ndarray
    radius_px: np.ndarray
    tile_radius: np.ndarray
    depth: np.ndarray


@dataclass
class GradientBuffer:
    """grad.GradientBuffer (grad.py:55-101) with float64 host arrays."""

    d_mean: np.ndarray
    d_quat: np.ndarray
    d_log_scale: np.ndarray
    d_trans_mag: np.ndarray
    d_trans_phase: np.ndarray
    d_coeffs: np.ndarray
    d_cov: np.ndarray

    def add(self, other: "GradientBuffer") -> None:
        for k in ("d_mean", "d_quat", "d_log_scale", "d_trans_mag", "d_trans_phase", "d_coeffs", "d_cov"):
            setattr(self, k, getattr(self, k) + getattr(other, k))

    def all_finite(self) -> bool:
        return all(np.all(np.isfinite(getattr(self, k))) for k in
                   ("d_mean", "d_quat", "d_log_scale", "d_trans_mag", "d_trans_phase", "d_coeffs", "d_cov"))

    @classmethod
    def from_device(cls, g: dict) -> "GradientBuffer":
        h = lambda t: t.detach().cpu().numpy()
        return cls(
            h(g["d_mean"]).astype(np.float64), h(g["d_quat"]).astype(np.float64),
            h(g["d_log_scale"]).astype(np.float64), h(g["d_trans_mag"]).astype(np.float64),
            h(g["d_trans_phase"]).astype(np.float64), h(g["d_coeffs"]).astype(np.complex128),
            h(g["d_cov"]).astype(np.float64),
        )


@dataclass
class RenderContextGPU:
    """Device analogue of render.RenderContext (render.py:191-214): the
    transmitter-independent geometry of a scene, reusable across TX."""

    scene: raster.DeviceScene
    geometry: raster.Geometry


def _device_scene(scene) -> raster.DeviceScene:
    if isinstance(scene, raster.DeviceScene):
        return scene
    return raster.DeviceScene.from_host(HostScene.from_any(scene))


def prepare_context(scene, tx=None, want_proj: bool = False, sort_backend: str = "hand") -> RenderContextGPU:
    ds = _device_scene(scene)
    return RenderContextGPU(ds, raster.build_geometry(ds, sort_backend=sort_backend, want_proj=want_proj))


def _tx_tensor(tx, dev) -> torch.Tensor:
    t = torch.as_tensor(np.asarray(tx, dtype=np.float32), device=dev)
    return t.reshape(-1, 3)


def render_complex_frames(scene, txs, ctx: RenderContextGPU | None = None) -> np.ndarray:
    """Complex frames for a TX batch, shape (B, n_az, n_el)."""
    ctx = ctx or prepare_context(scene)
    tx = _tx_tensor(txs, ctx.scene.means.device)
    psi = raster.compute_psi(ctx.scene, tx, ctx.geometry.used)
    return raster.forward(ctx.geometry, psi).cpu().numpy().astype(np.complex128)


def render_complex_frame(scene, tx, workers: int = 1, tiled: bool = True,
                         ctx: RenderContextGPU | None = None) -> np.ndarray:
    """render.render_complex_frame (render.py:282-289)."""
    return render_complex_frames(scene, np.asarray(tx, dtype=np.float64).reshape(1, 3), ctx)[0]


@dataclass
class SpectrumFrame:
    """render.SpectrumFrame (render.py:84-100): power per direction, (n_az, n_el) float64."""

    data: np.ndarray

    def __post_init__(self):
        self.data = np.asarray(self.data, dtype=np.float64)
        if self.data.ndim != 2:
            raise ShapeError("spectrum frame must be 2-dimensional")

    @property
    def n_az(self) -> int:
        return self.data.shape[0]

    @property
    def n_el(self) -> int:
        return self.data.shape[1]


def render_spectrum(scene, tx, workers: int = 1, ctx: RenderContextGPU | None = None) -> SpectrumFrame:
    """render.render_spectrum (render.py:292-298): SpectrumFrame(|S|^2)."""
    return SpectrumFrame(np.abs(render_complex_frame(scene, tx, workers, ctx=ctx)) ** 2)


def render_scalar(scene, tx, workers: int = 1, ctx: RenderContextGPU | None = None) -> complex:
    """render.render_scalar (render.py:301-307): coherent sum over rays."""
    return complex(render_complex_frame(scene, tx, workers, ctx=ctx).sum())


def upstream_to_ray(dL_dpower, s_frame) -> np.ndarray:
    """grad.upstream_to_ray (grad.py:104-120)."""
    if s_frame is None:
        raise ContractViolationError("forward complex frame was not cached")
    dL_dpower = np.asarray(dL_dpower, dtype=np.float64)
    s_frame = np.asarray(s_frame, dtype=np.complex128)
    if dL_dpower.shape != s_frame.shape:
        raise ContractViolationError("gradient frame and forward frame shapes differ")
    return 2.0 * dL_dpower * s_frame


def backward_frames(scene, txs, upstreams, include_direction_chain: bool = True,
                    ctx: RenderContextGPU | None = None, deterministic: bool = False) -> GradientBuffer:
    """Gradients summed over a TX batch (GradientBuffer.add semantics, grad.py:85-92).

    deterministic=True makes the buffer bitwise reproducible (the reference's
    fixed-order reduction) at some cost in speed."""
    ctx = ctx or prepare_context(scene)
    dev = ctx.scene.means.device
    tx = _tx_tensor(txs, dev)
    up = np.asarray(upstreams, dtype=np.complex64)
    if up.ndim == 2:
        up = up[None]
    if up.shape != (tx.shape[0], ctx.geometry.n_az, ctx.geometry.n_el):
        raise ShapeError("upstream frame shape does not match the scene grid")
    g = raster.backward(ctx.scene, ctx.geometry, tx, torch.as_tensor(up, device=dev), include_direction_chain,
                        deterministic=deterministic)
    return GradientBuffer.from_device(g)


def backward_frame(scene, tx, upstream, workers: int = 1, include_direction_chain: bool = True,
                   ctx: RenderContextGPU | None = None, deterministic: bool = False) -> GradientBuffer:
    """grad.backward_frame (grad.py:192-259)."""
    upstream = np.asarray(upstream)
    if upstream.ndim != 2:
        raise ShapeError("upstream frame shape does not match the scene grid")
    return backward_frames(scene, np.asarray(tx, dtype=np.float64).reshape(1, 3), upstream[None],
                           include_direction_chain, ctx, deterministic)


SCENE_FIELDS = ("means", "quats", "log_scales", "trans_mag_raw", "trans_phase", "coeffs")
OUT_GRADS = ("d_mean", "d_quat", "d_log_scale", "d_trans_mag", "d_trans_mag_raw", "d_trans_phase", "d_coeffs",
             "d_cov")


def pinned_host_scene(scene) -> dict:
    """fp32 / complex64 pinned host copies of a scene's parameters."""
    s = HostScene.from_any(scene)
    f = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a, dtype=dt)).pin_memory()
    return {"means": f(s.means, np.float32), "quats": f(s.quats, np.float32), "log_scales": f(s.log_scales, np.float32),
            "trans_mag_raw": f(s.trans_mag_raw, np.float32), "trans_phase": f(s.trans_phase, np.float32),
            "coeffs": f(s.coeffs, np.complex64)}


def alloc_host_outputs(n: int, k: int, b: int, n_az: int, n_el: int) -> dict:
    z = lambda shape, dt: torch.empty(shape, dtype=dt).pin_memory()
    return {"S": z((b, n_az, n_el), torch.complex64), "d_mean": z((n, 3), torch.float32),
            "d_quat": z((n, 4), torch.float32), "d_log_scale": z((n, 3), torch.float32),
            "d_trans_mag": z((n,), torch.float32), "d_trans_mag_raw": z((n,), torch.float32),
            "d_trans_phase": z((n,), torch.float32), "d_coeffs": z((n, k), torch.complex64),
            "d_cov": z((n, 3, 3), torch.float32)}


def fwd_bwd_host(host_scene: dict, tx_host: torch.Tensor, lam_host: torch.Tensor, out: dict, rx, ress_radius: float,
                 n_az: int, n_el: int, fle_degree: int = 3, include_direction_chain: bool = True,
                 sort_backend: str = "hand", reduce_fn=None) -> tuple:
    """One fwd+bwd step from HOST (pinned) buffers to HOST buffers.

    The drop-in for a caller holding the scene and upstream frames on the
    host, i.e. render_complex_frame + backward_frame of the reference
    (render.py:282-289, grad.py:192-259) for a TX batch.  Copies are
    stream-ordered (non_blocking) with respect to the current stream; the caller
    synchronizes.  Inside, the upstream frames travel on a copy stream while the
    geometry and the forward run, and the frames come back on another while
    the backward runs.  `reduce_fn`
    (optional) all-reduces the device gradient dict before the D2H copy.
    Returns (h2d_bytes, d2h_bytes).
    """
    dev = torch.device("cuda", torch.cuda.current_device())
    main = torch.cuda.current_stream(dev)
    d = {k: host_scene[k].to(dev, non_blocking=True) for k in SCENE_FIELDS}
    ds = raster.DeviceScene(d["means"], d["quats"], d["log_scales"], d["trans_mag_raw"], d["trans_phase"],
                            d["coeffs"], tuple(float(x) for x in rx), float(ress_radius), n_az, n_el, fle_degree)
    tx = tx_host.to(dev, non_blocking=True)
    # the upstream frames (the largest input) on the H2D copy stream, overlapping
    # the TX-independent geometry and the forward; the backward waits for them
    lam = torch.empty(tuple(lam_host.shape), dtype=lam_host.dtype, device=dev)
    up = _copy_stream(dev)
    up.wait_stream(main)
    with torch.cuda.stream(up):
        lam.copy_(lam_host, non_blocking=True)
        lam_ready = torch.cuda.Event()
        lam_ready.record(up)
    lam.record_stream(up)
    geo = raster.build_geometry(ds, sort_backend=sort_backend, psi_tx=tx, index=True, forward=True)
    psi = geo.psi
    S = raster.forward(geo, psi)
    # the frames back on the D2H copy stream while the backward runs (the other
    # copy engine: the two directions overlap too)
    down = _copy_stream_d2h(dev)
    down.wait_stream(main)
    with torch.cuda.stream(down):
        out["S"].copy_(S, non_blocking=True)
    S.record_stream(down)
    main.wait_event(lam_ready)
    g = raster.backward(ds, geo, tx, lam, include_direction_chain, psi=psi)
    if reduce_fn is not None:
        reduce_fn(g)
    down.wait_stream(main)
    with torch.cuda.stream(down):
        for k in OUT_GRADS:
            out[k].copy_(g[k], non_blocking=True)
    for k in OUT_GRADS:
        g[k].record_stream(down)
    main.wait_stream(down)  # stream-ordered for the caller, as before
    h2d = sum(host_scene[k].numel() * host_scene[k].element_size() for k in SCENE_FIELDS)
    h2d += tx_host.numel() * tx_host.element_size() + lam_host.numel() * lam_host.element_size()
    d2h = sum(out[k].numel() * out[k].element_size() for k in ("S",) + OUT_GRADS)
    return h2d, d2h


def fwd_bwd_device(ds: raster.DeviceScene, tx: torch.Tensor, lam: torch.Tensor | None = None,
                   include_direction_chain: bool = True, sort_backend: str = "hand", marks: list | None = None,
                   lamT: torch.Tensor | None = None, grads=None, group=None, deferred: dict | None = None) -> tuple:
    """The benched step (bench.py): render + backward of a device-resident
    scene for a TX batch [B, 3] under a fixed upstream.

    render_complex_frame + backward_frame (render.py:282-289, grad.py:192-259)
    for the whole batch, with psi queued behind the geometry's first host
    read, the composite behind the second, and the by-Gaussian index on the
    side stream.  The upstream is lam [B, n_az, n_el] (transposed for the
    backward behind the composite) or lamT [n_az*n_el, B], the loss kernel's
    own output layout (loss.spectrum_loss_frames(lam_layout="rays")).
    `grads` (optional parallel.GradBuffer): the backward writes into it and,
    under torch.distributed with more than one rank, all-reduces it in two
    buckets overlapped with the epilogue (this rank's `tx` is its TX shard).
    `deferred` (optional dict, see raster.build_geometry): the host-sync-free
    steady-state form (StepGraph captures it).
    Returns (S [B, n_az, n_el], grads).
    """
    b = int(tx.shape[0])
    early_t = None
    if lamT is None and b <= raster.MAX_TX_PER_LAUNCH:
        early_t = lambda S: raster.transpose_upstream(lam)
    geo = raster.build_geometry(ds, sort_backend=sort_backend, marks=marks, psi_tx=tx, forward=True, index=True,
                                after_forward=early_t, deferred=deferred)
    lt = lamT if lamT is not None else geo.after_result
    if grads is not None:
        from . import parallel

        g = parallel.backward_reduced(ds, geo, tx, lam, grads, include_direction_chain, psi=geo.psi, lamT=lt,
                                      group=group, marks=marks)
    else:
        g = raster.backward(ds, geo, tx, lam, include_direction_chain, psi=geo.psi, marks=marks, lamT=lt)
    return geo.S, g


class StepGraph:
    """The steady-state fwd+bwd step (fwd_bwd_device) captured as one CUDA graph.

    The step has two host reads when run eagerly (the incidence count M and
    the hit-list statistics); in the steady state every capacity they size is
    known from earlier steps, so the captured form reads nothing back during
    the step: the statistics land in pinned buffers and `ok()` validates them
    afterwards (a False answer means the capacities were exceeded -- rerun the
    step eagerly with `eager()`, which also grows them, and capture again).
    Replays launch the ~30 kernels of the step (two streams) with no host
    work in between.  Inputs: the static TX buffer `tx` [B, 3] (copy new
    positions into it, `set_tx`) and the ray-major upstream `lamT`; outputs:
    `S` and the gradient buffer `grads` (parallel.GradBuffer views).
    Single process (the multi-rank all-reduce stays eager)."""

    def __init__(self, ds: raster.DeviceScene, tx: torch.Tensor, lamT: torch.Tensor, grads,
                 include_direction_chain: bool = True, sort_backend: str = "hand", warmup: int = 3):
        self.ds, self.lamT, self.grads = ds, lamT, grads
        self.tx = tx.to(torch.float32).contiguous().clone()
        self.dc, self.sort_backend = include_direction_chain, sort_backend
        for _ in range(max(1, warmup)):  # capacities, persistent buffers, kernel attributes
            self.eager()
        torch.cuda.synchronize()
        self.deferred = {"stats": torch.zeros(16, dtype=torch.int32).pin_memory(),
                         "status": torch.zeros(8, dtype=torch.int32).pin_memory()}
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            self.S, self.g = fwd_bwd_device(ds, self.tx, None, self.dc, sort_backend, lamT=lamT, grads=grads,
                                            deferred=self.deferred)

    def set_tx(self, tx: torch.Tensor) -> None:
        self.tx.copy_(tx, non_blocking=True)

    def replay(self) -> None:
        self.graph.replay()

    def ok(self) -> bool:
        """After a synchronize: did the last replay stay within the capacities?"""
        return raster.deferred_ok(self.deferred)

    def eager(self):
        return fwd_bwd_device(self.ds, self.tx, None, self.dc, self.sort_backend, lamT=self.lamT, grads=self.grads)


class TrainStepGraph:
    """train_step_host captured as one CUDA graph (see StepGraph): each replay
    copies the TX positions and measured power frames from the given pinned
    host buffers (fill them before replaying), renders, runs the spectrum loss
    and the backward into `grads`, and copies the per-frame loss report into
    `report_host` -- no host work inside the step.  `ok()` validates the
    deferred statistics after a synchronize.  Single process."""

    def __init__(self, ds: raster.DeviceScene, tx_host: torch.Tensor, gt_host: torch.Tensor,
                 report_host: torch.Tensor, grads, w_ssim: float = 0.2, w_fourier: float = 0.2,
                 include_direction_chain: bool = True, sort_backend: str = "hand", warmup: int = 3):
        args = (ds, tx_host, gt_host, report_host, w_ssim, w_fourier, include_direction_chain, sort_backend)
        for _ in range(max(1, warmup)):
            train_step_host(*args, grads=grads)
        torch.cuda.synchronize()
        self.deferred = {"stats": torch.zeros(16, dtype=torch.int32).pin_memory(),
                         "status": torch.zeros(8, dtype=torch.int32).pin_memory()}
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            self.g, self.h2d, self.d2h = train_step_host(*args, grads=grads, deferred=self.deferred)

    def replay(self) -> None:
        self.graph.replay()

    def ok(self) -> bool:
        return raster.deferred_ok(self.deferred)


_COPY: dict = {}


def _copy_stream(dev) -> torch.cuda.Stream:
    k = str(dev)
    if k not in _COPY:
        _COPY[k] = torch.cuda.Stream(device=dev)
    return _COPY[k]


def _copy_stream_d2h(dev) -> torch.cuda.Stream:
    k = "d2h:" + str(dev)
    if k not in _COPY:
        _COPY[k] = torch.cuda.Stream(device=dev)
    return _COPY[k]


def train_step_host(ds: raster.DeviceScene, tx_host: torch.Tensor, gt_host: torch.Tensor, report_host: torch.Tensor,
                    w_ssim: float = 0.2, w_fourier: float = 0.2, include_direction_chain: bool = True,
                    sort_backend: str = "hand", reduce_fn=None, grads=None, group=None,
                    deferred: dict | None = None) -> tuple:
    """One training step of a device-resident scene on a TX batch from HOST buffers.

    The batched counterpart of the reference iteration (train.py:266-281,
    324-336): render, spectrum loss against the measured power frames,
    upstream_to_ray, backward_frame.  Per step the TX positions [B, 3] and the
    ground-truth power frames [B, n_az, n_el] (pinned host float32) go to the
    device, and the per-frame loss report [B, 4] = (total, L1, SSIM, Fourier)
    comes back into `report_host` (pinned float64); the gradient dict stays on
    the device for the optimizer.  Copies are stream-ordered (non_blocking);
    the caller synchronizes.  `grads` (optional parallel.GradBuffer) receives
    the gradients, all-reduced over the ranks as in fwd_bwd_device;
    `reduce_fn(g)` (optional) is applied to a plain gradient dict instead.
    `deferred` (optional dict, see raster.build_geometry): the host-sync-free
    steady-state form (TrainStepGraph captures it).
    Returns (grads, h2d_bytes, d2h_bytes).
    """
    from . import loss as _loss

    dev = ds.means.device
    main = torch.cuda.current_stream(dev)
    cs = _copy_stream(dev)
    cs.wait_stream(main)
    with torch.cuda.stream(cs):  # H2D on the copy engine, overlapping the TX-independent geometry
        tx = tx_host.to(dev, non_blocking=True)
        tx_ready = torch.cuda.Event()
        tx_ready.record(cs)
        gt = gt_host.to(dev, non_blocking=True)
        gt_rng = _loss.frame_range(gt)  # SSIM's dynamic range, off the critical path
        gt_ready = torch.cuda.Event()
        gt_ready.record(cs)
    raster._keep(tx, main)
    raster._keep(gt, main)
    raster._keep(gt_rng, main)
    main.wait_event(tx_ready)

    def loss_and_upstream(S):  # queued behind the geometry's hit-statistics read
        main.wait_event(gt_ready)
        if S.shape[0] <= raster.MAX_TX_PER_LAUNCH:  # the loss writes the backward's ray-major layout
            rep, lamT, _ = _loss.spectrum_loss_frames(S, gt, w_ssim, w_fourier, lam_layout="rays", gt_range=gt_rng)
            return rep, None, lamT
        rep, lam, _ = _loss.spectrum_loss_frames(S, gt, w_ssim, w_fourier, gt_range=gt_rng)
        return rep, lam, None

    geo = raster.build_geometry(ds, sort_backend=sort_backend, psi_tx=tx, index=True, forward=True,
                                after_forward=loss_and_upstream, deferred=deferred)
    rep, lam, lamT = geo.after_result
    if grads is not None:
        from . import parallel

        g = parallel.backward_reduced(ds, geo, tx, lam, grads, include_direction_chain, psi=geo.psi, lamT=lamT,
                                      group=group)
    else:
        g = raster.backward(ds, geo, tx, lam, include_direction_chain, psi=geo.psi, lamT=lamT)
        if reduce_fn is not None:
            reduce_fn(g)
    report_host.copy_(rep, non_blocking=True)
    h2d = tx_host.numel() * tx_host.element_size() + gt_host.numel() * gt_host.element_size()
    d2h = report_host.numel() * report_host.element_size()
    return g, h2d, d2h


def build_tiles_for_render(scene, proj=None, sort_backend: str = "hand") -> TileIndex:
    """splat.build_tiles_for_render (splat.py:374-380), bit-exact TileIndex."""
    ctx = prepare_context(scene, sort_backend=sort_backend)
    g = ctx.geometry
    keys, idx, rg = raster.tile_index_host(g)
    return TileIndex(g.n_az, g.n_el, g.tiles_u, g.tiles_v, keys, idx, rg)


def project_scene(scene) -> SceneProjection:
    """splat.project_scene (splat.py:212-268)."""
    ctx = prepare_context(scene, want_proj=True)
    p = ctx.geometry.proj.cpu().numpy()[: ctx.scene.n]
    return SceneProjection(p[:, 5] > 0.5, p[:, 0], p[:, 1], p[:, 2], p[:, 3], p[:, 4])
