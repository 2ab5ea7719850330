"""Optimizer and adaptive density control on the device (reference train.py:48-245).

    TrainConfig, lr_mean                      train.py:48-93 (same fields, defaults, validation)
    TrainState                                train.py:96-121 (grad_ema / last_dmean on the device)
    sgd_step(scene, grads, iteration, config, state)        train.py:145-162
    densify(scene, state, iteration, config, seed) -> DensifyReport   train.py:165-222
    prune(scene, state, iteration, config) -> PruneReport            train.py:225-245

`scene` is a raster.DeviceScene, updated in place (its tensors are replaced
when the Gaussian count changes, as the reference's RFScene.keep/append do);
`grads` is the gradient dict of raster.backward.  Densify / prune need one
host read (the new count) per call -- every 100 iterations by default.
Split children are sampled with a counter-based Philox stream keyed by
(seed, iteration, parent, child), so every data-parallel rank draws the same
children with no communication; they are not numpy's multivariate_normal
draws, so split parity with the reference is decision-level (which parents
split, the children's attributes and count), SURVEY.md §7 H8.
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native, raster
from .errors import ConfigError, NonFiniteGradientError

__all__ = ["TrainConfig", "TrainState", "DensifyReport", "PruneReport", "lr_mean", "sgd_step", "densify", "prune"]

_CLASSES = ("mean", "quat", "log_scale", "trans_mag", "trans_phase", "coeffs")
_FIELDS = ("means", "quats", "log_scales", "trans_mag_raw", "trans_phase", "coeffs")
_NO_BAD = 0x7F7F7F7F7F7F7F7F
_NO_OVF = 1 << 62
_LOOP_HOOKS: dict = {}  # test seam: "before_capture" runs before each capture of the training iteration


@dataclass
class TrainConfig:
    """Hyperparameters; defaults follow the reference operating point (train.py:48-76)."""

    iterations: int = 30000
    lr_transmittance: float = 0.01
    lr_radiance: float = 0.0025
    lr_scale: float = 0.01
    lr_rotation: float = 0.005
    lr_mean_start: float = 0.00016
    lr_mean_end: float = 1.6e-6
    densify_grad_threshold: float = 0.0002
    densify_radius_threshold: float = 10.0
    prune_threshold: float = 0.004
    densify_every: int = 100
    prune_every: int = 100
    split_factor: float = 1.6
    w_ssim: float = 0.2
    w_fourier: float = 0.2
    ema_decay: float = 0.9
    checkpoint_every: int = 0
    workers: int = 1
    direction_chain: bool = True
    csi_subcarrier: int = 0

    def validate(self) -> None:
        for name in ("lr_transmittance", "lr_radiance", "lr_scale", "lr_rotation", "lr_mean_start", "lr_mean_end"):
            if getattr(self, name) <= 0.0:
                raise ConfigError(f"{name} must be positive")
        if not 0.0 < self.w_ssim + self.w_fourier < 1.0:
            raise ConfigError("loss weights must satisfy 0 < w_ssim + w_fourier < 1")
        if self.iterations < 0:
            raise ConfigError("iterations must be non-negative")


def lr_mean(config: TrainConfig, iteration: int) -> float:
    """Exponential schedule from lr_mean_start to lr_mean_end (train.py:86-93)."""
    if config.iterations <= 0:
        return config.lr_mean_start
    frac = min(max(iteration / config.iterations, 0.0), 1.0)
    return config.lr_mean_start * (config.lr_mean_end / config.lr_mean_start) ** frac


@dataclass
class TrainState:
    """Per-Gaussian gradient statistics on the device (train.py:96-121)."""

    grad_ema: torch.Tensor    # f32 [N]
    last_dmean: torch.Tensor  # f32 [N, 3]

    @classmethod
    def zeros(cls, n: int, device="cuda") -> "TrainState":
        return cls(torch.zeros(n, dtype=torch.float32, device=device),
                   torch.zeros((n, 3), dtype=torch.float32, device=device))


@dataclass
class DensifyReport:
    cloned: list = field(default_factory=list)
    split: list = field(default_factory=list)


@dataclass
class PruneReport:
    removed: list = field(default_factory=list)


def _ptr(t):
    return None if t is None else t.data_ptr()


def sgd_step(scene: raster.DeviceScene, grads: dict, iteration: int, config: TrainConfig,
             state: TrainState | None = None, check: bool = True, prior: torch.Tensor | None = None,
             lr_dev: torch.Tensor | None = None) -> None:
    """One descent step on the device (train.py:145-162), plus TrainState.observe
    when `state` is given.  A non-finite gradient row leaves the scene untouched;
    with check=True the error is raised here (one 8-byte read), else it can be
    read later from `sgd_step.last_bad`.  `prior` (optional device i64, the
    first bad value of earlier unchecked steps) skips the update once set.
    `lr_dev` (optional device f32 [1]) replaces lr_mean(config, iteration):
    the captured training iteration reads its schedule value there."""
    n, K = scene.n, scene.coeffs.shape[1]
    dev = scene.means.device
    bad = torch.empty(1, dtype=torch.int64, device=dev)
    lrs = (_native.C.c_float * 5)(lr_mean(config, iteration), config.lr_rotation, config.lr_scale,
                                  config.lr_transmittance, config.lr_radiance)
    st = raster._stream()
    _native.call("rfs_sgd_step", n, K, lrs, float(config.ema_decay), _ptr(grads["d_mean"]), _ptr(grads["d_quat"]),
                 _ptr(grads["d_log_scale"]), _ptr(grads["d_trans_mag"]), _ptr(grads["d_trans_phase"]),
                 _ptr(grads["d_coeffs"]), _ptr(scene.means), _ptr(scene.quats), _ptr(scene.log_scales),
                 _ptr(scene.trans_mag_raw), _ptr(scene.trans_phase), _ptr(scene.coeffs),
                 _ptr(state.grad_ema if state else None), _ptr(state.last_dmean if state else None), _ptr(bad),
                 _ptr(prior), _ptr(lr_dev), st)
    sgd_step.last_bad = bad
    if check:
        raise_if_bad(bad, n)


def raise_if_bad(bad: torch.Tensor, n: int) -> None:
    v = int(bad.item())
    if v != _NO_BAD:
        raise NonFiniteGradientError(v % max(n, 1), _CLASSES[v // max(n, 1)])


def _compact(scene: raster.DeviceScene, state: TrainState, mode: int, iteration: int, config: TrainConfig,
             seed: int):
    n, K = scene.n, scene.coeffs.shape[1]
    dev = scene.means.device
    st = raster._stream()
    lib = _native.load()
    keep, clone, split = (torch.empty(max(n, 1), dtype=torch.int32, device=dev) for _ in range(3))
    _native.call("rfs_density_flags", n, mode, _ptr(state.grad_ema), _ptr(scene.log_scales),
                 _ptr(scene.trans_mag_raw), float(config.densify_grad_threshold),
                 float(config.densify_radius_threshold), float(config.prune_threshold), _ptr(keep), _ptr(clone),
                 _ptr(split), st)
    offs = [torch.empty(max(n, 1), dtype=torch.int32, device=dev) for _ in range(3)]
    totals = torch.zeros(4, dtype=torch.int32, device=dev)
    temp = torch.empty(int(lib.rfs_scan_temp_elems(max(n, 1))), dtype=torch.int32, device=dev)
    for i, f in enumerate((keep, clone, split)):
        _native.call("rfs_exclusive_scan_u32", _ptr(f), n, _ptr(offs[i]), totals.data_ptr() + 4 * i, _ptr(temp), st)
    n_keep, n_clone, n_split = (int(x) for x in totals[:3].tolist())  # the one host read
    if (mode == 0 and n_clone == 0 and n_split == 0) or (mode == 1 and n_keep == n):
        # nothing to do: the reference returns before touching the scene or the
        # statistics (train.py:184-186 -- no state.reset() when nothing is hot)
        return keep, clone, split, (n_keep, n_clone, n_split)
    n_new = n_keep + n_clone + 2 * n_split
    new = {k: torch.empty((n_new,) + tuple(getattr(scene, k).shape[1:]), dtype=getattr(scene, k).dtype, device=dev)
           for k in _FIELDS}
    ema = torch.empty(n_new, dtype=torch.float32, device=dev)
    last = torch.empty((n_new, 3), dtype=torch.float32, device=dev)
    _native.call("rfs_density_apply", n, K, mode, _ptr(keep), _ptr(clone), _ptr(split), _ptr(offs[0]), _ptr(offs[1]),
                 _ptr(offs[2]), _ptr(totals), float(lr_mean(config, iteration)), float(math.log(config.split_factor)),
                 int(seed) & 0xFFFFFFFFFFFFFFFF, int(iteration), _ptr(scene.means), _ptr(scene.quats),
                 _ptr(scene.log_scales), _ptr(scene.trans_mag_raw), _ptr(scene.trans_phase), _ptr(scene.coeffs),
                 _ptr(state.grad_ema), _ptr(state.last_dmean), _ptr(new["means"]), _ptr(new["quats"]),
                 _ptr(new["log_scales"]), _ptr(new["trans_mag_raw"]), _ptr(new["trans_phase"]), _ptr(new["coeffs"]),
                 _ptr(ema), _ptr(last), st)
    for k, v in new.items():
        setattr(scene, k, v)
    state.grad_ema, state.last_dmean = ema, last
    return keep, clone, split, (n_keep, n_clone, n_split)


def densify(scene: raster.DeviceScene, state: TrainState, iteration: int, config: TrainConfig,
            seed: int = 0) -> DensifyReport:
    """Clone small / split large Gaussians whose mean-gradient EMA runs hot (train.py:165-222)."""
    if scene.n == 0:
        return DensifyReport()
    keep, clone, split, (nk, nc, ns) = _compact(scene, state, 0, iteration, config, seed)
    if nc == 0 and ns == 0:
        return DensifyReport()
    c = clone[: len(keep)].cpu().numpy()
    s = split[: len(keep)].cpu().numpy()
    return DensifyReport(np.nonzero(c)[0].tolist(), np.nonzero(s)[0].tolist())


def prune(scene: raster.DeviceScene, state: TrainState, iteration: int, config: TrainConfig) -> PruneReport:
    """Remove Gaussians whose transmittance magnitude is below the floor (train.py:225-245)."""
    if scene.n == 0:
        return PruneReport()
    n = scene.n
    keep, _, _, (nk, _, _) = _compact(scene, state, 1, iteration, config, 0)
    if nk == n:
        return PruneReport()
    k = keep[:n].cpu().numpy()
    return PruneReport(np.nonzero(k == 0)[0].tolist())


@dataclass
class TraceRow:
    """train.TraceRow (train.py:248-255); losses averaged over the iteration's TX batch."""

    iteration: int
    total: float
    l1: float
    ssim: float
    fourier: float
    n_primitives: int


def train_loop(scene: raster.DeviceScene, txs: torch.Tensor, frames: torch.Tensor, config: TrainConfig,
               batch: int = 1, seed: int = 0, timings: list | None = None, mode: str = "spectrum",
               check_every: int = 50, group=None, graph: bool = False):
    """Batched counterpart of train.train_loop (train.py:284-361) on the device.

    Each iteration draws `batch` samples (TX position + measured target) with a
    seeded generator, renders, evaluates the loss and its upstream, runs the
    backward, the SGD step and TrainState.observe; density control runs on the
    reference schedule during the first half of training.  The scene stays in
    HBM throughout; the loss trace is read back once at the end.  `timings`
    (optional list) receives (iteration, milliseconds, n_gaussians, event,
    idle milliseconds since the previous iteration ended) per iteration from
    CUDA events.  `mode` is the dataset mode (train.py:266-291):
    "spectrum" (frames = power frames [S, n_az, n_el]), "rssi" (frames = dBm
    [S]) or "csi" (frames = complex targets [S] or [S, subcarriers]; the
    config's csi_subcarrier is used, train.py:282).

    Non-finite gradients: the reference raises at the first bad step and
    leaves the scene as it was (train.py:145-150, 324-336).  Here the steps
    are not synchronised one by one: a bad step sets a device flag that makes
    every later update a no-op, and the flag is read every `check_every`
    iterations and before each densify / prune, raising
    NonFiniteGradientError for the first bad step -- the scene the caller
    sees is the one after the last good step.

    Data parallel (`group`, or the default process group when
    torch.distributed is initialised with more than one rank): every rank
    draws the same samples, renders its contiguous shard of the batch and
    all-reduces the gradients (parallel.GradBuffer, two buckets overlapped
    with the epilogue), so every rank applies the same update and takes the
    same densify / prune decisions (Philox children keyed by seed and
    iteration); the loss trace is summed over the ranks once at the end.
    Captured iterations (`graph=True`, single process; for host-bound loops --
    small grids or batches -- since each capture costs milliseconds and a
    device-bound loop such as config 5 gains nothing from it): after
    one eager iteration at the current Gaussian count -- which sizes every
    capacity -- the iteration is captured as one CUDA graph and replayed: the
    samples and the learning rate are drawn up front and indexed on the
    device by an iteration counter, the geometry runs in its host-read-free
    form (raster.build_geometry(deferred=...)), and a capacity overflow found
    on the device halts the following updates the way a bad step does; at the
    next sync point the loop rewinds to the overflowing iteration and redoes
    it eagerly (which grows the capacities) before capturing again.  Density
    control runs eagerly and is followed by a new capture when it changed the
    scene.  Results are bitwise those of the eager loop.
    Returns (trace, densify_reports, prune_reports).
    """
    import torch.distributed as dist

    from . import loss as _loss
    from . import parallel

    config.validate()
    dev = scene.means.device
    if mode not in ("spectrum", "rssi", "csi"):
        raise ConfigError(f"unknown sample mode {mode!r}")
    if mode == "spectrum" and tuple(frames.shape[1:]) != (scene.n_az, scene.n_el):
        raise ConfigError(f"dataset grid {tuple(frames.shape[1:])} does not match scene grid "
                          f"{(scene.n_az, scene.n_el)}")
    if mode == "csi" and frames.dim() == 2:  # [S, subcarriers]: the configured one (train.py:282)
        if not 0 <= config.csi_subcarrier < frames.shape[1]:
            raise ConfigError(f"csi_subcarrier {config.csi_subcarrier} out of range")
        frames = frames[:, config.csi_subcarrier].contiguous()
    world = dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1
    rank = dist.get_rank(group) if world > 1 else 0
    rng = np.random.default_rng(seed)
    state = TrainState.zeros(scene.n, dev)
    first_bad = torch.full((1,), _NO_BAD, dtype=torch.int64, device=dev)
    first_n = torch.zeros(1, dtype=torch.int64, device=dev)  # Gaussian count of the first bad step
    gb = None
    reports_d, reports_p, rows = [], [], []

    def check():
        v = int(first_bad.item())
        if v != _NO_BAD:
            n0 = max(int(first_n.item()), 1)
            raise NonFiniteGradientError(v % n0, _CLASSES[v // n0])

    lo, hi = parallel.shard_bounds(batch, rank, world)
    iters = config.iterations
    if graph and world > 1:
        raise ConfigError("captured iterations need a single process (graph=False under torch.distributed)")
    # the samples of every iteration (row it) and the learning-rate schedule, drawn up front
    draws = [rng.integers(len(txs), size=batch)[lo:hi] for _ in range(iters)]
    idx_all = torch.as_tensor(np.stack([np.zeros(hi - lo, dtype=np.int64)] + draws).astype(np.int64), device=dev)
    lr_all = torch.tensor([0.0] + [lr_mean(config, i) for i in range(1, iters + 1)], dtype=torch.float32, device=dev)
    ctr = torch.zeros(1, dtype=torch.int64, device=dev)  # the iteration a replay runs
    ovf_at = torch.full((1,), _NO_OVF, dtype=torch.int64, device=dev)  # first replay past a capacity
    halt = torch.full((1,), _NO_BAD, dtype=torch.int64, device=dev)
    trace_buf = None
    n_at = [0] * (iters + 1)
    has_row = [False] * (iters + 1)

    def loss_up(S, gt):
        if mode == "spectrum":
            if S.shape[0] <= raster.MAX_TX_PER_LAUNCH:  # the upstream written ray-major for the backward
                rep, lamT, _ = _loss.spectrum_loss_frames(S, gt, config.w_ssim, config.w_fourier, lam_layout="rays")
                return rep, None, lamT
            rep, lam, _ = _loss.spectrum_loss_frames(S, gt, config.w_ssim, config.w_fourier)
            return rep, lam, None
        rep, _, lam = _loss.scalar_loss_frames(S, gt, "real_power" if mode == "rssi" else "complex")
        return rep, lam, None

    def step(it, deferred=None):
        """One iteration; `deferred` = the captured form (indexes by ctr)."""
        nonlocal gb, trace_buf
        idx = idx_all[it] if deferred is None else idx_all.index_select(0, ctr).view(-1)
        tx, gt = txs.index_select(0, idx), frames.index_select(0, idx)
        geo = raster.build_geometry(scene, psi_tx=tx, forward=True, index=True,
                                    after_forward=lambda S: loss_up(S, gt), deferred=deferred)
        rep, lam, lamT = geo.after_result
        if world > 1:
            if gb is None or gb.n != scene.n:
                gb = parallel.GradBuffer(scene.n, scene.fle_degree, dev)
            g = parallel.backward_reduced(scene, geo, tx, lam, gb, config.direction_chain, psi=geo.psi, lamT=lamT,
                                          group=group)
        else:
            g = raster.backward(scene, geo, tx, lam, config.direction_chain, psi=geo.psi, lamT=lamT)
        n_now = scene.n
        if deferred is None:
            prior, lr_dev = first_bad, None
        else:  # a capacity overflow of this or an earlier replay halts the updates like a bad step
            c, sv, zv = deferred["caps"], deferred["stats"], deferred["status"]
            over = (((zv[0:1] & 2) != 0) | ((zv[1:2].long() & 0xFFFFFFFF) > c["m_cap"]) | (sv[0:1] != 0)
                    | (sv[1:2] != 0) | (sv[3:4] > c["h_cap"]) | (sv[8:9] > c["u_cap"]))
            ovf_at.copy_(torch.where(over & (ovf_at == _NO_OVF), ctr, ovf_at))
            halt.copy_(torch.where((first_bad != _NO_BAD) | (ovf_at != _NO_OVF), torch.zeros_like(halt),
                                   torch.full_like(halt, _NO_BAD)))
            prior, lr_dev = halt, lr_all.index_select(0, ctr)
        sgd_step(scene, g, it, config, state, check=False, prior=prior, lr_dev=lr_dev)
        fresh = (prior == _NO_BAD) & (sgd_step.last_bad != _NO_BAD)
        first_n.copy_(torch.where(fresh, torch.full_like(first_n, n_now), first_n))
        first_bad.copy_(torch.where(fresh, sgd_step.last_bad, first_bad))
        if trace_buf is None:
            trace_buf = torch.zeros((iters + 1, rep.shape[1]), dtype=rep.dtype, device=dev)
        if deferred is None:
            trace_buf[it].copy_(rep.sum(0))
        else:
            trace_buf.index_copy_(0, ctr, rep.sum(0, keepdim=True))
            ctr.add_(1)

    def signature():
        return (scene.n,) + tuple(getattr(scene, k).data_ptr() for k in _FIELDS) + (
            state.grad_ema.data_ptr(), state.last_dmean.data_ptr())

    def capture():
        hook = _LOOP_HOOKS.get("before_capture")
        if hook is not None:
            hook()
        deferred = {"stats": torch.zeros(16, dtype=torch.int32, device=dev),
                    "status": torch.zeros(8, dtype=torch.int32, device=dev)}
        # capture_begin / capture_end on a side stream: no synchronize, gc pass
        # or allocator flush per capture (torch.cuda.graph does all three)
        g = torch.cuda.CUDAGraph()
        cur = torch.cuda.current_stream(dev)
        cap_stream.wait_stream(cur)
        try:
            with torch.cuda.stream(cap_stream):
                g.capture_begin()
                try:
                    step(0, deferred)
                finally:
                    g.capture_end()
        except ValueError:  # capacities not known for this scene (see raster._geometry_deferred)
            return None
        finally:
            cur.wait_stream(cap_stream)
        return g, signature()

    cg = None  # (graph, scene signature)
    cap_stream = torch.cuda.Stream(dev) if graph else None
    graph_off = False  # captures kept overflowing at their first replay: eager until the scene changes
    fails = tries = 0  # overflowing captures in a row / captures refused for missing capacities
    since_sync = []  # iterations replayed since the last sync point
    counts = train_loop.last_counts = {"replays": 0, "captures": 0, "rewinds": 0, "redone": 0, "capture_ms": 0.0}
    it = 1
    while it <= iters:
        e0 = torch.cuda.Event(enable_timing=True) if timings is not None else None
        if e0 is not None:
            e0.record()
        event = ""
        if scene.n > 0:
            if cg is not None and cg[1] == signature():
                cg[0].replay()
                since_sync.append(it)
                counts["replays"] += 1
            else:
                if cg is not None:
                    cg[0].reset()
                cg = None
                step(it)
                ctr.fill_(it + 1)
                if graph and not graph_off and it < iters and tries < 3:
                    t_cap = time.perf_counter()
                    cg = capture()
                    counts["capture_ms"] += (time.perf_counter() - t_cap) * 1e3
                    tries = 0 if cg is not None else tries + 1
                    counts["captures"] += cg is not None
            n_at[it], has_row[it] = scene.n, True
        dens = it < iters / 2 and scene.n > 0 and (it % config.densify_every == 0 or it % config.prune_every == 0)
        if since_sync and ((check_every > 0 and it % check_every == 0) or dens or it == iters):
            o = int(ovf_at.item())
            if o != _NO_OVF:  # iterations o..it were halted: redo them, o eagerly (capacities grow)
                fails = fails + 1 if o == since_sync[0] else 0
                graph_off = graph_off or fails >= 2
                ovf_at.fill_(_NO_OVF)
                counts["rewinds"] += 1
                counts["redone"] += it - o + 1
                cg[0].reset()
                cg = None
                if timings is not None:
                    timings[:] = [t for t in timings if t[0] < o]
                tries = 0
                since_sync = []
                it = o
                continue
            since_sync = []
        if check_every > 0 and it % check_every == 0:
            check()
        if it < iters / 2:
            if it % config.densify_every == 0 and scene.n > 0:
                check()  # no density control after a bad step
                r = densify(scene, state, it, config, seed)
                if r.cloned or r.split:
                    reports_d.append((it, r))
                    event += "densify "
                    graph_off, fails, tries = False, 0, 0
            if it % config.prune_every == 0 and scene.n > 0:
                check()
                r = prune(scene, state, it, config)
                if r.removed:
                    reports_p.append((it, r))
                    event += "prune "
                    graph_off, fails, tries = False, 0, 0
        if e0 is not None:
            e1 = torch.cuda.Event(enable_timing=True)
            e1.record()
            timings.append((it, e0, e1, scene.n, event.strip()))
        it += 1
    if cg is not None:
        cg[0].reset()
    torch.cuda.synchronize()
    check()
    if timings is not None:
        timings[:] = [(i, a.elapsed_time(b), n, ev, timings[j - 1][2].elapsed_time(a) if j else 0.0)
                      for j, (i, a, b, n, ev) in enumerate(timings)]
    rows = [i for i in range(1, iters + 1) if has_row[i]]
    if rows:
        sums = trace_buf[rows]
        if world > 1:
            dist.all_reduce(sums, op=dist.ReduceOp.SUM, group=group)
        means = (sums / max(batch, 1)).tolist()
    else:
        means = []
    trace = [TraceRow(i, *(float(x) for x in m), n_at[i]) for i, m in zip(rows, means)]
    return trace, reports_d, reports_p
