"""Data parallelism over the transmitter batch.

One process per GPU (torch.distributed, backend "nccl" on B200, "gloo" in the
CPU tests).  Every rank holds the full scene (Gaussians replicated), builds
the transmitter-independent geometry (projection, tile index, hit lists)
itself -- it is deterministic, so all ranks build the same one -- and runs the
TX-dependent kernels on its own contiguous shard of the TX batch.  The only
exchange is an all-reduce (sum) of the per-Gaussian gradient buffer per step:
the batch semantics of the reference are a sum over transmitters
(GradientBuffer.add, grad.py:85-92), and every gradient term is linear in the
upstream frames, so the sum of the per-shard buffers is the full-batch buffer.
After the all-reduce every rank holds identical gradients, so optimizer
updates and densify / prune decisions (train.py:167-245) taken from them are
identical on every rank without further communication.

Strong scaling (`tile_step`, SURVEY.md §8(e) "Scaling risk" fallback): with
few TX per rank the replicated TX-independent geometry -- above all the hit
lists K6 -- dominates, so the ray space is sharded instead: each rank traces
only the rays of a contiguous range of tiles (balanced by the tiles'
incidence counts), composites all B TX for them, and the frames are summed
over the ranks (disjoint supports: an all-reduce of S, which the loss needs
whole); the backward of its own hits gives a partial gradient buffer, reduced
as above (every gradient term is a sum over hits).

The reduced payload is 44 fp32 per Gaussian: d_coeffs 32,
d_mean 3, d_quat 4, d_log_scale 3, d_trans_mag 1, d_trans_phase 1.  The
backward writes straight into `GradBuffer`, one persistent flat fp32 buffer
whose fields are views (no pack / unpack copies), in two buckets:
  bucket 0 = d_coeffs, complete when K9b (k_grad_tx) finishes -- its
             all-reduce is issued then and overlaps K9a / K9c;
  bucket 1 = the geometry fields, complete after K9c (k_geom_final).
d_trans_mag_raw = d_trans_mag * sigma(1 - sigma) is elementwise in the
reduced d_trans_mag and is recomputed after the reduce; d_cov (not used by
the optimizer) is reduced only on request (`with_cov`).
"""

from __future__ import annotations

import torch
import torch.distributed as dist

__all__ = ["shard_bounds", "shard_tx", "flatten_grads", "unflatten_grads", "allreduce_grads", "GradBuffer",
           "dp_step", "GRAD_ORDER", "REDUCED_FLOATS", "tile_shards", "TileSharder", "tile_step"]

# gradient buffer fields in the order they are packed by flatten_grads
GRAD_ORDER = ("d_mean", "d_quat", "d_log_scale", "d_trans_mag", "d_trans_mag_raw", "d_trans_phase", "d_coeffs",
              "d_cov")
REDUCED_FLOATS = 44  # per Gaussian at fle_degree 3 (d_coeffs 2 * 16)


def shard_bounds(n_tx: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced [start, end) of rank's TX shard (sizes differ by <= 1)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("invalid rank / world size")
    base, extra = divmod(n_tx, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def shard_tx(txs, rank: int, world: int):
    a, b = shard_bounds(len(txs), rank, world)
    return txs[a:b]


def _world(group=None) -> int:
    return dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1


class GradBuffer:
    """Persistent flat gradient buffer of one rank; `views` is the gradient
    dict raster.backward(out=...) writes into.

    Layout (fp32): [d_coeffs 2K·N | d_mean 3N | d_quat 4N | d_log_scale 3N |
    d_trans_mag N | d_trans_phase N | d_cov 9N | d_trans_mag_raw N]; the first
    (2K + 12)·N floats are the all-reduced payload, d_cov joins it with
    `with_cov`.
    """

    def __init__(self, n: int, fle_degree: int = 3, device="cuda", with_cov: bool = False):
        K = (fle_degree + 1) ** 2
        self.n, self.K, self.with_cov = n, K, with_cov
        sizes = [("d_coeffs", 2 * K * n), ("d_mean", 3 * n), ("d_quat", 4 * n), ("d_log_scale", 3 * n),
                 ("d_trans_mag", n), ("d_trans_phase", n), ("d_cov", 9 * n), ("d_trans_mag_raw", n)]
        total = sum(s for _, s in sizes)
        self.flat = torch.zeros(max(total, 1), dtype=torch.float32, device=device)
        self.views, off, self._off = {}, 0, {}
        shapes = {"d_coeffs": (n, K, 2), "d_mean": (n, 3), "d_quat": (n, 4), "d_log_scale": (n, 3),
                  "d_trans_mag": (n,), "d_trans_phase": (n,), "d_cov": (n, 3, 3), "d_trans_mag_raw": (n,)}
        for name, size in sizes:
            v = self.flat[off:off + size].view(shapes[name])
            self.views[name] = torch.view_as_complex(v) if name == "d_coeffs" else v
            self._off[name] = (off, off + size)
            off += size
        self.bucket0 = self.flat[0:2 * K * n]                       # d_coeffs
        end1 = self._off["d_cov" if with_cov else "d_trans_phase"][1]
        self.bucket1 = self.flat[2 * K * n:end1]                    # geometry fields (+ d_cov)
        self.payload_floats = end1 // max(n, 1)

    @property
    def reduced_bytes(self) -> int:
        return 4 * (self.bucket0.numel() + self.bucket1.numel())


def flatten_grads(g: dict, order=GRAD_ORDER) -> torch.Tensor:
    """One contiguous fp32 buffer (complex fields viewed as pairs of floats)."""
    parts = []
    for k in order:
        t = g[k].contiguous()
        parts.append((torch.view_as_real(t) if t.is_complex() else t).reshape(-1).to(torch.float32))
    return torch.cat(parts)


def unflatten_grads(flat: torch.Tensor, like: dict, order=GRAD_ORDER) -> dict:
    out, o = {}, 0
    for k in order:
        t = like[k]
        n = t.numel() * (2 if t.is_complex() else 1)
        v = flat[o:o + n]
        o += n
        if t.is_complex():
            out[k] = torch.view_as_complex(v.reshape(*t.shape, 2).contiguous())
        else:
            out[k] = v.reshape(t.shape).clone()
    return out


def _raw_chain(gb: GradBuffer, trans_mag_raw: torch.Tensor) -> None:
    """d_trans_mag_raw = d|rho| sigma (1 - sigma) (train.py:161-162) from the reduced d|rho|."""
    sg = torch.sigmoid(trans_mag_raw.to(torch.float32))
    torch.mul(gb.views["d_trans_mag"], sg * (1.0 - sg), out=gb.views["d_trans_mag_raw"])


def allreduce_grads(g, group=None, order=GRAD_ORDER, trans_mag_raw: torch.Tensor | None = None):
    """Sum the gradient buffer over ranks.

    With a GradBuffer: in place, the two buckets (44 floats per Gaussian),
    then d_trans_mag_raw from the reduced d_trans_mag (needs `trans_mag_raw`,
    the scene's logits).  With a plain dict: one packed all-reduce of every
    field (returns a new dict).
    """
    if _world(group) == 1:
        return g
    if isinstance(g, GradBuffer):
        dist.all_reduce(g.bucket0, op=dist.ReduceOp.SUM, group=group)
        dist.all_reduce(g.bucket1, op=dist.ReduceOp.SUM, group=group)
        if trans_mag_raw is not None:
            _raw_chain(g, trans_mag_raw)
        return g
    flat = flatten_grads(g, order)
    dist.all_reduce(flat, op=dist.ReduceOp.SUM, group=group)
    return unflatten_grads(flat, g, order)


class _OverlappedReduce:
    """raster.backward hook: all-reduce bucket 0 (d_coeffs) on a communication
    stream as soon as K9b has produced it, overlapping K9a / K9c; bucket 1 after
    the backward.  `finish()` makes the current stream wait for both."""

    def __init__(self, gb: GradBuffer, group=None):
        self.gb, self.group = gb, group
        self.works = []

    def coeffs_ready(self, event: torch.cuda.Event) -> None:
        s = _comm_stream(self.gb.flat.device)
        s.wait_event(event)
        with torch.cuda.stream(s):
            self.works.append(dist.all_reduce(self.gb.bucket0, op=dist.ReduceOp.SUM, group=self.group,
                                              async_op=True))

    def finish(self, trans_mag_raw: torch.Tensor) -> None:
        s = _comm_stream(self.gb.flat.device)
        s.wait_stream(torch.cuda.current_stream(self.gb.flat.device))
        with torch.cuda.stream(s):
            self.works.append(dist.all_reduce(self.gb.bucket1, op=dist.ReduceOp.SUM, group=self.group,
                                              async_op=True))
        for w in self.works:
            w.wait()  # the current stream waits for the collectives (NCCL); gloo blocks
        torch.cuda.current_stream(self.gb.flat.device).wait_stream(s)
        self.works = []
        _raw_chain(self.gb, trans_mag_raw)


_COMM: dict = {}


def _comm_stream(dev) -> torch.cuda.Stream:
    k = str(dev)
    if k not in _COMM:
        _COMM[k] = torch.cuda.Stream(device=dev)
    return _COMM[k]


def backward_reduced(scene, geo, tx, grad_S, gb: GradBuffer, include_direction_chain: bool = True, psi=None,
                     lamT=None, group=None, marks=None) -> dict:
    """raster.backward into `gb` followed by the bucketed all-reduce (overlapped
    with the epilogue when the process group runs on CUDA streams)."""
    from . import raster

    if _world(group) == 1:
        return raster.backward(scene, geo, tx, grad_S, include_direction_chain, psi=psi, lamT=lamT, out=gb.views,
                               marks=marks)
    red = _OverlappedReduce(gb, group)
    g = raster.backward(scene, geo, tx, grad_S, include_direction_chain, psi=psi, lamT=lamT, out=gb.views,
                        on_coeffs=red.coeffs_ready, marks=marks)
    red.finish(scene.trans_mag_raw)
    return g


def dp_step(scene, txs_global, lam_global, include_direction_chain: bool = True, group=None,
            sort_backend: str = "hand", gb: GradBuffer | None = None) -> tuple:
    """One data-parallel fwd+bwd step on this rank's TX shard.

    scene is a raster.DeviceScene (replicated); txs_global [B,3] and
    lam_global [B,n_az,n_el] are the full batch (each rank slices its shard).
    Returns (S_shard, all-reduced gradient dict -- the views of `gb`).
    """
    from . import raster

    world = _world(group)
    rank = dist.get_rank(group) if world > 1 else 0
    a, b = shard_bounds(int(txs_global.shape[0]), rank, world)
    tx = txs_global[a:b].contiguous()
    if gb is None:
        gb = GradBuffer(scene.n, scene.fle_degree, scene.means.device)
    geo = raster.build_geometry(scene, sort_backend=sort_backend, psi_tx=tx, index=True, forward=True)
    S = geo.S
    g = backward_reduced(scene, geo, tx, lam_global[a:b].contiguous(), gb, include_direction_chain, psi=geo.psi,
                         group=group)
    return S, g


def tile_shards(lengths, world: int) -> list:
    """Contiguous tile ranges [(lo, hi)] for `world` ranks with balanced total
    list length (the K6 cost is ~ the candidates its rays walk)."""
    lengths = [max(int(x), 0) for x in lengths]
    n = len(lengths)
    total = sum(lengths) or 1
    out, lo, acc = [], 0, 0
    for r in range(world):
        if r == world - 1:
            out.append((lo, n))
            break
        target = total * (r + 1) / world
        hi = lo
        while hi < n and acc + lengths[hi] <= target:
            acc += lengths[hi]
            hi += 1
        if hi < n and hi == lo and n - lo > world - 1 - r:  # at least one tile
            acc += lengths[hi]
            hi += 1
        out.append((lo, hi))
        lo = hi
    return out


class TileSharder:
    """The tile shard of each rank, balanced by the last step's tile list
    lengths (an asynchronous 2 KB copy of the ranges, read at the next step);
    equal tile counts until then.  Every rank computes the same (deterministic)
    binning, hence the same shards."""

    def __init__(self, world: int, rank: int):
        self.world, self.rank = world, rank
        self._pending = None
        self._lengths = None

    def bounds(self, n_tiles: int) -> tuple:
        if self._pending is not None:
            ev, host = self._pending
            ev.synchronize()
            self._lengths = (host[:, 1] - host[:, 0]).tolist()
            self._pending = None
        if self._lengths is None or len(self._lengths) != n_tiles:
            return tile_shards([1] * n_tiles, self.world)[self.rank]
        return tile_shards(self._lengths, self.world)[self.rank]

    def update(self, geo) -> None:
        host = torch.empty(tuple(geo.ranges.shape), dtype=geo.ranges.dtype).pin_memory()
        host.copy_(geo.ranges, non_blocking=True)
        ev = torch.cuda.Event()
        ev.record()
        self._pending = (ev, host)


def tile_step(scene, tx, lamT, gb: GradBuffer, sharder: TileSharder, include_direction_chain: bool = True,
              group=None, sort_backend: str = "hand", marks=None) -> tuple:
    """One strong-scaling fwd+bwd step: every rank gets the WHOLE TX batch
    `tx` [B, 3] and upstream lamT [R, B] (the loss kernel's layout), traces its
    tile shard, all-reduces S (the full frames, as the loss needs them) and the
    gradient buffer.  Returns (S [B, n_az, n_el], gradient dict)."""
    from . import raster

    world = _world(group)
    n_tiles = ((scene.n_az + raster.TILE - 1) // raster.TILE) * ((scene.n_el + raster.TILE - 1) // raster.TILE)
    tiles = sharder.bounds(n_tiles) if world > 1 else None
    geo = raster.build_geometry(scene, sort_backend=sort_backend, marks=marks, psi_tx=tx, forward=True,
                                index=True, tiles=tiles)
    if world > 1:
        sharder.update(geo)
    S = geo.S
    if world > 1:
        s = _comm_stream(S.device)
        s.wait_stream(torch.cuda.current_stream(S.device))
        with torch.cuda.stream(s):  # the frames are summed while the backward runs
            work = dist.all_reduce(torch.view_as_real(S), op=dist.ReduceOp.SUM, group=group, async_op=True)
    g = backward_reduced(scene, geo, tx, None, gb, include_direction_chain, psi=geo.psi, lamT=lamT, group=group,
                         marks=marks)
    if world > 1:
        work.wait()
        torch.cuda.current_stream(S.device).wait_stream(s)
        S.record_stream(s)
    return S, g
