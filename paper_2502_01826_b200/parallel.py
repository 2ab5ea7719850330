"""Data parallelism over the transmitter batch.

One process per GPU (torch.distributed, backend "nccl" on B200, "gloo" in the
CPU tests).  Every rank holds the full scene (Gaussians replicated), builds
the transmitter-independent geometry (projection, tile index, hit lists)
itself -- it is deterministic, so all ranks build the same one -- and runs the
TX-dependent kernels on its own contiguous shard of the TX batch.  The only
exchange is one all-reduce (sum) of the per-Gaussian gradient buffer per step:
the batch semantics of the reference are a sum over transmitters
(GradientBuffer.add, grad.py:85-92), and every gradient term is linear in the
upstream frames, so the sum of the per-shard buffers is the full-batch buffer.
After the all-reduce every rank holds identical gradients, so optimizer
updates and densify / prune decisions (train.py:167-245) taken from them are
identical on every rank without further communication.
"""

from __future__ import annotations

import torch
import torch.distributed as dist

__all__ = ["shard_bounds", "shard_tx", "flatten_grads", "unflatten_grads", "allreduce_grads", "dp_step"]

# gradient buffer fields in the order they are packed for the all-reduce
GRAD_ORDER = ("d_mean", "d_quat", "d_log_scale", "d_trans_mag", "d_trans_mag_raw", "d_trans_phase", "d_coeffs",
              "d_cov")


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


def allreduce_grads(g: dict, group=None, order=GRAD_ORDER) -> dict:
    """Sum the gradient buffer over ranks: one collective per step."""
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size(group) == 1:
        return g
    flat = flatten_grads(g, order)
    dist.all_reduce(flat, op=dist.ReduceOp.SUM, group=group)
    return unflatten_grads(flat, g, order)


def dp_step(scene, txs_global, lam_global, include_direction_chain: bool = True, group=None,
            sort_backend: str = "hand") -> tuple:
    """One data-parallel fwd+bwd step on this rank's TX shard.

    scene is a raster.DeviceScene (replicated); txs_global [B,3] and
    lam_global [B,n_az,n_el] are the full batch (each rank slices its shard).
    Returns (S_shard, all-reduced gradient dict).
    """
    from . import raster

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    a, b = shard_bounds(int(txs_global.shape[0]), rank, world)
    tx = txs_global[a:b].contiguous()
    geo = raster.build_geometry(scene, sort_backend=sort_backend, psi_tx=tx, index=True, forward=True)
    psi = geo.psi
    S = raster.forward(geo, psi)
    g = raster.backward(scene, geo, tx, lam_global[a:b].contiguous(), include_direction_chain, psi=psi)
    return S, allreduce_grads(g, group)
