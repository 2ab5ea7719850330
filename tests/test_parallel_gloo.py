"""Multi-process (world_size 2, gloo, CPU) tests of the TX-sharded data parallelism.

The per-shard gradients come from the CPU oracle (test infrastructure); the
code under test is the product's sharding and all-reduce plumbing
(paper_2502_01826_b200/parallel.py): the all-reduced buffer of the shards
must equal the full-batch buffer (sum over TX, grad.py:85-92) on every rank.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2502_01826_b200.parallel import (
    GRAD_ORDER, allreduce_grads, flatten_grads, shard_bounds, shard_tx, unflatten_grads,
)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_shard_bounds_cover_batch_once():
    for n in (0, 1, 5, 64, 67):
        for world in (1, 2, 3, 8):
            seen = []
            for r in range(world):
                a, b = shard_bounds(n, r, world)
                seen.extend(range(a, b))
                assert abs((b - a) - n / world) < 1
            assert seen == list(range(n))


def test_flatten_roundtrip():
    rng = np.random.default_rng(0)
    g = {k: torch.tensor(rng.normal(size=(5, 3)), dtype=torch.float32) for k in GRAD_ORDER}
    g["d_coeffs"] = torch.tensor(rng.normal(size=(5, 16)) + 1j * rng.normal(size=(5, 16)), dtype=torch.complex64)
    back = unflatten_grads(flatten_grads(g), g)
    for k in GRAD_ORDER:
        assert torch.equal(back[k], g[k])


def _oracle_grads(scene, txs, ups):
    import oracle

    ctx = oracle.OracleContext(scene)
    tot = None
    for t, u in zip(txs, ups):
        ctx.set_tx(t)
        g = ctx.backward(u)
        tot = g if tot is None else {k: tot[k] + g[k] for k in tot}
    return tot


def _to_torch(g):
    return {
        "d_mean": torch.tensor(g["d_mean"], dtype=torch.float32),
        "d_quat": torch.tensor(g["d_quat"], dtype=torch.float32),
        "d_log_scale": torch.tensor(g["d_log_scale"], dtype=torch.float32),
        "d_trans_mag": torch.tensor(g["d_trans_mag"], dtype=torch.float32),
        "d_trans_mag_raw": torch.zeros(len(g["d_trans_mag"]), dtype=torch.float32),
        "d_trans_phase": torch.tensor(g["d_trans_phase"], dtype=torch.float32),
        "d_coeffs": torch.tensor(g["d_coeffs"], dtype=torch.complex64),
        "d_cov": torch.tensor(g["d_cov"], dtype=torch.float32),
    }


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2502_01826_b200.scene import bench_scene, default_txs, round_to_f32

        scene = round_to_f32(bench_scene(np.random.default_rng(3), 600, 48, 24))
        txs = default_txs(5, seed=2)
        rng = np.random.default_rng(4)
        ups = (rng.normal(size=(5, 48, 24)) + 1j * rng.normal(size=(5, 48, 24))) * 1e-2
        mine = shard_tx(np.arange(5), rank, world)
        g_local = _to_torch(_oracle_grads(scene, txs[mine], ups[mine]))
        g_sum = allreduce_grads(g_local)
        q.put((rank, {k: v.numpy() for k, v in g_sum.items()}))
    finally:
        dist.destroy_process_group()


def test_allreduce_of_shards_equals_full_batch():
    from paper_2502_01826_b200.scene import bench_scene, default_txs, round_to_f32

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    scene = round_to_f32(bench_scene(np.random.default_rng(3), 600, 48, 24))
    txs = default_txs(5, seed=2)
    rng = np.random.default_rng(4)
    ups = (rng.normal(size=(5, 48, 24)) + 1j * rng.normal(size=(5, 48, 24))) * 1e-2
    full = _to_torch(_oracle_grads(scene, txs, ups))
    for k in GRAD_ORDER:
        if k == "d_trans_mag_raw":
            continue
        ref = full[k].numpy()
        scale = max(np.abs(ref).max(), 1e-30)
        for r in (0, 1):
            np.testing.assert_allclose(res[r][k], ref, atol=1e-5 * scale, rtol=1e-5)
        np.testing.assert_array_equal(res[0][k], res[1][k])  # replicas stay identical
