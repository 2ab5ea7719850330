"""Data-parallel step on the GPU: 2 ranks (gloo) sharing cuda:0 run
parallel.dp_step -- each its TX shard, the backward writing into a
GradBuffer, the bucketed all-reduce overlapped with the epilogue -- and the
reduced gradients must equal the full-batch backward and the oracle's sum
over all TX (grad.py:85-92).  (NCCL cannot put two ranks on one GPU; the
driver's multi-GPU runs use NCCL through the same code.)"""

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

import oracle  # noqa: E402
from helpers import GRAD_KEYS, class_rel, l1_upstream  # noqa: E402

from paper_2502_01826_b200.scene import bench_scene, default_txs, round_to_f32  # noqa: E402

pytestmark = pytest.mark.gpu

N, AZ, EL, B = 8_000, 180, 90, 6


def _case():
    s = round_to_f32(bench_scene(np.random.default_rng(5), N, AZ, EL))
    txs = default_txs(B, seed=2)
    oc = oracle.OracleContext(s)
    lams, ref = [], None
    for t in txs:
        oc.set_tx(t)
        lam = l1_upstream(oc.forward())
        lams.append(lam)
        g = oc.backward(lam)
        ref = g if ref is None else {k: ref[k] + g[k] for k in ref}
    return s, txs, np.stack(lams), ref


def _worker(rank, world, port, s, txs, lams, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2502_01826_b200 import api, parallel, raster

        ds = raster.DeviceScene.from_host(s, "cuda:0")
        tx = torch.as_tensor(txs, dtype=torch.float32, device="cuda:0")
        lam = torch.as_tensor(lams.astype(np.complex64), device="cuda:0")
        gb = parallel.GradBuffer(ds.n, ds.fle_degree, "cuda:0")
        for _ in range(2):  # second step: the early side-stream index, reused buffer
            S, g = parallel.dp_step(ds, tx, lam, gb=gb)
        torch.cuda.synchronize()
        q.put((rank, api.GradientBuffer.from_device(g).__dict__, g["d_trans_mag_raw"].cpu().numpy(),
               gb.payload_floats))
    finally:
        dist.destroy_process_group()


def test_dp_step_two_ranks_equals_full_batch_and_oracle():
    from paper_2502_01826_b200 import api, raster

    s, txs, lams, ref = _case()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, s, txs, lams, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = {}
    for _ in procs:
        r, g, raw, pf = q.get(timeout=300)
        out[r] = (g, raw, pf)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    full = api.backward_frames(s, txs, lams)
    for k in ("d_mean", "d_quat", "d_log_scale", "d_trans_mag", "d_trans_phase", "d_coeffs"):
        # identical on both ranks, equal to the single-process batch, and to the oracle
        np.testing.assert_array_equal(out[0][0][k], out[1][0][k])
        # (the shard sums are rounded to fp32 before the reduce: d(phase), a sum
        # of strongly cancelling terms, shows it most)
        assert class_rel(out[0][0][k], getattr(full, k)) <= 2e-4, k
        assert class_rel(out[0][0][k], ref[k]) <= 1e-3, k
    sg = 1 / (1 + np.exp(-s.trans_mag_raw.astype(np.float64)))
    assert class_rel(out[0][1], ref["d_trans_mag"] * sg * (1 - sg)) <= 1e-3
    assert out[0][2] == 44  # reduced floats per Gaussian


def _train_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank,) + _train_run())
    finally:
        dist.destroy_process_group()


def _train_run():
    from paper_2502_01826_b200 import raster
    from paper_2502_01826_b200 import train as T
    from paper_2502_01826_b200.scene import cube_init, default_txs, round_to_f32

    init = round_to_f32(cube_init([-15] * 3, [15] * 3, 4.0, 72, 36, c00=30.0))
    txs = torch.as_tensor(default_txs(8, seed=5), dtype=torch.float32, device="cuda:0")
    geo = raster.build_geometry(raster.DeviceScene.from_host(init, "cuda:0"), psi_tx=txs, forward=True)
    frames = (1.2 * geo.S.abs() ** 2 + 0.01).float().contiguous()
    ds = raster.DeviceScene.from_host(init, "cuda:0")
    cfg = T.TrainConfig(iterations=12, densify_every=5, prune_every=5, densify_grad_threshold=1e-10,
                        lr_radiance=0.05, lr_transmittance=0.05)
    trace, dens, _ = T.train_loop(ds, txs, frames, cfg, batch=4, seed=3)
    return ds.means.cpu().numpy(), [r.total for r in trace], len(dens)


def test_train_loop_data_parallel_two_ranks():
    """train_loop over 2 ranks (each half of every batch, gradients
    all-reduced): both ranks end with the same scene, the same densify
    decisions and the loss trace of the single-process run."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    procs = [ctx.Process(target=_train_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = {}
    for _ in procs:
        r, means, trace, nd = q.get(timeout=600)
        out[r] = (means, trace, nd)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    np.testing.assert_array_equal(out[0][0], out[1][0])
    assert out[0][2] == out[1][2] > 0
    means1, trace1, nd1 = _train_run()
    assert nd1 == out[0][2] and out[0][0].shape == means1.shape
    np.testing.assert_allclose(out[0][0], means1, rtol=0, atol=1e-4)
    np.testing.assert_allclose(out[0][1], trace1, rtol=1e-4)


def _tile_worker(rank, world, port, s, txs, lams, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2502_01826_b200 import api, parallel, raster

        ds = raster.DeviceScene.from_host(s, "cuda:0")
        tx = torch.as_tensor(txs, dtype=torch.float32, device="cuda:0")
        lamT = raster.transpose_upstream(torch.as_tensor(lams.astype(np.complex64), device="cuda:0"))
        gb = parallel.GradBuffer(ds.n, ds.fle_degree, "cuda:0")
        sharder = parallel.TileSharder(world, rank)
        for _ in range(2):  # second step: shards balanced by the first step's tile lists
            S, g = parallel.tile_step(ds, tx, lamT, gb, sharder)
        torch.cuda.synchronize()
        q.put((rank, S.cpu().numpy(), api.GradientBuffer.from_device(g).__dict__, None))
    finally:
        dist.destroy_process_group()


def test_tile_sharded_step_two_ranks_equals_unsharded():
    """Strong scaling (parallel.tile_step): 2 ranks each trace half of the
    tiles; the all-reduced frames equal the unsharded frames bitwise (disjoint
    supports), the reduced gradients equal the unsharded backward and the
    oracle."""
    from paper_2502_01826_b200 import api, raster

    s, txs, lams, ref = _case()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    procs = [ctx.Process(target=_tile_worker, args=(r, 2, port, s, txs, lams, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = {}
    for _ in procs:
        r, S, g, _b = q.get(timeout=300)
        out[r] = (S, g)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ds = raster.DeviceScene.from_host(s, "cuda")
    tx = torch.as_tensor(txs, dtype=torch.float32, device="cuda")
    S_full, g_full = api.fwd_bwd_device(ds, tx, torch.as_tensor(lams.astype(np.complex64), device="cuda"))
    S_full = S_full.cpu().numpy()
    np.testing.assert_array_equal(out[0][0], S_full)
    np.testing.assert_array_equal(out[1][0], S_full)
    full = api.GradientBuffer.from_device(g_full)
    for k in ("d_mean", "d_quat", "d_log_scale", "d_trans_mag", "d_trans_phase", "d_coeffs"):
        np.testing.assert_array_equal(out[0][1][k], out[1][1][k])
        assert class_rel(out[0][1][k], getattr(full, k)) <= 2e-4, k
        assert class_rel(out[0][1][k], ref[k]) <= 1e-3, k
