"""api.StepGraph: the steady-state step captured as a CUDA graph must give
bitwise the eager step's frames and gradients, validate its deferred
statistics, and follow a new TX batch copied into its input buffer."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from paper_2502_01826_b200 import api, parallel, raster
from paper_2502_01826_b200.scene import bench_scene, default_txs, round_to_f32

pytestmark = pytest.mark.gpu


def _upstream(ds, tx):
    geo = raster.build_geometry(ds)
    S = raster.forward(geo, raster.compute_psi(ds, tx, geo.used))
    P = S.abs() ** 2
    lam = (2.0 * torch.sign(P - (1.3 * P + 0.05)) / P[0].numel() * S).to(torch.complex64).contiguous()
    return raster.transpose_upstream(lam)


def test_step_graph_equals_eager_step():
    s = round_to_f32(bench_scene(np.random.default_rng(3), 20_000, 120, 60))
    ds = raster.DeviceScene.from_host(s, "cuda")
    tx = torch.as_tensor(default_txs(64, seed=5), dtype=torch.float32, device="cuda")
    lamT = _upstream(ds, tx)
    gb_e = parallel.GradBuffer(ds.n, ds.fle_degree, "cuda")
    S_e, g_e = api.fwd_bwd_device(ds, tx, None, lamT=lamT, grads=gb_e)
    S_e = S_e.clone()
    flat_e = gb_e.flat.clone()
    gb_g = parallel.GradBuffer(ds.n, ds.fle_degree, "cuda")
    sg = api.StepGraph(ds, tx, lamT, gb_g)
    gb_g.flat.zero_()
    sg.replay()
    torch.cuda.synchronize()
    assert sg.ok()
    assert torch.equal(sg.S, S_e)
    assert torch.equal(gb_g.flat, flat_e)
    # a new TX batch through the input buffer: equals the eager step on it
    tx2 = torch.as_tensor(default_txs(64, seed=9), dtype=torch.float32, device="cuda")
    sg.set_tx(tx2)
    sg.replay()
    torch.cuda.synchronize()
    assert sg.ok()
    gb_2 = parallel.GradBuffer(ds.n, ds.fle_degree, "cuda")
    S_2, _ = api.fwd_bwd_device(ds, tx2, None, lamT=lamT, grads=gb_2)
    assert torch.equal(sg.S, S_2)
    assert torch.equal(gb_g.flat, gb_2.flat)


def test_train_step_graph_equals_eager_step():
    s = round_to_f32(bench_scene(np.random.default_rng(4), 20_000, 120, 60))
    ds = raster.DeviceScene.from_host(s, "cuda")
    tx = torch.as_tensor(default_txs(64, seed=6), dtype=torch.float32, device="cuda")
    geo = raster.build_geometry(ds)
    S = raster.forward(geo, raster.compute_psi(ds, tx, geo.used))
    gt = (S.abs() ** 2 * 1.2 + 0.01).float()
    txh = tx.cpu().pin_memory()
    gth = gt.cpu().pin_memory()
    rep_e = torch.empty((64, 4), dtype=torch.float64).pin_memory()
    gb_e = parallel.GradBuffer(ds.n, ds.fle_degree, "cuda")
    api.train_step_host(ds, txh, gth, rep_e, grads=gb_e)
    torch.cuda.synchronize()
    rep_g = torch.empty((64, 4), dtype=torch.float64).pin_memory()
    gb_g = parallel.GradBuffer(ds.n, ds.fle_degree, "cuda")
    tg = api.TrainStepGraph(ds, txh, gth, rep_g, gb_g)
    rep_g.zero_()
    gb_g.flat.zero_()
    tg.replay()
    torch.cuda.synchronize()
    assert tg.ok()
    assert torch.equal(rep_g, rep_e)
    assert torch.equal(gb_g.flat, gb_e.flat)
    # new host data in the same pinned buffers is picked up by the next replay
    gth.mul_(1.5)
    tg.replay()
    torch.cuda.synchronize()
    rep_2 = torch.empty((64, 4), dtype=torch.float64).pin_memory()
    api.train_step_host(ds, txh, gth, rep_2, grads=parallel.GradBuffer(ds.n, ds.fle_degree, "cuda"))
    torch.cuda.synchronize()
    assert torch.equal(rep_g, rep_2)


def test_dropin_host_call_equals_device_step():
    """api.fwd_bwd_host (host buffers in and out, the upstream's H2D and the
    frames' D2H on their own copy streams) returns bitwise the device step's
    frames and gradients."""
    s = round_to_f32(bench_scene(np.random.default_rng(5), 20_000, 120, 60))
    ds = raster.DeviceScene.from_host(s, "cuda")
    tx = torch.as_tensor(default_txs(64, seed=7), dtype=torch.float32, device="cuda")
    geo = raster.build_geometry(ds)
    S0 = raster.forward(geo, raster.compute_psi(ds, tx, geo.used))
    lam = (S0 * 0.37 - 0.1j * S0.abs()).to(torch.complex64).contiguous()
    S_d, g_d = api.fwd_bwd_device(ds, tx, lam)
    S_d = S_d.clone()
    g_d = {k: v.clone() for k, v in g_d.items()}
    hs = api.pinned_host_scene(s)
    out = api.alloc_host_outputs(ds.n, (ds.fle_degree + 1) ** 2, 64, 120, 60)
    for _ in range(2):  # the second call: known capacities (the timed path)
        for v in out.values():
            v.zero_()
        api.fwd_bwd_host(hs, tx.cpu().pin_memory(), lam.cpu().pin_memory(), out, s.rx, s.ress_radius, 120, 60,
                         ds.fle_degree)
        torch.cuda.current_stream().synchronize()
        assert torch.equal(out["S"], S_d.cpu())
        for k in api.OUT_GRADS:
            assert torch.equal(out[k], g_d[k].cpu()), k
