"""Optimizer and density control on the device vs the reference train.py
(golden vectors from tests/golden/make_golden_train.py)."""

import numpy as np
import pytest

from helpers import load
from paper_2502_01826_b200 import train as T
from paper_2502_01826_b200.errors import ConfigError


def test_config_validation_and_lr_schedule():
    z = load("train_golden.npz")
    cfg = T.TrainConfig(iterations=int(z["it"][1]))
    cfg.validate()
    got = [T.lr_mean(cfg, i) for i in (0, 1, 700, 1500, 3000, 4000)]
    np.testing.assert_allclose(got, z["lr_mean"], rtol=1e-15)
    with pytest.raises(ConfigError):
        T.TrainConfig(lr_scale=0.0).validate()
    with pytest.raises(ConfigError):
        T.TrainConfig(w_ssim=0.6, w_fourier=0.5).validate()


def _device_setup(z):
    import torch

    from paper_2502_01826_b200 import raster

    f = lambda k: torch.as_tensor(np.asarray(z[k], np.float32), device="cuda").contiguous()
    ds = raster.DeviceScene(f("means"), f("quats"), f("log_scales"), f("raw"), f("phase"),
                            torch.as_tensor(z["coeffs"], device="cuda").contiguous(), (0.0, 0.0, 0.0), 1.0, 90, 45, 3)
    grads = {"d_mean": f("g_mean"), "d_quat": f("g_quat"), "d_log_scale": f("g_log_scale"), "d_trans_mag": f("g_mag"),
             "d_trans_phase": f("g_phase"), "d_coeffs": torch.as_tensor(z["g_coeffs"], device="cuda").contiguous()}
    state = T.TrainState(f("ema"), f("last"))
    cfg = T.TrainConfig(iterations=int(z["it"][1]))
    return ds, grads, state, cfg


@pytest.mark.gpu
def test_gpu_sgd_step_and_observe():
    z = load("train_golden.npz")
    ds, grads, state, cfg = _device_setup(z)
    T.sgd_step(ds, grads, int(z["it"][0]), cfg, state)
    for k, ref in (("means", "sgd_means"), ("quats", "sgd_quats"), ("log_scales", "sgd_log_scales"),
                   ("trans_mag_raw", "sgd_raw"), ("trans_phase", "sgd_phase")):
        np.testing.assert_allclose(getattr(ds, k).cpu().numpy(), z[ref], rtol=2e-6, atol=2e-7, err_msg=k)
    np.testing.assert_allclose(ds.coeffs.cpu().numpy(), z["sgd_coeffs"], rtol=2e-6, atol=2e-7)
    np.testing.assert_allclose(state.grad_ema.cpu().numpy(), z["obs_ema"], rtol=2e-6, atol=1e-10)
    np.testing.assert_allclose(state.last_dmean.cpu().numpy(), z["obs_last"], rtol=0, atol=0)


@pytest.mark.gpu
def test_gpu_sgd_step_nonfinite_leaves_scene_untouched():
    from paper_2502_01826_b200.errors import NonFiniteGradientError

    z = load("train_golden.npz")
    ds, grads, state, cfg = _device_setup(z)
    grads["d_quat"][7, 2] = float("nan")
    grads["d_coeffs"][3, 1] = complex(float("inf"), 0.0)
    before = ds.means.clone()
    with pytest.raises(NonFiniteGradientError) as e:
        T.sgd_step(ds, grads, 1, cfg, state)
    assert e.value.args[0] == 7 or "quat" in str(e.value)  # first bad class in train.py:133-142 order
    assert bool((ds.means == before).all())


@pytest.mark.gpu
def test_gpu_densify_decisions_and_layout():
    z = load("train_golden.npz")
    ds, _, state, cfg = _device_setup(z)
    n = ds.n
    rep = T.densify(ds, state, int(z["it"][0]), cfg, seed=11)
    assert rep.cloned == z["dens_cloned"].tolist()
    assert rep.split == z["dens_split"].tolist()
    assert ds.n == int(z["dens_n"][0])
    nk, nc = n - len(rep.split), len(rep.cloned)
    # kept + clones: deterministic, compare with the reference
    m = ds.means.cpu().numpy()
    np.testing.assert_allclose(m[: nk + nc], z["dens_means"][: nk + nc], rtol=1e-6, atol=1e-7)
    for k, ref in (("quats", "dens_quats"), ("log_scales", "dens_log_scales"), ("trans_mag_raw", "dens_raw")):
        np.testing.assert_allclose(getattr(ds, k).cpu().numpy(), z[ref], rtol=1e-6, atol=1e-7, err_msg=k)
    # split children: two per parent with the parent's attributes, scales / 1.6, means ~ N(mu, Sigma)
    ls = z["log_scales"]
    q = z["quats"]
    for j, p in enumerate(rep.split):
        qq = q[p] / np.linalg.norm(q[p])
        w, x, y, zq = qq
        R = np.array([[1 - 2 * (y * y + zq * zq), 2 * (x * y - w * zq), 2 * (x * zq + w * y)],
                      [2 * (x * y + w * zq), 1 - 2 * (x * x + zq * zq), 2 * (y * zq - w * x)],
                      [2 * (x * zq - w * y), 2 * (y * zq + w * x), 1 - 2 * (x * x + y * y)]])
        for c in range(2):
            d = m[nk + nc + 2 * j + c] - z["means"][p]
            maha = np.linalg.norm((R.T @ d) / np.exp(ls[p]))
            assert maha < 6.0
    assert float(state.grad_ema.abs().sum()) == 0.0 and float(state.last_dmean.abs().sum()) == 0.0
    # counter-based sampling: same seed -> same children; another seed -> different
    ds2, _, st2, _ = _device_setup(z)
    T.densify(ds2, st2, int(z["it"][0]), cfg, seed=11)
    np.testing.assert_array_equal(ds2.means.cpu().numpy(), m)
    ds3, _, st3, _ = _device_setup(z)
    T.densify(ds3, st3, int(z["it"][0]), cfg, seed=12)
    assert not np.array_equal(ds3.means.cpu().numpy()[nk + nc:], m[nk + nc:])


@pytest.mark.gpu
def test_gpu_prune():
    z = load("train_golden.npz")
    ds, _, state, cfg = _device_setup(z)
    rep = T.prune(ds, state, int(z["it"][0]), cfg)
    assert rep.removed == z["prune_removed"].tolist()
    assert ds.n == int(z["prune_n"][0])
    np.testing.assert_array_equal(ds.means.cpu().numpy(), z["prune_means"].astype(np.float32))
    np.testing.assert_array_equal(state.grad_ema.cpu().numpy(), z["prune_ema"].astype(np.float32))


@pytest.mark.gpu
def test_gpu_train_loop_fits_and_densifies():
    """A short device training run: the loss falls, density control fires on
    schedule, and the run is bitwise reproducible (deterministic backward,
    counter-based split sampling)."""
    import torch

    from paper_2502_01826_b200 import raster
    from paper_2502_01826_b200.scene import bench_scene, cube_init, default_txs, round_to_f32

    # target: a perturbed copy of the initial scene (the reference's multipath
    # dataset simulator is outside this tier), so the fit is well posed
    init = cube_init([-15] * 3, [15] * 3, 2.5, 72, 36, c00=30.0)
    rng = np.random.default_rng(2)
    tgt = init.copy()
    tgt.means = tgt.means + rng.normal(0, 0.3, tgt.means.shape)
    tgt.trans_mag_raw = rng.normal(0, 1, tgt.n)
    tgt.coeffs = tgt.coeffs * rng.uniform(0.5, 1.5, (tgt.n, 1)) * np.exp(1j * rng.uniform(-1, 1, (tgt.n, 1)))
    tgt = round_to_f32(tgt)
    txs = torch.as_tensor(default_txs(16, seed=5), dtype=torch.float32, device="cuda")
    tds = raster.DeviceScene.from_host(tgt, "cuda")
    geo = raster.build_geometry(tds, psi_tx=txs, forward=True)
    frames = (geo.S.abs() ** 2).float().contiguous()

    def run():
        ds = raster.DeviceScene.from_host(round_to_f32(init), "cuda")
        cfg = T.TrainConfig(iterations=60, densify_every=10, prune_every=10, densify_grad_threshold=1e-9,
                            lr_radiance=0.05, lr_transmittance=0.05)
        trace, dens, pr = T.train_loop(ds, txs, frames, cfg, batch=4, seed=3)
        return trace, dens, ds

    trace, dens, ds = run()
    assert len(trace) == 60
    assert dens, "densify never fired"
    assert trace[-1].n_primitives == ds.n > trace[0].n_primitives
    def full_loss(scene):  # all 16 TX, fixed: the fit must improve
        from paper_2502_01826_b200 import loss as L

        g = raster.build_geometry(scene, psi_tx=txs, forward=True)
        return float(L.spectrum_loss_frames(g.S, frames)[0][:, 0].mean())

    assert full_loss(ds) < full_loss(raster.DeviceScene.from_host(round_to_f32(init), "cuda"))
    trace2, _, ds2 = run()
    assert [r.total for r in trace] == [r.total for r in trace2]
    assert torch.equal(ds.means, ds2.means)


def _small_fit_setup(n_tx=8):
    import torch

    from paper_2502_01826_b200 import raster
    from paper_2502_01826_b200.scene import cube_init, default_txs, round_to_f32

    init = round_to_f32(cube_init([-15] * 3, [15] * 3, 4.0, 72, 36, c00=30.0))
    txs = torch.as_tensor(default_txs(n_tx, seed=5), dtype=torch.float32, device="cuda")
    geo = raster.build_geometry(raster.DeviceScene.from_host(init, "cuda"), psi_tx=txs, forward=True)
    frames = (1.2 * geo.S.abs() ** 2 + 0.01).float().contiguous()
    return init, txs, frames


@pytest.mark.gpu
def test_gpu_train_loop_stops_at_first_nonfinite_step():
    """A non-finite gradient from step 1 on: train_loop raises
    NonFiniteGradientError and the scene is the one before that step
    (reference train.py:145-150) -- no later update, densify or prune."""
    import torch

    from paper_2502_01826_b200 import raster
    from paper_2502_01826_b200.errors import NonFiniteGradientError

    init, txs, frames = _small_fit_setup()
    ds = raster.DeviceScene.from_host(init, "cuda")
    ds.coeffs[:, 3] = complex(float("nan"), 0.0)  # NaN coefficients: every live hit's gradients are NaN
    before = {k: getattr(ds, k).clone() for k in ("means", "quats", "log_scales", "trans_mag_raw", "coeffs")}
    cfg = T.TrainConfig(iterations=30, densify_every=10, prune_every=10, densify_grad_threshold=1e-12)
    with pytest.raises(NonFiniteGradientError):
        T.train_loop(ds, txs, frames, cfg, batch=2, seed=1, check_every=7)
    for k, v in before.items():
        assert torch.equal(getattr(ds, k), v) or (k == "coeffs" and torch.equal(torch.nan_to_num(getattr(ds, k)),
                                                                                  torch.nan_to_num(v))), k


@pytest.mark.gpu
def test_gpu_densify_without_hot_gaussians_keeps_statistics():
    """Nothing above the threshold: densify returns before touching the scene
    or the EMA statistics (reference train.py:184-186, no state.reset())."""
    import torch

    from paper_2502_01826_b200 import raster

    init, txs, frames = _small_fit_setup()
    ds = raster.DeviceScene.from_host(init, "cuda")
    state = T.TrainState(torch.rand(ds.n, device="cuda") * 1e-6, torch.rand((ds.n, 3), device="cuda"))
    ema, last, means = state.grad_ema.clone(), state.last_dmean.clone(), ds.means.clone()
    rep = T.densify(ds, state, 10, T.TrainConfig(densify_grad_threshold=1.0, densify_radius_threshold=1e9))
    assert not rep.cloned and not rep.split
    assert torch.equal(state.grad_ema, ema) and torch.equal(state.last_dmean, last) and torch.equal(ds.means, means)


@pytest.mark.gpu
def test_gpu_train_loop_csi_subcarrier():
    """CSI targets [S, 26] train on config.csi_subcarrier (train.py:282)."""
    import torch

    from paper_2502_01826_b200 import raster

    init, txs, _ = _small_fit_setup()
    tg = (torch.randn((txs.shape[0], 26), device="cuda") + 1j * torch.randn((txs.shape[0], 26), device="cuda"))
    tg = tg.to(torch.complex64)
    out = {}
    for sub in (0, 7):
        ds = raster.DeviceScene.from_host(init, "cuda")
        cfg = T.TrainConfig(iterations=3, csi_subcarrier=sub, lr_transmittance=1e-7, lr_radiance=1e-7,
                            lr_scale=1e-7, lr_rotation=1e-7, lr_mean_start=1e-7, lr_mean_end=1e-8)
        trace, _, _ = T.train_loop(ds, txs, tg, cfg, batch=2, seed=4, mode="csi")
        ds1 = raster.DeviceScene.from_host(init, "cuda")
        trace1, _, _ = T.train_loop(ds1, txs, tg[:, sub].contiguous(), cfg, batch=2, seed=4, mode="csi")
        assert [r.total for r in trace] == [r.total for r in trace1]
        out[sub] = trace[0].total
    assert out[0] != out[7]
    with pytest.raises(ConfigError):
        T.train_loop(raster.DeviceScene.from_host(init, "cuda"), txs, tg, T.TrainConfig(iterations=1, csi_subcarrier=26),
                     mode="csi")


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["spectrum", "rssi"])
def test_gpu_train_loop_captured_matches_eager(mode):
    """The captured training iteration (CUDA graph replays, samples and
    learning rate indexed on the device) gives bitwise the eager loop's trace,
    density decisions and scene -- including a rewind: the first capture is
    made with a too-small hit capacity, its replay overflows, the loop redoes
    that iteration eagerly and captures again."""
    import torch

    from paper_2502_01826_b200 import raster

    init, txs, frames = _small_fit_setup(12)
    if mode == "rssi":
        frames = 10 * torch.log10(frames.sum((1, 2)) + 1e-3) - 30
    cfg = T.TrainConfig(iterations=40, densify_every=10, prune_every=15, densify_grad_threshold=1e-9)
    out = {}
    for g in (False, True):
        shrink = {"left": 1}

        def hook():
            if shrink["left"]:
                shrink["left"] -= 1
                for k in raster._CAPS["h_cap"]:
                    raster._CAPS["h_cap"][k] = 64
        T._LOOP_HOOKS["before_capture"] = hook
        try:
            ds = raster.DeviceScene.from_host(init, "cuda")
            tim = []
            trace, dens, pr = T.train_loop(ds, txs, frames, cfg, batch=3, seed=7, timings=tim, mode=mode,
                                           check_every=9, graph=g)
        finally:
            T._LOOP_HOOKS.pop("before_capture", None)
        out[g] = (trace, dens, pr, ds, dict(T.train_loop.last_counts), tim)
    (t0, d0, p0, s0, c0, _), (t1, d1, p1, s1, c1, tim1) = out[False], out[True]
    assert c0["replays"] == 0
    assert c1["replays"] >= 20 and c1["rewinds"] >= 1 and c1["captures"] >= 2, c1
    assert [(r.iteration, r.total, r.n_primitives) for r in t0] == [(r.iteration, r.total, r.n_primitives) for r in t1]
    assert [(i, r.cloned, r.split) for i, r in d0] == [(i, r.cloned, r.split) for i, r in d1]
    assert [(i, r.removed) for i, r in p0] == [(i, r.removed) for i, r in p1]
    for k in ("means", "quats", "log_scales", "trans_mag_raw", "trans_phase", "coeffs"):
        assert torch.equal(getattr(s0, k), getattr(s1, k)), k
    assert [t[0] for t in tim1] == list(range(1, 41))
