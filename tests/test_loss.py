"""Spectrum loss (reference loss.py:65-155): oracle pinned to the reference's
golden vectors on CPU; the CUDA loss against them on the GPU."""

import numpy as np
import pytest

import oracle.loss_ref as LR
from helpers import load

CASES = [str(x) for x in load("loss_frames.npz")["names"]]


def _case(name):
    z = load("loss_frames.npz")
    S = z[name + "_S"].astype(np.complex128)
    return S, z[name + "_gt"].astype(np.float64), z[name + "_w"], z[name + "_vals"], z[name + "_grad"]


def _grad_rel(a, r):
    return float(np.max(np.abs(a - r)) / max(np.max(np.abs(r)), 1e-300))


@pytest.mark.parametrize("name", CASES)
def test_oracle_loss_matches_reference(name):
    S, gt, w, vals, grad = _case(name)
    tot, l1, ss, fo, g = LR.spectrum_loss(np.abs(S) ** 2, gt, w[0], w[1])
    np.testing.assert_allclose([tot, l1, ss, fo], vals, rtol=1e-12, atol=1e-15)
    assert _grad_rel(g, grad) < 1e-10


@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
def test_gpu_loss_matches_reference(name):
    import torch

    from paper_2502_01826_b200 import loss

    S, gt, w, vals, grad = _case(name)
    St = torch.as_tensor(S.astype(np.complex64), device="cuda").unsqueeze(0)
    gtt = torch.as_tensor(gt.astype(np.float32), device="cuda").unsqueeze(0)
    rep, lam, g = loss.spectrum_loss_frames(St, gtt, float(w[0]), float(w[1]), want_grad=True)
    rep = rep[0].cpu().numpy()
    # values: fp64 statistics over fp32 power -> ~1e-6 relative
    np.testing.assert_allclose(rep, vals, rtol=2e-5, atol=1e-9)
    assert _grad_rel(g[0].cpu().numpy(), grad) < 1e-4
    lam_ref = 2.0 * grad * S  # upstream_to_ray (grad.py:119)
    assert _grad_rel(lam[0].cpu().numpy(), lam_ref) < 1e-4


@pytest.mark.gpu
def test_gpu_loss_batch_equals_frames_and_reference_api():
    import torch

    from paper_2502_01826_b200 import loss

    names = [n for n in CASES if n.startswith("r72") or n in ("same", "flat")]
    Ss, gts = [], []
    for n in names:
        S, gt, *_ = _case(n)
        Ss.append(S)
        gts.append(gt)
    St = torch.as_tensor(np.stack(Ss).astype(np.complex64), device="cuda")
    gtt = torch.as_tensor(np.stack(gts).astype(np.float32), device="cuda")
    rep, lam, _ = loss.spectrum_loss_frames(St, gtt, 0.2, 0.2)
    for i, n in enumerate(names):
        r1, l1, _ = loss.spectrum_loss_frames(St[i:i + 1], gtt[i:i + 1], 0.2, 0.2)
        np.testing.assert_array_equal(rep[i].cpu().numpy(), r1[0].cpu().numpy())
        np.testing.assert_array_equal(lam[i].cpu().numpy(), l1[0].cpu().numpy())
    # reference-shaped single-frame API (power frame in, LossReport out)
    S, gt, w, vals, grad = _case("r360")
    rep1 = loss.spectrum_loss(np.abs(S) ** 2, gt, float(w[0]), float(w[1]))
    np.testing.assert_allclose([rep1.total, rep1.l1, rep1.ssim, rep1.fourier], vals, rtol=2e-5)
    assert _grad_rel(rep1.grad_frame, grad) < 1e-4
    v, g = loss.l1_loss(np.abs(S) ** 2, gt)
    assert abs(v - vals[1]) <= 1e-5 * vals[1]


@pytest.mark.gpu
def test_gpu_loss_shape_error():
    from paper_2502_01826_b200 import loss
    from paper_2502_01826_b200.errors import ShapeError

    with pytest.raises(ShapeError):
        loss.spectrum_loss(np.zeros((8, 4)), np.zeros((4, 8)))


@pytest.mark.gpu
def test_gpu_train_step_matches_oracle():
    """render -> spectrum loss -> upstream -> backward through api.train_step_host
    vs the oracle chain (train.py:266-281 for a TX batch, gradients summed)."""
    import torch

    import oracle
    from helpers import GRAD_KEYS, class_rel
    from paper_2502_01826_b200 import api, raster
    from paper_2502_01826_b200.scene import bench_scene, default_txs, round_to_f32

    s = round_to_f32(bench_scene(np.random.default_rng(5), 4_000, 90, 45))
    txs = default_txs(3, seed=4)
    oc = oracle.OracleContext(s)
    gts, vals, ref = [], [], None
    rng = np.random.default_rng(1)
    for t in txs:
        oc.set_tx(t)
        S = oc.forward()
        gt = (np.abs(S) ** 2 * rng.uniform(0.5, 1.5, S.shape) + 1e-4).astype(np.float32)
        tot, l1, ss, fo, gframe = LR.spectrum_loss(np.abs(S) ** 2, gt.astype(np.float64))
        vals.append([tot, l1, ss, fo])
        gts.append(gt)
        g = oc.backward(LR.upstream_to_ray(gframe, S))
        ref = g if ref is None else {k: ref[k] + g[k] for k in ref}
    ds = raster.DeviceScene.from_host(s, "cuda")
    txh = torch.as_tensor(txs, dtype=torch.float32).pin_memory()
    gth = torch.as_tensor(np.stack(gts)).pin_memory()
    reph = torch.empty((3, 4), dtype=torch.float64).pin_memory()
    grads, h2d, d2h = api.train_step_host(ds, txh, gth, reph)
    torch.cuda.synchronize()
    np.testing.assert_allclose(reph.numpy(), np.array(vals), rtol=1e-4, atol=1e-9)
    assert h2d == txh.numel() * 4 + gth.numel() * 4 and d2h == 3 * 4 * 8
    for k in GRAD_KEYS:
        a = grads[k].cpu().numpy()
        assert class_rel(a, ref[k]) <= 1e-3, k


@pytest.mark.gpu
def test_gpu_scalar_loss_matches_reference():
    import torch

    from paper_2502_01826_b200 import loss

    z = load("loss_frames.npz")
    for p, g, m, v, u in zip(z["scalar_pred"], z["scalar_gt"], z["scalar_mode"], z["scalar_value"], z["scalar_up"]):
        gt = complex(g) if str(m) == "complex" else float(np.real(g))
        val, up = loss.scalar_loss(complex(p), gt, str(m))
        assert abs(val - v) <= 1e-5 * max(abs(v), 1e-6), (m, val, v)
        assert abs(up - u) <= 1e-4 * max(abs(u), 1e-9), (m, up, u)
    # batched frames: the total is the coherent frame sum, lam is constant per frame
    S = torch.randn(3, 20, 10, dtype=torch.complex64, device="cuda")
    rep, total, lam = loss.scalar_loss_frames(S, torch.tensor([0.1 + 0.2j, -1.0, 2.0j]), "complex")
    np.testing.assert_allclose(total.cpu().numpy(), S.sum(dim=(1, 2)).cpu().numpy(), rtol=1e-5, atol=1e-5)
    ref_up = 2.0 * (S.sum(dim=(1, 2)) - torch.tensor([0.1 + 0.2j, -1.0, 2.0j], device="cuda"))
    np.testing.assert_allclose(lam[:, 7, 3].cpu().numpy(), ref_up.cpu().numpy(), rtol=1e-4, atol=1e-5)
    assert bool((lam == lam[:, :1, :1]).all())
