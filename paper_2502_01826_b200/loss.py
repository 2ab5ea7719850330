"""Spectrum loss on the device, drop-in for the reference's loss.py.

    loss.spectrum_loss(pred, gt, w_ssim, w_fourier) -> LossReport   loss.py:149-155
    loss.l1_loss / ssim_loss / fourier_loss(pred, gt) -> (value, grad) loss.py:65-146

run the hand-written kernels of csrc/loss.cu (rfs_spectrum_loss) on one frame
and return float64 numpy results like the reference.  The batched device
entry point `spectrum_loss_frames(S, gt)` evaluates B frames at once from the
complex frames S of the rasterizer and also returns the chained upstream
lam = 2 dL/dP S (upstream_to_ray, grad.py:104-120) that the backward
consumes; `SpectrumLoss` wraps it as a torch.autograd.Function.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _native
from .errors import ShapeError

__all__ = ["LossReport", "spectrum_loss_frames", "spectrum_loss", "l1_loss", "ssim_loss", "fourier_loss",
           "SpectrumLoss", "scalar_loss_frames", "scalar_loss"]


@dataclass
class LossReport:
    """loss.LossReport (loss.py:49-56)."""

    total: float
    l1: float
    ssim: float
    fourier: float
    grad_frame: np.ndarray


def _ptr(t):
    return None if t is None else t.data_ptr()


def frame_range(gt: torch.Tensor) -> torch.Tensor:
    """Per-frame (min, max) partials of measured power frames gt [B, n_az, n_el]
    (float32, on the device): SSIM's dynamic range (loss.py:108), computed
    ahead of the loss, e.g. right behind the frames' H2D copy on its stream;
    pass it to spectrum_loss_frames(gt_range=...)."""
    b, n_az, n_el = (int(x) for x in gt.shape)
    lib = _native.load()
    out = torch.empty(2 * int(lib.rfs_frame_range_elems(b)), dtype=torch.float32, device=gt.device)
    _native.call("rfs_frame_range", b, n_az, n_el, _ptr(gt), _ptr(out), torch.cuda.current_stream(gt.device).cuda_stream)
    return out


def spectrum_loss_frames(S: torch.Tensor | None, gt: torch.Tensor, w_ssim: float = 0.2, w_fourier: float = 0.2,
                         pred: torch.Tensor | None = None, want_lam: bool = True, want_grad: bool = False,
                         lam_layout: str = "frames", gt_range: torch.Tensor | None = None):
    """Loss of B frames on the device.

    S: complex64 [B, n_az, n_el] (the predicted power is |S|^2) or None with
    `pred` float32 [B, n_az, n_el] given; gt: float32 [B, n_az, n_el].
    Returns (report float64 [B, 4] = total, L1, SSIM, Fourier per frame,
    lam or None, grad float32 [B, n_az, n_el] or None).  lam is complex64
    [B, n_az, n_el] (lam_layout "frames"), or [n_az*n_el, B] ("rays": the
    backward's layout, raster.backward(lamT=...), written directly by the
    loss kernel -- no transpose pass).  `gt_range` (optional): frame_range(gt),
    precomputed.
    """
    if lam_layout not in ("frames", "rays"):
        raise ValueError("lam_layout must be 'frames' or 'rays'")
    ref = S if S is not None else pred
    if ref is None:
        raise ShapeError("spectrum_loss_frames needs S or pred")
    if ref.dim() == 2:
        ref = ref.unsqueeze(0)
    b, n_az, n_el = (int(x) for x in ref.shape)
    dev = ref.device
    gt = gt.reshape(-1, n_az, n_el) if gt.numel() == b * n_az * n_el else gt
    if tuple(gt.shape) != (b, n_az, n_el):
        raise ShapeError(f"frame shapes differ: {tuple(ref.shape)} vs {tuple(gt.shape)}")
    gt = gt.to(device=dev, dtype=torch.float32).contiguous()
    if S is not None:
        S = S.reshape(b, n_az, n_el).to(torch.complex64).contiguous()
        want_lam = bool(want_lam)
    else:
        want_lam = False
    if pred is not None:
        pred = pred.reshape(b, n_az, n_el).to(device=dev, dtype=torch.float32).contiguous()
    report = torch.empty((b, 4), dtype=torch.float64, device=dev)
    rays = lam_layout == "rays"
    lam = None
    if want_lam:
        shape = (n_az * n_el, b) if rays else (b, n_az, n_el)
        lam = torch.empty(shape, dtype=torch.complex64, device=dev)
    grad = torch.empty((b, n_az, n_el), dtype=torch.float32, device=dev) if want_grad else None
    lib = _native.load()
    nbytes = int(lib.rfs_loss_scratch_bytes(b, n_az, n_el))
    scratch = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    _native.call("rfs_spectrum_loss", b, n_az, n_el, _ptr(S), _ptr(pred), _ptr(gt), float(w_ssim), float(w_fourier),
                 _ptr(report), _ptr(grad), None if rays else _ptr(lam), _ptr(lam) if rays else None, _ptr(scratch),
                 nbytes, _ptr(gt_range), torch.cuda.current_stream(dev).cuda_stream)
    return report, lam, grad


def _one(pred, gt, w_ssim, w_fourier):
    pred = np.asarray(pred, dtype=np.float64)
    gt = np.asarray(gt, dtype=np.float64)
    if pred.shape != gt.shape:  # loss.py:59-62
        raise ShapeError(f"frame shapes differ: {pred.shape} vs {gt.shape}")
    if pred.ndim != 2:
        raise ShapeError("frames must be 2-D (n_az, n_el)")
    dev = torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() else None
    if dev is None:
        _native.load()  # raises NativeLibraryError: no CPU fallback
    p = torch.as_tensor(pred, dtype=torch.float32, device=dev)
    g = torch.as_tensor(gt, dtype=torch.float32, device=dev)
    rep, _, grad = spectrum_loss_frames(None, g.unsqueeze(0), w_ssim, w_fourier, pred=p.unsqueeze(0),
                                        want_grad=True)
    r = rep[0].cpu().numpy()
    return r, grad[0].cpu().numpy().astype(np.float64)


def spectrum_loss(pred, gt, w_ssim: float = 0.2, w_fourier: float = 0.2) -> LossReport:
    """loss.spectrum_loss (loss.py:149-155) on the device."""
    r, grad = _one(pred, gt, w_ssim, w_fourier)
    return LossReport(float(r[0]), float(r[1]), float(r[2]), float(r[3]), grad)


def l1_loss(pred, gt):
    """loss.l1_loss (loss.py:65-72)."""
    r, grad = _one(pred, gt, 0.0, 0.0)
    return float(r[1]), grad


def ssim_loss(pred, gt):
    """loss.ssim_loss (loss.py:92-128)."""
    r, grad = _one(pred, gt, 1.0, 0.0)
    return float(r[2]), grad


def fourier_loss(pred, gt):
    """loss.fourier_loss (loss.py:131-146)."""
    r, grad = _one(pred, gt, 0.0, 1.0)
    return float(r[3]), grad


class SpectrumLoss(torch.autograd.Function):
    """Per-frame blended loss of complex frames S [B, n_az, n_el] against power targets.

    forward returns the B per-frame totals (float32); backward returns
    lam * grad_output per frame, lam = 2 dL/dP S -- PyTorch's gradient
    convention for a complex input (dL/dRe S + i dL/dIm S).
    """

    @staticmethod
    def forward(ctx, S, gt, w_ssim: float = 0.2, w_fourier: float = 0.2):
        report, lam, _ = spectrum_loss_frames(S.detach(), gt, w_ssim, w_fourier)
        ctx.save_for_backward(lam)
        return report[:, 0].to(torch.float32)

    @staticmethod
    def backward(ctx, grad_out):
        (lam,) = ctx.saved_tensors
        return lam * grad_out.to(torch.float32).reshape(-1, 1, 1), None, None, None


_SCALAR_MODES = {"complex": 0, "real_power": 1}


def scalar_loss_frames(S: torch.Tensor, target: torch.Tensor, mode: str, want_lam: bool = True):
    """Single-antenna loss of B frames on the device (render_scalar + scalar_loss,
    render.py:301-307, loss.py:158-180; mode 'complex' = CSI, 'real_power' = RSSI dBm).

    S complex64 [B, n_az, n_el]; target complex64 [B] ('complex') or float [B]
    of dBm ('real_power').  Returns (report float64 [B, 4] = (value, value, 0,
    0), total complex64 [B], lam complex64 [B, n_az, n_el] or None) -- lam is
    the per-frame constant upstream of the coherent sum (train.py:288).
    """
    if mode not in _SCALAR_MODES:
        raise ValueError(f"unknown scalar loss mode {mode!r}")
    b, n_az, n_el = (int(x) for x in S.shape)
    dev = S.device
    S = S.to(torch.complex64).contiguous()
    t = torch.as_tensor(target, device=dev).reshape(-1)
    if t.numel() != b:
        raise ShapeError("one scalar target per frame")
    t = t.to(torch.complex64).contiguous()
    report = torch.empty((b, 4), dtype=torch.float64, device=dev)
    total = torch.empty(b, dtype=torch.complex64, device=dev)
    lam = torch.empty((b, n_az, n_el), dtype=torch.complex64, device=dev) if want_lam else None
    _native.call("rfs_scalar_loss", b, n_az * n_el, _SCALAR_MODES[mode], _ptr(S), _ptr(t), _ptr(report), _ptr(total),
                 _ptr(lam), torch.cuda.current_stream(dev).cuda_stream)
    return report, total, lam


def scalar_loss(pred: complex, gt, mode: str):
    """loss.scalar_loss (loss.py:158-180) for one complex prediction, on the device."""
    if mode not in _SCALAR_MODES:
        raise ValueError(f"unknown scalar loss mode {mode!r}")
    dev = torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() else None
    if dev is None:
        _native.load()  # raises NativeLibraryError: no CPU fallback
    S = torch.tensor([[[complex(pred)]]], dtype=torch.complex64, device=dev)
    tgt = complex(gt) if mode == "complex" else complex(float(gt), 0.0)
    rep, total, lam = scalar_loss_frames(S, torch.tensor([tgt], dtype=torch.complex64), mode)
    return float(rep[0, 0]), complex(lam[0, 0, 0].item())
