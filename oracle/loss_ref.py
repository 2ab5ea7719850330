"""CPU restatement of the reference spectrum loss (test infrastructure only).

Follows /root/reference/pkg/src/rfsplat/loss.py: l1_loss (loss.py:65-72),
the 11-tap sigma-1.5 window (loss.py:75-81), the zero-padded separable blur
(loss.py:87-89, scipy correlate1d mode="constant" restated with numpy),
ssim_loss (loss.py:92-128), fourier_loss (loss.py:131-146, Parseval form),
spectrum_loss (loss.py:149-155) and upstream_to_ray (grad.py:104-120).
fp64 throughout.  Pinned against tests/golden/loss_frames.npz, which the
reference itself produced (tests/golden/make_golden_loss.py).  Only tests/
and bench.py's CPU legs use this module; the product path never does.
"""

from __future__ import annotations

import numpy as np

_K1, _K2, _FLOOR = 0.01, 0.03, 1e-6


def window() -> np.ndarray:
    x = np.arange(-5, 6, dtype=np.float64)
    g = np.exp(-(x * x) / (2.0 * 1.5 ** 2))
    return g / g.sum()


_W = window()


def _corr(a: np.ndarray, axis: int) -> np.ndarray:
    """correlate1d(a, W, axis, mode='constant', cval=0): out[i] = sum_j W[j] a[i + j - 5]."""
    a = np.moveaxis(a, axis, -1)
    pad = np.zeros(a.shape[:-1] + (a.shape[-1] + 10,))
    pad[..., 5:-5] = a
    out = np.zeros_like(a)
    n = a.shape[-1]
    for j in range(11):
        out += _W[j] * pad[..., j:j + n]
    return np.moveaxis(out, -1, axis)


def blur(a: np.ndarray) -> np.ndarray:
    """Axis 0 then axis 1 of the last two dimensions (loss.py:87-89)."""
    return _corr(_corr(a, a.ndim - 2), a.ndim - 1)


def spectrum_loss(pred, gt, w_ssim: float = 0.2, w_fourier: float = 0.2):
    """(total, l1, ssim, fourier, grad_frame) of one frame (loss.py:149-155)."""
    x = np.asarray(pred, dtype=np.float64)
    y = np.asarray(gt, dtype=np.float64)
    d = x - y
    n = d.size
    l1 = float(np.mean(np.abs(d)))
    g1 = np.sign(d) / n
    D = max(float(y.max() - y.min()), _FLOOR)
    c1, c2 = (_K1 * D) ** 2, (_K2 * D) ** 2
    mx, my = blur(x), blur(y)
    vx, vy, wxy = blur(x * x), blur(y * y), blur(x * y)
    a1 = 2.0 * mx * my + c1
    a2 = 2.0 * (wxy - mx * my) + c2
    b1 = mx * mx + my * my + c1
    b2 = (vx - mx * mx) + (vy - my * my) + c2
    s = (a1 * a2) / (b1 * b2)
    ss = 1.0 - float(np.mean(s))
    ds_dmu = 2.0 * my * (a2 - a1) / (b1 * b2) - 2.0 * mx * s * (1.0 / b1 - 1.0 / b2)
    ds_dv = -s / b2
    ds_dw = 2.0 * a1 / (b1 * b2)
    g2 = -(blur(ds_dmu) + blur(ds_dv) * 2.0 * x + blur(ds_dw) * y) / n
    fo = float(np.sum(d * d))
    g3 = 2.0 * d
    w1 = 1.0 - w_ssim - w_fourier
    return w1 * l1 + w_ssim * ss + w_fourier * fo, l1, ss, fo, w1 * g1 + w_ssim * g2 + w_fourier * g3


def upstream_to_ray(dL_dpower, s_frame) -> np.ndarray:
    return 2.0 * np.asarray(dL_dpower, np.float64) * np.asarray(s_frame, np.complex128)
