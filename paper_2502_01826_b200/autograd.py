"""`RFSplat`: torch.autograd.Function over the sm_100a rasterizer.

The reference exposes plain functions (render.render_complex_frame,
grad.backward_frame); this Function binds the same forward
and backward to autograd for a TX batch:

    S = RFSplat.apply(means, quats, log_scales, trans_mag_raw, trans_phase,
                      coeffs, rx, tx, n_az, n_el, ress_radius,
                      include_direction_chain)          -> complex64 [B, n_az, n_el]

grad_S arrives as PyTorch's complex gradient dL/dRe S + i dL/dIm S, which is
exactly the reference's packed upstream lambda (grad.py:4-8, 104-120), and
coeffs.grad comes back in the same packing as GradientBuffer.d_coeffs
(grad.py:59-61).  trans_mag_raw receives d|rho| * sigma (1 - sigma), the
logit chain the reference applies in sgd_step (train.py:161-162).  Gradients
are summed over the TX batch (GradientBuffer.add, grad.py:85-92).
"""

from __future__ import annotations

import torch

from . import raster

__all__ = ["RFSplat", "rfsplat"]


class RFSplat(torch.autograd.Function):
    @staticmethod
    def forward(ctx, means, quats, log_scales, trans_mag_raw, trans_phase, coeffs, rx, tx, n_az: int, n_el: int,
                ress_radius: float = 1.0, include_direction_chain: bool = True):
        k = int(coeffs.shape[1])
        degree = int(round(k ** 0.5)) - 1
        rx_t = tuple(float(v) for v in torch.as_tensor(rx, dtype=torch.float64).reshape(3).tolist())
        scene = raster.DeviceScene(
            means.detach().contiguous(), quats.detach().contiguous(), log_scales.detach().contiguous(),
            trans_mag_raw.detach().contiguous(), trans_phase.detach().contiguous(), coeffs.detach().contiguous(),
            rx_t, float(ress_radius), int(n_az), int(n_el), degree,
        )
        txc = tx.detach().to(device=means.device, dtype=torch.float32).contiguous()
        # psi and the composite are queued behind the geometry's two host reads
        geo = raster.build_geometry(scene, psi_tx=txc, index=True, forward=True)
        psi = geo.psi
        S = raster.forward(geo, psi)
        ctx.scene, ctx.geo, ctx.psi, ctx.tx = scene, geo, psi, txc
        ctx.include_direction_chain = bool(include_direction_chain)
        return S

    @staticmethod
    def backward(ctx, grad_S):
        g = raster.backward(ctx.scene, ctx.geo, ctx.tx, grad_S.contiguous(), ctx.include_direction_chain, psi=ctx.psi)
        ctx.last_grads = g
        return (g["d_mean"], g["d_quat"], g["d_log_scale"], g["d_trans_mag_raw"], g["d_trans_phase"], g["d_coeffs"],
                None, None, None, None, None, None)


def rfsplat(means, quats, log_scales, trans_mag_raw, trans_phase, coeffs, rx, tx, n_az=360, n_el=180,
            ress_radius=1.0, include_direction_chain=True):
    """Functional form of RFSplat.apply."""
    return RFSplat.apply(means, quats, log_scales, trans_mag_raw, trans_phase, coeffs, rx, tx, n_az, n_el,
                         ress_radius, include_direction_chain)
