"""Small end-to-end driver for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck): every kernel family of the rasterizer path at a size
the sanitizers finish in minutes -- geometry (project, bucket binning,
streaming hit lists incl. the slow path), psi, forward, the early
side-stream by-Gaussian index, backward (paired-TX kernel with straddling
Gaussians, generic kernel), loss with the ray-major upstream, the radix-sort
binning path, a short training loop with densify / prune, and the dataset
generator.

    compute-sanitizer --tool memcheck python tools/sanitize_step.py
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2502_01826_b200 import api, datagen, loss, raster  # noqa: E402
from paper_2502_01826_b200 import train as T  # noqa: E402
from paper_2502_01826_b200.scene import bench_scene, cube_init, default_txs, round_to_f32  # noqa: E402


def main():
    torch.cuda.set_device(0)
    s = bench_scene(np.random.default_rng(17), 4000, 90, 45)
    s.means[0] = [3.0, 0.5, -0.2]  # a Gaussian around the receiver: hits on most rays
    s.log_scales[0] = np.log([2.5, 2.0, 2.2])
    s = round_to_f32(s)
    ds = raster.DeviceScene.from_host(s, "cuda")
    for b in (64, 5):
        tx = torch.as_tensor(default_txs(b, seed=3), dtype=torch.float32, device="cuda")
        lam = (torch.randn((b, 90, 45), device="cuda") + 1j * torch.randn((b, 90, 45), device="cuda")).to(torch.complex64)
        for _ in range(2):  # second: known capacities, early index on the side stream
            S, g = api.fwd_bwd_device(ds, tx, lam)
        rep, lamT, _ = loss.spectrum_loss_frames(S, (S.abs() ** 2 * 1.1).float(), lam_layout="rays")
        if b <= 256:
            api.fwd_bwd_device(ds, tx, None, lamT=lamT)
    raster._CAPS["tile_sort"] = "radix"
    raster.build_geometry(ds, psi_tx=tx, forward=True, index=True)
    raster._CAPS["tile_sort"] = "bucket"
    raster._CAPS["pcap"] = 16
    c = round_to_f32(cube_init([-15] * 3, [15] * 3, 2.5, 72, 36, c00=30.0))
    cds = raster.DeviceScene.from_host(c, "cuda")
    tx8 = torch.as_tensor(default_txs(8, seed=5), dtype=torch.float32, device="cuda")
    frames = (raster.build_geometry(cds, psi_tx=tx8, forward=True).S.abs() ** 2 * 1.2 + 0.01).float()
    T.train_loop(cds, tx8, frames, T.TrainConfig(iterations=6, densify_every=2, prune_every=3,
                                                 densify_grad_threshold=1e-10), batch=4, seed=1)
    datagen.spectrum_frames([datagen.PathSpec(), datagen.PathSpec([3.0, 4.0, 1.0], 0.5, 0.3)],
                            default_txs(4, seed=2), [0, 0, 0], 2.4e9, 90, 45)
    torch.cuda.synchronize()
    print("sanitize_step done")


if __name__ == "__main__":
    main()
