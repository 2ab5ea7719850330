"""Generate golden parity vectors by running the REFERENCE package itself.

Run in the build container only (it imports `rfsplat` from /root/reference,
which does not exist on the GPU box):

    NUMBA_CACHE_DIR=/tmp/nb python tests/golden/make_golden.py

Every scene is rounded to float32-representable values first (SURVEY.md
§8(c) parity protocol), so the fp32-parameter GPU path and the fp64 oracle
see identical inputs.  Outputs are .npz files next to this script; the CPU
test tests/test_oracle_golden.py pins the oracle against them and the GPU
tests pin the CUDA path against them where sizes allow.
"""

from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/nb")

import rfsplat  # noqa: E402
from rfsplat import fle, grad, render, splat  # noqa: E402
from rfsplat.scene import Box, RFScene, covariance  # noqa: E402

from paper_2502_01826_b200.scene import (  # noqa: E402
    HostScene, bench_scene, cube_init, random_scene, round_to_f32,
)

GRAD_KEYS = ("d_mean", "d_quat", "d_log_scale", "d_trans_mag", "d_trans_phase", "d_coeffs", "d_cov")


def to_ref(s: HostScene) -> RFScene:
    return RFScene(
        s.means, s.quats, s.log_scales, s.trans_mag_raw, s.trans_phase, s.coeffs,
        s.rx, s.ress_radius, 2.4e9, Box([-60] * 3, [60] * 3), s.n_az, s.n_el, s.fle_degree,
    )


def scene_arrays(s: HostScene, prefix: str = "") -> dict:
    return {
        prefix + "means": s.means, prefix + "quats": s.quats, prefix + "log_scales": s.log_scales,
        prefix + "trans_mag_raw": s.trans_mag_raw, prefix + "trans_phase": s.trans_phase,
        prefix + "coeffs": s.coeffs, prefix + "rx": s.rx,
        prefix + "cfg": np.array([s.ress_radius, s.n_az, s.n_el, s.fle_degree], np.float64),
    }


def sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def l1_upstream(frame):
    p = np.abs(frame) ** 2
    return grad.upstream_to_ray(np.sign(p - (1.3 * p + 0.05)) / p.size, frame)


def full_case(s: HostScene, tx, prefix: str, grads_subset=None, with_tiles=True) -> dict:
    rs = to_ref(s)
    ctx = render.prepare_context(rs, tx)
    S = render.render_complex_frame(rs, tx, ctx=ctx, workers=8)
    lam = l1_upstream(S)
    buf = grad.backward_frame(rs, tx, lam, ctx=ctx, workers=8)
    counts = np.zeros(s.n_az * s.n_el, np.int64)
    from rfsplat import _kernels
    _kernels.count_hits_tiled(
        ctx.ray_dirs, rs.means, ctx.inv_covs, ctx.norm_consts, ctx.rho,
        ctx.projection.center_u, ctx.projection.center_v, ctx.splat_r2,
        ctx.tiles.indices, ctx.tiles.ranges, ctx.tiles.tiles_u,
        rs.rx, rs.ress_radius, rs.n_az, rs.n_el, counts,
    )
    out = {prefix + "tx": np.asarray(tx, np.float64), prefix + "frame": S, prefix + "live": counts.astype(np.int32)}
    if with_tiles:
        out[prefix + "keys"] = ctx.tiles.keys
        out[prefix + "indices"] = ctx.tiles.indices
        out[prefix + "ranges"] = ctx.tiles.ranges
    p = ctx.projection
    out[prefix + "proj"] = np.stack([p.center_u, p.center_v, p.radius_px, p.tile_radius, p.depth, p.active.astype(float)], 1)
    sel = np.arange(s.n) if grads_subset is None else grads_subset
    out[prefix + "grad_sel"] = sel
    for k in GRAD_KEYS:
        a = getattr(buf, k)
        out[prefix + k] = a[sel]
        out[prefix + k + "_sum"] = np.array(a.sum(axis=0))
    return out


def main():
    os.makedirs(HERE, exist_ok=True)

    # 1. known-answer tests from SPEC.md, evaluated by the reference
    kat = {}
    kat["cov_diag"] = covariance(rfsplat.GaussianPrimitive(
        np.zeros(3), np.array([1.0, 0, 0, 0]), np.array([0.0, np.log(2), np.log(3)]), 0.0, 0.0, np.zeros(16)))
    kat["p20_half"] = np.array(fle.assoc_legendre(2, 0, 0.5))
    kat["p11_zero"] = np.array(fle.assoc_legendre(1, 1, 0.0))
    sp = splat.project_gaussian((5.0, 0.0, 0.0), np.eye(3), np.zeros(3))
    kat["proj_5_0_0"] = np.array([sp.center_u, sp.center_v, sp.radius_px, sp.depth])
    kat["pack_key_3_1"] = np.array(splat.pack_key(3, 1.0), np.uint64)
    kat["upstream_1_3p4j"] = np.array(grad.upstream_to_ray(np.array([[1.0]]), np.array([[3 + 4j]])))
    ray = render.Ray(np.zeros(3), np.array([1.0, 0, 0]))
    kat["ray_sphere_10"] = np.array(render.ray_ellipsoid_intersect(ray, (10.0, 0, 0), np.eye(3)))
    kat["fle_basis_l3"] = fle.fle_basis(0.7, -0.3, 3)
    b, da, db = fle.fle_basis_with_derivs(np.array([0.7, 2.0, 5.5]), np.array([-0.3, 0.0, 1.2]), 3)
    kat["fle_with_derivs"] = np.stack([b, da, db])
    two = splat.build_tiles(
        [splat.Splat2D(0, 392.0 % 360, 24.0, 0.5, 2.0), splat.Splat2D(1, 392.0 % 360, 24.0, 0.5, 1.0)], 360, 180)
    kat["two_splats_keys"] = two.keys
    kat["two_splats_idx"] = two.indices
    np.savez_compressed(os.path.join(HERE, "kat.npz"), **kat)

    # 2. config 1: 10k bench scene, 360x180, tx (5,3,1) -- full tiles + frame
    s10k = round_to_f32(bench_scene(np.random.default_rng(0), 10_000, 360, 180))
    sel = np.sort(np.random.default_rng(7).choice(10_000, 400, replace=False))
    c1 = full_case(s10k, np.array([5.0, 3.0, 1.0]), "", grads_subset=sel)
    c1["scene_sha"] = np.array(sha(*scene_arrays(s10k).values()))
    np.savez_compressed(os.path.join(HERE, "config1_10k.npz"), **c1)

    # 3. gradient-check scenes (gradcheck.py:82-110), 16x8, full buffers
    rng = np.random.default_rng(0)
    gc = {}
    for i in range(20):
        n = int(rng.integers(4, 21))
        s = round_to_f32(random_scene(rng, n))
        tx = rng.uniform(-6.0, 6.0, 3)
        gc.update(scene_arrays(s, f"s{i}_"))
        gc.update(full_case(s, tx, f"s{i}_"))
    np.savez_compressed(os.path.join(HERE, "gradcheck_scenes.npz"), **gc)

    # 4. edge scenes: cube_init (receiver inside ellipsoids -> clamped hits,
    #    inactive primitives), polar / wraparound / inside-RESS splats,
    #    coarse and hemisphere grids with partial tiles
    edge = {}
    cub = round_to_f32(cube_init([-3.0] * 3, [3.0] * 3, 1.0, n_az=90, n_el=45, c00=0.1 + 0.05j))
    rng = np.random.default_rng(3)
    cub.coeffs = (cub.coeffs + (rng.normal(0, 0.05, cub.coeffs.shape) + 1j * rng.normal(0, 0.05, cub.coeffs.shape))
                  ).astype(np.complex64).astype(np.complex128)
    cub.trans_mag_raw = rng.normal(0, 1, cub.n).astype(np.float32).astype(np.float64)
    cub.trans_phase = rng.uniform(-np.pi, np.pi, cub.n).astype(np.float32).astype(np.float64)
    edge.update(scene_arrays(cub, "cube_"))
    edge.update(full_case(cub, np.array([2.0, -1.5, 0.7]), "cube_"))

    sp = bench_scene(np.random.default_rng(11), 300, 72, 18)
    sp.means[0] = [0.0, 0.0, 6.0]     # polar (straight up)
    sp.means[1] = [0.0, 0.0, -4.0]    # polar (straight down)
    sp.means[2] = [0.5, 0.2, 0.1]     # inside the RESS -> inactive
    sp.means[3] = [7.0, -0.05, -2.0]  # azimuth wraparound near 0/360
    sp.means[4] = [1.2, 0.3, -0.4]    # receiver inside its 3-sigma ball
    sp.log_scales[4] = np.log([0.6, 0.5, 0.7])
    sp = round_to_f32(sp)
    edge.update(scene_arrays(sp, "special_"))
    edge.update(full_case(sp, np.array([-3.0, 4.0, -1.0]), "special_"))

    hemi = round_to_f32(bench_scene(np.random.default_rng(5), 2000, 360, 90))
    edge.update(scene_arrays(hemi, "hemi_"))
    edge.update(full_case(hemi, np.array([1.0, -6.0, 2.0]), "hemi_", grads_subset=np.arange(0, 2000, 5)))
    np.savez_compressed(os.path.join(HERE, "edge_scenes.npz"), **edge)

    # 5. binning at config-2 / config-3 scale: hashes of the reference TileIndex
    big = {}
    for n in (100_000, 500_000):
        s = round_to_f32(bench_scene(np.random.default_rng(0), n, 360, 180))
        rs = to_ref(s)
        proj = splat.project_scene(rs)
        t = splat.build_tiles_for_render(rs, proj)
        big[f"n{n}_m"] = np.array(t.keys.size)
        big[f"n{n}_sha_keys"] = np.array(sha(t.keys))
        big[f"n{n}_sha_indices"] = np.array(sha(t.indices))
        big[f"n{n}_sha_ranges"] = np.array(sha(t.ranges))
        big[f"n{n}_scene_sha"] = np.array(sha(*scene_arrays(s).values()))
        print(n, t.keys.size)
    np.savez_compressed(os.path.join(HERE, "tile_hashes.npz"), **big)
    print("golden vectors written to", HERE)


if __name__ == "__main__":
    main()
