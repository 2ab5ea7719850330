"""Pin the CPU oracle (oracle/) against golden vectors produced by the reference.

CPU-only.  The oracle is the checker for every GPU parity test, so it must
first reproduce the reference's own outputs: the tile index bit for bit, and
frames / gradient buffers to fp64 round-off.
"""

import numpy as np
import pytest

import oracle
from helpers import GRAD_KEYS, config1_scene, load, rel_err, scene_from, scene_sha, sha

from paper_2502_01826_b200.scene import bench_scene, round_to_f32


def _check_case(z, prefix, scene, grad_tol=1e-9, tiles=True):
    ctx = oracle.OracleContext(scene, threads=0)
    if tiles:
        np.testing.assert_array_equal(ctx.keys, z[prefix + "keys"])
        np.testing.assert_array_equal(ctx.indices, z[prefix + "indices"])
        np.testing.assert_array_equal(ctx.ranges, z[prefix + "ranges"])
    proj = np.stack([ctx.center_u, ctx.center_v, ctx.radius_px, ctx.tile_radius, ctx.depth, ctx.active.astype(float)], 1)
    np.testing.assert_allclose(proj, z[prefix + "proj"], rtol=1e-12, atol=1e-12)
    ctx.set_tx(z[prefix + "tx"])
    frame = ctx.forward()
    ref = z[prefix + "frame"]
    assert rel_err(frame, ref) < 1e-12
    np.testing.assert_array_equal(ctx.live_counts().ravel(), z[prefix + "live"])
    lam = oracle.l1_upstream(ref)
    g = ctx.backward(lam)
    sel = z[prefix + "grad_sel"]
    for k in GRAD_KEYS:
        r = z[prefix + k]
        a = g[k][sel]
        scale = max(np.abs(r).max(), 1e-300)
        assert np.abs(a - r).max() / scale < grad_tol, k
        np.testing.assert_allclose(g[k].sum(axis=0), z[prefix + k + "_sum"], rtol=1e-8, atol=1e-12 * scale)


def test_kat():
    z = load("kat.npz")
    np.testing.assert_allclose(z["cov_diag"], np.diag([1.0, 4.0, 9.0]), atol=1e-12)
    assert abs(float(z["p20_half"]) + 0.125) < 1e-15
    assert abs(float(z["p11_zero"]) + 1.0) < 1e-15
    np.testing.assert_allclose(z["proj_5_0_0"], [0.0, 90.0, 3 * 180 / (5 * np.pi), 5.0], rtol=1e-12)
    assert int(z["pack_key_3_1"]) == 0x33F800000
    np.testing.assert_allclose(z["upstream_1_3p4j"], [[6 + 8j]])
    np.testing.assert_allclose(z["ray_sphere_10"], [7.0, 13.0])


def test_kat_projection_through_oracle():
    """project_gaussian((5,0,0), I) through the oracle's vectorized projection."""
    from paper_2502_01826_b200.scene import HostScene

    s = HostScene(np.array([[5.0, 0, 0]]), np.array([[1.0, 0, 0, 0]]), np.zeros((1, 3)),
                  np.zeros(1), np.zeros(1), np.zeros((1, 16)), np.zeros(3), 1.0, 360, 180, 3)
    ctx = oracle.OracleContext(s)
    assert ctx.center_u[0] == 0.0 and ctx.center_v[0] == 90.0
    assert abs(ctx.radius_px[0] - 3 * 180 / (5 * np.pi)) < 1e-12
    assert ctx.depth[0] == 5.0


def test_bench_scene_generator_matches_reference():
    z = load("config1_10k.npz")
    assert scene_sha(config1_scene()) == str(z["scene_sha"])


def test_config1_oracle_vs_reference():
    z = load("config1_10k.npz")
    _check_case(z, "", config1_scene())


@pytest.mark.parametrize("i", range(20))
def test_gradcheck_scene_oracle_vs_reference(i):
    z = load("gradcheck_scenes.npz")
    _check_case(z, f"s{i}_", scene_from(z, f"s{i}_"))


@pytest.mark.parametrize("prefix", ["cube_", "special_", "hemi_"])
def test_edge_scene_oracle_vs_reference(prefix):
    z = load("edge_scenes.npz")
    _check_case(z, prefix, scene_from(z, prefix))


@pytest.mark.parametrize("n", [100_000, 500_000])
def test_tile_index_hash_large(n):
    z = load("tile_hashes.npz")
    s = round_to_f32(bench_scene(np.random.default_rng(0), n, 360, 180))
    assert scene_sha(s) == str(z[f"n{n}_scene_sha"])
    ctx = oracle.OracleContext(s)
    assert ctx.m == int(z[f"n{n}_m"])
    assert sha(ctx.keys) == str(z[f"n{n}_sha_keys"])
    assert sha(ctx.indices) == str(z[f"n{n}_sha_indices"])
    assert sha(ctx.ranges) == str(z[f"n{n}_sha_ranges"])


def test_tiled_equals_naive():
    """Render equivalence (SPEC.md acceptance #4) on the oracle."""
    s = round_to_f32(bench_scene(np.random.default_rng(4), 400, 360, 90))
    ctx = oracle.OracleContext(s)
    ctx.set_tx([1.0, 2.0, -1.0])
    a = ctx.forward(tiled=True)
    b = ctx.forward(tiled=False)
    np.testing.assert_array_equal(a, b)
