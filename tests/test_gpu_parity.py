"""GPU parity: the sm_100a path against the reference-pinned oracle / golden vectors.

Bars (BASELINE.json north_star):
- tile index (keys, indices, ranges): bit-exact;
- live hit counts per ray: exact (fp64 geometry reproduces the hit sets);
- spectra P = |S|^2: normwise rel <= 1e-4 and per-ray |dP| <= 1e-4 * max(P, 1e-3 max P);
- gradients: per class |a-r| / max(|a|, |r|, 1e-3 class_max) <= 1e-3.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle
from helpers import GRAD_KEYS, class_rel, config1_scene, l1_upstream, load, rel_err, scene_from, sha

from paper_2502_01826_b200 import api, raster
from paper_2502_01826_b200.scene import bench_scene, default_txs, random_scene, round_to_f32

pytestmark = pytest.mark.gpu

SPEC_TOL = 1e-4
GRAD_TOL = 1e-3


def _spectrum_ok(S, ref):
    P, Pr = np.abs(S) ** 2, np.abs(ref) ** 2
    assert rel_err(P, Pr) <= SPEC_TOL, rel_err(P, Pr)
    floor = 1e-3 * Pr.max() if Pr.size else 0.0
    bad = np.abs(P - Pr) > SPEC_TOL * np.maximum(Pr, floor) + 1e-30
    assert not bad.any(), f"{bad.sum()} rays outside tolerance"


def _grads_ok(g: api.GradientBuffer, z, prefix, sel=None):
    sel = z[prefix + "grad_sel"] if sel is None else sel
    for k in GRAD_KEYS:
        a = getattr(g, k)[sel]
        r = z[prefix + k]
        e = class_rel(a, r)
        assert e <= GRAD_TOL, (k, e)


# ---------------------------------------------------------------- binning
@pytest.mark.parametrize("backend", ["hand", "cub"])
def test_tile_index_config1_bit_exact(backend):
    z = load("config1_10k.npz")
    t = api.build_tiles_for_render(config1_scene(), sort_backend=backend)
    np.testing.assert_array_equal(t.keys, z["keys"])
    np.testing.assert_array_equal(t.indices, z["indices"])
    np.testing.assert_array_equal(t.ranges, z["ranges"])


@pytest.mark.parametrize("n", [100_000, 500_000])
def test_tile_index_large_bit_exact(n):
    z = load("tile_hashes.npz")
    s = round_to_f32(bench_scene(np.random.default_rng(0), n, 360, 180))
    t = api.build_tiles_for_render(s)
    assert t.keys.size == int(z[f"n{n}_m"])
    assert sha(t.keys) == str(z[f"n{n}_sha_keys"])
    assert sha(t.indices) == str(z[f"n{n}_sha_indices"])
    assert sha(t.ranges) == str(z[f"n{n}_sha_ranges"])


@pytest.mark.parametrize("prefix", ["cube_", "special_", "hemi_"])
def test_tile_index_edge_scenes(prefix):
    z = load("edge_scenes.npz")
    t = api.build_tiles_for_render(scene_from(z, prefix))
    np.testing.assert_array_equal(t.keys, z[prefix + "keys"])
    np.testing.assert_array_equal(t.indices, z[prefix + "indices"])
    np.testing.assert_array_equal(t.ranges, z[prefix + "ranges"])


def test_projection_matches_reference():
    z = load("config1_10k.npz")
    p = api.project_scene(config1_scene())
    got = np.stack([p.center_u, p.center_v, p.radius_px, p.tile_radius, p.depth, p.active.astype(float)], 1)
    np.testing.assert_allclose(got[:, [0, 1, 3, 4, 5]], z["proj"][:, [0, 1, 3, 4, 5]], rtol=1e-12, atol=1e-11)
    np.testing.assert_allclose(got[:, 2], z["proj"][:, 2], rtol=1e-9)


def test_sort_hand_vs_cub_random_keys():
    dev = "cuda"
    rng = np.random.default_rng(3)
    for m in (1, 2, 1000, 4097, 300_000):
        k = rng.integers(0, 1 << 40, m, dtype=np.int64)
        k[rng.integers(0, m, m // 3)] = k[0]  # many ties
        v = np.arange(m, dtype=np.int32)
        kt, vt = torch.as_tensor(k, device=dev), torch.as_tensor(v, device=dev)
        a = raster.sort_pairs(kt.clone(), vt.clone(), 40, "hand")
        b = raster.sort_pairs(kt.clone(), vt.clone(), 40, "cub")
        order = np.argsort(k, kind="stable")
        np.testing.assert_array_equal(a[0].cpu().numpy(), k[order])
        np.testing.assert_array_equal(a[1].cpu().numpy(), v[order])
        np.testing.assert_array_equal(b[1].cpu().numpy(), v[order])


# ---------------------------------------------------------------- hit lists
def test_live_counts_config1_exact():
    z = load("config1_10k.npz")
    ctx = api.prepare_context(config1_scene())
    np.testing.assert_array_equal(ctx.geometry.ray_counts.cpu().numpy(), z["live"])


@pytest.mark.parametrize("n", [100_000])
def test_live_counts_large_vs_oracle(n):
    s = round_to_f32(bench_scene(np.random.default_rng(0), n, 360, 180))
    ctx = api.prepare_context(s)
    oc = oracle.OracleContext(s)
    np.testing.assert_array_equal(ctx.geometry.ray_counts.cpu().numpy(), oc.live_counts().ravel())


# ---------------------------------------------------------------- forward
def test_forward_config1():
    z = load("config1_10k.npz")
    S = api.render_complex_frame(config1_scene(), z["tx"])
    _spectrum_ok(S, z["frame"])


@pytest.mark.parametrize("i", range(20))
def test_forward_gradcheck_scenes(i):
    z = load("gradcheck_scenes.npz")
    S = api.render_complex_frame(scene_from(z, f"s{i}_"), z[f"s{i}_tx"])
    _spectrum_ok(S, z[f"s{i}_frame"])


@pytest.mark.parametrize("prefix", ["cube_", "special_", "hemi_"])
def test_forward_edge_scenes(prefix):
    z = load("edge_scenes.npz")
    S = api.render_complex_frame(scene_from(z, prefix), z[prefix + "tx"])
    _spectrum_ok(S, z[prefix + "frame"])


def test_forward_tx_batch_vs_oracle():
    s = round_to_f32(bench_scene(np.random.default_rng(2), 20_000, 360, 180))
    txs = default_txs(70, seed=5)  # > 64: exercises the second TX block
    S = api.render_complex_frames(s, txs)
    oc = oracle.OracleContext(s)
    for b in (0, 33, 64, 69):
        oc.set_tx(txs[b])
        _spectrum_ok(S[b], oc.forward())


# ---------------------------------------------------------------- backward
def test_backward_config1():
    z = load("config1_10k.npz")
    lam = l1_upstream(z["frame"])
    g = api.backward_frame(config1_scene(), z["tx"], lam)
    _grads_ok(g, z, "")


@pytest.mark.parametrize("i", range(20))
def test_backward_gradcheck_scenes(i):
    z = load("gradcheck_scenes.npz")
    p = f"s{i}_"
    g = api.backward_frame(scene_from(z, p), z[p + "tx"], l1_upstream(z[p + "frame"]))
    _grads_ok(g, z, p)


@pytest.mark.parametrize("prefix", ["cube_", "special_", "hemi_"])
def test_backward_edge_scenes(prefix):
    z = load("edge_scenes.npz")
    g = api.backward_frame(scene_from(z, prefix), z[prefix + "tx"], l1_upstream(z[prefix + "frame"]))
    _grads_ok(g, z, prefix)


def test_backward_deterministic_config1():
    """Atomic-free fixed-order backward: parity, and bitwise identical buffers across runs."""
    z = load("config1_10k.npz")
    lam = l1_upstream(z["frame"])
    s = config1_scene()
    g1 = api.backward_frame(s, z["tx"], lam)
    _grads_ok(g1, z, "")
    g2 = api.backward_frame(s, z["tx"], lam)
    for k in GRAD_KEYS:
        np.testing.assert_array_equal(getattr(g1, k), getattr(g2, k))


def test_backward_multi_launch_batch():
    """A batch wider than one launch (256 TX) accumulates C and d_coeffs across launches."""
    s = round_to_f32(bench_scene(np.random.default_rng(12), 8_000, 180, 90))
    txs = default_txs(300, seed=3)
    rng = np.random.default_rng(0)
    up = (rng.normal(size=(300, 180, 90)) + 1j * rng.normal(size=(300, 180, 90))) * 1e-3
    a = api.backward_frames(s, txs, up)
    d = api.backward_frames(s, txs[:150], up[:150])
    d.add(api.backward_frames(s, txs[150:], up[150:]))
    for k in GRAD_KEYS:
        assert class_rel(getattr(a, k), getattr(d, k)) <= 1e-4, k


def test_backward_tx_batch_is_sum_of_singles():
    """Batch semantics = sum over TX (GradientBuffer.add, grad.py:85-92) vs the oracle."""
    s = round_to_f32(bench_scene(np.random.default_rng(8), 5_000, 180, 90))
    txs = default_txs(5, seed=9)
    oc = oracle.OracleContext(s)
    ups, ref = [], None
    for t in txs:
        oc.set_tx(t)
        lam = l1_upstream(oc.forward())
        ups.append(lam)
        g = oc.backward(lam)
        ref = g if ref is None else {k: ref[k] + g[k] for k in ref}
    got = api.backward_frames(s, txs, np.stack(ups))
    for k in GRAD_KEYS:
        assert class_rel(getattr(got, k), ref[k]) <= GRAD_TOL, k


def test_autograd_matches_backward_frame():
    from paper_2502_01826_b200 import RFSplat

    z = load("gradcheck_scenes.npz")
    s = scene_from(z, "s3_")
    ds = raster.DeviceScene.from_host(s)
    leaves = [t.clone().requires_grad_(True) for t in
              (ds.means, ds.quats, ds.log_scales, ds.trans_mag_raw, ds.trans_phase, ds.coeffs)]
    tx = torch.as_tensor(z["s3_tx"], dtype=torch.float32, device="cuda").reshape(1, 3)
    S = RFSplat.apply(*leaves, torch.tensor(s.rx), tx, s.n_az, s.n_el, s.ress_radius, True)
    P = (S.abs() ** 2)
    loss = (P - (1.3 * P.detach() + 0.05)).abs().mean()
    loss.backward()
    lam = l1_upstream(S.detach().cpu().numpy()[0].astype(np.complex128))
    ref = oracle.backward_frame(s, z["s3_tx"], lam)
    assert class_rel(leaves[0].grad.cpu().numpy(), ref["d_mean"]) <= GRAD_TOL
    assert class_rel(leaves[1].grad.cpu().numpy(), ref["d_quat"]) <= GRAD_TOL
    assert class_rel(leaves[2].grad.cpu().numpy(), ref["d_log_scale"]) <= GRAD_TOL
    sg = 1 / (1 + np.exp(-s.trans_mag_raw))
    assert class_rel(leaves[3].grad.cpu().numpy(), ref["d_trans_mag"] * sg * (1 - sg)) <= GRAD_TOL
    assert class_rel(leaves[4].grad.cpu().numpy(), ref["d_trans_phase"]) <= GRAD_TOL
    assert class_rel(leaves[5].grad.cpu().numpy(), ref["d_coeffs"]) <= GRAD_TOL


def test_geometry_error_raised():
    from paper_2502_01826_b200.errors import GeometryError

    s = round_to_f32(random_scene(np.random.default_rng(0), 5))
    s.means[2] = 0.0
    with pytest.raises(GeometryError):
        api.build_tiles_for_render(s)


def test_empty_scene_renders_zero():
    s = round_to_f32(random_scene(np.random.default_rng(0), 5))
    s.means[:] = [[0.2, 0.1, 0.0]] * 5  # all inside the RESS -> inactive
    S = api.render_complex_frame(s, [1.0, 2.0, 3.0])
    assert np.all(S == 0)
    t = api.build_tiles_for_render(s)
    assert t.keys.size == 0 and np.all(t.ranges == 0)


@pytest.mark.gpu
def test_slow_path_bitwise_equals_ring_path():
    """Rays whose pending ring overflows are redone by the global-memory slow
    path; both must give bitwise the same hit lists (run-to-run determinism
    must not depend on the adaptive ring size) and match the oracle."""
    import torch

    from paper_2502_01826_b200 import raster
    from paper_2502_01826_b200.scene import HostScene, cube_init

    c = cube_init([-15] * 3, [15] * 3, 2.5, 72, 36, c00=1.0)
    rng = np.random.default_rng(4)
    dup = lambda a, eps=0.0: np.concatenate([a, a + eps * rng.normal(size=a.shape)])  # near-duplicates (clones)
    s = round_to_f32(HostScene(dup(c.means, 1e-3), dup(c.quats), dup(c.log_scales), dup(c.trans_mag_raw),
                               dup(c.trans_phase), dup(c.coeffs), c.rx, c.ress_radius, 72, 36, 3))
    ds = raster.DeviceScene.from_host(s, "cuda")
    tx = torch.as_tensor(default_txs(2, seed=3), dtype=torch.float32, device="cuda")
    saved = dict(raster._CAPS)
    try:
        out = {}
        for pc in (16, 64):
            raster._CAPS["pcap"] = pc
            g = raster.build_geometry(ds, psi_tx=tx, forward=True)
            out[pc] = (g.S.cpu().numpy(), g.ray_counts.cpu().numpy(), g.stats[0])
    finally:
        raster._CAPS.update(saved)
    assert out[16][2] > 0 and out[16][2] >= out[64][2]  # the small ring was not enough (slow path taken)
    np.testing.assert_array_equal(out[16][0], out[64][0])
    np.testing.assert_array_equal(out[16][1], out[64][1])
    ref = oracle.render_complex_frame(s, default_txs(2, seed=3)[0])
    P, Pr = np.abs(out[64][0][0]) ** 2, np.abs(ref) ** 2
    assert np.linalg.norm(P - Pr) / np.linalg.norm(Pr) <= 1e-4


@pytest.mark.gpu
def test_full_ring_keeps_smallest_pending_hits():
    """Config-5 geometry (cube_init at 360x180, the receiver inside the cloud),
    opaque Gaussians: rays hold up to 22 pending hits but terminate after 7
    emitted ones.  A full 16-entry ring keeps the 16 smallest (t_mid, g) and
    remembers the smallest dropped hit, so every ray finishes in the ring (no
    slow path): bitwise the hit lists and frames of a 64-entry ring, and the
    oracle's live counts."""
    import torch

    from paper_2502_01826_b200 import raster
    from paper_2502_01826_b200.scene import cube_init

    s = cube_init([-15] * 3, [15] * 3, 0.65, 360, 180)
    s.trans_mag_raw[:] = -2.0
    s = round_to_f32(s)
    ds = raster.DeviceScene.from_host(s, "cuda")
    tx = torch.as_tensor(default_txs(2, seed=3), dtype=torch.float32, device="cuda")
    saved = dict(raster._CAPS)
    try:
        out = {}
        for pc in (16, 64):
            raster._CAPS["pcap"] = pc
            raster._CAPS["ring_evict"] = True
            g = raster.build_geometry(ds, psi_tx=tx, forward=True)
            out[pc] = (g.S.cpu().numpy(), *_hit_lists(g), list(g.stats))
        raster._CAPS["pcap"], raster._CAPS["ring_evict"] = 16, False  # without: the ring overflows
        g = raster.build_geometry(ds, psi_tx=tx, forward=True)
        out["plain"] = (g.S.cpu().numpy(), *_hit_lists(g), list(g.stats))
    finally:
        raster._CAPS.update(saved)
    st16, st64 = out[16][3], out[64][3]
    assert st16[5] == 16 and st64[5] > 16  # the small rings filled up
    assert st16[0] == 0, st16  # ... without sending a ray to the slow path
    assert out["plain"][3][0] > 0.1 * 64800  # (a ring that does not keep them: the slow path)
    for i in range(3):
        np.testing.assert_array_equal(out[16][i], out[64][i])
        np.testing.assert_array_equal(out["plain"][i], out[64][i])
    oc = oracle.OracleContext(s)
    np.testing.assert_array_equal(out[16][1], oc.live_counts().ravel())


@pytest.mark.gpu
def _cone_scene(n: int):
    """n Gaussians within ~3 degrees of one direction: a few tile lists of ~n
    entries (beyond the 4-CTA cluster class: the global-memory passes)."""
    rng = np.random.default_rng(11)
    s = bench_scene(rng, n, 360, 180)
    d = rng.uniform(3.0, 15.0, n)
    az = np.deg2rad(40.0 + rng.uniform(-1.5, 1.5, n))
    el = np.deg2rad(-20.0 + rng.uniform(-1.5, 1.5, n))
    s.means = np.stack([d * np.cos(el) * np.cos(az), d * np.cos(el) * np.sin(az), d * np.sin(el)], axis=1)
    return round_to_f32(s)


@pytest.mark.parametrize("which", ["config1", "cube_", "special_", "hemi_", "bench20k", "bench100k", "bench500k",
                                   "bench1000k", "cone60k"])
def test_bucket_binning_bitwise_equals_radix(which):
    """bucket.cu (per-tile buckets sorted in shared memory) must give bitwise
    the sorted keys, ids, ranges and emission bounds of the radix-sort path
    (K2b + K3 + K4 + K4b), hence the same hit lists and spectra."""
    import torch

    if which == "config1":
        s = config1_scene()
    elif which.endswith("_"):
        s = scene_from(load("edge_scenes.npz"), which)
    elif which == "cone60k":
        s = _cone_scene(60_000)
    else:  # bench500k / 1000k: tile lists beyond one block (the 4-CTA cluster class)
        n = {"bench20k": 20_000, "bench100k": 100_000, "bench500k": 500_000, "bench1000k": 1_000_000}[which]
        s = round_to_f32(bench_scene(np.random.default_rng(7), n, 360, 180))
    ds = raster.DeviceScene.from_host(s, "cuda")
    tx = torch.as_tensor(default_txs(2, seed=9), dtype=torch.float32, device="cuda")
    saved = dict(raster._CAPS)
    out = {}
    try:
        for mode in ("radix", "bucket"):
            raster._CAPS["tile_sort"] = mode
            raster._CAPS["m_cap"] = {}
            raster._CAPS["tile_max"] = {}  # the bucket path even for long lists
            g = raster.build_geometry(ds, psi_tx=tx, forward=True)
            m = g.m
            out[mode] = [g.ckeys[:m].cpu().numpy(), g.vals[:m].cpu().numpy(), g.ranges.cpu().numpy(),
                         g.S.cpu().numpy(), *_hit_lists(g)]
    finally:
        raster._CAPS.update(saved)
    for a, b in zip(out["radix"], out["bucket"]):
        np.testing.assert_array_equal(a, b)
    rg = out["bucket"][2]
    if which in ("bench500k", "bench1000k"):
        assert 12288 < (rg[:, 1] - rg[:, 0]).max() <= 4 * 12288  # the cluster class
    if which == "cone60k":
        assert (rg[:, 1] - rg[:, 0]).max() > 4 * 12288  # the global-memory class


def _huge_gaussian_scene():
    """bench scene + one Gaussian whose 3-sigma ball holds the receiver: it is
    hit by (nearly) every ray: one by-Gaussian segment of ~R hits."""
    s = bench_scene(np.random.default_rng(17), 20_000, 360, 180)
    s.means[0] = [3.0, 0.5, -0.2]
    s.log_scales[0] = np.log([2.5, 2.0, 2.2])
    s.trans_mag_raw[0] = -2.0
    return round_to_f32(s)


@pytest.mark.gpu
def test_two_live_geometries_backward():
    """The early by-Gaussian index lives in buffers reused by the next
    geometry; a backward on an older geometry must rebuild its index, not read
    the newer one's."""
    import torch

    s = round_to_f32(bench_scene(np.random.default_rng(3), 5_000, 72, 36))
    s2 = round_to_f32(bench_scene(np.random.default_rng(4), 5_000, 72, 36))
    ds, ds2 = raster.DeviceScene.from_host(s, "cuda"), raster.DeviceScene.from_host(s2, "cuda")
    tx = torch.as_tensor(default_txs(2, seed=2), dtype=torch.float32, device="cuda")
    for _ in range(2):  # second round: capacities known, the early index path is taken
        g1 = raster.build_geometry(ds, psi_tx=tx, forward=True, index=True)
        lam = (g1.S * 1e-3).contiguous()
        ref = raster.backward(ds, g1, tx, lam, True, psi=g1.psi)
        ref = {k: v.clone() for k, v in ref.items()}
        g1b = raster.build_geometry(ds, psi_tx=tx, forward=True, index=True)
        g2 = raster.build_geometry(ds2, psi_tx=tx, forward=True, index=True)  # reuses the buffers
        out = raster.backward(ds, g1b, tx, lam, True, psi=g1b.psi)
        for k in ref:
            torch.testing.assert_close(out[k], ref[k], rtol=0, atol=0)
        raster.backward(ds2, g2, tx, (g2.S * 1e-3).contiguous(), True, psi=g2.psi)


def _hit_lists(g):
    counts = g.ray_counts.cpu().numpy()
    slab = g.slab.view(-1, g.hcap, 16).cpu().numpy()
    keep = np.arange(g.hcap)[None, :] < counts[:, None]
    return counts, slab[keep]


@pytest.mark.gpu
def test_psi_large_scene_grid():
    """psi for > 262,140 Gaussians (the launch grid must not overflow a 65,535 dimension)
    vs the oracle's directional response (render.py:229-238)."""
    import torch

    s = round_to_f32(bench_scene(np.random.default_rng(21), 300_000, 36, 18))
    ds = raster.DeviceScene.from_host(s, "cuda")
    tx = default_txs(2, seed=4)
    psi = raster.compute_psi(ds, torch.as_tensor(tx, dtype=torch.float32, device="cuda")).cpu().numpy()
    oc = oracle.OracleContext(s)
    oc.set_tx(tx[1])
    ref = oc.psi
    assert np.max(np.abs(psi[:, 1] - ref)) <= 1e-4 * np.max(np.abs(ref))


@pytest.mark.gpu
def test_config4_1m_tile_index_and_spectrum():
    """Config 4 scale (1M Gaussians, 4.77M incidences, tile lists up to 30k,
    pending sets past the small ring): bit-exact tile index and live counts,
    spectrum within the 1e-4 bar, all vs the oracle."""
    s = round_to_f32(bench_scene(np.random.default_rng(0), 1_000_000, 360, 180))
    oc = oracle.OracleContext(s)
    t = api.build_tiles_for_render(s)
    np.testing.assert_array_equal(t.keys, oc.keys)
    np.testing.assert_array_equal(t.indices, oc.indices)
    np.testing.assert_array_equal(t.ranges, oc.ranges)
    tx = np.array([5.0, 3.0, 1.0])
    oc.set_tx(tx)
    ref = oc.forward()
    got = api.render_complex_frame(s, tx)
    P, Pr = np.abs(got) ** 2, np.abs(ref) ** 2
    assert np.linalg.norm(P - Pr) / np.linalg.norm(Pr) <= 1e-4
    ctx = api.prepare_context(s)
    counts, *_ = raster.hit_lists_host(ctx.geometry)
    np.testing.assert_array_equal(counts.reshape(360, 180), oc.live_counts())
