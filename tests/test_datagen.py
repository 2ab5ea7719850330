"""GPU synthetic datasets (paper_2502_01826_b200/datagen.py, datagen.cu) vs the
reference's multipath oracles (oracle.py:100-177) and cli.cmd_generate
(cli.py:82-113), through tests/golden/datagen.npz (made by the reference,
tests/golden/make_golden_datagen.py)."""

import json

import numpy as np
import pytest

from helpers import load

CASES = {
    "direct": ([(None, 1.0, 0.0)], [0.0, 0.0, 0.0], 90, 45, 2.0, False),
    "multi": ([(None, 1.0, 0.0), ([4.0, -3.0, 2.5], 0.6, np.pi / 3), ([-6.0, 1.0, -1.0], 0.35, 1.1)],
              [0.5, -0.25, 0.1], 360, 180, 2.0, True),
    "delta": ([(None, 0.8, 0.2), ([2.0, 7.0, 1.0], 0.5, 0.0)], [0.0, 0.0, 0.0], 72, 36, 0.0, False),
    "wide": ([(None, 1.0, 0.0), ([-5.0, -5.0, 0.5], 0.9, 2.0)], [0.0, 0.0, 0.0], 180, 90, 7.5, False),
}


def _paths(specs):
    from paper_2502_01826_b200.datagen import PathSpec

    return [PathSpec(None if r is None else np.asarray(r, float), a, ph) for r, a, ph in specs]


@pytest.mark.parametrize("mode", ["spectrum", "csi", "rssi"])
def test_tx_sampling_matches_cmd_generate(mode):
    from paper_2502_01826_b200.datagen import sample_txs

    z = load("datagen.npz")
    gen = json.loads(str(z[f"gen_{mode}_cfg"]))
    txs = sample_txs(gen["n_samples"], gen.get("tx_box", {"lo": [-8, -8, -3], "hi": [8, 8, 3]}), 11)
    np.testing.assert_array_equal(txs, z[f"gen_{mode}_tx"])


def test_path_validation():
    from paper_2502_01826_b200.datagen import PathSpec, path_length
    from paper_2502_01826_b200.errors import GeometryError

    with pytest.raises(ValueError):
        PathSpec(None, -1.0)
    with pytest.raises(GeometryError):
        path_length(PathSpec(), [1.0, 2.0, 3.0], [1.0, 2.0, 3.0])
    assert path_length(PathSpec([0.0, 4.0, 0.0]), [3.0, 0.0, 0.0], [0.0, 0.0, 0.0]) == 9.0


@pytest.mark.gpu
@pytest.mark.parametrize("name", list(CASES))
def test_gpu_oracles_match_reference(name):
    from paper_2502_01826_b200 import datagen

    z = load("datagen.npz")
    specs, rx, n_az, n_el, sigma, rolloff = CASES[name]
    paths = _paths(specs)
    txs = z[name + "_tx"]
    spec = datagen.spectrum_frames(paths, txs, rx, 2.4e9, n_az, n_el, sigma, rolloff, dtype=__import__("torch").float64)
    ref = z[name + "_spec"]
    assert np.abs(spec.cpu().numpy() - ref).max() <= 1e-9 * ref.max()
    assert np.abs(datagen.rssi_values(paths, txs, rx, 2.4e9, rolloff).cpu().numpy() - z[name + "_rssi"]).max() <= 1e-9
    csi = datagen.csi_values(paths, txs, rx, 2.4e9, rolloff=rolloff).cpu().numpy()
    assert np.abs(csi - z[name + "_csi"]).max() <= 1e-9 * np.abs(z[name + "_csi"]).max()
    # single-sample drop-ins (oracle.spectrum_oracle / multipath_signal / rssi / csi)
    fr = datagen.spectrum_oracle(paths, txs[0], rx, 2.4e9, n_az, n_el, sigma, rolloff)
    assert fr.data.shape == (n_az, n_el) and np.abs(fr.data - ref[0]).max() <= 1e-9 * ref.max()
    assert abs(datagen.multipath_signal(paths, txs[0], rx, 2.4e9, rolloff) - z[name + "_sig"][0]) <= 1e-9
    assert abs(datagen.rssi_oracle(paths, txs[0], rx, 2.4e9, rolloff) - z[name + "_rssi"][0]) <= 1e-9
    assert np.abs(datagen.csi_oracle(paths, txs[0], rx, 2.4e9, rolloff=rolloff) - z[name + "_csi"][0]).max() <= 1e-9


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["spectrum", "csi", "rssi"])
def test_gpu_generate_dataset_matches_cmd_generate(mode, tmp_path):
    from paper_2502_01826_b200 import datagen, io

    z = load("datagen.npz")
    gen = json.loads(str(z[f"gen_{mode}_cfg"]))
    ds = datagen.generate_dataset(gen, seed=11)
    io.write_dataset(str(tmp_path), ds)  # the reference's on-disk format (float32 payloads)
    back = io.load_dataset(str(tmp_path))
    ref = z[f"gen_{mode}_payload"]
    got = np.stack([np.asarray(s.payload) for s in back.samples])
    np.testing.assert_array_equal(np.stack([s.tx for s in back.samples]), z[f"gen_{mode}_tx"])
    # float32 payloads: equal up to one float32 ulp
    np.testing.assert_allclose(got, ref, rtol=2.5e-7, atol=1e-30)
    txs, tgt = datagen.generate_dataset(gen, seed=11, device=True)
    assert tgt.is_cuda and tgt.shape[0] == gen["n_samples"]
