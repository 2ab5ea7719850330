"""Dataset / checkpoint formats vs files written by the reference io.py."""

import filecmp
import os

import numpy as np
import pytest

from helpers import GOLDEN
from paper_2502_01826_b200 import io, train
from paper_2502_01826_b200.errors import DataError

G = os.path.join(GOLDEN, "io")


@pytest.mark.parametrize("mode", ["spectrum", "rssi", "csi"])
def test_dataset_roundtrip_byte_identical(mode, tmp_path):
    ds = io.load_dataset(os.path.join(G, mode))
    assert ds.mode == mode and len(ds.samples) == 3 and ds.n_az == 12 and ds.n_el == 6
    io.write_dataset(str(tmp_path), ds)
    names = sorted(os.listdir(os.path.join(G, mode)))
    assert sorted(os.listdir(tmp_path)) == names
    match, mismatch, errors = filecmp.cmpfiles(os.path.join(G, mode), str(tmp_path), names, shallow=False)
    assert not mismatch and not errors, (mismatch, errors)


def test_dataset_errors(tmp_path):
    import json
    import shutil

    d = tmp_path / "bad"
    shutil.copytree(os.path.join(G, "spectrum"), d)
    m = json.loads((d / "manifest.json").read_text())
    m["n_az"] = 400
    (d / "manifest.json").write_text(json.dumps(m))
    with pytest.raises(DataError, match=r"\$\.n_az"):
        io.load_dataset(str(d))
    m["n_az"] = 12
    m["format_version"] = 2
    (d / "manifest.json").write_text(json.dumps(m))
    with pytest.raises(DataError, match="version"):
        io.load_dataset(str(d))
    m["format_version"] = 1
    (d / "manifest.json").write_text(json.dumps(m))
    (d / "s001.bin").write_bytes(b"\0" * 8)
    with pytest.raises(DataError, match="expected 72 float32 values"):
        io.load_dataset(str(d))
    with pytest.raises(DataError, match="no manifest"):
        io.load_dataset(str(tmp_path))


def test_checkpoint_roundtrip_byte_identical(tmp_path):
    scene, it, cfg = io.load_checkpoint(os.path.join(G, "checkpoint.json"))
    assert it == 1234 and scene.n == 5 and cfg == io.config_to_dict(train.TrainConfig())
    p = tmp_path / "c.json"
    io.save_checkpoint(str(p), scene, it, cfg)
    assert filecmp.cmp(os.path.join(G, "checkpoint.json"), str(p), shallow=False)
    (tmp_path / "v.json").write_text('{"format_version": 9}')
    with pytest.raises(DataError, match="version"):
        io.load_checkpoint(str(tmp_path / "v.json"))
    assert io.checkpoint_path("d", 42).endswith("checkpoint_0000042.json")


def test_trace_csv_identical(tmp_path):
    rows = [train.TraceRow(i, 0.1 * i + 1e-3, 0.05 * i, 0.2, 3.0 / (i + 1), 5 + i) for i in range(1, 4)]
    io.write_trace_csv(str(tmp_path / "t.csv"), rows)
    assert filecmp.cmp(os.path.join(G, "trace.csv"), str(tmp_path / "t.csv"), shallow=False)


@pytest.mark.gpu
def test_dataset_to_device_and_checkpoint_of_device_scene(tmp_path):
    import torch

    from paper_2502_01826_b200 import raster

    txs, frames, meta = io.load_dataset_device(os.path.join(G, "spectrum"), "cuda")
    ref = io.load_dataset(os.path.join(G, "spectrum"))
    np.testing.assert_array_equal(frames.cpu().numpy(), np.stack([s.payload for s in ref.samples]).astype(np.float32))
    np.testing.assert_array_equal(txs.cpu().numpy(), np.stack([s.tx for s in ref.samples]).astype(np.float32))
    _, csi, _ = io.load_dataset_device(os.path.join(G, "csi"), "cuda")
    np.testing.assert_array_equal(csi.cpu().numpy(),
                                  np.stack([s.payload for s in io.load_dataset(os.path.join(G, "csi")).samples])
                                  .astype(np.complex64))
    scene, _, _ = io.load_checkpoint(os.path.join(G, "checkpoint.json"))
    ds = io.device_scene_from_checkpoint(scene)
    assert isinstance(ds, raster.DeviceScene) and ds.n == 5
    back = io.checkpoint_from_device(ds)
    np.testing.assert_array_equal(back.means, scene.means.astype(np.float32).astype(np.float64))
    # the scene metadata survives the device round trip (not replaced by defaults)
    assert back.carrier_freq == scene.carrier_freq
    np.testing.assert_array_equal(back.bounds_lo, scene.bounds_lo)
    np.testing.assert_array_equal(back.bounds_hi, scene.bounds_hi)
    assert torch.cuda.is_available()
