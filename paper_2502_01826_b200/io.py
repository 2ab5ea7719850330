"""Dataset and checkpoint formats of the reference (io.py:1-310), plus device loading.

Byte-compatible with the reference: a dataset is `manifest.json` plus one
little-endian float32 payload file per sample (spectrum: row-major n_az x n_el;
rssi: one value; csi: 26 interleaved (re, im) pairs); a checkpoint is one JSON
document with every primitive attribute at full float64 precision (shortest
round-trip repr), a config echo and the iteration -- save / load / save gives
byte-identical files, version mismatches raise DataError.

B200 addition: `load_dataset_device` reads every spectrum payload straight into
one pinned host buffer and moves the whole dataset to HBM with a single copy
(TX positions [S, 3] and frames [S, n_az, n_el] float32), the layout
`train.train_loop` draws its batches from; `checkpoint_from_device` /
`device_scene_from_checkpoint` connect checkpoints with raster.DeviceScene.
"""

from __future__ import annotations

import dataclasses
import json
import os
from dataclasses import dataclass

import numpy as np

from .errors import DataError

__all__ = [
    "DATASET_VERSION", "CHECKPOINT_VERSION", "CSI_SUBCARRIERS", "TrainSample", "Dataset", "write_dataset",
    "load_dataset", "load_dataset_device", "save_checkpoint", "load_checkpoint", "checkpoint_path",
    "write_trace_csv", "config_to_dict", "CheckpointScene", "checkpoint_from_device", "device_scene_from_checkpoint",
]

DATASET_VERSION = 1
CHECKPOINT_VERSION = 1
CSI_SUBCARRIERS = 26
_MODES = ("spectrum", "rssi", "csi")


@dataclass
class TrainSample:
    """io.TrainSample (io.py:81-91)."""

    id: str
    tx: np.ndarray
    payload: object
    mode: str

    def __post_init__(self):
        self.tx = np.asarray(self.tx, dtype=np.float64).reshape(3)


@dataclass
class Dataset:
    """io.Dataset (io.py:94-111)."""

    mode: str
    rx: np.ndarray
    n_az: int
    n_el: int
    carrier_freq: float
    samples: list

    def __post_init__(self):
        self.rx = np.asarray(self.rx, dtype=np.float64).reshape(3)

    def check_mode(self) -> None:
        bad = [s.id for s in self.samples if s.mode != self.mode]
        if bad:
            raise DataError(f"samples with inconsistent mode: {bad[:5]}")


def _payload_bytes(sample: TrainSample) -> bytes:
    if sample.mode == "spectrum":
        return np.asarray(sample.payload, dtype="<f4").tobytes(order="C")
    if sample.mode == "rssi":
        return np.asarray([sample.payload], dtype="<f4").tobytes()
    if sample.mode == "csi":
        vec = np.asarray(sample.payload, dtype=np.complex128).reshape(-1)
        inter = np.empty(2 * vec.size, dtype="<f4")
        inter[0::2] = vec.real
        inter[1::2] = vec.imag
        return inter.tobytes()
    raise DataError(f"unknown sample mode {sample.mode!r}")


def _expected_values(mode: str, n_az: int, n_el: int) -> int:
    return {"spectrum": n_az * n_el, "rssi": 1, "csi": 2 * CSI_SUBCARRIERS}[mode]


def _payload_from_bytes(raw: bytes, mode: str, n_az: int, n_el: int, path: str):
    data = np.frombuffer(raw, dtype="<f4")
    want = _expected_values(mode, n_az, n_el)
    if data.size != want:
        unit = "value" if want == 1 else "values"
        raise DataError(f"{path}: expected {want} float32 {unit}, found {data.size}")
    if mode == "spectrum":
        return data.reshape(n_az, n_el).astype(np.float64)
    if mode == "rssi":
        return float(data[0])
    return (data[0::2] + 1j * data[1::2]).astype(np.complex128)


def write_dataset(directory, dataset: Dataset) -> None:
    """Write manifest.json plus one payload file per sample (io.py:147-167)."""
    os.makedirs(directory, exist_ok=True)
    entries = []
    for sample in dataset.samples:
        name = f"{sample.id}.bin"
        with open(os.path.join(directory, name), "wb") as f:
            f.write(_payload_bytes(sample))
        entries.append({"id": sample.id, "tx": sample.tx.tolist(), "payload": name})
    manifest = {
        "format_version": DATASET_VERSION, "mode": dataset.mode, "n_az": dataset.n_az, "n_el": dataset.n_el,
        "carrier_freq": float(dataset.carrier_freq), "rx": dataset.rx.tolist(), "samples": entries,
    }
    with open(os.path.join(directory, "manifest.json"), "w", encoding="utf-8") as f:
        json.dump(manifest, f, indent=1)
        f.write("\n")


def _validate_manifest(m) -> None:
    """The checks of MANIFEST_SCHEMA (io.py:47-78), reported with their JSON path."""
    if not isinstance(m, dict):
        raise DataError("manifest invalid at $: not an object")
    for key in ("format_version", "mode", "n_az", "n_el", "carrier_freq", "rx", "samples"):
        if key not in m:
            raise DataError(f"manifest invalid at $: '{key}' is a required property")
    num = lambda x: isinstance(x, (int, float)) and not isinstance(x, bool)
    integer = lambda x: isinstance(x, int) and not isinstance(x, bool)
    if not integer(m["format_version"]):
        raise DataError("manifest invalid at $.format_version: not an integer")
    if m["mode"] not in _MODES:
        raise DataError(f"manifest invalid at $.mode: {m['mode']!r} is not one of {list(_MODES)}")
    for key, hi in (("n_az", 360), ("n_el", 180)):
        if not integer(m[key]) or not 1 <= m[key] <= hi:
            raise DataError(f"manifest invalid at $.{key}: must be an integer in [1, {hi}]")
    if not num(m["carrier_freq"]) or not m["carrier_freq"] > 0:
        raise DataError("manifest invalid at $.carrier_freq: must be a number > 0")
    if not isinstance(m["rx"], list) or len(m["rx"]) != 3 or not all(num(x) for x in m["rx"]):
        raise DataError("manifest invalid at $.rx: must be an array of 3 numbers")
    if not isinstance(m["samples"], list):
        raise DataError("manifest invalid at $.samples: not an array")
    for i, e in enumerate(m["samples"]):
        if not isinstance(e, dict):
            raise DataError(f"manifest invalid at $.samples[{i}]: not an object")
        for key in ("id", "tx", "payload"):
            if key not in e:
                raise DataError(f"manifest invalid at $.samples[{i}]: '{key}' is a required property")
        if not isinstance(e["id"], str) or not isinstance(e["payload"], str):
            raise DataError(f"manifest invalid at $.samples[{i}]: id and payload must be strings")
        if not isinstance(e["tx"], list) or len(e["tx"]) != 3 or not all(num(x) for x in e["tx"]):
            raise DataError(f"manifest invalid at $.samples[{i}].tx: must be an array of 3 numbers")


def _read_manifest(directory):
    path = os.path.join(directory, "manifest.json")
    if not os.path.exists(path):
        raise DataError(f"no manifest.json in {directory}")
    with open(path, encoding="utf-8") as f:
        manifest = json.load(f)
    _validate_manifest(manifest)
    if manifest["format_version"] != DATASET_VERSION:
        raise DataError(f"dataset format version {manifest['format_version']} is not {DATASET_VERSION}; "
                        "refusing to guess")
    return manifest


def load_dataset(directory) -> Dataset:
    """Load and validate a dataset directory (io.py:183-212)."""
    m = _read_manifest(directory)
    samples = []
    for e in m["samples"]:
        path = os.path.join(directory, e["payload"])
        if not os.path.exists(path):
            raise DataError(f"payload file missing: {path}")
        with open(path, "rb") as f:
            samples.append(TrainSample(e["id"], e["tx"], _payload_from_bytes(f.read(), m["mode"], m["n_az"],
                                                                             m["n_el"], path), m["mode"]))
    return Dataset(m["mode"], m["rx"], m["n_az"], m["n_el"], m["carrier_freq"], samples)


def load_dataset_device(directory, device="cuda"):
    """A dataset straight into HBM for train.train_loop.

    Returns (txs float32 [S, 3], targets, meta): targets are float32
    [S, n_az, n_el] power frames ('spectrum'), float32 [S] dBm ('rssi') or
    complex64 [S, 26] ('csi').  Payloads are read into one pinned buffer and
    copied with a single transfer.
    """
    import torch

    m = _read_manifest(directory)
    mode, n_az, n_el = m["mode"], m["n_az"], m["n_el"]
    per = _expected_values(mode, n_az, n_el)
    s = len(m["samples"])
    host = torch.empty(s * per, dtype=torch.float32).pin_memory()
    buf = host.numpy()
    for i, e in enumerate(m["samples"]):
        path = os.path.join(directory, e["payload"])
        if not os.path.exists(path):
            raise DataError(f"payload file missing: {path}")
        raw = np.fromfile(path, dtype="<f4")
        if raw.size != per:
            raise DataError(f"{path}: expected {per} float32 values, found {raw.size}")
        buf[i * per:(i + 1) * per] = raw
    txs = torch.as_tensor(np.asarray([e["tx"] for e in m["samples"]], dtype=np.float32).reshape(s, 3), device=device)
    dev = host.to(device, non_blocking=True)
    if mode == "spectrum":
        targets = dev.view(s, n_az, n_el)
    elif mode == "rssi":
        targets = dev.view(s)
    else:
        targets = torch.view_as_complex(dev.view(s, CSI_SUBCARRIERS, 2).contiguous())
    meta = {"mode": mode, "n_az": n_az, "n_el": n_el, "rx": tuple(float(x) for x in m["rx"]),
            "carrier_freq": float(m["carrier_freq"]), "ids": [e["id"] for e in m["samples"]]}
    return txs, targets, meta


def config_to_dict(config) -> dict:
    """Dataclass config to a JSON-ready dict (io.py:215-217)."""
    return dataclasses.asdict(config)


def checkpoint_path(directory, iteration) -> str:
    name = "checkpoint_final.json" if iteration is None else f"checkpoint_{iteration:07d}.json"
    return os.path.join(directory, name)


@dataclass
class CheckpointScene:
    """The scene fields a checkpoint carries (RFScene, scene.py:205-246)."""

    means: np.ndarray
    quats: np.ndarray
    log_scales: np.ndarray
    trans_mag_raw: np.ndarray
    trans_phase: np.ndarray
    coeffs: np.ndarray
    rx: np.ndarray
    ress_radius: float = 1.0
    carrier_freq: float = 2.4e9
    bounds_lo: np.ndarray = None
    bounds_hi: np.ndarray = None
    n_az: int = 360
    n_el: int = 180
    fle_degree: int = 3

    @property
    def n(self) -> int:
        return int(np.asarray(self.means).shape[0])


def save_checkpoint(path, scene, iteration: int, config: dict) -> None:
    """Serialize a scene at full precision, byte-stable (io.py:225-254).

    `scene` is any object with the RFScene fields; the box may be given as
    `bounds` (with .lo / .hi) or `bounds_lo` / `bounds_hi`.
    """
    if getattr(scene, "bounds", None) is not None:
        lo, hi = np.asarray(scene.bounds.lo, np.float64), np.asarray(scene.bounds.hi, np.float64)
    else:
        lo, hi = np.asarray(scene.bounds_lo, np.float64), np.asarray(scene.bounds_hi, np.float64)
    f64 = lambda a: np.asarray(a, dtype=np.float64)
    coeffs = np.asarray(scene.coeffs, dtype=np.complex128)
    doc = {
        "format_version": CHECKPOINT_VERSION,
        "iteration": int(iteration),
        "config": config,
        "scene": {
            "rx": f64(scene.rx).tolist(),
            "ress_radius": float(scene.ress_radius),
            "carrier_freq": float(scene.carrier_freq),
            "bounds": {"lo": lo.tolist(), "hi": hi.tolist()},
            "n_az": int(scene.n_az),
            "n_el": int(scene.n_el),
            "fle_degree": int(scene.fle_degree),
            "primitives": {
                "means": f64(scene.means).tolist(),
                "quats": f64(scene.quats).tolist(),
                "log_scales": f64(scene.log_scales).tolist(),
                "trans_mag_raw": f64(scene.trans_mag_raw).tolist(),
                "trans_phase": f64(scene.trans_phase).tolist(),
                "coeffs_re": coeffs.real.tolist(),
                "coeffs_im": coeffs.imag.tolist(),
            },
        },
    }
    tmp = f"{path}.tmp"
    with open(tmp, "w", encoding="utf-8") as f:
        json.dump(doc, f, indent=1)
        f.write("\n")
    os.replace(tmp, path)


def load_checkpoint(path):
    """Load a checkpoint; returns (CheckpointScene, iteration, config dict) (io.py:257-299)."""
    try:
        with open(path, encoding="utf-8") as f:
            doc = json.load(f)
    except (OSError, json.JSONDecodeError) as e:
        raise DataError(f"cannot read checkpoint {path}: {e}") from e
    version = doc.get("format_version")
    if version != CHECKPOINT_VERSION:
        raise DataError(f"checkpoint format version {version} is not {CHECKPOINT_VERSION}; refusing to coerce")
    sc = doc["scene"]
    p = sc["primitives"]
    n = len(p["means"])
    k = (sc["fle_degree"] + 1) ** 2
    if n == 0:
        coeffs = np.zeros((0, k), dtype=np.complex128)
    else:
        coeffs = np.asarray(p["coeffs_re"], dtype=np.float64) + 1j * np.asarray(p["coeffs_im"], dtype=np.float64)
    a = lambda key, shape: np.asarray(p[key], dtype=np.float64).reshape(shape)
    scene = CheckpointScene(a("means", (n, 3)), a("quats", (n, 4)), a("log_scales", (n, 3)), a("trans_mag_raw", (n,)),
                            a("trans_phase", (n,)), coeffs.reshape(n, k), np.asarray(sc["rx"], np.float64),
                            float(sc["ress_radius"]), float(sc["carrier_freq"]),
                            np.asarray(sc["bounds"]["lo"], np.float64), np.asarray(sc["bounds"]["hi"], np.float64),
                            int(sc["n_az"]), int(sc["n_el"]), int(sc["fle_degree"]))
    return scene, doc["iteration"], doc["config"]


def checkpoint_from_device(ds, carrier_freq: float | None = None, bounds=None) -> CheckpointScene:
    """A raster.DeviceScene (fp32 in HBM) as a checkpointable scene (values widened to float64).

    carrier_freq / bounds default to the scene's own metadata (kept by
    device_scene_from_checkpoint / DeviceScene.from_host), so a checkpoint
    round trip through training keeps them; a scene without them needs both.
    """
    carrier_freq = carrier_freq if carrier_freq is not None else getattr(ds, "carrier_freq", None)
    bounds = bounds if bounds is not None else getattr(ds, "bounds", None)
    if carrier_freq is None or bounds is None:
        raise DataError("checkpoint_from_device: the scene carries no carrier_freq / bounds; pass them")
    c = lambda t: t.detach().cpu().numpy()
    return CheckpointScene(c(ds.means).astype(np.float64), c(ds.quats).astype(np.float64),
                           c(ds.log_scales).astype(np.float64), c(ds.trans_mag_raw).astype(np.float64),
                           c(ds.trans_phase).astype(np.float64), c(ds.coeffs).astype(np.complex128),
                           np.asarray(ds.rx, np.float64), float(ds.ress_radius), float(carrier_freq),
                           np.asarray(bounds[0], np.float64), np.asarray(bounds[1], np.float64), int(ds.n_az),
                           int(ds.n_el), int(ds.fle_degree))


def device_scene_from_checkpoint(scene: CheckpointScene, device="cuda"):
    """Checkpoint scene -> raster.DeviceScene (fp32 parameters in HBM)."""
    from . import raster

    return raster.DeviceScene.from_host(scene, device)


def write_trace_csv(path, trace) -> None:
    """Loss trace as CSV: iter,total,l1,ssim,fourier,n_primitives (io.py:302-310)."""
    with open(path, "w", encoding="utf-8") as f:
        f.write("iter,total,l1,ssim,fourier,n_primitives\n")
        for row in trace:
            f.write(f"{row.iteration},{row.total!r},{row.l1!r},{row.ssim!r},{row.fourier!r},{row.n_primitives}\n")
