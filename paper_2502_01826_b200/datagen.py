"""Synthetic training data on the GPU: the reference's multipath oracles.

Mirrors rfsplat.oracle (oracle.py:49-177) -- `PathSpec`, `SyntheticScene`,
`path_length`, `multipath_signal`, `spectrum_oracle`, `rssi_oracle`,
`csi_oracle` -- with the per-sample work done by datagen.cu for whole TX
batches, and `generate_dataset`, the batched counterpart of
`cli.cmd_generate` (cli.py:82-113): TX positions drawn exactly as the
reference draws them (numpy default_rng(seed).uniform(lo, hi) per sample, on
the host), the frames computed on the device.  The result is the reference's
`io.Dataset` (byte-compatible through io.write_dataset) or, with
`device=True`, the device tensors the training loop consumes directly.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _native
from .errors import GeometryError

__all__ = ["SPEED_OF_LIGHT", "PathSpec", "SyntheticScene", "path_length", "multipath_signal", "spectrum_oracle",
           "rssi_oracle", "csi_oracle", "spectrum_frames", "rssi_values", "csi_values", "paths_from_config",
           "sample_txs", "generate_dataset"]

SPEED_OF_LIGHT = 3.0e8  # oracle.py:46


@dataclass
class PathSpec:
    """oracle.PathSpec (oracle.py:49-66): direct (reflector None) or single bounce."""

    reflector: np.ndarray | None = None
    amplitude: float = 1.0
    extra_phase: float = 0.0

    def __post_init__(self):
        if self.reflector is not None:
            self.reflector = np.asarray(self.reflector, dtype=np.float64).reshape(3)
        if self.amplitude < 0.0:
            raise ValueError("path amplitude must be non-negative")


@dataclass
class SyntheticScene:
    """oracle.SyntheticScene (oracle.py:69-83)."""

    tx_positions: list
    rx: np.ndarray
    paths: list
    carrier_freq: float = 2.4e9
    rolloff: bool = False

    def __post_init__(self):
        self.rx = np.asarray(self.rx, dtype=np.float64).reshape(3)
        self.tx_positions = [np.asarray(p, dtype=np.float64).reshape(3) for p in self.tx_positions]


def path_length(path: PathSpec, tx, rx) -> float:
    """oracle.path_length (oracle.py:86-99)."""
    tx = np.asarray(tx, dtype=np.float64).reshape(3)
    rx = np.asarray(rx, dtype=np.float64).reshape(3)
    if path.reflector is None:
        d = float(np.linalg.norm(tx - rx))
    else:
        d = float(np.linalg.norm(tx - path.reflector) + np.linalg.norm(path.reflector - rx))
    if d <= 0.0:
        raise GeometryError("zero-length propagation path")
    return d


def _pack_paths(paths, dev) -> torch.Tensor:
    size = int(_native.load().rfs_datagen_path_bytes())
    if size != 48:
        raise RuntimeError(f"unexpected PathRec size {size}")
    buf = np.zeros(len(paths), dtype=[("refl", "<f8", 3), ("amp", "<f8"), ("phase", "<f8"), ("direct", "<i4"),
                                      ("pad", "<i4")])
    for i, p in enumerate(paths):
        if p.reflector is not None:
            buf["refl"][i] = p.reflector
        buf["amp"][i] = p.amplitude
        buf["phase"][i] = p.extra_phase
        buf["direct"][i] = 1 if p.reflector is None else 0
    return torch.as_tensor(buf.view(np.uint8).copy(), device=dev)


def _check(status: torch.Tensor) -> None:
    code = int(status.item())
    if code & 1:
        raise GeometryError("zero-length propagation path")
    if code & 2:
        raise GeometryError("point coincides with the receiver")


def _dev(device):
    return torch.device(device if device is not None else "cuda")


def spectrum_frames(paths, txs, rx, f_c: float, n_az: int, n_el: int, sigma_beam: float = 2.0,
                    rolloff: bool = False, dtype=torch.float32, device=None) -> torch.Tensor:
    """spectrum_oracle for a TX batch [S, 3] -> power frames [S, n_az, n_el] on the device."""
    dev = _dev(device)
    if not paths:
        raise ValueError("at least one path is required")
    tx = torch.as_tensor(np.asarray(txs, dtype=np.float64).reshape(-1, 3), device=dev).contiguous()
    s, p = int(tx.shape[0]), len(paths)
    pk = _pack_paths(paths, dev)
    gain = torch.empty((max(s * p, 1), 2), dtype=torch.float64, device=dev)
    cell = torch.empty((max(s * p, 1), 2), dtype=torch.int32, device=dev)
    out = torch.empty((s, n_az, n_el), dtype=dtype, device=dev)
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    rxa = (C.c_double * 3)(*np.asarray(rx, dtype=np.float64).reshape(3))
    _native.call("rfs_spectrum_dataset", s, tx.data_ptr(), p, pk.data_ptr(), rxa, float(f_c), int(n_az), int(n_el),
                 float(sigma_beam), int(bool(rolloff)), gain.data_ptr(), cell.data_ptr(),
                 out.data_ptr() if dtype == torch.float32 else None,
                 out.data_ptr() if dtype == torch.float64 else None, status.data_ptr(),
                 torch.cuda.current_stream(dev).cuda_stream)
    _check(status)
    return out


def _scalar(paths, txs, rx, f_c, mode, n_sub, spacing, rolloff, device):
    dev = _dev(device)
    tx = torch.as_tensor(np.asarray(txs, dtype=np.float64).reshape(-1, 3), device=dev).contiguous()
    s = int(tx.shape[0])
    pk = _pack_paths(paths, dev)
    rssi = torch.empty(max(s, 1), dtype=torch.float64, device=dev) if mode == 0 else None
    csi = torch.empty((s, n_sub), dtype=torch.complex128, device=dev) if mode == 1 else None
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    rxa = (C.c_double * 3)(*np.asarray(rx, dtype=np.float64).reshape(3))
    _native.call("rfs_scalar_dataset", s, tx.data_ptr(), len(paths), pk.data_ptr(), rxa, float(f_c), mode,
                 int(n_sub), float(spacing), int(bool(rolloff)), rssi.data_ptr() if rssi is not None else None,
                 csi.data_ptr() if csi is not None else None, status.data_ptr(),
                 torch.cuda.current_stream(dev).cuda_stream)
    _check(status)
    return rssi[:s] if mode == 0 else csi


def rssi_values(paths, txs, rx, f_c: float, rolloff: bool = False, device=None) -> torch.Tensor:
    """rssi_oracle for a TX batch -> dBm [S] (float64, device)."""
    return _scalar(paths, txs, rx, f_c, 0, 1, 0.0, rolloff, device)


def csi_values(paths, txs, rx, f_c: float, n_subcarriers: int = 26, spacing: float = 312.5e3,
               rolloff: bool = False, device=None) -> torch.Tensor:
    """csi_oracle for a TX batch -> complex128 [S, n_subcarriers] (device)."""
    return _scalar(paths, txs, rx, f_c, 1, n_subcarriers, spacing, rolloff, device)


def multipath_signal(paths, tx, rx, f_c: float, rolloff: bool = False) -> complex:
    """oracle.multipath_signal (oracle.py:100-108)."""
    return complex(csi_values(paths, [tx], rx, f_c, 1, 0.0, rolloff)[0, 0].item())


def spectrum_oracle(paths, tx, rx, f_c: float, n_az: int, n_el: int, sigma_beam: float = 2.0,
                    rolloff: bool = False):
    """oracle.spectrum_oracle (oracle.py:118-147) -> api.SpectrumFrame."""
    from .api import SpectrumFrame

    return SpectrumFrame(spectrum_frames(paths, [tx], rx, f_c, n_az, n_el, sigma_beam, rolloff,
                                         dtype=torch.float64)[0].cpu().numpy())


def rssi_oracle(paths, tx, rx, f_c: float, rolloff: bool = False) -> float:
    """oracle.rssi_oracle (oracle.py:156-162)."""
    return float(rssi_values(paths, [tx], rx, f_c, rolloff)[0].item())


def csi_oracle(paths, tx, rx, f_c: float, n_subcarriers: int = 26, spacing: float = 312.5e3,
               rolloff: bool = False) -> np.ndarray:
    """oracle.csi_oracle (oracle.py:165-177)."""
    return csi_values(paths, [tx], rx, f_c, n_subcarriers, spacing, rolloff)[0].cpu().numpy()


def paths_from_config(generate: dict) -> list:
    """cli._paths_from_config (cli.py:67-79)."""
    out = []
    for spec in generate.get("paths", [{"reflector": None, "amplitude": 1.0}]):
        refl = spec.get("reflector")
        out.append(PathSpec(None if refl is None else np.asarray(refl, dtype=np.float64),
                            float(spec.get("amplitude", 1.0)), float(spec.get("extra_phase", 0.0))))
    return out


def sample_txs(n: int, tx_box: dict, seed: int) -> np.ndarray:
    """TX positions of cli.cmd_generate (cli.py:93-100): one rng.uniform(lo, hi) per sample."""
    rng = np.random.default_rng(seed)
    lo, hi = np.asarray(tx_box["lo"], dtype=np.float64), np.asarray(tx_box["hi"], dtype=np.float64)
    return np.stack([rng.uniform(lo, hi) for _ in range(n)]) if n else np.zeros((0, 3))


def generate_dataset(generate: dict, seed: int = 0, device: bool = False, dev=None):
    """cli.cmd_generate (cli.py:82-113) with the frames computed on the GPU.

    `generate` is the config's generate section (mode, n_samples, n_az, n_el,
    carrier_freq, rx, tx_box, sigma_beam, rolloff, paths).  TX positions are
    drawn on the host exactly as the reference does (one rng.uniform per
    sample), so the same seed gives the same dataset.  Returns io.Dataset
    (host; float32 payloads as written by the reference), or with device=True
    (txs f32 [S, 3], targets) on the device: spectrum -> f32 [S, n_az, n_el],
    rssi -> f32 [S], csi -> complex64 [S, 26].
    """
    from . import io

    mode = generate.get("mode", "spectrum")
    n = int(generate.get("n_samples", 10))
    n_az, n_el = int(generate.get("n_az", 90)), int(generate.get("n_el", 45))
    f_c = float(generate.get("carrier_freq", 2.4e9))
    rx = np.asarray(generate.get("rx", [0.0, 0.0, 0.0]), dtype=np.float64)
    box = generate.get("tx_box", {"lo": [-8, -8, -3], "hi": [8, 8, 3]})
    sigma_beam = float(generate.get("sigma_beam", 2.0))
    rolloff = bool(generate.get("rolloff", False))
    paths = paths_from_config(generate)
    txs = sample_txs(n, box, seed)
    d = _dev(dev)
    if mode == "spectrum":
        tgt = spectrum_frames(paths, txs, rx, f_c, n_az, n_el, sigma_beam, rolloff, torch.float32, d)
    elif mode == "rssi":
        tgt = rssi_values(paths, txs, rx, f_c, rolloff, d)
    elif mode == "csi":
        tgt = csi_values(paths, txs, rx, f_c, rolloff=rolloff, device=d)
    else:
        from .errors import ConfigError

        raise ConfigError(f"unknown generate mode {mode!r}")
    if device:
        t = tgt.to(torch.complex64) if mode == "csi" else tgt.to(torch.float32)
        return torch.as_tensor(txs, dtype=torch.float32, device=d), t
    host = tgt.cpu().numpy()
    samples = [io.TrainSample(f"sample_{i:05d}", txs[i], host[i], mode) for i in range(n)]
    return io.Dataset(mode, rx, n_az, n_el, f_c, samples)
