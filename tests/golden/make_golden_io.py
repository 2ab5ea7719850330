"""Golden files for the dataset / checkpoint formats, written by the REFERENCE io.py.

    python tests/golden/make_golden_io.py      (build container only)

tests/golden/io/{spectrum,rssi,csi}/ (manifest.json + payloads), checkpoint.json
(a 5-Gaussian scene with a TrainConfig echo) and trace.csv.
"""

from __future__ import annotations

import os
import shutil
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/nb")

from rfsplat import io, train  # noqa: E402
from rfsplat.scene import Box, RFScene  # noqa: E402


def main():
    out = os.path.join(HERE, "io")
    shutil.rmtree(out, ignore_errors=True)
    os.makedirs(out)
    rng = np.random.default_rng(11)
    n_az, n_el = 12, 6
    for mode in ("spectrum", "rssi", "csi"):
        samples = []
        for i in range(3):
            tx = rng.uniform(-8, 8, 3)
            if mode == "spectrum":
                payload = rng.random((n_az, n_el))
            elif mode == "rssi":
                payload = float(rng.uniform(-80, -20))
            else:
                payload = rng.normal(size=26) + 1j * rng.normal(size=26)
            samples.append(io.TrainSample(f"s{i:03d}", tx, payload, mode))
        io.write_dataset(os.path.join(out, mode), io.Dataset(mode, [0.5, -0.25, 1.0], n_az, n_el, 2.4e9, samples))
    n = 5
    q = rng.normal(size=(n, 4))
    scene = RFScene(rng.normal(size=(n, 3)) * 5, q / np.linalg.norm(q, axis=1, keepdims=True),
                    rng.uniform(-2, 0, (n, 3)), rng.normal(size=n), rng.uniform(-3, 3, n),
                    rng.normal(size=(n, 16)) + 1j * rng.normal(size=(n, 16)), np.array([0.5, -0.25, 1.0]), 1.0, 2.4e9,
                    Box([-15] * 3, [15] * 3), n_az, n_el, 3)
    io.save_checkpoint(os.path.join(out, "checkpoint.json"), scene, 1234, io.config_to_dict(train.TrainConfig()))
    rows = [train.TraceRow(i, 0.1 * i + 1e-3, 0.05 * i, 0.2, 3.0 / (i + 1), 5 + i) for i in range(1, 4)]
    io.write_trace_csv(os.path.join(out, "trace.csv"), rows)
    print("wrote", out)


if __name__ == "__main__":
    main()
