"""Golden vectors for the GPU dataset generator, made by the REFERENCE itself.

    NUMBA_CACHE_DIR=/tmp/nb python tests/golden/make_golden_datagen.py

Runs rfsplat.oracle (oracle.py:100-177) and cli.cmd_generate's TX sampling
(cli.py:82-113) on a few path sets; the GPU generator
(paper_2502_01826_b200/datagen.py) is tested against datagen.npz.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/nb")

from rfsplat import oracle  # noqa: E402

CASES = {
    # name: (paths [(reflector or None, amplitude, extra_phase)], rx, n_az, n_el, sigma_beam, rolloff, n_samples)
    "direct": ([(None, 1.0, 0.0)], [0.0, 0.0, 0.0], 90, 45, 2.0, False, 4),
    "multi": ([(None, 1.0, 0.0), ([4.0, -3.0, 2.5], 0.6, np.pi / 3), ([-6.0, 1.0, -1.0], 0.35, 1.1)],
              [0.5, -0.25, 0.1], 360, 180, 2.0, True, 2),
    "delta": ([(None, 0.8, 0.2), ([2.0, 7.0, 1.0], 0.5, 0.0)], [0.0, 0.0, 0.0], 72, 36, 0.0, False, 3),
    "wide": ([(None, 1.0, 0.0), ([-5.0, -5.0, 0.5], 0.9, 2.0)], [0.0, 0.0, 0.0], 180, 90, 7.5, False, 2),
}


def main():
    z = {}
    for name, (specs, rx, n_az, n_el, sigma, rolloff, n) in CASES.items():
        paths = [oracle.PathSpec(None if r is None else np.asarray(r, float), a, ph) for r, a, ph in specs]
        rng = np.random.default_rng(7)
        txs = np.stack([rng.uniform(np.array([-8.0, -8.0, -3.0]), np.array([8.0, 8.0, 3.0])) for _ in range(n)])
        z[name + "_tx"] = txs
        z[name + "_spec"] = np.stack([oracle.spectrum_oracle(paths, t, rx, 2.4e9, n_az, n_el, sigma, rolloff).data
                                      for t in txs])
        z[name + "_rssi"] = np.array([oracle.rssi_oracle(paths, t, rx, 2.4e9, rolloff) for t in txs])
        z[name + "_csi"] = np.stack([oracle.csi_oracle(paths, t, rx, 2.4e9, rolloff=rolloff) for t in txs])
        z[name + "_sig"] = np.array([oracle.multipath_signal(paths, t, rx, 2.4e9, rolloff) for t in txs])
    # cli.cmd_generate end to end (TX sampling + payload files), spectrum and csi
    import json
    import tempfile
    from types import SimpleNamespace

    from rfsplat import cli, io

    for mode in ("spectrum", "csi", "rssi"):
        gen = {"mode": mode, "n_samples": 5, "n_az": 90, "n_el": 45, "rx": [0.2, 0.1, -0.3],
               "paths": [{"reflector": None, "amplitude": 1.0},
                         {"reflector": [3.0, 4.0, 1.0], "amplitude": 0.7, "extra_phase": 0.4}],
               "sigma_beam": 3.0, "rolloff": True}
        with tempfile.TemporaryDirectory() as d:
            cfg = os.path.join(d, "cfg.json")
            json.dump({"generate": gen}, open(cfg, "w"))
            cli.cmd_generate(SimpleNamespace(config=cfg, seed=11, out=os.path.join(d, "ds")))
            ds = io.load_dataset(os.path.join(d, "ds"))
        z["gen_" + mode + "_cfg"] = np.array(json.dumps(gen))
        z["gen_" + mode + "_tx"] = np.stack([s_.tx for s_ in ds.samples])
        z["gen_" + mode + "_payload"] = np.stack([np.asarray(s_.payload) for s_ in ds.samples])
    np.savez_compressed(os.path.join(HERE, "datagen.npz"), **z)


if __name__ == "__main__":
    main()
