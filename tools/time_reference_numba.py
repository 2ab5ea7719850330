"""Calibration (run in the build container only: it imports the reference
package from /root/reference, which does not travel to the GPU box): the
reference's own CPU path -- numba kernels, render.prepare_context +
render_complex_frame + grad.backward_frame per TX, as BASELINE.md §2
specifies -- on config 2 (100k Gaussians, 360x180), with a per-stage
breakdown, beside the oracle port (oracle/, C + OpenMP, the `--impl
reference` arm of bench.py) on the same TX and cores.  The ratio calibrates
the port against the reference itself.

    NUMBA_CACHE_DIR=/tmp/numba_cache python tools/time_reference_numba.py [n_tx] > profiles/r2_reference_numba.json
"""
import json
import os
import platform
import subprocess
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)

from rfsplat import cli, grad, loss, render  # noqa: E402  (the reference)

import oracle  # noqa: E402  (the port, test infrastructure)
from paper_2502_01826_b200.scene import default_txs  # noqa: E402


def main():
    n_tx = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    workers = os.cpu_count() or 1
    scene = cli._bench_scene(np.random.default_rng(0), 100_000, 360, 180)
    txs = default_txs(n_tx + 1, seed=1)
    # warm-up: numba JIT of every kernel on the first TX
    ctx = render.prepare_context(scene, txs[0])
    S = render.render_complex_frame(scene, txs[0], workers=workers, tiled=True, ctx=ctx)
    P = np.abs(S) ** 2
    lam = grad.upstream_to_ray(loss.spectrum_loss(P, 1.3 * P + 0.05).grad_frame, S)
    grad.backward_frame(scene, txs[0], lam, workers=workers, ctx=ctx)
    stages = {"prepare_context": [], "render_complex_frame": [], "backward_frame": [], "loss (not in the step)": []}
    for tx in txs[1:]:
        t0 = time.perf_counter()
        ctx = render.prepare_context(scene, tx)
        t1 = time.perf_counter()
        S = render.render_complex_frame(scene, tx, workers=workers, tiled=True, ctx=ctx)
        t2 = time.perf_counter()
        P = np.abs(S) ** 2
        rep = loss.spectrum_loss(P, 1.3 * P + 0.05)
        lam = grad.upstream_to_ray(rep.grad_frame, S)
        t3 = time.perf_counter()
        grad.backward_frame(scene, tx, lam, workers=workers, ctx=ctx)
        t4 = time.perf_counter()
        for k, dt in zip(stages, (t1 - t0, t2 - t1, t4 - t3, t3 - t2)):
            stages[k].append(dt)
    med = {k: float(np.median(v)) for k, v in stages.items()}
    step = med["prepare_context"] + med["render_complex_frame"] + med["backward_frame"]
    # the port on the same TX and threads (bench.py's cpu_baseline / --impl reference)
    oracle.lib()
    port = []
    for tx in txs[1:]:
        t0 = time.perf_counter()
        c = oracle.OracleContext(scene, workers)
        c.set_tx(tx)
        Sp = c.forward()
        c.backward(oracle.l1_upstream(Sp))
        port.append(time.perf_counter() - t0)
    port_s = float(np.median(port))
    model = subprocess.run(["bash", "-c", "lscpu | grep 'Model name' | sed 's/.*: *//'"], capture_output=True,
                           text=True).stdout.strip()
    print(json.dumps({
        "what": "reference CPU path (rfsplat numba kernels) vs the oracle port, config 2: 100k Gaussians "
                "(cli._bench_scene seed 0), 360x180, one TX per step as the reference trains (train.py:268-335)",
        "host": {"cpu": model, "nproc": workers, "machine": platform.machine()},
        "numba_workers": workers, "tx_timed": n_tx,
        "reference_stage_median_s": {k: round(v, 4) for k, v in med.items()},
        "reference_spectra_per_s": round(1.0 / step, 4),
        "port_spectra_per_s": round(1.0 / port_s, 4),
        "port_over_reference": round(step / port_s, 2),
    }))


if __name__ == "__main__":
    main()
