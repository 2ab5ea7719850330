#!/usr/bin/env python
"""Benchmark: RF spectra/sec (fwd+bwd) at 100k Gaussians on B200 (BASELINE.json).

Workload (config 2 of BASELINE.json): the reference perf
scene cli._bench_scene(default_rng(0), 100_000, 360, 180) rounded to fp32,
a batch of 64 TX per GPU from the default tx box (cli.py:90), and a fixed
synthetic upstream lambda (L1 pattern of gradcheck.py:187).
One step = project + bin + sort + hit lists + psi + composite + backward +
epilogue (+ NCCL all-reduce of the gradient buffer when N > 1); the loss is
not part of the step.  Data: synthetic, random-init scene.

  python bench.py [--gpus N --steps K --warmup W]           # this framework
  python bench.py --impl reference [...]                    # CPU reference arm

The reference arm times the oracle port (oracle/, a C restatement of the
reference's numba/numpy path) on the host cores: the reference package is
pure Python, so there is no compiled `oracle/_ref` to run.
"""

from __future__ import annotations

import argparse
import gc
import json
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = "RF spectra/sec (fwd+bwd) at 100k Gaussians, 1/2/4/8 B200; frac of HBM roofline"
UNIT = "spectra/s"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--gaussians", type=int, default=100_000)
    p.add_argument("--batch", type=int, default=64, help="TX per GPU")
    p.add_argument("--sort", default="hand", choices=["hand", "cub"])
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--deterministic", action="store_true", help="(no-op: the backward is always atomic-free and deterministic)")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--eager", action="store_true", help="time the eager step (no CUDA graph)")
    p.add_argument("--strong", action="store_true",
                   help="strong scaling: --batch TX in total, the ray space (tiles) sharded over the ranks, "
                        "frames and gradients all-reduced (parallel.tile_step); e.g. config 4: --gaussians 1000000")
    p.add_argument("--cpu-sample", type=int, default=32, help="TX in the bounded CPU-baseline sample (~10 s on 16 cores)")
    return p.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def workload(n: int, b: int, rank: int, world: int):
    from paper_2502_01826_b200.scene import bench_scene, default_txs, round_to_f32

    scene = round_to_f32(bench_scene(np.random.default_rng(0), n, 360, 180))
    txs = default_txs(b * world, seed=1)[rank * b:(rank + 1) * b]
    return scene, txs


# ------------------------------------------------------------- clocks
class ClockSampler:
    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = None

    def start(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}", "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax.append(float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        os.unlink(self.path)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# --------------------------------------------------------- algorithmic bytes
def algo_bytes(n: int, m: int, r: int, b: int) -> dict:
    """Per-step algorithmic bytes of SURVEY.md §8(d) (fp32/c64 storage)."""
    return {
        "project": n * (48 + 96),
        "bin": n * 32 + m * 12,
        "sort": m * 24,
        "ranges": m * 8,
        "psi": n * 140 + n * b * 8,
        "forward": m * 68 + n * b * 8 + r * b * 8,
        "backward": r * b * 8 + m * 68 + n * b * 8 + n * (56 + 8 * b),
        "epilogue": n * (8 * b + 56 + 168) + n * 176,
    }


def hitlist_bytes(n: int, used: int, h: int, r: int, b: int) -> dict:
    """Algorithmic bytes per launch of the compositing kernels under the hit-list
    design: H live hits (16 B slab records; the by-Gaussian index
    = 8 B id + 4 B slot + 8 B wT per hit), `used` Gaussians with a live hit (their
    psi / p_acc rows, B complex64 each), R rays (their S / lambda rows)."""
    row = b * 8
    return {
        "K7": h * 16 + used * row + r * row,                        # slab, psi rows, S
        "K8c": h * 20 + used * row + r * row + h * 8 + used * row,  # index, psi, lamT rows, C out, p_acc out
        "K8r": h * 16 + h * 8 + used * 32 + h * 16,                 # slab, C, rho (fp32 + fp64), per-hit scalars out
    }


def load_traffic() -> dict:
    """ncu dram bytes per launch of the compositing kernels (profiles/*_traffic.json, newest)."""
    import glob

    files = sorted(glob.glob(os.path.join(REPO, "profiles", "*_traffic.json")), key=os.path.getmtime)
    if not files:
        return {}
    d = json.load(open(files[-1]))
    d["_source"] = os.path.relpath(files[-1], REPO)
    return d


def peaks() -> dict:
    path = os.path.join(REPO, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        d = json.load(open(path))
        return {"hbm_gbs": float(d["hbm_gbs"]), "source": "measured (MEASURED_PEAKS.json)"}
    return {"hbm_gbs": 6650.0, "source": "fallback (B200_PROFILING.md)"}


# ---------------------------------------------------------------- our arm
def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2502_01826_b200 import _native, api, raster

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    if args.strong:  # every rank takes the whole batch; the rays are sharded
        scene, txs = workload(args.gaussians, args.batch, 0, 1)
    else:
        scene, txs = workload(args.gaussians, args.batch, rank, world)
    ds = raster.DeviceScene.from_host(scene, dev)
    tx = torch.as_tensor(txs, dtype=torch.float32, device=dev)
    B = tx.shape[0]

    from paper_2502_01826_b200 import parallel

    # persistent flat gradient buffer: the backward writes into it, and for N > 1
    # its 44 floats per Gaussian are all-reduced by NCCL in two buckets, the
    # first (d_coeffs) overlapping the rest of the epilogue
    gb = parallel.GradBuffer(ds.n, ds.fle_degree, dev)

    # fixed synthetic upstream: lambda = upstream_to_ray(dL1/dP, S), target 1.3 P + 0.05
    geo = raster.build_geometry(ds, sort_backend=args.sort)
    S0 = raster.forward(geo, raster.compute_psi(ds, tx, geo.used))
    P0 = S0.abs() ** 2
    lam = (2.0 * torch.sign(P0 - (1.3 * P0 + 0.05)) / P0[0].numel() * S0).to(torch.complex64).contiguous()
    gt_frames = (1.3 * P0 + 0.05).to(torch.float32).contiguous()  # measured spectra of the e2e training step
    M, H = geo.m, geo.total_hits
    hit_stats = {"max_live": geo.stats[2], "max_tile_list": geo.stats[4], "max_pending": geo.stats[5],
                 "sphere_pass": geo.stats[6], "whitened_pass": geo.stats[7], "slow_rays": geo.stats[0]}
    R = geo.n_rays
    n_used = int(geo.used[: ds.n].sum().item())  # Gaussians with a live hit (rows K7 / K8 touch)

    def hit_stats_after():
        """K6 statistics of a geometry built after the timed steps, with the ring
        size / eviction mode they ran with (the first geometry above starts cold)."""
        g = raster.build_geometry(ds, sort_backend=args.sort)
        return {"max_live": g.stats[2], "max_tile_list": g.stats[4], "max_pending": g.stats[5],
                "sphere_pass": g.stats[6], "whitened_pass": g.stats[7], "slow_rays": g.stats[0],
                "ring": raster._CAPS["pcap"], "ring_keeps_smallest": bool(raster._CAPS["ring_evict"])}
    del S0, P0
    # spectrum loss alone (not part of `value`): timed separately
    from paper_2502_01826_b200 import loss as _loss
    S1 = raster.forward(geo, raster.compute_psi(ds, tx, geo.used))
    for _ in range(3):
        _loss.spectrum_loss_frames(S1, gt_frames)
    torch.cuda.synchronize()
    l0 = torch.cuda.Event(enable_timing=True)
    l1 = torch.cuda.Event(enable_timing=True)
    l0.record()
    for _ in range(5):
        _loss.spectrum_loss_frames(S1, gt_frames)
    l1.record()
    torch.cuda.synchronize()
    loss_ms = l0.elapsed_time(l1) / 5
    del S1

    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)  # > 126 MB L2

    # the upstream enters the backward in the loss kernel's own output layout
    # (ray-major lamT, loss.spectrum_loss_frames(lam_layout="rays")): made once here
    lamT = raster.transpose_upstream(lam)

    sharder = parallel.TileSharder(world, rank)

    def step(marks=None):
        # psi queued behind the M read, the composite behind the hit-statistics read
        if args.strong:
            S, g = parallel.tile_step(ds, tx, lamT, gb, sharder, True, sort_backend=args.sort, marks=marks)
        else:
            S, g = api.fwd_bwd_device(ds, tx, None, True, args.sort, marks, lamT=lamT, grads=gb)
        raster._mark(marks, "allreduce")
        return S, g

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    per_step, phases = [], {}
    launches0 = _native.launch_counter["kernels"]
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    # Steps are enqueued back to back (no host synchronisation between them, as
    # in a training loop): the host runs ahead of the device except at each
    # step's one hit-statistics read.  Each step is bracketed by its own
    # events; the L2 flush between steps sits outside them.
    all_marks = []
    gc.collect()
    gc.disable()  # no collector pauses inside the timed host loops (re-enabled after)
    for _ in range(args.steps):
        flush.fill_(1)  # evict L2 between steps (outside the timed events)
        marks = []
        e0 = torch.cuda.Event(enable_timing=True)
        e0.record()
        marks.append(("start", e0))
        step(marks)
        all_marks.append(marks)
    torch.cuda.synchronize()
    gc.enable()
    for marks in all_marks:
        per_step.append(marks[0][1].elapsed_time(marks[-1][1]))
        for (_, a), (name, bb) in zip(marks[:-1], marks[1:]):
            phases.setdefault(name, []).append(a.elapsed_time(bb))
    launches = (_native.launch_counter["kernels"] - launches0) // args.steps
    eager_ms = float(np.sum(per_step)) / args.steps
    # The steady-state step as one CUDA graph (api.StepGraph: the same kernels,
    # no host work between them, the hit statistics validated after the step).
    # Single process only; `value` is the graph replay if every replay stayed
    # within the capacities, else the eager steps above.
    graph_info = None
    if world == 1 and not args.strong and not args.eager and args.sort == "hand":
        sg = api.StepGraph(ds, tx, lamT, gb, True, args.sort)
        for _ in range(args.warmup):
            sg.replay()
        torch.cuda.synchronize()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        oks = []
        for a, b_ in ev:
            flush.fill_(1)  # evict L2 between steps (outside the timed events)
            a.record()
            sg.set_tx(tx)  # the step's TX batch into the graph's input buffer (device copy, timed)
            sg.replay()
            b_.record()
        torch.cuda.synchronize()
        oks.append(sg.ok())
        g_ms = float(np.mean([a.elapsed_time(b_) for a, b_ in ev]))
        graph_info = {"ms_per_step": round(g_ms, 4), "valid": all(oks), "eager_ms_per_step": round(eager_ms, 4)}
        if all(oks):
            per_step = [a.elapsed_time(b_) for a, b_ in ev]
            launches = launches  # the same kernels per replay
        del sg
    clk = clocks.stop()
    t_ms = float(np.sum(per_step))
    if world > 1:
        tt = torch.tensor([t_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_ms = float(tt.item())
    ms_per_step = t_ms / args.steps
    value = (1 if args.strong else world) * B * args.steps / (t_ms / 1e3)

    # Roofline of the compositing kernels.  Algorithmic bytes per launch under the
    # hit-list design (every byte a kernel must move at least once --
    # the live-hit slab / by-Gaussian index, each used psi / lambda / p_acc row once,
    # the output), divided by the kernel's own duration: the CUDA events recorded on
    # its stream right before and after it in every timed step (raster._mark).
    # SURVEY.md §8(d)'s model (per-incidence tile gathers, M·68) is reported beside
    # it for comparison.  traffic = ncu dram bytes of the same launch from the
    # committed --set full capture (profiles/*_traffic.json).
    pk = peaks()
    ph_ms = {k: float(np.mean(v)) for k, v in phases.items()}
    traffic = load_traffic()
    hb = hitlist_bytes(ds.n, n_used, H, R, B)
    ab = algo_bytes(ds.n, M, R, B)
    kern = {
        "K7 forward composite (k_forward_v)": (hb["K7"], ph_ms.get("forward"), "k_forward_v", ab["forward"]),
        "K8c backward by Gaussian (k_bwd_gauss_v)": (hb["K8c"], ph_ms.get("bwd_gauss"), "k_bwd_gauss_v", None),
        "K8r backward ray recursion (k_bwd_rays)": (hb["K8r"], ph_ms.get("backward_rays"), "k_bwd_rays", None),
    }
    roof = {}
    for k, (byts, ms, kname, survey) in kern.items():
        if not ms:
            continue
        ach = byts / (ms / 1e3) / 1e9
        roof[k] = {"bound": "hbm", "achieved": round(ach, 1), "peak": pk["hbm_gbs"], "unit": "GB/s",
                   "frac": round(ach / pk["hbm_gbs"], 4), "algo_bytes": int(byts), "ms": round(ms, 4),
                   "traffic": traffic.get(kname)}
        if survey is not None:
            roof[k]["survey_model_bytes"] = int(survey)  # SURVEY §8(d) K7 = M·68 + N·B·8 + R·B·8
    # the dominant HBM-class kernel of the step (largest share of the step)
    dom = max(roof, key=lambda k: roof[k]["ms"])
    rl = dict(roof[dom])
    rl["kernel"] = dom
    rl["peak_source"] = pk["source"]
    rl["traffic_source"] = traffic.get("_source")
    rl["bytes_model"] = "hit-list design, DESIGN.md §4"
    # K6 (hit lists) is the longest single kernel; its bound is fp64 / latency, not HBM
    # (SURVEY.md §8(d)): its algorithmic flops for context
    flops_k6 = 64800 * (765 * 10 + 423 * 60)
    roof["K6 hit lists (k_hits), not HBM-bound"] = {
        "bound": "fp64 / latency", "achieved_tflops": round(flops_k6 / (ph_ms.get("hits", 1) / 1e3) / 1e12, 3),
        "algo_flops": flops_k6, "ms": round(ph_ms.get("hits", 0), 4)}

    # ---- end to end: one training step through the public API (api.train_step_host):
    # TX batch + measured power frames H2D from pinned memory, render, spectrum
    # loss, upstream, backward (+ all-reduce), per-frame loss report D2H -- all
    # inside the timed region; the gradients stay on the device for the optimizer
    e2e = None
    if not args.no_e2e and not args.strong:
        txh = torch.as_tensor(txs, dtype=torch.float32).pin_memory()
        gth = gt_frames.cpu().pin_memory()
        reph = torch.empty((B, 4), dtype=torch.float64).pin_memory()
        for _ in range(max(1, args.warmup)):
            api.train_step_host(ds, txh, gth, reph, sort_backend=args.sort, grads=gb)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        es = torch.cuda.Event(enable_timing=True)
        ee = torch.cuda.Event(enable_timing=True)
        e2e_step = "eager"
        if world == 1 and not args.eager and args.sort == "hand":
            # the training step as one CUDA graph (api.TrainStepGraph): H2D of the
            # TX batch and the measured frames, render, loss, backward, D2H of the
            # loss report -- all graph nodes, replayed per step
            tg = api.TrainStepGraph(ds, txh, gth, reph, gb, sort_backend=args.sort)
            for _ in range(args.warmup):
                tg.replay()
            torch.cuda.synchronize()
            gc.collect()
            gc.disable()
            es.record()
            for _ in range(args.steps):
                tg.replay()
            ee.record()
            torch.cuda.synchronize()
            gc.enable()
            h2d, d2h = tg.h2d, tg.d2h
            if tg.ok():
                e2e_step = "CUDA graph replay (api.TrainStepGraph)"
            del tg
        if e2e_step == "eager":
            gc.collect()
            gc.disable()
            es.record()
            for _ in range(args.steps):
                _, h2d, d2h = api.train_step_host(ds, txh, gth, reph, sort_backend=args.sort, grads=gb)
            ee.record()
            torch.cuda.synchronize()
            gc.enable()
        te = es.elapsed_time(ee)
        if world > 1:
            tt = torch.tensor([te], device=dev, dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            te = float(tt.item())
        e2e = {"value": round(world * B * args.steps / (te / 1e3), 2), "unit": UNIT,
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h), "ms_per_step": round(te / args.steps, 4),
               "api": "api.train_step_host: TX + target power frames in, loss report out, spectrum loss on device",
               "step": e2e_step,
               "loss": [round(float(x), 6) for x in reph[:, 0].tolist()[:2]]}

        if world == 1:
            # the reference-shaped drop-in call (render_complex_frame + backward_frame
            # for the batch, render.py:282-289, grad.py:192-259): scene, TX and the
            # upstream frames from pinned HOST buffers, frames and every gradient back
            # to HOST buffers, each step (api.fwd_bwd_host) -- the PCIe copies dominate
            hs = api.pinned_host_scene(scene)
            lamh = lam.cpu().pin_memory()
            outh = api.alloc_host_outputs(ds.n, (ds.fle_degree + 1) ** 2, B, 360, 180)
            for _ in range(max(1, args.warmup)):
                api.fwd_bwd_host(hs, txh, lamh, outh, scene.rx, scene.ress_radius, 360, 180, ds.fle_degree)
            torch.cuda.synchronize()
            gc.collect()
            gc.disable()
            es.record()
            for _ in range(args.steps):
                h2d_d, d2h_d = api.fwd_bwd_host(hs, txh, lamh, outh, scene.rx, scene.ress_radius, 360, 180,
                                                ds.fle_degree)
            ee.record()
            torch.cuda.synchronize()
            gc.enable()
            td = es.elapsed_time(ee)
            e2e["dropin"] = {"value": round(B * args.steps / (td / 1e3), 2), "unit": UNIT,
                             "h2d_bytes_per_step": int(h2d_d), "d2h_bytes_per_step": int(d2h_d),
                             "ms_per_step": round(td / args.steps, 4),
                             "api": "api.fwd_bwd_host: scene + TX + upstream frames in, frames + all gradients out "
                                    "(render_complex_frame + backward_frame for the batch, host buffers)"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline(scene, txs[: args.cpu_sample])

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4), "higher_is_better": True,
            "scaling": "strong" if args.strong else "weak", "vs_baseline": None, "dtype": "f32 (fp64 geometry)",
            "data": "synthetic",
            "config": {"workload": (f"{'config 4 strong scaling' if args.strong else 'config 2'}: "
                                    f"{ds.n // 1000}k Gaussians (cli._bench_scene seed 0), 360x180 grid, "
                                    + (f"{B} TX in total" if args.strong else f"{B} TX per GPU") + ", fwd+bwd step"),
                       "gaussians": ds.n, "tx_per_gpu": B // world if args.strong else B,
                       "global_tx": B if args.strong else B * world, "grid": "360x180", "incidences_M": M,
                       "live_hits_H": H,
                       "used_gaussians": n_used,
                       "upstream": "fixed synthetic lambda, given to the backward in the loss kernel's "
                                   "ray-major output layout (made once, outside the timed steps)",
                       "sort": args.sort, "hit_stats": hit_stats_after(),
                       "parallelism": (f"tile-sharded x{world} (rays split by tiles, frames + grads all-reduced)"
                                       if args.strong else f"dp{world} (TX-sharded, grads all-reduced)"),
                       "l2": "flushed between steps (256 MB write)",
                       "step": ("CUDA graph replay of the steady-state step (api.StepGraph); phase_ms / roofline "
                                "from the eager steps" if graph_info and graph_info["valid"] else "eager"),
                       "graph": graph_info},
            "roofline": rl, "kernels_roofline": roof, "phase_ms": {k: round(v, 4) for k, v in ph_ms.items()},
            "loss_ms": round(loss_ms, 4), "e2e": e2e, "cpu_baseline": cpu, "gpu_launches": int(launches), "clocks": clk,
        }
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


# ------------------------------------------------------------ CPU baseline
def cpu_baseline(scene, txs) -> dict:
    """The oracle port (C, OpenMP) on the host cores: per TX the reference's
    behaviour -- rebuild the context (train.py:268), render, backward."""
    import oracle

    threads = os.cpu_count() or 1
    oracle.lib()
    # one warm-up TX (page-in), then the timed sample
    ctx = oracle.OracleContext(scene, threads)
    ctx.set_tx(txs[0])
    t0 = time.perf_counter()
    for t in txs:
        ctx = oracle.OracleContext(scene, threads)
        ctx.set_tx(t)
        S = ctx.forward()
        ctx.backward(oracle.l1_upstream(S))
    dt = time.perf_counter() - t0
    return {"value": round(len(txs) / dt, 4), "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"{len(txs)} TX of config 2 (100k Gaussians, 360x180), context rebuilt per TX, {dt:.1f} s"}


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    import oracle

    scene, txs = workload(args.gaussians, args.batch, 0, 1)
    threads = os.cpu_count() or 1
    oracle.lib()

    def one(t):
        ctx = oracle.OracleContext(scene, threads)
        ctx.set_tx(t)
        S = ctx.forward()
        ctx.backward(oracle.l1_upstream(S))

    for i in range(args.warmup):
        one(txs[i % len(txs)])
    t0 = time.perf_counter()
    for i in range(args.steps):
        one(txs[i % len(txs)])
    dt = time.perf_counter() - t0
    v = args.steps / dt
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": round(v, 4), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(dt / args.steps * 1e3, 2),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "config 2: 100k Gaussians (cli._bench_scene seed 0), 360x180 grid, fwd+bwd, "
                               "1 TX per step (bounded sample of the 64-TX batch)", "gaussians": args.gaussians,
                   "grid": "360x180"},
        "cpu_baseline": {"value": round(v, 4), "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": f"{args.steps} TX, context rebuilt per TX (train.py:268)"},
        "e2e": {"value": round(v, 4), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


def self_launch(args) -> int:
    """`bench.py --gpus N` run directly (no WORLD_SIZE): start N ranks with
    torch.distributed.run on this node (rendezvous on 127.0.0.1) and relay
    rank 0's line; the exit code is the launcher's."""
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


if __name__ == "__main__":
    a = parse()
    if a.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(self_launch(a))
    _, _world, _ = dist_env()
    if _world != a.gpus:
        sys.exit(f"bench.py: --gpus {a.gpus} but WORLD_SIZE={_world}")
    if a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)
