import sys, os
sys.path.insert(0, "/root/repo")
import numpy as np, torch
from paper_2502_01826_b200 import raster, train as T, loss as L
from paper_2502_01826_b200.scene import cube_init, default_txs, round_to_f32
init = cube_init([-15] * 3, [15] * 3, 2.5, 72, 36, c00=30.0)
rng = np.random.default_rng(2)
tgt = init.copy()
tgt.means = tgt.means + rng.normal(0, 0.3, tgt.means.shape)
tgt.trans_mag_raw = rng.normal(0, 1, tgt.n)
tgt.coeffs = tgt.coeffs * rng.uniform(0.5, 1.5, (tgt.n, 1)) * np.exp(1j * rng.uniform(-1, 1, (tgt.n, 1)))
tgt = round_to_f32(tgt)
txs = torch.as_tensor(default_txs(16, seed=5), dtype=torch.float32, device="cuda")
tds = raster.DeviceScene.from_host(tgt, "cuda")
geo = raster.build_geometry(tds, psi_tx=txs, forward=True)
frames = (geo.S.abs() ** 2).float().contiguous()
def run(iters):
    ds = raster.DeviceScene.from_host(round_to_f32(init), "cuda")
    cfg = T.TrainConfig(iterations=60, densify_every=10, prune_every=10, densify_grad_threshold=1e-9, lr_radiance=0.05, lr_transmittance=0.05)
    cfg.iterations = 60
    # replicate train_loop but stop at iters
    import types
    trace, d, p = [], [], []
    rng = np.random.default_rng(3)
    state = T.TrainState.zeros(ds.n, "cuda")
    out = []
    for it in range(1, iters + 1):
        idx = torch.as_tensor(rng.integers(16, size=4), device="cuda")
        tx, gt = txs[idx].contiguous(), frames[idx].contiguous()
        g0 = raster.build_geometry(ds, psi_tx=tx, forward=True)
        rep, lam, _ = L.spectrum_loss_frames(g0.S, gt)
        g = raster.backward(ds, g0, tx, lam, True, psi=g0.psi)
        out.append({"S": g0.S.clone(), "lam": lam.clone(), **{k: v.clone() for k, v in g.items()},
                    "means": ds.means.clone(), "quats": ds.quats.clone(), "log_scales": ds.log_scales.clone(),
                    "raw": ds.trans_mag_raw.clone(), "phase": ds.trans_phase.clone(), "coeffs": ds.coeffs.clone(),
                    "ema": state.grad_ema.clone(), "last": state.last_dmean.clone(), "m": g0.m, "h": g0.total_hits, "hcap": g0.hcap})
        T.sgd_step(ds, g, it, cfg, state, check=False)
        if it % 10 == 0 and it < 30:
            T.densify(ds, state, it, cfg, 0)
            T.prune(ds, state, it, cfg)
    return out
a = run(14); b = run(14)
for it, (x, y) in enumerate(zip(a, b), 1):
    diffs = [k for k in x if isinstance(x[k], torch.Tensor) and not torch.equal(x[k], y[k])]
    print(it, "m", x["m"], y["m"], "h", x["h"], y["h"], "hcap", x["hcap"], y["hcap"], "diff:", diffs)


x, y = a[10], b[10]
for k in ("quats", "log_scales", "raw", "phase", "coeffs"):
    d = (x[k] != y[k])
    if d.dim() > 1:
        d = d.any(dim=1)
    idx = torch.nonzero(d).flatten()
    print(k, "rows differing", idx.numel(), idx[:10].tolist(), "n", x[k].shape[0])

# ring vs slow path on the post-densify scene of iteration 10
ds = raster.DeviceScene.from_host(round_to_f32(init), "cuda")
cfg = T.TrainConfig(iterations=60, densify_grad_threshold=1e-9, lr_radiance=0.05, lr_transmittance=0.05)
rng = np.random.default_rng(3)
state = T.TrainState.zeros(ds.n, "cuda")
for it in range(1, 11):
    idx = torch.as_tensor(rng.integers(16, size=4), device="cuda")
    tx, gt = txs[idx].contiguous(), frames[idx].contiguous()
    g0 = raster.build_geometry(ds, psi_tx=tx, forward=True)
    rep, lam, _ = L.spectrum_loss_frames(g0.S, gt)
    g = raster.backward(ds, g0, tx, lam, True, psi=g0.psi)
    T.sgd_step(ds, g, it, cfg, state, check=False)
T.densify(ds, state, 10, cfg, 0)
T.prune(ds, state, 10, cfg)
tx = txs[:4].contiguous()
res = {}
for pc in (16, 32, 64):
    raster._CAPS["pcap"] = pc
    g0 = raster.build_geometry(ds, psi_tx=tx, forward=True)
    print("pcap", pc, "stats", g0.stats, "pcap now", raster._CAPS["pcap"])
    res[pc] = (g0.S.clone(), g0.ray_counts.clone())
for pc in (32, 64):
    print(pc, "S equal to pcap16:", torch.equal(res[16][0], res[pc][0]), "counts equal:", torch.equal(res[16][1], res[pc][1]),
          "max|dS|", float((res[16][0] - res[pc][0]).abs().max()))
import oracle
from paper_2502_01826_b200.scene import HostScene
hs = HostScene(ds.means.cpu().numpy().astype(np.float64), ds.quats.cpu().numpy().astype(np.float64), ds.log_scales.cpu().numpy().astype(np.float64),
               ds.trans_mag_raw.cpu().numpy().astype(np.float64), ds.trans_phase.cpu().numpy().astype(np.float64), ds.coeffs.cpu().numpy().astype(np.complex128),
               np.zeros(3), 1.0, 72, 36, 3)
oc = oracle.OracleContext(hs)
oc.set_tx(tx[0].cpu().numpy().astype(np.float64))
ref = oc.forward().reshape(-1)
lc = oc.live_counts().reshape(-1)
for pc in (16, 32, 64):
    S = res[pc][0][0].reshape(-1).cpu().numpy()
    print(pc, "vs oracle rel", float(np.linalg.norm(np.abs(S)**2 - np.abs(ref)**2) / np.linalg.norm(np.abs(ref)**2)),
          "live count mismatches", int((res[pc][1].cpu().numpy() != np.minimum(lc, 64)).sum()))
