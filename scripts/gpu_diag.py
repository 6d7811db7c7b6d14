"""First-light diagnostics on a B200: kernels vs numpy/oracle, golden parity, C2 timing."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2104_04726_b200 as tb  # noqa: E402
from paper_2104_04726_b200 import _lib as L  # noqa: E402
from paper_2104_04726_b200.pipeline import encode_stack_device  # noqa: E402
from paper_2104_04726_b200.synth import CONFIGS, make_stack  # noqa: E402
import oracle  # noqa: E402

G = ROOT / "tests" / "golden"


def angle(u, v):
    d = u - v @ (v.T @ u)
    return float(np.arcsin(min(1.0, np.linalg.norm(d, 2))))


def section(name):
    print(f"\n=== {name}", flush=True)


def t0():
    torch.cuda.synchronize()
    return time.perf_counter()


section("colour KAT")
kat = np.load(G / "colour.npz")
u8 = kat["u8"]
for space in ("ycbcr", "ipt"):
    imgs = u8.reshape(1, 1, 1, -1, 3)
    t = tb.coding_tensor(imgs, space).cpu().numpy().reshape((1, u8.shape[0], 3, 1), order="F")[0, :, :, 0]
    ref = kat[f"{space}_u8"].astype(np.float32)
    print(space, "u8 max|d| vs fp32(ref):", np.abs(t - ref).max(), "exact:", np.mean(t == ref))
    px = kat["fpx"]
    got = tb.to_coding_space(tb.ColorImage(px), space).pixels
    print(space, "f64 max|d|:", np.abs(got - kat[f"{space}_f"]).max())

section("ttm / gram / eig small")
rng = np.random.default_rng(0)
x = rng.standard_normal((7, 9, 5, 4))
m = rng.standard_normal((3, 9))
print("ttm mode1", np.abs(tb.ttm(tb.DenseTensor(x), m, 1).array - oracle.ttm(x, m, 1)).max())
m0 = rng.standard_normal((6, 7))
print("ttm mode0", np.abs(tb.ttm(tb.DenseTensor(x), m0, 0).array - oracle.ttm(x, m0, 0)).max())
a = rng.standard_normal((150, 300))
print("gram 150x300", np.abs(tb.gram(a) - oracle.gram(a)).max() / np.abs(oracle.gram(a)).max())
for n, k in [(6, 3), (40, 40), (64, 10)]:
    b = rng.standard_normal((n, n)); g = b @ b.T
    v, w = tb.leading_eigvecs(g, k)
    vr, wr = oracle.leading_eigvecs(g, k)
    print(f"eig jacobi n={n} k={k}: vec {np.abs(v - vr).max():.2e} val {np.abs(w - wr).max() / wr[0]:.2e}")

section("eig tridiagonal path")
for n, k, decay in [(100, 20, 1.0), (300, 60, 2.0), (1080, 270, 3.0)]:
    q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    lam = np.exp(-decay * np.linspace(0, 12, n)) * 1e3
    g = (q * lam) @ q.T
    g = 0.5 * (g + g.T)
    ts = t0()
    try:
        v, w = tb.leading_eigvecs(g, k)
        dt = time.perf_counter() - ts
        vr, wr = oracle.leading_eigvecs(g, k)
        orth = np.abs(v.T @ v - np.eye(k)).max()
        print(f"n={n} k={k}: angle {angle(v, vr):.2e} colmax {np.abs(v - vr).max():.2e} "
              f"val rel {np.abs(w - wr).max() / wr[0]:.2e} orth {orth:.2e} ({dt*1e3:.1f} ms incl H2D)")
    except Exception as ex:  # noqa: BLE001
        print(f"n={n} k={k}: FAILED {ex}")

section("golden parity")
for name in ("c1", "c2q", "c3q"):
    z = np.load(G / f"{name}.npz")
    ranks = tuple(int(r) for r in z["ranks"])
    ts = t0()
    res = tb.encode_stack(z["images"], str(z["space"]), ranks, int(z["sweeps"]), int(z["qp"]))
    dt = time.perf_counter() - ts
    ang = [angle(res.model.factors[n], z[f"factor{n}"]) for n in range(4)]
    ours = np.array([r.fit for r in res.trace.records]); ref = z["trace_fit"]; nn = min(len(ours), len(ref))
    fit_d = np.abs(ours[:nn] - ref[:nn]).max()
    print(f"{name}: trace len ours {len(ours)} ref {len(ref)} converged ours {res.trace.converged} ref {bool(z['converged'])}; "
          f"fit deltas ours {np.diff(ours)[-3:]} ref {np.diff(ref)[-3:]}")
    lv = res.levels
    diff = int((lv != z["levels"]).sum())
    print(f"{name}: {dt:.2f}s angles {['%.1e' % a for a in ang]} fit|d| {fit_d:.2e} rel_err {res.rel_err:.6f} "
          f"(ref {float(z['rel_err']):.6f}) step rel {res.step / float(z['step']) - 1:.1e} levels diff {diff}/{lv.size}"
          f" max|dl| {np.abs(lv - z['levels']).max()}")

section("C2 timing (device-resident)")
cfg = CONFIGS["c2"]
imgs = make_stack(cfg, seed=0)
dev = torch.from_numpy(imgs).cuda()
sc = tb.SolveConfig(ranks=cfg.ranks, max_sweeps=cfg.sweeps, fit_tol=1e-300, pp_enter_tol=0.0)
bufs = None
for it in range(3):
    ts = t0()
    n0 = L.launch_count()
    bufs, tr, step, rel = encode_stack_device(dev, cfg.space, cfg.ranks, sc, cfg.qp, rel_err=True, bufs=bufs)
    dt = t0() - ts
    print(f"run {it}: {dt*1e3:.1f} ms  launches {L.launch_count() - n0}  fit {tr.fit[tr.n_records-1]:.8f} rel {rel:.6f}")
