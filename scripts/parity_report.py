"""Parity numbers of the device path against the reference goldens for every
BASELINE config (the values DESIGN §5 quotes; the asserts live in
tests/test_gpu_parity.py and tests/test_gpu_configs.py).

    python scripts/parity_report.py [c2 c3 c4 c5]
"""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2104_04726_b200 as tb  # noqa: E402
from paper_2104_04726_b200.synth import CONFIGS, make_stack  # noqa: E402

G = ROOT / "tests" / "golden"


def sketch(u):
    w = np.random.default_rng(1000 + u.shape[0]).standard_normal((u.shape[0], 16)) / np.sqrt(u.shape[0])
    p = w.T @ u
    return p @ p.T


def report(label, res, z, tag=""):
    fits = np.array([r.fit for r in res.trace.records])
    ref = z[f"{tag}trace_fit"]
    m = min(len(fits), len(ref))
    out = [f"{label}: trace len {len(fits)}/{len(ref)}",
           f"max|dfit| {np.abs(fits[:m] - ref[:m]).max():.1e}",
           f"|drel| {abs(res.rel_err - float(z[f'{tag}rel_err'])):.1e}"]
    out.append("sketch " + "/".join(f"{np.abs(sketch(u) - z[f'{tag}sketch{n}']).max():.0e}"
                                    for n, u in enumerate(res.model.factors)))
    out.append("head " + "/".join(f"{np.abs(u[:, :8] - z[f'{tag}head{n}']).max():.0e}"
                                  for n, u in enumerate(res.model.factors)))
    if f"{tag}levels" in z or f"{tag}levels_idx" in z:
        lv = res.levels.ravel(order="F").astype(np.int64)
        if f"{tag}levels" in z:
            r = z[f"{tag}levels"].astype(np.int64)
            mine = lv if r.ndim == 1 else res.levels.astype(np.int64)
            r, mine = r.ravel(), mine.ravel()
        else:
            r = z[f"{tag}levels_sample"].astype(np.int64)
            mine = lv[z[f"{tag}levels_idx"]]
        d = mine != r
        out.append(f"levels {int(d.sum())}/{r.size} differ (max {int(np.abs(mine - r).max())} LSB)")
    print(", ".join(out), flush=True)


names = sys.argv[1:] or ["c2", "c3", "c4", "c5"]
if "c2" in names:
    z = dict(np.load(G / "c2_full.npz"))
    cfg = CONFIGS["c2"]
    res = tb.encode_stack(make_stack(cfg, seed=0), cfg.space, cfg.ranks, cfg.sweeps, cfg.qp)
    report("c2 full (20 sweeps)", res, z)
if "c3" in names:
    z = dict(np.load(G / "c3_full.npz"))
    cfg = CONFIGS["c3"]
    res = tb.encode_stack(make_stack(cfg, seed=0, frame=0), cfg.space, cfg.ranks, cfg.sweeps, cfg.qp)
    report("c3 full (10 sweeps)", res, z)
    report("c3 vs reference chain from u8 (f64 colour, App. B.1(ii))", res, z, "f64in_")
if "c4" in names:
    z = dict(np.load(G / "c4_curve.npz"))
    images = make_stack(CONFIGS["c4_8"], seed=0)
    for name in ("c4_8", "c4_4", "c4_2"):
        cfg = CONFIGS[name]
        res = tb.encode_stack(images, cfg.space, cfg.ranks, 2, 51)
        report(f"{name} ranks {cfg.ranks} (2 sweeps) rel_err {res.rel_err:.6e}", res, z, f"{name}_")
if "c5" in names:
    z = dict(np.load(G / "c5_2sweeps.npz"))
    cfg = CONFIGS["c5"]
    res = tb.encode_stack(make_stack(cfg, seed=0), cfg.space, cfg.ranks, 2, cfg.qp)
    report("c5 (T-HOSVD + 2 sweeps)", res, z)
