"""Print the full-size C2 parity numbers against tests/golden/c2_full.npz (the
reference run in the build container): fit/rel-err deltas, sketch and leading
eigenvector deltas, differing quantised levels."""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2104_04726_b200 as tb  # noqa: E402
from paper_2104_04726_b200.synth import CONFIGS, make_stack  # noqa: E402

z = np.load(ROOT / "tests" / "golden" / "c2_full.npz")
cfg = CONFIGS["c2"]
res = tb.encode_stack(make_stack(cfg, seed=0), cfg.space, cfg.ranks, cfg.sweeps, cfg.qp)
fits = np.array([r.fit for r in res.trace.records])
print(f"trace fit max |d| {np.abs(fits - z['trace_fit']).max():.2e}; rel_err |d| {abs(res.rel_err - float(z['rel_err'])):.2e}")
for n in range(4):
    u = res.model.factors[n]
    w = np.random.default_rng(1000 + u.shape[0]).standard_normal((u.shape[0], 16)) / np.sqrt(u.shape[0])
    p = w.T @ u
    h = z[f"head{n}"]
    print(f"mode {n}: sketch max |d| {np.abs(p @ p.T - z[f'sketch{n}']).max():.2e}; leading columns max |d| "
          f"{np.abs(u[:, :h.shape[1]] - h).max():.2e}")
lv, ref = res.levels.astype(np.int64), z["levels"].astype(np.int64)
d = lv != ref
print(f"levels differing: {int(d.sum())} of {lv.size}, max |d| {int(np.abs(lv - ref).max())}; step rel |d| "
      f"{abs(res.step / float(z['step']) - 1):.2e}")
