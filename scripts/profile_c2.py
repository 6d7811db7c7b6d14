"""One C2 stack through the fused device path (for ncu launch lists / captures)."""
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2104_04726_b200 as tb  # noqa: E402
from paper_2104_04726_b200.pipeline import encode_stack_device  # noqa: E402
from paper_2104_04726_b200.synth import CONFIGS, make_stack  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
sweeps = int(sys.argv[2]) if len(sys.argv) > 2 else None
cfg = CONFIGS[name]
dev = torch.from_numpy(make_stack(cfg, seed=0)).cuda()
sc = tb.SolveConfig(ranks=cfg.ranks, max_sweeps=sweeps or cfg.sweeps, fit_tol=1e-300, pp_enter_tol=0.0)
bufs, tr, step, rel = encode_stack_device(dev, cfg.space, cfg.ranks, sc, cfg.qp or 51, rel_err=True)
torch.cuda.synchronize()
print("fit", tr.fit[tr.n_records - 1], "rel", rel)
