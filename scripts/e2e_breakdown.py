"""Where the end-to-end (host API) time of one C2 stack goes beyond the
device-resident solve, phase by phase inside encode_stack's own sequence
(wall clock with a device synchronise after each phase; diagnostic only)."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2104_04726_b200 as tb  # noqa: E402
from paper_2104_04726_b200 import _lib as L  # noqa: E402
from paper_2104_04726_b200.pipeline import _trace_from_c, encode_stack_device  # noqa: E402
from paper_2104_04726_b200.synth import CONFIGS, make_stack  # noqa: E402

cfg = CONFIGS["c2"]
images = make_stack(cfg, seed=0)
pinned = torch.from_numpy(images).pin_memory()
for _ in range(2):
    tb.encode_stack(pinned, cfg.space, cfg.ranks, cfg.sweeps, cfg.qp)
torch.cuda.synchronize()
dims = (1080, 1920, 3, 10)
ranks = cfg.ranks
n = int(np.prod(ranks))
for rep in range(5):
    t = [time.perf_counter()]
    imgs = pinned.to("cuda", non_blocking=True)
    sc = tb.SolveConfig(ranks=tuple(ranks), max_sweeps=cfg.sweeps, fit_tol=1e-300, pp_enter_tol=0.0)
    torch.cuda.synchronize(); t.append(time.perf_counter())
    bufs, tr, step, rel = encode_stack_device(imgs, cfg.space, ranks, sc, cfg.qp, rel_err=True)
    torch.cuda.synchronize(); t.append(time.perf_counter())
    levels = np.reshape(bufs["levels"][:n].cpu().numpy(), ranks, order="F")
    t.append(time.perf_counter())
    core = tb.DenseTensor(L.host_f(bufs["core"], ranks))
    facs = [L.host_f(f, (dims[i], ranks[i])) for i, f in enumerate(bufs["factors"])]
    t.append(time.perf_counter())
    model = tb.TuckerModel(core, facs, dims)
    trace = _trace_from_c(tr)
    t.append(time.perf_counter())
    e = [1e3 * (b - a) for a, b in zip(t, t[1:])]
    print(f"rep {rep}: h2d {e[0]:.2f} | device {e[1]:.2f} | levels d2h {e[2]:.2f} | core+factors d2h {e[3]:.2f} | "
          f"model+trace {e[4]:.2f} | total {1e3 * (t[-1] - t[0]):.2f} ms", flush=True)
s, e_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
w0 = time.perf_counter()
for _ in range(5):
    tb.encode_stack(pinned, cfg.space, cfg.ranks, cfg.sweeps, cfg.qp)
e_.record(); torch.cuda.synchronize()
print(f"5 x encode_stack: events {s.elapsed_time(e_) / 5:.2f} ms/stack, wall {1e3 * (time.perf_counter() - w0) / 5:.2f}")
