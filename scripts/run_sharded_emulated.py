"""Row-sharded solve (sharded.py) at a BASELINE config's full size, with G
host-thread ranks on ONE GPU (ThreadComm: host-side collectives, no device-side
waiting), against the unsharded device solver on the same stack.
Usage: run_sharded_emulated.py [config=c5] [ranks=2] [sweeps]"""
import sys
import threading
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2104_04726_b200 as tb  # noqa: E402
from paper_2104_04726_b200.pipeline import coding_tensor  # noqa: E402
from paper_2104_04726_b200.sharded import ThreadComm, row_ranges, sharded_tucker_als  # noqa: E402
from paper_2104_04726_b200.synth import CONFIGS, make_stack  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c5"
world = int(sys.argv[2]) if len(sys.argv) > 2 else 2
cfg0 = CONFIGS[name]
sweeps = int(sys.argv[3]) if len(sys.argv) > 3 else cfg0.sweeps
t0 = time.time()
t = coding_tensor(make_stack(cfg0, seed=0), cfg0.space)
dims = tuple(int(d) for d in cfg0.dims)
print(f"{name} {dims} ranks {cfg0.ranks} sweeps {sweeps}, stack ready in {time.time() - t0:.0f} s", flush=True)
sc = tb.SolveConfig(ranks=cfg0.ranks, max_sweeps=sweeps, fit_tol=1e-300, pp_enter_tol=0.0)
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
ref_model, ref_trace = tb.tucker.solve_device(t, tb._lib.F32, dims, sc)
e.record()
torch.cuda.synchronize()
print(f"unsharded: {s.elapsed_time(e) / 1e3:.2f} s, fit {ref_trace.records[-1].fit:.12f}", flush=True)
full = t.view(int(np.prod(dims[1:])), dims[0])
comm = ThreadComm(world)
results = [None] * world


def run(rank):
    torch.cuda.set_device(0)
    a, b = row_ranges(dims[0], world)[rank]
    xl = full[:, a:b].contiguous().view(-1)
    results[rank] = sharded_tucker_als(xl, dims, sc, comm.bind(rank))


t1 = time.time()
th = [threading.Thread(target=run, args=(r,)) for r in range(world)]
for x in th:
    x.start()
for x in th:
    x.join()
torch.cuda.synchronize()
m0, tr0 = results[0]
same = all(np.array_equal(a, b) for r in results[1:] for a, b in zip(m0.factors, r[0].factors))
angles = []
for a, b in zip(m0.factors, ref_model.factors):
    d = a - b @ (b.T @ a)
    angles.append(float(np.arcsin(min(1.0, np.linalg.norm(d, 2)))))
dfit = max(abs(x.fit - y.fit) for x, y in zip(tr0.records, ref_trace.records))
print(f"sharded over {world} thread-ranks on 1 GPU: {time.time() - t1:.2f} s wall, ranks identical {same}, "
      f"max principal angle vs unsharded {max(angles):.2e}, max |dfit| {dfit:.2e}, "
      f"fit {tr0.records[-1].fit:.12f}", flush=True)
