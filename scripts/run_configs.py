"""One stack of each BASELINE config end to end on one GPU (encode_stack: u8
images in pinned host memory -> colour -> tucker_als -> quantise -> rel. error),
timed with CUDA events after one warm-up solve. Usage: run_configs.py c3 c4_8 ..."""
import sys
import time
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2104_04726_b200 as tb  # noqa: E402
from paper_2104_04726_b200.synth import CONFIGS, make_stack  # noqa: E402

for name in sys.argv[1:]:
    cfg = CONFIGS[name]
    t0 = time.time()
    images = torch.from_numpy(make_stack(cfg, seed=0)).pin_memory()
    gen = time.time() - t0
    qp = cfg.qp or 51
    tb.encode_stack(images, cfg.space, cfg.ranks, 1, qp)  # warm-up (allocations, module load)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    res = tb.encode_stack(images, cfg.space, cfg.ranks, cfg.sweeps, qp)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e)
    print(f"{name}: dims {cfg.dims} ranks {cfg.ranks} sweeps {cfg.sweeps} qp {qp}: {ms / 1e3:.3f} s/stack "
          f"({1e3 / ms:.3f} stacks/s), fit {res.trace.records[-1].fit:.6f}, rel_err {res.rel_err:.3e} "
          f"[generation {gen:.0f} s on host]", flush=True)
