"""Per-kernel-family device time of one stack of a BASELINE config (libtmb's
live CUDA-event launch timing, tmb_timing), after a 1-sweep warm-up.
Usage: config_families.py c5 [c4_2 ...]"""
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2104_04726_b200 as tb  # noqa: E402
from paper_2104_04726_b200 import _lib as L  # noqa: E402
from paper_2104_04726_b200.synth import CONFIGS, make_stack  # noqa: E402

FAM = ((0, "gemm_dmma"), (1, "sytrd"), (2, "tridiag_vectors"), (3, "color_u8"), (4, "eig_gemm_dmma"),
       (5, "ttm_ozaki_i8"))
for name in sys.argv[1:]:
    cfg = CONFIGS[name]
    images = torch.from_numpy(make_stack(cfg, seed=0)).pin_memory()
    qp = cfg.qp or 51
    tb.encode_stack(images, cfg.space, cfg.ranks, 1, qp)
    h = L.ctx()
    L.check(L.LIB.tmb_timing(h, 1), h)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    tb.encode_stack(images, cfg.space, cfg.ranks, cfg.sweeps, qp)
    e.record()
    torch.cuda.synchronize()
    out = []
    for tag, nm in FAM:
        cnt, tms, work = L.C.c_int64(), L.C.c_double(), L.C.c_double()
        L.check(L.LIB.tmb_timing_read(h, tag, L.C.byref(cnt), L.C.byref(tms), L.C.byref(work)), h)
        out.append(f"{nm} {tms.value:.0f} ms/{cnt.value}")
    L.check(L.LIB.tmb_timing(h, 0), h)
    print(f"{name}: total {s.elapsed_time(e):.0f} ms | " + " | ".join(out), flush=True)
