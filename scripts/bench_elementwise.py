"""HBM-bound kernels through the C ABI (device resident): the u8 -> coding-space
colour kernel at the BASELINE stack sizes (both spaces) and the decode-side
to_rgb + SSE kernel, timed with CUDA events on the context's stream and
reported as algorithmic GB/s against MEASURED_PEAKS.json hbm_gbs.

    python scripts/bench_elementwise.py [reps] [filter]
"""
import json
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2104_04726_b200 import _lib as L  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
which = sys.argv[2] if len(sys.argv) > 2 else ""
peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
hbm = float(peaks.get("hbm_gbs", 6443.8))
h = L.ctx()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")  # 256 MB > L2: written between reps


def timed(fn):
    ts = []
    for _ in range(reps):
        flush.fill_(1)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        L.check(fn(), h)
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    return float(np.median(ts))


shapes = {"c2": (10, 1080, 1920), "c4": (14, 2160, 3840), "c5": (18, 4320, 7680)}
for cname, (n_img, hh, ww) in shapes.items():
    px = n_img * hh * ww
    rgb = torch.randint(0, 256, (px * 3,), dtype=torch.uint8, device="cuda")
    out = torch.empty(px * 3, dtype=torch.float32, device="cuda")
    for space in ("ycbcr", "ipt"):
        name = f"color_u8 {cname} {space}"
        if which and which not in name:
            continue
        ms = timed(lambda: L.LIB.tmb_color_u8(h, L.ptr(rgb), n_img, hh, ww, L.SPACES[space], L.ptr(out)))
        gbs = 15.0 * px / (ms / 1e3) / 1e9
        print(f"{name}: {ms:.3f} ms  {gbs:.0f} GB/s = {gbs / hbm:.1%} of {hbm:.0f} (15 B/px)", flush=True)
    del rgb, out
    torch.cuda.empty_cache()
