"""C2-shaped TTM / Gram GEMMs through the C ABI (device resident), for A/B timing and ncu captures."""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2104_04726_b200 import _lib as L  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
which = sys.argv[2] if len(sys.argv) > 2 else "all"
h = L.ctx()
dims = (1080, 1920, 3, 10)
x = torch.rand(int(np.prod(dims)), dtype=torch.float32, device="cuda")
xd = x.double()
s1 = torch.rand(1920 * 480, dtype=torch.float64, device="cuda")
s0 = torch.rand(1080 * 270, dtype=torch.float64, device="cuda")
y = L.empty_f64(1080 * 1920 * 30)
dy0, dy1 = (1080, 480, 3, 5), (270, 1920, 3, 5)
y0 = torch.rand(int(np.prod(dy0)), dtype=torch.float64, device="cuda")
y1 = torch.rand(int(np.prod(dy1)), dtype=torch.float64, device="cuda")
cases = {
    "ttm1": (lambda: L.LIB.tmb_ttm(h, L.ptr(x), L.F32, 4, L.i64s(dims), 1, L.ptr(s1), 480, L.ptr(y)), 2 * 480 * np.prod(dims)),
    "ttm0": (lambda: L.LIB.tmb_ttm(h, L.ptr(x), L.F32, 4, L.i64s(dims), 0, L.ptr(s0), 270, L.ptr(y)), 2 * 270 * np.prod(dims)),
    "gram1": (lambda: L.LIB.tmb_mode_gram(h, L.ptr(x), L.F32, 4, L.i64s(dims), 1, L.ptr(y)), 1921 * np.prod(dims)),
    "ttm1_f64": (lambda: L.LIB.tmb_ttm(h, L.ptr(xd), L.F64, 4, L.i64s(dims), 1, L.ptr(s1), 480, L.ptr(y)), 2 * 480 * np.prod(dims)),
    "gram1_f64": (lambda: L.LIB.tmb_mode_gram(h, L.ptr(xd), L.F64, 4, L.i64s(dims), 1, L.ptr(y)), 1921 * np.prod(dims)),
    # HOOI sweep Grams at C2: Y0 = 1080 x (480*3*5), Y1 = 1920 x (270*3*5), fp64
    "gram_y0": (lambda: L.LIB.tmb_mode_gram(h, L.ptr(y0), L.F64, 4, L.i64s(dy0), 0, L.ptr(y)), 1080 * 1081 * 7200),
    "gram_y1": (lambda: L.LIB.tmb_mode_gram(h, L.ptr(y1), L.F64, 4, L.i64s(dy1), 1, L.ptr(y)), 1920 * 1921 * 4050),
    # cuBLAS DGEMM on the same ttm1 contraction (30 batched 480x1920 @ 1920x1080), for scale
    "cublas_ttm1": (lambda: torch.matmul(s1.view(480, 1920), xd.view(30, 1920, 1080)), 2 * 480 * np.prod(dims)),
    "cublas_gram1": (lambda: torch.matmul(xd.view(1920, -1), xd.view(1920, -1).T), 2 * 1920 * np.prod(dims)),
}
for name, (fn, flops) in cases.items():
    if which != "all" and which != name:
        continue
    ts = []
    for _ in range(reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); rc = fn(); e.record(); torch.cuda.synchronize()
        L.check(rc, h) if isinstance(rc, int) else None
        ts.append(s.elapsed_time(e))
    t = min(ts)
    print(f"{name}: {t:.3f} ms  {flops / t / 1e9:.1f} TFLOP/s")
