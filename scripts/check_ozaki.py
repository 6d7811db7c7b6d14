"""Ozaki tcgen05 TTM vs fp64 references on the C2 full-pass shapes: accuracy
(against torch float64 matmul) and time. Run with TMB_OZAKI=0 for the DMMA path."""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2104_04726_b200 import _lib as L  # noqa: E402

torch.manual_seed(0)
dims = (1080, 1920, 3, 10)
x = torch.rand(int(np.prod(dims)), dtype=torch.float32, device="cuda") ** 3  # skewed values, exact fp32
h = L.ctx()
for mode, r in ((1, 480), (0, 270)):
    s = dims[mode]
    u = torch.linalg.qr(torch.randn(s, r, dtype=torch.float64, device="cuda"))[0]  # orthonormal columns
    m = u.contiguous().view(-1)   # C-order (s, r) == u^T column-major (r x s)
    nd = list(dims)
    nd[mode] = r
    y = torch.empty(int(np.prod(nd)), dtype=torch.float64, device="cuda")
    times = []
    for _ in range(4):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        L.check(L.LIB.tmb_ttm(h, L.ptr(x), L.F32, 4, L.i64s(dims), mode, L.ptr(m), r, L.ptr(y)), h)
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
    # reference: float64 matmul of the same contraction
    xt = x.double().view(dims[3], dims[2], dims[1], dims[0])  # C-order view of the F-order tensor
    if mode == 1:
        ref = torch.einsum("lcji,jr->lcri", xt, u)
    else:
        ref = torch.einsum("lcji,ir->lcjr", xt, u)
    yv = y.view(*reversed(nd))
    err = (yv - ref).abs()
    scale = torch.einsum("lcji,jr->lcri", xt.abs(), u.abs()) if mode == 1 else torch.einsum("lcji,ir->lcjr", xt.abs(), u.abs())
    flops = 2 * np.prod(dims) * r
    print(f"mode {mode}: {min(times):.3f} ms ({flops / min(times) / 1e9:.1f} TFLOP/s fp64-eq), "
          f"max |err| / (|x||u|) = {(err / scale.clamp_min(1e-300)).max().item():.2e}, "
          f"normwise rel err = {(err.norm() / ref.norm()).item():.2e}")
