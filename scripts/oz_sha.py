"""sha1 of the Ozaki TTM output on the C2 mode-1 full pass (to compare kernel variants bit for bit)."""
import hashlib
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2104_04726_b200 import _lib as L  # noqa: E402

torch.manual_seed(0)
dims = (1080, 1920, 3, 10)
x = torch.rand(int(np.prod(dims)), dtype=torch.float32, device="cuda") ** 3
u = torch.linalg.qr(torch.randn(1920, 480, dtype=torch.float64, device="cuda"))[0]
y = torch.empty(1080 * 480 * 30, dtype=torch.float64, device="cuda")
h = L.ctx()
L.check(L.LIB.tmb_ttm(h, L.ptr(x), L.F32, 4, L.i64s(dims), 1, L.ptr(u.contiguous().view(-1)), 480, L.ptr(y)), h)
torch.cuda.synchronize()
print("sha1", hashlib.sha1(y.cpu().numpy().tobytes()).hexdigest()[:16])
