"""One two-stage leading_eigvecs call at size n (for ncu launch lists)."""
import os
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
os.environ.setdefault("TMB_EIG_2STAGE", "1")
from paper_2104_04726_b200 import _lib as L  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2160
k = int(sys.argv[2]) if len(sys.argv) > 2 else n // 4
rng = np.random.default_rng(0)
q, _ = np.linalg.qr(rng.standard_normal((n, n)))
g = (q * (1e3 * np.exp(-np.linspace(0, 20, n)))) @ q.T
g = 0.5 * (g + g.T)
gd = L.dev_f64(g)
vecs, vals = L.empty_f64(n * k), L.empty_f64(k)
h = L.ctx()
for _ in range(int(sys.argv[3]) if len(sys.argv) > 3 else 1):
    L.check(L.LIB.tmb_leading_eigvecs(h, L.ptr(gd), n, k, L.ptr(vecs), L.ptr(vals)), h)
torch.cuda.synchronize()
print("ok", n, k)
