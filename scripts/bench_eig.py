"""Device-resident leading_eigvecs timing on C2-like Grams (n, k) -- for ncu captures and A/B runs."""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2104_04726_b200 import _lib as L  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
sizes = [(1080, 270), (1920, 480)] if len(sys.argv) <= 2 else [tuple(map(int, s.split("x"))) for s in sys.argv[2:]]
rng = np.random.default_rng(0)
for n, k in sizes:
    q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    lam = 1e3 * np.exp(-np.linspace(0, 20, n))
    g = (q * lam) @ q.T
    g = 0.5 * (g + g.T)
    gd = L.dev_f64(g)
    vecs = L.empty_f64(n * k)
    vals = L.empty_f64(k)
    h = L.ctx()
    times = []
    for r in range(reps):
        s = torch.cuda.Event(enable_timing=True)
        e = torch.cuda.Event(enable_timing=True)
        s.record()
        L.check(L.LIB.tmb_leading_eigvecs(h, L.ptr(gd), n, k, L.ptr(vecs), L.ptr(vals)), h)
        e.record()
        torch.cuda.synchronize()
        times.append(s.elapsed_time(e))
    import hashlib
    digest = hashlib.sha1(vecs.cpu().numpy().tobytes() + vals.cpu().numpy().tobytes()).hexdigest()[:12]
    w = np.linalg.eigvalsh(g)[::-1][:k]
    err = np.abs(vals.cpu().numpy() - w).max() / w[0]
    L.check(L.LIB.tmb_timing(h, 1), h)
    L.check(L.LIB.tmb_leading_eigvecs(h, L.ptr(gd), n, k, L.ptr(vecs), L.ptr(vals)), h)
    torch.cuda.synchronize()
    fam = []
    for tag, nm in ((1, "sytrd"), (2, "tridiag"), (4, "wy_gemm")):
        cnt, tms, work = L.C.c_int64(), L.C.c_double(), L.C.c_double()
        L.check(L.LIB.tmb_timing_read(h, tag, L.C.byref(cnt), L.C.byref(tms), L.C.byref(work)), h)
        fam.append(f"{nm} {tms.value:.2f}")
    L.check(L.LIB.tmb_timing(h, 0), h)
    print(f"n={n} k={k}: [" + ", ".join(fam) + "] " + " ".join(f"{t:.2f}" for t in times) + f" ms  sha1 {digest}  val err {err:.1e}")
