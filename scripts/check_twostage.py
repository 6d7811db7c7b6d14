"""Two-stage tridiagonalisation / eigen-solver check against LAPACK (research + GPU validation).

    TMB_EIG_2STAGE=1 python scripts/check_twostage.py [n ...]

For each n: T from tmb_tridiagonalize (eigenvalues vs numpy.linalg.eigvalsh of G),
then tmb_leading_eigvecs (k = n/4) vs numpy.linalg.eigh: eigenvalue error,
residual, orthogonality, largest principal angle; plus device timings.
"""
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2104_04726_b200 import _lib as L  # noqa: E402


def gram(n, kind, rng):
    if kind == "decay":
        q, _ = np.linalg.qr(rng.standard_normal((n, n)))
        lam = 1e3 * np.exp(-np.linspace(0, 20, n))
        g = (q * lam) @ q.T
    else:
        y = rng.standard_normal((n, n + 7))
        g = y @ y.T
    return 0.5 * (g + g.T)


def main():
    sizes = [int(a) for a in sys.argv[1:]] or [100, 257, 700, 1000, 2160]
    rng = np.random.default_rng(0)
    h = L.ctx()
    for n in sizes:
        for kind in (("decay", "wishart") if n < 3000 else ("decay",)):
            g = gram(n, kind, rng)
            gd = L.dev_f64(g)
            d = L.empty_f64(n)
            e = L.empty_f64(max(n - 1, 1))
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            L.check(L.LIB.tmb_tridiagonalize(h, L.ptr(gd), n, L.ptr(d), L.ptr(e)), h)
            torch.cuda.synchronize()
            t_tri = (time.perf_counter() - t0) * 1e3
            dh, eh = d.cpu().numpy(), e.cpu().numpy()[: n - 1]
            wt = np.linalg.eigvalsh(np.diag(dh) + np.diag(eh, 1) + np.diag(eh, -1))
            wr = np.linalg.eigvalsh(g)
            nrm = np.abs(wr).max()
            tri_err = np.abs(wt - wr).max() / nrm
            k = max(1, n // 4)
            vecs = L.empty_f64(n * k)
            vals = L.empty_f64(k)
            times = []
            for _ in range(3):
                s = torch.cuda.Event(enable_timing=True)
                t = torch.cuda.Event(enable_timing=True)
                s.record()
                L.check(L.LIB.tmb_leading_eigvecs(h, L.ptr(gd), n, k, L.ptr(vecs), L.ptr(vals)), h)
                t.record()
                torch.cuda.synchronize()
                times.append(s.elapsed_time(t))
            x = vecs.cpu().numpy().reshape(k, n).T
            w = vals.cpu().numpy()
            wv, xv = np.linalg.eigh(g)
            wv, xv = wv[::-1][:k], xv[:, ::-1][:, :k]
            val_err = np.abs(w - wv).max() / nrm
            resid = np.abs(g @ x - x * w).max() / nrm
            orth = np.abs(x.T @ x - np.eye(k)).max()
            ang = float(np.arcsin(min(1.0, np.linalg.norm(x - xv @ (xv.T @ x), 2))))
            print(f"n={n} {kind}: tri eig err {tri_err:.1e} ({t_tri:.1f} ms host) | k={k} val err {val_err:.1e} "
                  f"resid {resid:.1e} orth {orth:.1e} angle {ang:.1e} | {' '.join(f'{v:.2f}' for v in times)} ms",
                  flush=True)


if __name__ == "__main__":
    main()
