"""Prototype: warm-started Ogita-Aishima eigenvector refinement for the HOOI Grams.

Records the mode-0/1 Grams of oracle HOOI sweeps on a (downscaled) synthetic
stack, then refines the previous sweep's full eigenvector basis against the
next Gram and compares the leading-k eigenvectors with numpy eigh.
"""
import sys
from dataclasses import replace
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from oracle import tucker_oracle as O  # noqa: E402
from paper_2104_04726_b200.synth import CONFIGS, make_stack  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 4
cfg = CONFIGS["c2"]
cfg = replace(cfg, height=cfg.height // scale, width=cfg.width // scale,
              ranks=(cfg.ranks[0] // scale, cfg.ranks[1] // scale, 3, 5))
imgs = make_stack(cfg, seed=0)
x = O.coding_tensor(imgs, cfg.space)
print("tensor", x.shape, "ranks", cfg.ranks)

grams = {0: [], 1: []}
core, f = O.t_hosvd(x, cfg.ranks)
for n in (0, 1):
    grams[n].append(O.gram(O.unfold(x, n)))
for s in range(8):
    f = list(f)
    for n in range(4):
        y = O.ttmc(x, f, skip=n)
        g = O.gram(O.unfold(y, n))
        if n < 2:
            grams[n].append(g)
        f[n] = O.leading_eigvecs(g, cfg.ranks[n])[0]


def refine(a, xh, iters=6, tag=""):
    n = a.shape[0]
    anorm = np.linalg.norm(a, 2)
    hist = []
    for it in range(iters):
        r = np.eye(n) - xh.T @ xh
        s = xh.T @ a @ xh
        lam = np.diag(s) / (1 - np.diag(r))
        dlt = 2 * (np.linalg.norm(s - np.diag(lam), 2) + anorm * np.linalg.norm(r, 2))
        dl = lam[None, :] - lam[:, None]       # lam_j - lam_i
        e = np.where(np.abs(dl) > dlt, (s + lam[None, :] * r) / np.where(dl == 0, 1, dl), r / 2)
        np.fill_diagonal(e, np.diag(r) / 2)
        xh = xh + xh @ e
        ncl = int((np.abs(dl) <= dlt).sum() - n)
        hist.append((np.abs(e).max(), dlt / anorm, ncl))
    return xh, lam, hist


for n in (0, 1):
    k = cfg.ranks[n]
    for t in range(1, len(grams[n])):
        a_prev, a = grams[n][t - 1], grams[n][t]
        w0, v0 = np.linalg.eigh(a_prev)
        w, v = np.linalg.eigh(a)
        xh, lam, hist = refine(a, v0[:, ::-1])
        order = np.argsort(-lam)
        xk = O.sign_fix(xh[:, order[:k]])
        vk = O.sign_fix(v[:, ::-1][:, :k])
        # leading-k subspace angle and per-vector agreement
        sv = np.linalg.svd(vk.T @ xk, compute_uv=False)
        ang = np.sqrt(max(0.0, 1 - sv.min() ** 2))
        colerr = np.abs(xk - vk).max()
        gaps = np.diff(w[::-1][: k + 1])
        print(f"mode {n} t {t}: start dV {np.abs(np.abs(v0[:, ::-1][:, :k]) - np.abs(v[:, ::-1][:, :k])).max():.1e} "
              f"hist {[f'{h[0]:.0e}/{h[2]}' for h in hist]} subspace {ang:.1e} col {colerr:.1e} "
              f"min rel gap(k) {np.abs(gaps).min() / w[-1]:.1e}")
