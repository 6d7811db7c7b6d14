"""Prototype (research only): warm-started subspace iteration for the HOOI
eigen-update, measured against the oracle's full eigh on the real per-sweep
Grams of a synthetic stack.

Iteration: Z = G Q diag(1/theta) (theta = Rayleigh quotients), Q = polar(Z)
by Newton-Schulz (Z is near-orthonormal when Q is near the eigenbasis), with a
per-column off-subspace residual check on the top-R columns; Rayleigh-Ritz at
the end. The HOOI trajectory follows the oracle (eigh) factors; each mode's
warm start is the previous sweep's SI Ritz block (R+p columns).

  python scripts/research/si_proto.py c2 1.0 --p 16 --tol 1e-12
"""
import argparse
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
from oracle.tucker_oracle import coding_tensor, gram, leading_eigvecs, sign_fix, ttmc, unfold  # noqa: E402
from paper_2104_04726_b200.synth import CONFIGS, make_stack  # noqa: E402


def ns_polar(z, tol=1e-15, max_steps=12):
    k = z.shape[1]
    eye = np.eye(k)
    for s in range(max_steps):
        a = z.T @ z
        e = np.abs(a - eye).max()
        if e < tol:
            return z, s, e
        z = z @ (1.5 * eye - 0.5 * a)
    return z, max_steps, e


def cholqr(z):
    c = np.linalg.cholesky(z.T @ z)
    return np.linalg.solve(c, z.T).T


def rr(g, q):
    h = q.T @ g @ q
    h = 0.5 * (h + h.T)
    w, v = np.linalg.eigh(h)
    order = np.argsort(w)[::-1]
    return q @ v[:, order], w[order]


def si(g, q, r, tol, max_it, stats):
    ns_total = 0
    res = np.inf
    # iteration 1: unscaled power step, CholQR2 (robust to the warm start's
    # components along far larger eigenvalues), then Rayleigh-Ritz
    q = cholqr(cholqr(g @ q))
    q, th = rr(g, q)
    it = 1
    dev_max = 0.0
    for it in range(2, max_it + 1):
        z = g @ q
        th = np.einsum("ij,ij->j", q, z)
        z = z / th
        zr = z[:, :r]
        res = np.linalg.norm(zr - q @ (q.T @ zr), axis=0).max()
        dev_max = max(dev_max, np.abs(z.T @ z - np.eye(z.shape[1])).max())
        q, s, e = ns_polar(z)
        ns_total += s
        if res < tol:
            break
    stats["dev"] = dev_max
    x, w = rr(g, q)
    return x, w, it, ns_total, res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("cfg")
    ap.add_argument("scale", type=float)
    ap.add_argument("--p", type=int, default=16)
    ap.add_argument("--tol", type=float, default=1e-12)
    ap.add_argument("--max-it", type=int, default=200)
    ap.add_argument("--sweeps", type=int, default=None)
    a = ap.parse_args()
    cfg = CONFIGS[a.cfg]
    h, w = int(cfg.height * a.scale), int(cfg.width * a.scale)
    ranks = [int(round(r * a.scale)) if i < 2 else r for i, r in enumerate(cfg.ranks)]
    images = make_stack(cfg, seed=1, height=h, width=w)
    x = np.asfortranarray(coding_tensor(images, cfg.space).astype(np.float32).astype(np.float64))
    print(f"{a.cfg} {x.shape} ranks {ranks} p {a.p} tol {a.tol}")
    sweeps = a.sweeps or cfg.sweeps
    big = [n for n in range(4) if x.shape[n] > 64]
    # T-HOSVD: full eigh, keep R+p for the warm start
    factors, warm = [], {}
    for n in range(4):
        g = gram(unfold(x, n))
        kp = min(ranks[n] + a.p, x.shape[n])
        v, _ = leading_eigvecs(g, kp)
        factors.append(v[:, :ranks[n]])
        warm[n] = v
    for sw in range(1, sweeps + 1):
        for n in range(4):
            y = ttmc(x, factors, skip=n)
            g = gram(unfold(y, n))
            ref, lam = leading_eigvecs(g, ranks[n])
            if n in big:
                t0 = time.time()
                st = {}
                xs, th, it, ns, res = si(g, warm[n], ranks[n], a.tol, a.max_it, st)
                dt = time.time() - t0
                mine = sign_fix(xs[:, :ranks[n]])
                cosv = np.abs(np.einsum("ij,ij->j", mine, ref))
                ang = np.arccos(np.clip(cosv, -1, 1)).max()
                sv = np.linalg.svd(mine.T @ ref, compute_uv=False)
                sub = np.arccos(np.clip(sv.min(), -1, 1))
                lw, _ = leading_eigvecs(g, ranks[n] + a.p + 1)
                rho = lw[-1] / lw[ranks[n] - 1]
                print(f"sweep {sw:2d} mode {n}: it {it:3d} ns {ns:3d} res {res:.1e} rho {rho:.3f} "
                      f"max vec angle {ang:.2e} subspace {sub:.2e} eig rel err {np.abs(th[:ranks[n]]/lam-1).max():.1e} "
                      f"dev {st['dev']:.1e} ({dt:.1f}s)", flush=True)
                warm[n] = xs
            factors[n] = ref


if __name__ == "__main__":
    main()
