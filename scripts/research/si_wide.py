"""Research only: warm-started subspace iteration with WIDE oversampling
(m = R + p columns, p ~ R/2..R) followed by one Rayleigh-Ritz, on the real
per-sweep HOOI Grams of a synthetic stack (oracle trajectory). Question: with
the block spanning well past the truncation rank, does lambda_{m+1}/lambda_R
get small enough that a handful of G.Q products pins the top-R subspace to
fp64 accuracy, so the full n x n tridiagonalisation can be replaced by an
m x m one?

  python scripts/research/si_wide.py c2 1.0 --pfrac 0.5 --iters 6 --sweeps 3
"""
import argparse
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
from oracle.tucker_oracle import coding_tensor, gram, leading_eigvecs, ttmc, unfold  # noqa: E402
from paper_2104_04726_b200.synth import CONFIGS, make_stack  # noqa: E402


def sub_angle(a, b):
    sv = np.linalg.svd(a.T @ b, compute_uv=False)
    return float(np.arccos(np.clip(sv.min(), -1, 1)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("cfg")
    ap.add_argument("scale", type=float)
    ap.add_argument("--pfrac", type=float, default=0.5)
    ap.add_argument("--iters", type=int, default=6)
    ap.add_argument("--sweeps", type=int, default=3)
    a = ap.parse_args()
    cfg = CONFIGS[a.cfg]
    h, w = int(cfg.height * a.scale), int(cfg.width * a.scale)
    ranks = [int(round(r * a.scale)) if i < 2 else r for i, r in enumerate(cfg.ranks)]
    images = make_stack(cfg, seed=1, height=h, width=w)
    x = np.asfortranarray(coding_tensor(images, cfg.space).astype(np.float32).astype(np.float64))
    print(f"{a.cfg} {x.shape} ranks {ranks} pfrac {a.pfrac}", flush=True)
    factors, warm = [], {}
    for n in range(4):
        g = gram(unfold(x, n))
        r = ranks[n]
        m = min(x.shape[n], r + int(a.pfrac * r))
        v, _ = leading_eigvecs(g, m)
        factors.append(v[:, :r])
        warm[n] = v
    for sw in range(1, a.sweeps + 1):
        for n in range(2):
            y = ttmc(x, factors, skip=n)
            g = gram(unfold(y, n))
            r = ranks[n]
            lam_all, vec_all = np.linalg.eigh(g)
            lam_all, vec_all = lam_all[::-1], vec_all[:, ::-1]
            ref = vec_all[:, :r]
            q = warm[n]
            m = q.shape[1]
            rho = lam_all[m] / lam_all[r - 1] if m < len(lam_all) else 0.0
            print(f"sweep {sw} mode {n}: n {g.shape[0]} R {r} m {m} lam1/lamR {lam_all[0]/lam_all[r-1]:.2e} "
                  f"lamR/lamR+1 {lam_all[r-1]/lam_all[r]:.6f} rho=lam(m+1)/lamR {rho:.3e} "
                  f"warm angle {sub_angle(q[:, :r], ref):.2e}", flush=True)
            for it in range(1, a.iters + 1):
                z = g @ q
                q, _ = np.linalg.qr(z)
                hq = q.T @ g @ q
                hq = 0.5 * (hq + hq.T)
                wv, vv = np.linalg.eigh(hq)
                vv = vv[:, ::-1]
                xs = q @ vv
                ang = sub_angle(xs[:, :r], ref)
                cosv = np.abs(np.einsum("ij,ij->j", xs[:, :r], ref))
                vang = np.arccos(np.clip(cosv, -1, 1)).max()
                print(f"   it {it}: top-R subspace angle {ang:.2e}  max vector angle {vang:.2e}  "
                      f"eig rel err {np.abs(wv[::-1][:r] / lam_all[:r] - 1).max():.1e}", flush=True)
            q = xs
            warm[n] = q
            factors[n] = ref


if __name__ == "__main__":
    main()
