"""numpy prototype of the two-stage tridiagonalisation (research; not product).

Stage 1 (dense -> band b): panels of b columns, Householder QR of the panel
below the band, compact-WY two-sided update of the trailing matrix.
Stage 2 (band -> tridiagonal): one-column-at-a-time bulge chasing; sweep s,
position j touches only rows block_j(s) = [s+1+jb, s+1+(j+1)b) (lower storage).
Back-transform: Q2 (reflector per (s, j)) then Q1 (WY panels).

Checks eigenvalues / eigenvectors against numpy.linalg.eigh.
"""
import sys

import numpy as np


def house(x):
    """LAPACK dlarfg: H x = beta e1, H = I - tau v v^T, v[0] = 1."""
    x = np.asarray(x, float)
    alpha = x[0]
    xn = np.linalg.norm(x[1:])
    v = np.zeros_like(x)
    v[0] = 1.0
    if xn == 0.0:
        return v, 0.0, alpha
    beta = -np.copysign(np.hypot(alpha, xn), alpha)
    tau = (beta - alpha) / beta
    v[1:] = x[1:] / (alpha - beta)
    return v, tau, beta


def sy2sb(A, b):
    A = A.copy()
    n = A.shape[0]
    panels = []
    p0 = 0
    while p0 + b < n - 1:
        r0 = p0 + b
        m = n - r0
        bw = min(b, n - p0)
        P = A[r0:, p0:p0 + bw].copy()
        nr = min(m, bw)
        if m == 1:
            break
        V = np.zeros((m, bw))
        taus = np.zeros(bw)
        for i in range(min(m - 1, bw)):
            v, tau, beta = house(P[i:, i])
            V[i:, i] = v
            taus[i] = tau
            P[i:, i + 1:] -= tau * np.outer(v, v @ P[i:, i + 1:])
            P[i, i] = beta
            P[i + 1:, i] = 0.0
        # T factor (dlarft, forward columnwise)
        T = np.zeros((bw, bw))
        for i in range(bw):
            T[i, i] = taus[i]
            if i:
                T[:i, i] = -taus[i] * T[:i, :i] @ (V[:, :i].T @ V[:, i])
        A[r0:, p0:p0 + bw] = P
        A[p0:p0 + bw, r0:] = P.T
        A22 = A[r0:, r0:]
        X = A22 @ V @ T
        M = V.T @ X
        W = X - 0.5 * V @ (T.T @ M)
        A[r0:, r0:] = A22 - V @ W.T - W @ V.T
        panels.append((r0, V, T))
        p0 += b
    return A, panels


def sb2st(Bd, b):
    """Band (dense array holding a band matrix) -> tridiagonal by bulge chasing.
    Returns d, e, reflectors dict (s, j) -> (row0, v, tau)."""
    A = Bd.copy()
    n = A.shape[0]
    refl = []
    for s in range(n - 2):
        # position 0: column s, rows [s+1, s+1+b)
        r0 = s + 1
        r1 = min(s + 1 + b, n)
        v, tau, beta = house(A[r0:r1, s])
        A[r0:r1, s] = 0.0
        A[r0, s] = beta
        A[s, r0:r1] = A[r0:r1, s]
        D = A[r0:r1, r0:r1]
        p = tau * D @ v
        K = 0.5 * tau * p @ v
        w = p - K * v
        A[r0:r1, r0:r1] = D - np.outer(v, w) - np.outer(w, v)
        refl.append((s, 0, r0, v, tau))
        j = 1
        while True:
            q0 = s + 1 + j * b
            if q0 >= n:
                break
            q1 = min(q0 + b, n)
            c0, c1 = r0, r1  # previous block columns
            B = A[q0:q1, c0:c1]
            B = B - tau * np.outer(B @ v, v)  # right apply H_{j-1}
            v2, tau2, beta2 = house(B[:, 0])
            B = B - tau2 * np.outer(v2, v2 @ B)
            B[1:, 0] = 0.0
            A[q0:q1, c0:c1] = B
            A[c0:c1, q0:q1] = B.T
            D = A[q0:q1, q0:q1]
            p = tau2 * D @ v2
            K = 0.5 * tau2 * p @ v2
            w = p - K * v2
            A[q0:q1, q0:q1] = D - np.outer(v2, w) - np.outer(w, v2)
            refl.append((s, j, q0, v2, tau2))
            r0, r1, v, tau = q0, q1, v2, tau2
            j += 1
    d = np.diag(A).copy()
    e = np.diag(A, -1).copy()
    off = np.tril(A, -2)
    return d, e, refl, np.abs(off).max()


def backtransform(n, refl, panels, Z):
    X = Z.copy()
    for (s, j, q0, v, tau) in reversed(refl):
        L = len(v)
        X[q0:q0 + L] -= tau * np.outer(v, v @ X[q0:q0 + L])
    for (r0, V, T) in reversed(panels):
        X[r0:] -= V @ (T @ (V.T @ X[r0:]))
    return X


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 200
    b = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    rng = np.random.default_rng(1)
    q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    lam = np.exp(-np.linspace(0, 20, n))
    G = (q * lam) @ q.T
    G = 0.5 * (G + G.T)
    Bd, panels = sy2sb(G, b)
    band_off = np.abs(np.tril(Bd, -b - 1)).max()
    d, e, refl, off = sb2st(Bd, b)
    T = np.diag(d) + np.diag(e, -1) + np.diag(e, 1)
    w, Z = np.linalg.eigh(T)
    X = backtransform(n, refl, panels, Z)
    wr, Xr = np.linalg.eigh(G)
    print(f"n={n} b={b}: band leak {band_off:.1e}, tri leak {off:.1e}, eig err {np.abs(w - wr).max():.1e}, "
          f"resid {np.abs(G @ X - X * w).max():.1e}, ortho {np.abs(X.T @ X - np.eye(n)).max():.1e}")


if __name__ == "__main__":
    main()


def sb2st_band(Bd, b, order="wave"):
    """Same algorithm on lower band storage L[r, o] = A[r, r - o], o in [0, 2b),
    tasks executed in wavefront order (key 2s + j): each task reads/writes only
    the rows of its block (the symmetric halves it needs are rebuilt locally)."""
    n = Bd.shape[0]
    W = 2 * b
    L = np.zeros((n, W))
    for r in range(n):
        for o in range(W):
            if r - o >= 0:
                L[r, o] = Bd[r, r - o]
    tasks = []
    for s in range(n - 2):
        j = 0
        while s + 1 + j * b < n:
            tasks.append((2 * s + j, s, j))
            j += 1
    if order == "wave":
        tasks.sort()
    H = {}
    refl = []
    for _, s, j in tasks:
        q0 = s + 1 + j * b
        q1 = min(q0 + b, n)
        m = q1 - q0
        if j == 0:
            x = np.array([L[r, r - s] for r in range(q0, q1)])
            v, tau, beta = house(x)
            for i, r in enumerate(range(q0, q1)):
                L[r, r - s] = beta if i == 0 else 0.0
        else:
            c0 = q0 - b
            vp, taup = H[(s, j - 1)]
            cw = len(vp)
            B = np.array([[L[r, r - c] for c in range(c0, c0 + cw)] for r in range(q0, q1)])
            B = B - taup * np.outer(B @ vp, vp)
            v, tau, beta = house(B[:, 0])
            B = B - tau * np.outer(v, v @ B)
            B[1:, 0] = 0.0
            for i, r in enumerate(range(q0, q1)):
                for jj, c in enumerate(range(c0, c0 + cw)):
                    L[r, r - c] = B[i, jj]
        D = np.array([[L[max(r, c), abs(r - c)] for c in range(q0, q1)] for r in range(q0, q1)])
        p = tau * D @ v
        K = 0.5 * tau * p @ v
        w = p - K * v
        D = D - np.outer(v, w) - np.outer(w, v)
        for i, r in enumerate(range(q0, q1)):
            for jj, c in enumerate(range(q0, r + 1)):
                L[r, r - c] = D[i, jj]
        H[(s, j)] = (v, tau)
        refl.append((s, j, q0, v, tau))
    refl.sort(key=lambda t: (t[0], t[1]))
    d = L[:, 0].copy()
    e = L[1:, 1].copy()
    return d, e, refl


def check_band(n=120, b=8):
    rng = np.random.default_rng(2)
    G = rng.standard_normal((n, n))
    G = G + G.T
    Bd, panels = sy2sb(G, b)
    d0, e0, r0, _ = sb2st(Bd, b)
    d1, e1, r1 = sb2st_band(Bd, b, "seq")
    d2, e2, r2 = sb2st_band(Bd, b, "wave")
    print("band seq vs dense:", np.abs(d1 - d0).max(), np.abs(e1 - e0).max(),
          "wave vs seq bitwise:", np.array_equal(d1, d2) and np.array_equal(e1, e2))
