"""float64 numpy restatement of the reference Tucker-ALS path (test oracle only).

Conventions follow the reference: tensors are ndarrays whose logical
linearisation is mode-0-fastest (Fortran order), the mode-n unfolding is
``s_n x prod(others)`` with the lowest remaining mode fastest
(``tensor.py:1-13``), factors are ``s_n x r_n`` with orthonormal columns.
Reference paths are relative to ``/root/reference/pkg/src/tmcodec/``.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

__all__ = [
    "unfold", "fold", "ttm", "ttmc", "gram", "leading_eigvecs", "sign_fix",
    "fro_norm", "hosvd", "t_hosvd", "hooi_sweep", "reconstruct", "fit",
    "pp_operators", "pp_sweep", "tucker_als", "Trace", "quantize_core",
    "dequantize_core", "preset_ranks", "rgb_to_ycbcr", "rgb_to_ipt",
    "ycbcr_to_rgb", "ipt_to_rgb", "coding_tensor", "dequantize_model", "decode_stack", "scene_mse",
    "varint_encode_ints", "varint_decode_ints", "serialize_latent_channel",
    "ORTHO_TOL", "PP_DIP_TOL",
]

ORTHO_TOL = 1e-8          # tucker.py:44
PP_DIP_TOL = 1e-6         # tucker.py:45


# ---------------------------------------------------------------- tensor.py
def unfold(x: np.ndarray, mode: int) -> np.ndarray:
    """Mode-n unfolding (tensor.py:89-94): rows = mode n, columns = the other
    modes in ascending order with the lowest fastest."""
    perm = [mode] + [m for m in range(x.ndim) if m != mode]
    return np.transpose(x, perm).reshape(x.shape[mode], -1, order="F")


def fold(m: np.ndarray, mode: int, dims) -> np.ndarray:
    """Inverse of unfold (tensor.py:97-108)."""
    dims = tuple(int(d) for d in dims)
    rest = [d for i, d in enumerate(dims) if i != mode]
    arr = np.reshape(m, [dims[mode]] + rest, order="F")
    inv = np.argsort([mode] + [i for i in range(len(dims)) if i != mode])
    return np.transpose(arr, inv)


def ttm(x: np.ndarray, m: np.ndarray, mode: int) -> np.ndarray:
    """Mode-n product, dims[mode] -> m.shape[0] (tensor.py:111-123)."""
    dims = list(x.shape)
    dims[mode] = m.shape[0]
    return fold(np.asarray(m, np.float64) @ unfold(x, mode), mode, dims)


def _greedy(x: np.ndarray, factors, modes, transpose: bool):
    """Most size-reducing mode first, stable on ties (tensor.py:126-135)."""
    def ratio(n):
        f = np.asarray(factors[n])
        return (f.shape[1] if transpose else f.shape[0]) / x.shape[n]
    return sorted(modes, key=ratio)


def ttmc(x: np.ndarray, factors, skip=None, transpose=True, order="ascending") -> np.ndarray:
    """Multi-mode product with every factor but ``skip`` (tensor.py:138-173)."""
    modes = [n for n in range(x.ndim) if n != skip]
    if order == "greedy":
        modes = _greedy(x, factors, modes, transpose)
    out = x
    for n in modes:
        f = np.asarray(factors[n], np.float64)
        out = ttm(out, f.T if transpose else f, n)
    return out


def gram(m: np.ndarray) -> np.ndarray:
    """m m^T with the upper triangle mirrored (tensor.py:176-180)."""
    g = m @ m.T
    up = np.triu(g)
    return up + np.triu(g, 1).T


def sign_fix(v: np.ndarray) -> np.ndarray:
    """Flip each column whose first max-|entry| is negative (tensor.py:203-209)."""
    v = v.copy()
    for j in range(v.shape[1]):
        i = int(np.argmax(np.abs(v[:, j])))
        if v[i, j] < 0:
            v[:, j] = -v[:, j]
    return v


def leading_eigvecs(g: np.ndarray, k: int):
    """Top-k eigenpairs, eigenvalues nonincreasing, sign rule (tensor.py:183-200)."""
    w, v = np.linalg.eigh(np.asarray(g, np.float64))
    n = g.shape[0]
    idx = list(range(n - 1, n - 1 - k, -1))
    return sign_fix(v[:, idx]), w[idx]


def fro_norm(x: np.ndarray) -> float:
    """sqrt of the sum of squares (tensor.py:212-214)."""
    return float(np.linalg.norm(np.ravel(x)))


# ---------------------------------------------------------------- tucker.py
def hosvd(x: np.ndarray):
    """Full HOSVD (tucker.py:120-127)."""
    return t_hosvd(x, x.shape)


def t_hosvd(x: np.ndarray, ranks, order="ascending"):
    """Truncated HOSVD: per-mode Gram eigenvectors, core by projection
    (tucker.py:130-148). Returns (core, factors)."""
    factors = [leading_eigvecs(gram(unfold(x, n)), int(ranks[n]))[0] for n in range(x.ndim)]
    return ttmc(x, factors, order=order), factors


def hooi_sweep(x: np.ndarray, factors, order="ascending"):
    """Gauss-Seidel HOOI sweep (tucker.py:151-163): factor n is replaced before
    mode n+1 is processed, then the core is re-projected."""
    factors = list(factors)
    for n in range(x.ndim):
        y = ttmc(x, factors, skip=n, order=order)
        factors[n] = leading_eigvecs(gram(unfold(y, n)), factors[n].shape[1])[0]
    return ttmc(x, factors, order=order), factors


def reconstruct(core: np.ndarray, factors) -> np.ndarray:
    """core x_0 S_0 x_1 S_1 ... in ascending order (tucker.py:166-171)."""
    out = core
    for n, f in enumerate(factors):
        out = ttm(out, f, n)
    return out


def fit(x: np.ndarray, core: np.ndarray, factors=None, method="core") -> float:
    """1 - ||x - x_hat|| / ||x|| (tucker.py:174-191)."""
    tn = fro_norm(x)
    if method == "core":
        cn = fro_norm(core)
        resid = math.sqrt(max(tn * tn - cn * cn, 0.0))
    else:
        resid = float(np.linalg.norm((x - reconstruct(core, factors)).ravel()))
    return 1.0 - resid / tn


# pairwise perturbation (tucker.py:199-311)
@dataclass
class PPOps:
    anchors: list
    single: list
    pair: dict
    count: int


def pp_operators(x: np.ndarray, anchors) -> PPOps:
    """Dimension tree keyed by the free-mode set; a node's parent re-adds the
    largest contracted mode, so every node is an ascending contraction
    (tucker.py:222-265)."""
    n_modes = x.ndim
    memo = {frozenset(range(n_modes)): x}
    count = [0]

    def node(free):
        if free in memo:
            return memo[free]
        m = max(i for i in range(n_modes) if i not in free)
        out = ttm(node(free | {m}), np.asarray(anchors[m], np.float64).T, m)
        count[0] += 1
        memo[free] = out
        return out

    single = [node(frozenset((n,))) for n in range(n_modes)]
    pair = {(i, n): node(frozenset((i, n))) for i in range(n_modes) for n in range(i + 1, n_modes)}
    return PPOps([np.asarray(a, np.float64) for a in anchors], single, pair, count[0])


def pp_sweep(ops: PPOps, factors, return_operands=False):
    """First-order PP sweep with entry deltas (tucker.py:268-311). Returns
    (pp_core, factors[, operands])."""
    deltas = [f - a for f, a in zip(factors, ops.anchors)]
    factors = list(factors)
    operands = []
    y = None
    for n in range(len(factors)):
        y = ops.single[n]
        acc = None
        for i in range(len(factors)):
            if i == n or not np.any(deltas[i]):
                continue
            p = ops.pair[(i, n) if i < n else (n, i)]
            corr = ttm(p, deltas[i].T, i)
            acc = corr if acc is None else acc + corr
        if acc is not None:
            y = y + acc
        operands.append(y)
        factors[n] = leading_eigvecs(gram(unfold(y, n)), factors[n].shape[1])[0]
    last = len(factors) - 1
    core = ttm(y, factors[last].T, last)
    if return_operands:
        return core, factors, operands
    return core, factors


@dataclass
class Trace:
    rows: list = field(default_factory=list)  # (index, kind, fit, max_change)
    converged: bool = False


def _max_change(new, old) -> float:
    """tucker.py:319-323."""
    out = 0.0
    for a, b in zip(new, old):
        out = max(out, float(np.linalg.norm(a - b)) / float(np.linalg.norm(b)))
    return out


def tucker_als(x: np.ndarray, ranks, max_sweeps=50, fit_tol=1e-5, pp_enter_tol=0.1,
               pp_exit_tol=0.3, sequential_reduction=True):
    """Driver (tucker.py:331-397): T-HOSVD init, standard sweeps, optional PP
    phase, stop on |dfit| < fit_tol, best-fit model when not converged.
    Returns (core, factors, Trace)."""
    if fro_norm(x) == 0.0:
        raise ValueError("cannot decompose the zero tensor")
    order = "ascending" if sequential_reduction else "greedy"
    trace = Trace()
    core, factors = t_hosvd(x, ranks, order)
    cur = fit(x, core)
    trace.rows.append((0, "init", cur, math.nan))
    best = (cur, core, factors)
    if cur >= 1.0 - fit_tol:
        trace.converged = True
        return core, factors, trace
    phase_pp, ops = False, None
    for sweep in range(1, max_sweeps + 1):
        if phase_pp:
            deltas_ok = max(float(np.linalg.norm(f - a)) / float(np.linalg.norm(a))
                            for f, a in zip(factors, ops.anchors)) <= pp_exit_tol
            cand = None
            if deltas_ok:
                _, fac_pp = pp_sweep(ops, factors)
                cand = (ttmc(x, fac_pp, order=order), fac_pp)
                if fit(x, cand[0]) < cur - PP_DIP_TOL:
                    cand = None
            if cand is None:
                new_core, new_fac = hooi_sweep(x, factors, order)
                kind = "standard"
                ops = pp_operators(x, new_fac)
            else:
                new_core, new_fac = cand
                kind = "pp"
        else:
            new_core, new_fac = hooi_sweep(x, factors, order)
            kind = "standard"
        change = _max_change(new_fac, factors)
        new_fit = fit(x, new_core)
        trace.rows.append((sweep, kind, new_fit, change))
        if new_fit > best[0]:
            best = (new_fit, new_core, new_fac)
        if kind == "standard" and not phase_pp and pp_enter_tol > 0 and change < pp_enter_tol:
            phase_pp = True
            ops = pp_operators(x, new_fac)
        done = abs(new_fit - cur) < fit_tol
        core, factors, cur = new_core, new_fac, new_fit
        if done:
            trace.converged = True
            break
    if not trace.converged:
        _, core, factors = best
    return core, factors, trace


# ---------------------------------------------------------------- codec.py
def preset_ranks(preset: int, dims):
    """RANK k -> (H, W, E, V) ranks (codec.py:86-95)."""
    h, w, e, v = dims

    def spatial(s):
        return min(s, max(1, math.ceil(math.ceil(preset * s / 5) * 0.25)))

    return (spatial(h), spatial(w), min(preset, e), min(preset, v))


def quantize_core(core: np.ndarray, qp: int):
    """Uniform quantiser, step = amax 2^((qp-51)/6) 2^-8, round half away
    (codec.py:98-99, 114-134). Returns (levels int64, step)."""
    amax = float(np.max(np.abs(core))) if core.size else 0.0
    step = amax * 2.0 ** ((qp - 51) / 6.0) * 2.0 ** -8 if amax > 0.0 else 1.0
    q = core / step
    levels = (np.sign(q) * np.floor(np.abs(q) + 0.5)).astype(np.int64)
    return levels, step


def dequantize_core(levels: np.ndarray, step: float) -> np.ndarray:
    """codec.py:137-148 (core part)."""
    return levels.astype(np.float64) * step


# ---------------------------------------------------------------- color.py
_KR, _KG, _KB = 0.299, 0.587, 0.114                    # color.py:40
_M_RGB_XYZ = np.array([[0.4124564, 0.3575761, 0.1804375],
                       [0.2126729, 0.7151522, 0.0721750],
                       [0.0193339, 0.1191920, 0.9503041]])   # color.py:43-49
_HPE = np.array([[0.4002, 0.7075, -0.0807],
                 [-0.2280, 1.1500, 0.0612],
                 [0.0000, 0.0000, 0.9184]])                   # color.py:54-60
_M_XYZ_LMS = _HPE / (_HPE @ (_M_RGB_XYZ @ np.ones(3)))[:, None]  # color.py:61-62
_M_LMS_IPT = np.array([[0.4000, 0.4000, 0.2000],
                       [4.4550, -4.8510, 0.3960],
                       [0.8056, 0.3572, -1.1628]])            # color.py:66-72


def rgb_to_ycbcr(px: np.ndarray) -> np.ndarray:
    """Full-range BT.601 + clip (color.py:111-119). px: (..., 3) in [0, 1]."""
    r, g, b = px[..., 0], px[..., 1], px[..., 2]
    y = _KR * r + _KG * g + _KB * b
    cb = 0.5 * (b - y) / (1.0 - _KB) + 0.5
    cr = 0.5 * (r - y) / (1.0 - _KR) + 0.5
    return np.clip(np.stack([y, cb, cr], axis=-1), 0.0, 1.0)


def ycbcr_to_rgb(px: np.ndarray) -> np.ndarray:
    """color.py:122-128."""
    y, cb, cr = px[..., 0], px[..., 1], px[..., 2]
    r = y + 2.0 * (1.0 - _KR) * (cr - 0.5)
    b = y + 2.0 * (1.0 - _KB) * (cb - 0.5)
    g = (y - _KR * r - _KB * b) / _KG
    return np.stack([r, g, b], axis=-1)


def _eotf(v):
    """sRGB decode (color.py:131-133)."""
    return np.where(v > 0.04045, ((v + 0.055) / 1.055) ** 2.4, v / 12.92)


def _oetf(v):
    """sRGB encode (color.py:136-138)."""
    return np.where(v > 0.0031308, 1.055 * np.maximum(v, 0.0) ** (1.0 / 2.4) - 0.055, 12.92 * v)


def rgb_to_ipt(px: np.ndarray) -> np.ndarray:
    """EOTF -> XYZ -> HPE LMS -> signed ^0.43 -> IPT, chroma*0.5+0.5
    (color.py:145-158)."""
    lms = _eotf(px) @ _M_RGB_XYZ.T @ _M_XYZ_LMS.T
    lmsp = np.sign(lms) * np.abs(lms) ** 0.43
    ipt = lmsp @ _M_LMS_IPT.T
    out = ipt.copy()
    out[..., 1:] = 0.5 * ipt[..., 1:] + 0.5
    return out


def ipt_to_rgb(px: np.ndarray, count_clamped=False):
    """Algebraic inverse with linear-RGB clamp (color.py:161-182)."""
    ipt = px.copy()
    ipt[..., 1:] = 2.0 * (px[..., 1:] - 0.5)
    lmsp = ipt @ np.linalg.inv(_M_LMS_IPT).T
    lms = np.sign(lmsp) * np.abs(lmsp) ** (1.0 / 0.43)
    lin = lms @ np.linalg.inv(_M_XYZ_LMS).T @ np.linalg.inv(_M_RGB_XYZ).T
    cl = np.clip(lin, 0.0, 1.0)
    out = _oetf(cl)
    if count_clamped:
        return out, int(np.count_nonzero(np.any(cl != lin, axis=-1)))
    return out


def coding_tensor(images_u8: np.ndarray, space: str) -> np.ndarray:
    """(V, E, H, W, 3) uint8 -> (H, W, 3, V*E) float64 coding-space tensor,
    index v*E + e (the BASELINE.json layout)."""
    v_, e_, h, w, _ = images_u8.shape
    fn = rgb_to_ycbcr if space == "ycbcr" else rgb_to_ipt
    out = np.empty((h, w, 3, v_ * e_), order="F")
    for v in range(v_):
        for e in range(e_):
            out[:, :, :, v * e_ + e] = fn(images_u8[v, e].astype(np.float64) / 255.0)
    return out


# ---------------------------------------------------------------- decode side
def dequantize_model(levels: np.ndarray, step: float, factors):
    """codec.py:137-148: core = levels * step, float32 factors upcast."""
    return levels.astype(np.float64) * step, [np.asarray(f, dtype=np.float32).astype(np.float64) for f in factors]


def decode_stack(core: np.ndarray, factors, space: str, views: int, exposures: int):
    """reconstruct (tucker.py:166-171) then to_rgb per image (color.py:197-205):
    (V, E, H, W, 3) float64 RGB from a (H, W, 3, V*E) model (tensor_to_stack's
    plane order)."""
    t = reconstruct(core, factors)
    h, w, _, _ = t.shape
    out = np.empty((views, exposures, h, w, 3))
    for v in range(views):
        for e in range(exposures):
            px = np.ascontiguousarray(t[:, :, :, v * exposures + e])
            if space == "ycbcr":
                out[v, e] = ycbcr_to_rgb(px)
            elif space == "ipt":
                out[v, e] = ipt_to_rgb(px)
            else:
                out[v, e] = px
    return out


def scene_mse(images_u8: np.ndarray, rgb: np.ndarray) -> np.ndarray:
    """metrics.mse(ref.pixels*255, test.pixels*255) per (view, exposure)
    (metrics.py:16-23, as scene_psnr calls it at :58-62)."""
    ref = images_u8.astype(np.float64) / 255.0 * 255.0
    d = ref - rgb * 255.0
    return np.mean(d * d, axis=(2, 3, 4))


# ---------------------------------------------------------------- latent block bytes
def varint_encode_ints(values: np.ndarray) -> bytes:
    """encode_ints (entropy.py:55-111): zigzag then LEB128, low group first."""
    out = bytearray()
    for v in np.asarray(values, dtype=np.int64).ravel():
        u = ((int(v) << 1) ^ (int(v) >> 63)) & 0xFFFFFFFFFFFFFFFF
        while True:
            b = u & 0x7F
            u >>= 7
            if u:
                out.append(b | 0x80)
            else:
                out.append(b)
                break
    return bytes(out)


def varint_decode_ints(data: bytes, count: int):
    """decode_ints (entropy.py:88-117): (int64 values, bytes consumed)."""
    vals, pos = [], 0
    for _ in range(count):
        u, shift, nb = 0, 0, 0
        while True:
            if pos >= len(data):
                raise ValueError("varint stream truncated")
            b = data[pos]
            pos += 1
            nb += 1
            u |= (b & 0x7F) << shift
            shift += 7
            if b < 0x80:
                break
        if nb > 10:
            raise ValueError("varint longer than 10 bytes")
        vals.append((u >> 1) ^ -(u & 1))
    return np.array(vals, dtype=np.int64), pos


def serialize_latent_channel(levels: np.ndarray, step: float, factors) -> bytes:
    """_serialize_latent_channel (codec.py:285-291)."""
    import struct

    out = bytearray()
    for f in factors:
        out += np.asarray(f, dtype="<f4").tobytes(order="F")
    out += varint_encode_ints(np.asarray(levels).ravel(order="F"))
    out += struct.pack("<d", step)
    return bytes(out)
