"""Tucker decomposition solvers on the B200 (drop-in for the reference's ``tucker.py``).

Same public surface (tucker.py:28-42): ``TuckerModel``, ``SolveConfig``,
``SweepRecord``, ``SolveTrace``, ``PPState``, ``hosvd``, ``t_hosvd``,
``hooi_sweep``, ``reconstruct``, ``fit``, ``pp_operators``, ``pp_sweep``,
``tucker_als``. The solve loop (T-HOSVD, memoised Gauss-Seidel HOOI sweeps,
fit trace, convergence, best-of) runs natively in libtmb
(``tmb_tucker_als``); tensors stay resident on the device for the whole solve.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Sequence

import numpy as np

from . import _lib as L
from .tensor import DenseTensor, fro_norm, gram, leading_eigvecs, ttm, unfold

__all__ = [
    "TuckerModel", "SolveConfig", "SweepRecord", "SolveTrace", "PPState", "hosvd", "t_hosvd",
    "hooi_sweep", "reconstruct", "fit", "pp_operators", "pp_sweep", "tucker_als",
]

ORTHO_TOL = 1e-8   # tucker.py:44
PP_DIP_TOL = 1e-6  # tucker.py:45


@dataclass
class TuckerModel:
    """Core tensor plus per-mode orthonormal factor matrices (tucker.py:48-71)."""

    core: DenseTensor
    factors: list[np.ndarray]
    source_dims: tuple[int, ...]

    @property
    def ranks(self) -> tuple[int, ...]:
        return self.core.dims

    def validate(self, ortho_tol: float = ORTHO_TOL) -> None:
        if len(self.factors) != self.core.ndim or len(self.factors) != len(self.source_dims):
            raise ValueError("factor count does not match tensor order")
        for n, f in enumerate(self.factors):
            s, r = self.source_dims[n], self.core.dims[n]
            if f.shape != (s, r):
                raise ValueError(f"mode {n}: factor shape {f.shape}, expected {(s, r)}")
            if r > s:
                raise ValueError(f"mode {n}: rank {r} exceeds dimension {s}")
            err = float(np.max(np.abs(_cross_gram(f) - np.eye(r))))
            if err >= ortho_tol:
                raise ValueError(f"mode {n}: factor columns not orthonormal (err={err:.2e})")


def _cross_gram(f: np.ndarray) -> np.ndarray:
    """f^T f on the device (gram of f^T)."""
    return gram(np.asarray(f, dtype=np.float64).T)


@dataclass
class SolveConfig:
    """Solver knobs (tucker.py:74-95)."""

    ranks: tuple[int, ...]
    max_sweeps: int = 50
    fit_tol: float = 1e-5
    pp_enter_tol: float = 0.1
    pp_exit_tol: float = 0.3
    sequential_reduction: bool = True
    seed: int = 0

    def validate(self, dims: Sequence[int]) -> None:
        if len(self.ranks) != len(dims):
            raise ValueError(f"{len(self.ranks)} ranks for an order-{len(dims)} tensor")
        for n, (r, s) in enumerate(zip(self.ranks, dims)):
            if not 1 <= r <= s:
                raise ValueError(f"mode {n}: rank {r} not in [1, {s}]")
        if self.fit_tol <= 0 or self.pp_exit_tol <= 0:
            raise ValueError("tolerances must be positive")
        if self.max_sweeps < 0:
            raise ValueError("max_sweeps must be >= 0")

    def to_c(self) -> L.SolveCfg:
        return L.SolveCfg(int(self.max_sweeps), float(self.fit_tol), float(self.pp_enter_tol),
                          float(self.pp_exit_tol), 1 if self.sequential_reduction else 0)


@dataclass
class SweepRecord:
    index: int
    kind: str
    fit: float
    max_change: float


@dataclass
class SolveTrace:
    records: list[SweepRecord] = field(default_factory=list)
    converged: bool = False

    def rows(self) -> list[tuple]:
        return [(r.index, r.kind, r.fit, r.max_change) for r in self.records]


def _order(order: str) -> int:
    if order not in ("ascending", "greedy"):
        raise ValueError(f"unknown contraction order {order!r}")
    return 1 if order == "greedy" else 0


def _check_ranks(ranks, dims) -> tuple[int, ...]:
    ranks = tuple(int(r) for r in ranks)
    if len(ranks) != len(dims):
        raise ValueError(f"{len(ranks)} ranks for an order-{len(dims)} tensor")
    for n, (r, s) in enumerate(zip(ranks, dims)):
        if not 1 <= r <= s:
            raise ValueError(f"mode {n}: rank {r} not in [1, {s}]")
    return ranks


def _model_from_dev(core_d, fac_d, ranks, dims) -> TuckerModel:
    core = DenseTensor(L.host_f(core_d, tuple(ranks)))
    factors = [L.host_f(f, (dims[n], ranks[n])) for n, f in enumerate(fac_d)]
    return TuckerModel(core, factors, tuple(dims))


def hosvd(t: DenseTensor) -> TuckerModel:
    """Full HOSVD (tucker.py:120-127)."""
    return t_hosvd(t, t.dims)


def t_hosvd(t: DenseTensor, ranks: Sequence[int], order: str = "ascending") -> TuckerModel:
    """Truncated HOSVD (tucker.py:130-148) on the device."""
    ranks = _check_ranks(ranks, t.dims)
    greedy = _order(order)
    h = L.ctx()
    x = L.dev_f64(t.array)
    core = L.empty_f64(int(np.prod(ranks)))
    facs = [L.empty_f64(s * r) for s, r in zip(t.dims, ranks)]
    L.check(L.LIB.tmb_t_hosvd(h, L.ptr(x), L.F64, t.ndim, L.i64s(t.dims), L.i64s(ranks), greedy, L.ptr(core),
                              L.ptrs(facs)), h)
    return _model_from_dev(core, facs, ranks, t.dims)


def hooi_sweep(t: DenseTensor, model: TuckerModel, order: str = "ascending") -> TuckerModel:
    """One Gauss-Seidel HOOI sweep (tucker.py:151-163) on the device."""
    if tuple(model.source_dims) != tuple(t.dims):
        raise ValueError(f"model dims {model.source_dims} do not match tensor dims {t.dims}")
    ranks = tuple(model.ranks)
    greedy = _order(order)
    h = L.ctx()
    x = L.dev_f64(t.array)
    fin = [L.dev_f64(f) for f in model.factors]
    core = L.empty_f64(int(np.prod(ranks)))
    fout = [L.empty_f64(s * r) for s, r in zip(t.dims, ranks)]
    L.check(L.LIB.tmb_hooi_sweep(h, L.ptr(x), L.F64, t.ndim, L.i64s(t.dims), L.i64s(ranks), L.ptrs(fin), greedy,
                                 L.ptr(core), L.ptrs(fout)), h)
    return _model_from_dev(core, fout, ranks, t.dims)


def reconstruct(model: TuckerModel) -> DenseTensor:
    """Core multiplied by each factor along its mode (tucker.py:166-171)."""
    ranks = tuple(model.core.dims)
    dims = tuple(f.shape[0] for f in model.factors)
    h = L.ctx()
    core = L.dev_f64(model.core.array)
    facs = [L.dev_f64(f) for f in model.factors]
    out = L.empty_f64(int(np.prod(dims)))
    L.check(L.LIB.tmb_reconstruct(h, len(ranks), L.i64s(ranks), L.i64s(dims), L.ptr(core), L.ptrs(facs),
                                  L.ptr(out)), h)
    return DenseTensor(L.host_f(out, dims))


def fit(t: DenseTensor, model: TuckerModel, method: str = "core") -> float:
    """1 - ||t - t_hat|| / ||t|| (tucker.py:174-191)."""
    tn = fro_norm(t)
    if tn == 0.0:
        raise ValueError("fit is undefined for the zero tensor")
    if method == "core":
        cn = fro_norm(model.core)
        resid = math.sqrt(max(tn * tn - cn * cn, 0.0))
    elif method == "residual":
        rec = reconstruct(model)
        if rec.dims != t.dims:
            raise ValueError(f"model reconstructs dims {rec.dims}, tensor is {t.dims}")
        h = L.ctx()
        x = L.dev_f64(t.array)
        r = L.dev_f64(rec.array)
        out = L.C.c_double()
        L.check(L.LIB.tmb_resid_sumsq(h, L.ptr(x), L.F64, L.ptr(r), t.size, L.C.byref(out)), h)
        resid = math.sqrt(out.value)
    else:
        raise ValueError(f"unknown fit method {method!r}")
    return 1.0 - resid / tn


# ---------------------------------------------------------------------------
# pairwise perturbation (tucker.py:199-311): dimension tree of device TTMs
# ---------------------------------------------------------------------------


class PPState:
    """Anchor factors, their drift and the skip-one / skip-two operators
    (tucker.py:199-219), held by libtmb's native ``tmb_pp`` handle on the
    device. ``op_single`` / ``op_pair`` are host views fetched on first access;
    ``deltas`` may be assigned as in the reference (it is uploaded before the
    next ``pp_sweep``)."""

    def __init__(self, handle, dims, ranks, anchors, count: int):
        self._h = L.C.c_void_p(handle)
        self._dims = tuple(dims)
        self._ranks = tuple(ranks)
        self.anchors = [np.asarray(a, dtype=np.float64) for a in anchors]
        self._deltas = [np.zeros_like(a) for a in self.anchors]
        self._dirty = False          # host deltas newer than the device copy
        self._max_rel = 0.0
        self.contraction_count = int(count)
        self._single = None
        self._pair = None

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            L.LIB.tmb_pp_destroy(h)

    def _op(self, mask: int) -> DenseTensor:
        d = (L.C.c_int64 * len(self._dims))()
        p = L.C.c_void_p()
        if L.LIB.tmb_pp_operator(self._h, mask, L.C.byref(p), d) != L.TMB_OK:
            raise RuntimeError(f"pp operator {mask} unavailable")
        dims = tuple(int(v) for v in d)
        out = L.empty_f64(int(np.prod(dims)))
        h = L.ctx()
        L.check(L.LIB.tmb_pp_operator_copy(h, self._h, mask, L.ptr(out)), h)
        return DenseTensor(L.host_f(out, dims))

    @property
    def op_single(self) -> list[DenseTensor]:
        if self._single is None:
            self._single = [self._op(1 << n) for n in range(len(self._dims))]
        return self._single

    @property
    def op_pair(self) -> dict[tuple[int, int], DenseTensor]:
        if self._pair is None:
            n_modes = len(self._dims)
            self._pair = {(i, n): self._op((1 << i) | (1 << n)) for i in range(n_modes) for n in range(i + 1, n_modes)}
        return self._pair

    def pair(self, i: int, n: int) -> DenseTensor:
        return self.op_pair[(i, n) if i < n else (n, i)]

    @property
    def deltas(self) -> list[np.ndarray]:
        return self._deltas

    @deltas.setter
    def deltas(self, value) -> None:
        self._deltas = [np.asarray(d, dtype=np.float64) for d in value]
        self._dirty = True

    def _upload(self, mats, are_factors: bool) -> float:
        h = L.ctx()
        dev = [L.dev_f64(m) for m in mats]
        mr = L.C.c_double()
        L.check(L.LIB.tmb_pp_set_deltas(h, self._h, L.ptrs(dev), 1 if are_factors else 0, L.C.byref(mr)), h)
        return float(mr.value)

    def set_current(self, factors: Sequence[np.ndarray]) -> None:
        """deltas = factors - anchors, on the device (tucker.py:212-213)."""
        self._max_rel = self._upload(factors, True)
        self._deltas = [np.asarray(f, dtype=np.float64) - a for f, a in zip(factors, self.anchors)]
        self._dirty = False

    def max_rel_delta(self) -> float:
        """max_n ||d_n|| / ||a_n|| (tucker.py:215-219)."""
        if self._dirty:
            self._max_rel = self._upload(self._deltas, False)
            self._dirty = False
        return self._max_rel


def pp_operators(t: DenseTensor, anchors: Sequence[np.ndarray]) -> PPState:
    """Skip-one and skip-two contractions through the memoised dimension tree
    whose parent re-adds the largest contracted mode (tucker.py:222-265), built
    natively in one call (``tmb_pp_operators``)."""
    n_modes = t.ndim
    if len(anchors) != n_modes:
        raise ValueError(f"expected {n_modes} anchors, got {len(anchors)}")
    for n, a in enumerate(anchors):
        a = np.asarray(a)
        if a.ndim != 2 or a.shape[0] != t.dims[n]:
            raise ValueError(f"mode {n}: anchor shape {a.shape} does not match dim {t.dims[n]}")
    ranks = tuple(int(np.asarray(a).shape[1]) for a in anchors)
    h = L.ctx()
    x = L.dev_f64(t.array)
    dev = [L.dev_f64(a) for a in anchors]
    out = L.C.c_void_p()
    L.check(L.LIB.tmb_pp_operators(h, L.ptr(x), L.F64, n_modes, L.i64s(t.dims), L.i64s(ranks), L.ptrs(dev),
                                   L.C.byref(out)), h)
    cnt = L.C.c_int()
    L.LIB.tmb_pp_info(out, None, L.C.byref(cnt))
    return PPState(out.value, t.dims, ranks, anchors, cnt.value)


def pp_sweep(state: PPState, model: TuckerModel, return_operands: bool = False):
    """One accelerated sweep from the precomputed operators and the entry
    deltas (tucker.py:285-311), one native call (``tmb_pp_sweep``); the core is
    the pp estimate Y_{N-1} x_{N-1} S_{N-1}^T, as in the reference."""
    if state._dirty:
        state.max_rel_delta()
    dims, ranks = state._dims, tuple(model.ranks)
    if ranks != state._ranks:
        raise ValueError(f"model ranks {ranks} do not match the pp operators' {state._ranks}")
    n_modes = len(dims)
    h = L.ctx()
    core = L.empty_f64(int(np.prod(ranks)))
    facs = [L.empty_f64(s * r) for s, r in zip(dims, ranks)]
    op_dims = [tuple(dims[m] if m == n else ranks[m] for m in range(n_modes)) for n in range(n_modes)]
    ops = [L.empty_f64(int(np.prod(d))) for d in op_dims] if return_operands else None
    L.check(L.LIB.tmb_pp_sweep(h, state._h, L.ptr(core), L.ptrs(facs), L.ptrs(ops) if ops else None), h)
    out = _model_from_dev(core, facs, ranks, model.source_dims)
    if return_operands:
        return out, [DenseTensor(L.host_f(o, d)) for o, d in zip(ops, op_dims)]
    return out


# ---------------------------------------------------------------------------
# full solve
# ---------------------------------------------------------------------------


def tucker_als(t: DenseTensor, cfg: SolveConfig) -> tuple[TuckerModel, SolveTrace]:
    """Tucker-ALS (tucker.py:331-397) solved end to end in libtmb."""
    cfg.validate(t.dims)
    return solve_device(L.dev_f64(t.array), L.F64, t.dims, cfg)


def solve_device(x_dev, dtype: int, dims: Sequence[int], cfg: SolveConfig) -> tuple[TuckerModel, SolveTrace]:
    """tucker_als on a tensor already resident on the device (F-order)."""
    dims = tuple(int(d) for d in dims)
    cfg.validate(dims)
    ranks = tuple(int(r) for r in cfg.ranks)
    h = L.ctx()
    core = L.empty_f64(int(np.prod(ranks)))
    facs = [L.empty_f64(s * r) for s, r in zip(dims, ranks)]
    tr, keep = _trace_buffers(cfg.max_sweeps + 1)
    c = cfg.to_c()
    L.check(L.LIB.tmb_tucker_als(h, L.ptr(x_dev), dtype, len(dims), L.i64s(dims), L.i64s(ranks), L.C.byref(c),
                                 L.ptr(core), L.ptrs(facs), L.C.byref(tr)), h)
    return _model_from_dev(core, facs, ranks, dims), _trace_from_c(tr)


def _trace_buffers(cap: int):
    kind = (L.C.c_int * cap)()
    fitv = (L.C.c_double * cap)()
    chg = (L.C.c_double * cap)()
    tr = L.Trace(cap, 0, 0, 0, L.C.cast(kind, L.C.POINTER(L.C.c_int)), L.C.cast(fitv, L.C.POINTER(L.C.c_double)),
                 L.C.cast(chg, L.C.POINTER(L.C.c_double)))
    tr._keep = (kind, fitv, chg)
    return tr, tr._keep


def _trace_from_c(tr) -> SolveTrace:
    out = SolveTrace()
    for i in range(tr.n_records):
        out.records.append(SweepRecord(i, L.KINDS[tr.kind[i]], float(tr.fit[i]), float(tr.max_change[i])))
    out.converged = bool(tr.converged)
    return out
