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


@dataclass
class PPState:
    anchors: list[np.ndarray]
    deltas: list[np.ndarray]
    op_single: list[DenseTensor]
    op_pair: dict[tuple[int, int], DenseTensor]
    contraction_count: int

    def pair(self, i: int, n: int) -> DenseTensor:
        return self.op_pair[(i, n) if i < n else (n, i)]

    def set_current(self, factors: Sequence[np.ndarray]) -> None:
        self.deltas = [np.asarray(f, dtype=np.float64) - a for f, a in zip(factors, self.anchors)]

    def max_rel_delta(self) -> float:
        out = 0.0
        for d, a in zip(self.deltas, self.anchors):
            out = max(out, _frob(d) / _frob(a))
        return out


def _frob(m: np.ndarray) -> float:
    return fro_norm(DenseTensor(np.asarray(m, dtype=np.float64)))


def pp_operators(t: DenseTensor, anchors: Sequence[np.ndarray]) -> PPState:
    """Skip-one and skip-two contractions through a memoised dimension tree
    whose parent re-adds the largest contracted mode (tucker.py:222-265), so
    every node is an ascending contraction. Each node is one device TTM."""
    n_modes = t.ndim
    if len(anchors) != n_modes:
        raise ValueError(f"expected {n_modes} anchors, got {len(anchors)}")
    for n, a in enumerate(anchors):
        a = np.asarray(a)
        if a.ndim != 2 or a.shape[0] != t.dims[n]:
            raise ValueError(f"mode {n}: anchor shape {a.shape} does not match dim {t.dims[n]}")
    cache: dict[frozenset, DenseTensor] = {frozenset(range(n_modes)): t}
    count = 0

    def node(free: frozenset) -> DenseTensor:
        nonlocal count
        got = cache.get(free)
        if got is not None:
            return got
        m = max(i for i in range(n_modes) if i not in free)
        out = ttm(node(free | {m}), np.asarray(anchors[m], dtype=np.float64).T, m)
        count += 1
        cache[free] = out
        return out

    op_single = [node(frozenset((n,))) for n in range(n_modes)]
    op_pair = {(i, n): node(frozenset((i, n))) for i in range(n_modes) for n in range(i + 1, n_modes)}
    anchors64 = [np.asarray(a, dtype=np.float64) for a in anchors]
    return PPState(anchors64, [np.zeros_like(a) for a in anchors64], op_single, op_pair, count)


def _pp_operand(state: PPState, n: int) -> DenseTensor:
    """First-order skip-n estimate (tucker.py:268-282); accumulation on the device."""
    y = state.op_single[n]
    acc_d = None
    for i in range(len(state.anchors)):
        if i == n:
            continue
        d = state.deltas[i]
        if not np.any(d):
            continue
        corr = ttm(state.pair(i, n), d.T, i)
        if acc_d is None:
            acc_d = L.dev_f64(corr.array)
        else:
            h = L.ctx()
            cd = L.dev_f64(corr.array)
            L.check(L.LIB.tmb_axpy(h, corr.size, 1.0, L.ptr(cd), L.ptr(acc_d)), h)
    if acc_d is None:
        return y
    h = L.ctx()
    yd = L.dev_f64(y.array)
    L.check(L.LIB.tmb_axpy(h, y.size, 1.0, L.ptr(yd), L.ptr(acc_d)), h)
    return DenseTensor(L.host_f(acc_d, y.dims))


def pp_sweep(state: PPState, model: TuckerModel, return_operands: bool = False):
    """One accelerated sweep from the precomputed operators (tucker.py:285-311)."""
    ranks = model.ranks
    factors = list(model.factors)
    operands: list[DenseTensor] = []
    last_y = None
    for n in range(len(factors)):
        y = _pp_operand(state, n)
        if return_operands:
            operands.append(y)
        factors[n] = leading_eigvecs(gram(unfold(y, n)), ranks[n])[0]
        last_y = y
    n_last = len(factors) - 1
    core = ttm(last_y, factors[n_last].T, n_last)
    out = TuckerModel(core, factors, model.source_dims)
    if return_operands:
        return out, operands
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
