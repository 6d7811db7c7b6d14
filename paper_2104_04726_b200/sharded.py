"""Row-sharded Tucker-ALS for one stack split over G ranks.

The reference solves one stack in one process (tucker.py:331-397). For a stack
whose working set should be split over GPUs (config 5: 4320x7680x3x18), rank i
holds the mode-0 rows [r_i, r_{i+1}) of every (colour, view-exposure) plane and
the solve exchanges one block per mode update, replacing the reference's
single-process ``t_hosvd`` + ``hooi_sweep`` (tucker.py:130-163) with:

* T-HOSVD: the mode-0 Gram by blocks -- the row shards are passed round the
  ranks one at a time (a broadcast per shard), rank i forms its column block
  G0[:, rows_i] = [T_j T_i^T]_j on the tensor pipe, and the column blocks are
  all-gathered (no rank ever holds the whole tensor, and the 4320^2 Gram is
  computed once, split G ways); modes n > 0 Grams are additive over row
  shards (all-reduce); core = sum_i t_i x_0 S_0,i^T x_1 ... (all-reduce of
  the partial core). The four T-HOSVD eigen-updates are independent, so mode
  n is solved on rank n mod G and broadcast.
* HOOI mode 0: Y0_i = t_i x_1 S_1^T x_2 S_2^T x_3 S_3^T is row-local; all-gather
  the rows, Gram and eigen-update replicated.
* HOOI modes 1..3 and the core: A_i = t_i x_0 S_0,i^T is a partial sum over
  shards; Y1 = all-reduce(A_i x_2 S_2^T x_3 S_3^T); B_i = A_i x_1 S_1^T;
  Y2 = all-reduce(B_i x_3 S_3^T); Y3 = all-reduce(B_i x_2 S_2^T); core =
  Y3 x_3 S_3^T locally. The Gauss-Seidel order of the reference is kept (each
  factor is replaced before the next mode).

The HOOI Grams and eigen-updates (sequential in the Gauss-Seidel order) are
computed redundantly on every rank from bitwise identical all-reduced inputs (ring collectives hand every rank the same
bits; the eigen-solver is deterministic), so all ranks hold identical factors.
The driver reproduces tucker_als's trace, fit, best-of and |dfit| < fit_tol
rules for standard sweeps; PP (pp_enter_tol > 0) is not sharded.

Compute goes through ``ops`` (``DeviceOps``: libtmb on CUDA tensors) and
communication through ``comm`` (``TorchComm``: torch.distributed, NCCL on the
GPU). Both are parameters so the exchange logic is testable on CPU (gloo) with
a checker backend, and on one GPU with threads standing in for ranks.
"""

from __future__ import annotations

import math
import threading
from typing import Sequence

import numpy as np

from .tensor import DenseTensor
from .tucker import SolveConfig, SolveTrace, SweepRecord, TuckerModel

__all__ = ["row_ranges", "TorchComm", "ThreadComm", "DeviceOps", "sharded_tucker_als"]


def row_ranges(h: int, world: int) -> list[tuple[int, int]]:
    """Balanced contiguous split of mode-0 rows: the first h % world ranks get one more."""
    base, extra = divmod(h, world)
    out, r = [], 0
    for i in range(world):
        n = base + (1 if i < extra else 0)
        out.append((r, r + n))
        r += n
    return out


class TorchComm:
    """SUM all-reduce / all-gather over torch.distributed (NCCL on CUDA tensors)."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self._dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)

    def allreduce_sum(self, t):
        self._dist.all_reduce(t, op=self._dist.ReduceOp.SUM, group=self.group)
        return t

    def allgather(self, t) -> list:
        import torch

        out = [torch.empty_like(t) for _ in range(self.world)]
        self._dist.all_gather(out, t.contiguous(), group=self.group)
        return out

    def broadcast(self, t, src: int):
        self._dist.broadcast(t, src=self._dist.get_global_rank(self.group, src) if self.group else src,
                             group=self.group)
        return t


class ThreadComm:
    """In-process ranks (one host thread each) for single-GPU emulation: every
    rank sums the deposited tensors in rank order, so all ranks get the same bits."""

    def __init__(self, world: int):
        self.world = world
        self._slots: list = [None] * world
        self._bar = threading.Barrier(world)
        self._local = threading.local()

    def bind(self, rank: int) -> "ThreadComm":
        self._local.rank = rank
        return self

    @property
    def rank(self) -> int:
        return self._local.rank

    def _sync(self):
        import torch

        if torch.cuda.is_available():
            torch.cuda.synchronize()
        self._bar.wait()

    def allreduce_sum(self, t):
        self._slots[self.rank] = t.clone()
        self._sync()
        acc = self._slots[0].clone()
        for i in range(1, self.world):
            acc += self._slots[i]
        self._sync()
        t.copy_(acc)
        return t

    def allgather(self, t) -> list:
        self._slots[self.rank] = t.clone()
        self._sync()
        out = [s.clone() for s in self._slots]
        self._sync()
        return out

    def broadcast(self, t, src: int):
        if self.rank == src:
            self._slots[src] = t.clone()
        self._sync()
        if self.rank != src:
            t.copy_(self._slots[src])
        self._sync()
        return t


class DeviceOps:
    """The per-rank arithmetic through the libtmb C ABI on CUDA tensors (F-order flat)."""

    def __init__(self):
        from . import _lib as L

        self.L = L

    def _dt(self, x) -> int:
        import torch

        return self.L.F32 if x.dtype == torch.float32 else self.L.F64

    def ttm_t(self, x, dims: Sequence[int], mode: int, u, r: int):
        """x x_mode u^T for u (dims[mode] x r, column-major); returns (y, new dims)."""
        import torch

        L = self.L
        s = dims[mode]
        m = u.view(r, s).t().contiguous().view(-1)  # u^T column-major (r x s)
        nd = list(dims)
        nd[mode] = r
        y = torch.empty(int(np.prod(nd)), dtype=torch.float64, device=x.device)
        h = L.ctx()
        L.check(L.LIB.tmb_ttm(h, L.ptr(x), self._dt(x), len(dims), L.i64s(dims), mode, L.ptr(m), r, L.ptr(y)), h)
        return y, tuple(nd)

    def gram(self, x, dims: Sequence[int], mode: int):
        import torch

        L = self.L
        n = dims[mode]
        g = torch.empty(n * n, dtype=torch.float64, device=x.device)
        h = L.ctx()
        L.check(L.LIB.tmb_mode_gram(h, L.ptr(x), self._dt(x), len(dims), L.i64s(dims), mode, L.ptr(g)), h)
        return g

    def cross_rows(self, xj, hj: int, xi64, hi: int, kdim: int):
        """X_j X_i^T (hj x hi, column-major) of two mode-0 row blocks given as
        F-order (h, K) matrices; xi64 float64 (the GEMM's factor operand)."""
        import torch

        L = self.L
        y = torch.empty(hj * hi, dtype=torch.float64, device=xj.device)
        h = L.ctx()
        L.check(L.LIB.tmb_ttm(h, L.ptr(xj), self._dt(xj), 2, L.i64s((hj, kdim)), 1, L.ptr(xi64), hi, L.ptr(y)), h)
        return y

    def to_f64(self, x):
        return x if self._dt(x) == self.L.F64 else x.double()

    def mirror_upper(self, g, n: int):
        """g <- triu(g) + triu(g, 1)^T in place: the exactly symmetric Gram of
        gram() (tensor.py:176-180) from independently computed blocks."""
        L = self.L
        h = L.ctx()
        L.check(L.LIB.tmb_mirror_upper(h, L.ptr(g), n), h)
        return g

    def eig(self, g, n: int, k: int):
        import torch

        L = self.L
        v = torch.empty(n * k, dtype=torch.float64, device=g.device)
        w = torch.empty(k, dtype=torch.float64, device=g.device)
        h = L.ctx()
        L.check(L.LIB.tmb_leading_eigvecs(h, L.ptr(g), n, k, L.ptr(v), L.ptr(w)), h)
        return v

    def sumsq(self, x) -> float:
        L = self.L
        out = L.C.c_double()
        h = L.ctx()
        L.check(L.LIB.tmb_sumsq(h, L.ptr(x), self._dt(x), x.numel(), L.C.byref(out)), h)
        return float(out.value)

    def rel_change(self, new, old) -> float:
        """||new - old||_F / ||old||_F (tucker.py:319-323) via axpy + sumsq."""
        L = self.L
        d = new.clone()
        h = L.ctx()
        L.check(L.LIB.tmb_axpy(h, d.numel(), -1.0, L.ptr(old), L.ptr(d)), h)
        return math.sqrt(self.sumsq(d)) / math.sqrt(self.sumsq(old))


def _gather_rows(comm, y, dims_local: Sequence[int], ranges) -> tuple:
    """All-gather row shards of an F-order tensor along mode 0 (padded to the
    largest shard, then trimmed): an F-order (h_i, K) block is C-order (K, h_i)."""
    import torch

    k = int(np.prod(dims_local[1:]))
    hmax = max(b - a for a, b in ranges)
    hi = dims_local[0]
    blk = y.view(k, hi)
    if hi < hmax:
        blk = torch.cat([blk, blk.new_zeros(k, hmax - hi)], dim=1)
    parts = comm.allgather(blk.contiguous())
    full = torch.cat([p[:, : b - a] for p, (a, b) in zip(parts, ranges)], dim=1)
    h = ranges[-1][1]
    return full.contiguous().view(-1), (h,) + tuple(dims_local[1:])


def _blocked_mode0_gram(comm, ops, x_local, dims, ranges):
    """Mode-0 Gram of a row-sharded tensor without gathering it: shard j is
    broadcast in turn, rank i forms the block X_j X_i^T of its column block
    G0[:, rows_i], the column blocks are all-gathered, and the upper triangle
    is mirrored (the reference's exactly symmetric gram, tensor.py:176-180)."""
    import torch

    n = dims[0]
    kdim = int(np.prod(dims[1:]))
    a0, b0 = ranges[comm.rank]
    hi = b0 - a0
    xi64 = ops.to_f64(x_local)
    hmax = max(b - a for a, b in ranges)
    col = torch.empty((hmax, n), dtype=torch.float64, device=x_local.device)  # C-order (hi, n) = column-major n x hi
    for j, (aj, bj) in enumerate(ranges):
        hj = bj - aj
        buf = x_local if j == comm.rank else torch.empty(hj * kdim, dtype=x_local.dtype, device=x_local.device)
        comm.broadcast(buf, j)
        y = ops.cross_rows(buf, hj, xi64, hi, kdim)                  # (hj x hi) column-major
        col[:hi, aj:bj] = y.view(hi, hj)                              # rows aj..bj of columns rows_i
        del buf
    parts = comm.allgather(col.contiguous().view(-1))
    g = torch.cat([p.view(hmax, n)[: b - a] for p, (a, b) in zip(parts, ranges)], dim=0).contiguous().view(-1)
    return ops.mirror_upper(g, n)


def _rows_of(u, s: int, r: int, a: int, b: int):
    """Rows [a, b) of a column-major s x r factor, column-major (b - a) x r."""
    return u.view(r, s)[:, a:b].contiguous().view(-1)


def _to_host(u, shape) -> np.ndarray:
    return u.detach().cpu().numpy().reshape(shape, order="F").copy()


def sharded_tucker_als(x_local, dims: Sequence[int], cfg: SolveConfig, comm, ops=None
                       ) -> tuple[TuckerModel, SolveTrace]:
    """tucker_als (tucker.py:331-397) on a mode-0 row-sharded 4-way tensor.

    ``x_local`` is this rank's F-order block of rows ``row_ranges(dims[0],
    comm.world)[comm.rank]`` (fp32 or fp64, flat). Every rank returns the same
    model and trace."""
    dims = tuple(int(d) for d in dims)
    if len(dims) != 4:
        raise ValueError("the row-sharded solver handles order-4 stacks (H, W, C, V*E)")
    cfg.validate(dims)
    if cfg.pp_enter_tol > 0:
        raise ValueError("pairwise perturbation is not available in the row-sharded solver (pp_enter_tol must be 0)")
    import torch

    ops = ops or DeviceOps()
    ranges = row_ranges(dims[0], comm.world)
    a0, b0 = ranges[comm.rank]
    dl = (b0 - a0,) + dims[1:]
    if x_local.numel() != int(np.prod(dl)):
        raise ValueError(f"rank {comm.rank}: local block has {x_local.numel()} entries, rows {a0}:{b0} need "
                         f"{int(np.prod(dl))}")
    r = tuple(int(v) for v in cfg.ranks)
    s = dims

    t2 = torch.tensor([ops.sumsq(x_local)], dtype=torch.float64, device=x_local.device)
    comm.allreduce_sum(t2)
    tnorm2 = float(t2[0])
    if tnorm2 == 0.0:
        raise ValueError("cannot decompose the zero tensor")

    def fit_of(core) -> float:
        c2 = ops.sumsq(core)
        return 1.0 - math.sqrt(max(tnorm2 - c2, 0.0)) / math.sqrt(tnorm2)

    def core_from_y3(y3, u3):
        return ops.ttm_t(y3, (r[0], r[1], r[2], s[3]), 3, u3, r[3])[0]

    # ---- T-HOSVD (tucker.py:130-148)
    g0 = _blocked_mode0_gram(comm, ops, x_local, dims, ranges)
    grams = [g0] + [comm.allreduce_sum(ops.gram(x_local, dl, n)) for n in (1, 2, 3)]
    u = []
    for n in range(4):   # independent eigen-updates: mode n on rank n mod G, then broadcast
        owner = n % comm.world
        if comm.rank == owner:
            v = ops.eig(grams[n], s[n], r[n])
        else:
            v = torch.empty(s[n] * r[n], dtype=torch.float64, device=x_local.device)
        u.append(comm.broadcast(v, owner))
    del grams, g0
    p, pd = ops.ttm_t(x_local, dl, 0, _rows_of(u[0], s[0], r[0], a0, b0), r[0])
    for n in (1, 2):
        p, pd = ops.ttm_t(p, pd, n, u[n], r[n])
    comm.allreduce_sum(p)
    core = core_from_y3(p, u[3])

    trace = SolveTrace()
    cur = fit_of(core)
    trace.records.append(SweepRecord(0, "init", cur, math.nan))
    best = (cur, core, list(u))
    if cur >= 1.0 - cfg.fit_tol:
        trace.converged = True
    else:
        for sweep in range(1, cfg.max_sweeps + 1):
            new = list(u)
            # mode 0: rows are local
            y, yd = x_local, dl
            for n in (1, 2, 3):
                y, yd = ops.ttm_t(y, yd, n, new[n], r[n])
            yf, yfd = _gather_rows(comm, y, yd, ranges)
            new[0] = ops.eig(ops.gram(yf, yfd, 0), s[0], r[0])
            # modes 1..3: partial sums over the row shards
            a, ad = ops.ttm_t(x_local, dl, 0, _rows_of(new[0], s[0], r[0], a0, b0), r[0])
            y1, y1d = ops.ttm_t(a, ad, 2, new[2], r[2])
            y1, y1d = ops.ttm_t(y1, y1d, 3, new[3], r[3])
            new[1] = ops.eig(ops.gram(comm.allreduce_sum(y1), y1d, 1), s[1], r[1])
            bt, bd = ops.ttm_t(a, ad, 1, new[1], r[1])
            del a
            y2, y2d = ops.ttm_t(bt, bd, 3, new[3], r[3])
            new[2] = ops.eig(ops.gram(comm.allreduce_sum(y2), y2d, 2), s[2], r[2])
            y3, y3d = ops.ttm_t(bt, bd, 2, new[2], r[2])
            comm.allreduce_sum(y3)
            new[3] = ops.eig(ops.gram(y3, y3d, 3), s[3], r[3])
            new_core = core_from_y3(y3, new[3])
            change = max(ops.rel_change(f, o) for f, o in zip(new, u))
            new_fit = fit_of(new_core)
            trace.records.append(SweepRecord(sweep, "standard", new_fit, change))
            if new_fit > best[0]:
                best = (new_fit, new_core, list(new))
            done = abs(new_fit - cur) < cfg.fit_tol
            core, u, cur = new_core, new, new_fit
            if done:
                trace.converged = True
                break
        if not trace.converged:
            _, core, u = best
    model = TuckerModel(DenseTensor(_to_host(core, r)), [_to_host(f, (s[n], r[n])) for n, f in enumerate(u)], dims)
    return model, trace
