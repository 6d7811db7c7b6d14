"""Row-sharded Tucker-ALS: the exchange logic.

CPU: world_size 2 over gloo, with the oracle as the per-rank arithmetic (test
infrastructure only -- the product's per-rank arithmetic is libtmb, exercised
by the GPU test below), checked against the single-process oracle solve.
GPU: two in-process ranks (host threads, ``ThreadComm``) on one device running
libtmb, checked against the unsharded device solver."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from paper_2104_04726_b200.sharded import ThreadComm, row_ranges

DIMS = (23, 18, 3, 4)
RANKS = (6, 5, 2, 3)
SWEEPS = 3


def _tensor():
    rng = np.random.default_rng(5)
    base = rng.standard_normal((23, 4)) @ rng.standard_normal((4, 18 * 3 * 4))
    x = base.reshape(DIMS, order="F") + 0.05 * rng.standard_normal(DIMS)
    return x


class OracleOps:
    """Per-rank arithmetic from the numpy oracle on flat F-order CPU tensors."""

    def __init__(self):
        import oracle.tucker_oracle as O

        self.O = O

    @staticmethod
    def _arr(x, dims):
        return x.detach().cpu().numpy().astype(np.float64).reshape(dims, order="F")

    @staticmethod
    def _flat(a):
        return torch.from_numpy(np.asfortranarray(a).ravel(order="F").copy())

    def ttm_t(self, x, dims, mode, u, r):
        uu = u.numpy().reshape((dims[mode], r), order="F")
        y = self.O.ttm(self._arr(x, dims), uu.T, mode)
        return self._flat(y), y.shape

    def gram(self, x, dims, mode):
        return self._flat(self.O.gram(self.O.unfold(self._arr(x, dims), mode)))

    def cross_rows(self, xj, hj, xi64, hi, kdim):
        a = xj.numpy().astype(np.float64).reshape((hj, kdim), order="F")
        b = xi64.numpy().reshape((hi, kdim), order="F")
        return self._flat(a @ b.T)

    def to_f64(self, x):
        return x.double()

    def mirror_upper(self, g, n):
        m = g.numpy().reshape((n, n), order="F")
        m = np.triu(m) + np.triu(m, 1).T
        return self._flat(m)

    def eig(self, g, n, k):
        v, _ = self.O.leading_eigvecs(g.numpy().reshape((n, n), order="F"), k)
        return self._flat(v)

    def sumsq(self, x):
        return float((x.double() ** 2).sum())

    def rel_change(self, new, old):
        return float(np.linalg.norm((new - old).numpy()) / np.linalg.norm(old.numpy()))


def test_row_ranges_cover_balanced():
    for h, w in [(4320, 8), (23, 2), (7, 3), (5, 5)]:
        rr = row_ranges(h, w)
        assert rr[0][0] == 0 and rr[-1][1] == h
        assert all(a[1] == b[0] for a, b in zip(rr, rr[1:]))
        sizes = [b - a for a, b in rr]
        assert max(sizes) - min(sizes) <= 1


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank: int, world: int, port: int, q):
    import torch.distributed as dist

    from paper_2104_04726_b200.sharded import TorchComm, sharded_tucker_als
    from paper_2104_04726_b200.tucker import SolveConfig

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    x = _tensor()
    a, b = row_ranges(DIMS[0], world)[rank]
    xl = torch.from_numpy(np.asfortranarray(x[a:b]).ravel(order="F").copy())
    cfg = SolveConfig(ranks=RANKS, max_sweeps=SWEEPS, fit_tol=1e-300, pp_enter_tol=0.0)
    model, trace = sharded_tucker_als(xl, DIMS, cfg, TorchComm(), OracleOps())
    q.put((rank, [f.copy() for f in model.factors], model.core.array.copy(), trace.rows()))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_two_ranks_match_single_process_oracle():
    import oracle.tucker_oracle as O

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (_, f0, c0, t0), (_, f1, c1, t1) = out
    # every rank holds the same model
    for a, b in zip(f0, f1):
        assert np.array_equal(a, b)
    assert np.array_equal(c0, c1)
    assert np.array_equal(np.array([r[2:] for r in t0]), np.array([r[2:] for r in t1]), equal_nan=True)
    core, factors, tr = O.tucker_als(_tensor(), RANKS, max_sweeps=SWEEPS, fit_tol=1e-300, pp_enter_tol=0.0)
    from conftest import principal_angle

    for a, b in zip(f0, factors):
        assert principal_angle(a, b) < 1e-8
        assert np.abs(np.abs(a) - np.abs(b)).max() < 1e-8
    assert np.abs(np.abs(c0) - np.abs(core)).max() < 1e-8 * np.abs(core).max()
    assert len(t0) == len(tr.rows) == SWEEPS + 1
    for (i, k, fit, _), (ri, rk, rfit, _) in zip(t0, tr.rows):
        assert i == ri and k == rk and abs(fit - rfit) < 1e-12


def test_pp_rejected():
    from paper_2104_04726_b200.sharded import sharded_tucker_als
    from paper_2104_04726_b200.tucker import SolveConfig

    comm = ThreadComm(1).bind(0)
    with pytest.raises(ValueError, match="pairwise perturbation"):
        sharded_tucker_als(torch.zeros(int(np.prod(DIMS))), DIMS, SolveConfig(ranks=RANKS), comm, OracleOps())


@pytest.mark.gpu
def test_two_thread_ranks_on_device_match_unsharded():
    import threading

    import paper_2104_04726_b200 as tb
    from paper_2104_04726_b200.sharded import sharded_tucker_als
    from paper_2104_04726_b200.synth import CONFIGS, make_stack
    from paper_2104_04726_b200.pipeline import coding_tensor

    cfg0 = CONFIGS["c1"]
    t = coding_tensor(make_stack(cfg0, seed=2), cfg0.space)  # (384, 512, 3, 6) fp32 device
    dims = tuple(int(d) for d in cfg0.dims)
    sc = tb.SolveConfig(ranks=cfg0.ranks, max_sweeps=4, fit_tol=1e-300, pp_enter_tol=0.0)
    ref_model, ref_trace = tb.tucker.solve_device(t, tb._lib.F32, dims, sc)
    world = 2
    comm = ThreadComm(world)
    full = t.view(int(np.prod(dims[1:])), dims[0])  # F-order (H, K) == C-order (K, H)
    results = [None] * world

    def run(rank):
        torch.cuda.set_device(0)
        a, b = row_ranges(dims[0], world)[rank]
        xl = full[:, a:b].contiguous().view(-1)
        results[rank] = sharded_tucker_als(xl, dims, sc, comm.bind(rank))

    th = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for x in th:
        x.start()
    for x in th:
        x.join()
    (m0, tr0), (m1, tr1) = results
    for a, b in zip(m0.factors, m1.factors):
        assert np.array_equal(a, b)
    from conftest import principal_angle

    for a, b in zip(m0.factors, ref_model.factors):
        assert principal_angle(a, b) < 1e-6
    for r0, r1 in zip(tr0.records, ref_trace.records):
        assert abs(r0.fit - r1.fit) < 1e-10


def _device_worker(rank: int, world: int, port: int, q):
    """One process per rank on the SAME GPU, the product's TorchComm (gloo on CUDA
    tensors -- NCCL refuses two ranks on one device) + DeviceOps (libtmb)."""
    import torch.distributed as dist

    import paper_2104_04726_b200 as tb
    from paper_2104_04726_b200.pipeline import coding_tensor
    from paper_2104_04726_b200.sharded import DeviceOps, TorchComm, sharded_tucker_als
    from paper_2104_04726_b200.synth import CONFIGS, make_stack

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg0 = CONFIGS["c1"]
    t = coding_tensor(make_stack(cfg0, seed=2), cfg0.space)
    dims = tuple(int(d) for d in cfg0.dims)
    full = t.view(int(np.prod(dims[1:])), dims[0])
    a, b = row_ranges(dims[0], world)[rank]
    xl = full[:, a:b].contiguous().view(-1)
    sc = tb.SolveConfig(ranks=cfg0.ranks, max_sweeps=3, fit_tol=1e-300, pp_enter_tol=0.0)
    model, trace = sharded_tucker_als(xl, dims, sc, TorchComm(), DeviceOps())
    q.put((rank, [f.copy() for f in model.factors], [r.fit for r in trace.records]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.gpu
def test_two_process_ranks_torchcomm_deviceops_match_unsharded():
    import paper_2104_04726_b200 as tb
    from paper_2104_04726_b200.pipeline import coding_tensor
    from paper_2104_04726_b200.synth import CONFIGS, make_stack

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_device_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    (_, f0, fit0), (_, f1, fit1) = out
    for a, b in zip(f0, f1):
        assert np.array_equal(a, b)          # every rank holds the same model
    assert fit0 == fit1
    cfg0 = CONFIGS["c1"]
    t = coding_tensor(make_stack(cfg0, seed=2), cfg0.space)
    dims = tuple(int(d) for d in cfg0.dims)
    sc = tb.SolveConfig(ranks=cfg0.ranks, max_sweeps=3, fit_tol=1e-300, pp_enter_tol=0.0)
    ref_model, ref_trace = tb.tucker.solve_device(t, tb._lib.F32, dims, sc)
    from conftest import principal_angle

    for a, b in zip(f0, ref_model.factors):
        assert principal_angle(a, b) < 1e-6
    for x, y in zip(fit0, [r.fit for r in ref_trace.records]):
        assert abs(x - y) < 1e-10
