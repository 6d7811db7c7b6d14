"""Pairwise-perturbation phase (tucker.py:199-311, 359-387) against the
reference's own traces (tests/golden/pp.npz): the reference DEFAULT
SolveConfig on random tensors, and config 1 forced to 25 sweeps."""

from __future__ import annotations

import numpy as np
import pytest

import oracle
from conftest import principal_angle

N_CASES = 5


def _cfg(z, k):
    return dict(max_sweeps=int(z[f"max_sweeps{k}"]), fit_tol=float(z[f"fit_tol{k}"]))


@pytest.mark.parametrize("k", range(N_CASES))
def test_oracle_pp_trace_matches_reference(golden, k):
    z = golden("pp")
    core, factors, trace = oracle.tucker_als(z[f"x{k}"], tuple(z[f"ranks{k}"]), **_cfg(z, k))
    assert "".join(r[1][0] for r in trace.rows) == str(z[f"kinds{k}"])
    assert np.abs(np.array([r[2] for r in trace.rows]) - z[f"fit{k}"]).max() < 1e-12
    for n, f in enumerate(factors):
        assert np.abs(f - z[f"f{k}_{n}"]).max() < 1e-8


@pytest.mark.gpu
@pytest.mark.parametrize("k", range(N_CASES))
def test_device_pp_trace_matches_reference(golden, k):
    import paper_2104_04726_b200 as tb

    z = golden("pp")
    t = tb.DenseTensor(z[f"x{k}"])
    model, trace = tb.tucker_als(t, tb.SolveConfig(ranks=tuple(int(r) for r in z[f"ranks{k}"]), **_cfg(z, k)))
    kinds = "".join(r.kind[0] for r in trace.records)
    assert kinds == str(z[f"kinds{k}"])
    assert np.abs(np.array([r.fit for r in trace.records]) - z[f"fit{k}"]).max() < 1e-10
    assert trace.converged == bool(z[f"converged{k}"])
    for n, f in enumerate(model.factors):
        assert principal_angle(f, z[f"f{k}_{n}"]) < 1e-7
    model.validate()


@pytest.mark.gpu
def test_device_pp_config1_matches_reference(golden):
    import paper_2104_04726_b200 as tb

    z = golden("pp")
    c1 = golden("c1")
    x = oracle.coding_tensor(c1["images"], "ycbcr").astype(np.float32).astype(np.float64)
    model, trace = tb.tucker_als(tb.DenseTensor(x), tb.SolveConfig(ranks=(48, 64, 3, 3), max_sweeps=25,
                                                                   fit_tol=1e-12))
    kinds = "".join(r.kind[0] for r in trace.records)
    assert kinds == str(z["c1_kinds"])
    assert np.abs(np.array([r.fit for r in trace.records]) - z["c1_fit"]).max() < 1e-9
    for n in range(4):
        assert principal_angle(model.factors[n], z[f"c1_f{n}"]) < 1e-6


@pytest.mark.gpu
def test_greedy_schedule_matches_sequential_default_config():  # tests/test_tucker.py:315-321 verbatim config
    import paper_2104_04726_b200 as tb

    t = tb.DenseTensor(np.random.default_rng(23).standard_normal((9, 7, 5, 3)))
    ranks = (3, 3, 2, 2)
    f_seq = tb.fit(t, tb.tucker_als(t, tb.SolveConfig(ranks=ranks, sequential_reduction=True))[0])
    f_greedy = tb.fit(t, tb.tucker_als(t, tb.SolveConfig(ranks=ranks, sequential_reduction=False))[0])
    assert abs(f_seq - f_greedy) < 1e-9
