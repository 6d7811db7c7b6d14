"""More drop-in contracts on the device path, in the reference test suite's
tolerance regime: tensor.py products and norms, the Tucker
invariants (tucker.py:120-397), PP (tucker.py:199-311) and the colour
transforms (color.py:111-205). Written independently of the reference's
tests; each cites the property it pins."""

from __future__ import annotations

import itertools
import math

import numpy as np
import pytest

import oracle
import paper_2104_04726_b200 as tb

pytestmark = pytest.mark.gpu


def orth(rng, rows, cols):
    return np.linalg.qr(rng.standard_normal((rows, cols)))[0]


def exact_tensor(rng, dims, ranks):
    core = tb.DenseTensor(rng.standard_normal(ranks))
    model = tb.TuckerModel(core, [orth(rng, s, r) for s, r in zip(dims, ranks)], tuple(dims))
    return tb.reconstruct(model), model


# ---------------------------------------------------------------- tensor.py
def test_ttm_rank1_outer_product():  # ttm of an outer product scales one factor
    rng = np.random.default_rng(30)
    a, b, c = rng.standard_normal(4), rng.standard_normal(5), rng.standard_normal(3)
    t = tb.DenseTensor(np.einsum("i,j,k->ijk", a, b, c))
    m = rng.standard_normal((6, 5))
    got = tb.ttm(t, m, 1).array
    assert np.abs(got - np.einsum("i,j,k->ijk", a, m @ b, c)).max() < 1e-12


def test_ttm_distinct_modes_commute():
    rng = np.random.default_rng(31)
    t = tb.DenseTensor(rng.standard_normal((5, 6, 7)))
    m0, m2 = rng.standard_normal((3, 5)), rng.standard_normal((4, 7))
    a = tb.ttm(tb.ttm(t, m0, 0), m2, 2).array
    b = tb.ttm(tb.ttm(t, m2, 2), m0, 0).array
    assert np.abs(a - b).max() < 1e-12


def test_ttmc_identity_and_projection_norm():
    rng = np.random.default_rng(32)
    t = tb.DenseTensor(rng.standard_normal((6, 5, 4)))
    assert np.abs(tb.ttmc(t, [np.eye(6), np.eye(5), np.eye(4)]).array - t.array).max() < 1e-14
    fs = [orth(rng, 6, 3), orth(rng, 5, 2), orth(rng, 4, 2)]
    for skip in (None, 0, 1, 2):
        assert tb.fro_norm(tb.ttmc(t, fs, skip=skip)) <= tb.fro_norm(t) * (1 + 1e-12)


def test_gram_identity_and_outer_product():
    assert np.array_equal(tb.gram(np.eye(5)), np.eye(5))
    v = np.random.default_rng(33).standard_normal((6, 1))
    assert np.abs(tb.gram(v) - v @ v.T).max() < 1e-14


def test_eig_rank_one():
    v = np.random.default_rng(34).standard_normal(9)
    vec, val = tb.leading_eigvecs(np.outer(v, v), 1)
    u = v / np.linalg.norm(v)
    assert abs(val[0] - v @ v) < 1e-12 * (v @ v)
    assert np.abs(np.abs(vec[:, 0]) - np.abs(u)).max() < 1e-12
    assert vec[np.argmax(np.abs(vec[:, 0])), 0] > 0   # sign rule


def test_fro_norm_cases():
    assert tb.fro_norm(tb.DenseTensor(np.zeros((3, 4)))) == 0.0
    z = np.zeros((2, 3, 4))
    z[1, 2, 3] = -7.5
    assert tb.fro_norm(tb.DenseTensor(z)) == 7.5
    assert abs(tb.fro_norm(tb.DenseTensor(np.ones((4, 5, 6)))) - math.sqrt(120)) < 1e-13


# ---------------------------------------------------------------- tucker.py
def test_hosvd_order2_is_svd():
    m = np.random.default_rng(35).standard_normal((7, 5))
    model = tb.hosvd(tb.DenseTensor(m))
    u, s, vt = np.linalg.svd(m)
    assert np.abs(np.abs(np.diag(model.core.array)[:5]) - s).max() < 1e-12
    assert np.abs(np.abs(model.factors[1]) - np.abs(vt.T)).max() < 1e-10


def test_thosvd_rank_one_bound_and_nested_truncation():
    rng = np.random.default_rng(36)
    t = tb.DenseTensor(rng.standard_normal((8, 7, 6)))
    tn2 = tb.fro_norm(t) ** 2
    err = []
    for r in [(1, 1, 1), (3, 3, 3), (5, 5, 5)]:
        m = tb.t_hosvd(t, r)
        resid2 = tn2 - tb.fro_norm(m.core) ** 2
        # bound: sum over modes of the discarded Gram eigenvalues (tucker.py:130-148 property)
        bound = sum(float(np.sum(np.linalg.eigvalsh(oracle.gram(oracle.unfold(t.array, n)))[:-r[n]]))
                    for n in range(3))
        assert resid2 <= bound * (1 + 1e-10)
        err.append(resid2)
    assert err[0] >= err[1] >= err[2]   # nested truncations never get worse


def test_hooi_order2_converges_to_svd_subspace():
    rng = np.random.default_rng(37)
    m = rng.standard_normal((12, 9))
    model, _ = tb.tucker_als(tb.DenseTensor(m), tb.SolveConfig(ranks=(3, 3), max_sweeps=30, fit_tol=1e-14,
                                                                pp_enter_tol=0.0))
    u = np.linalg.svd(m)[0][:, :3]
    from conftest import principal_angle

    assert principal_angle(model.factors[0], u) < 1e-8


def test_hooi_sweep_dimension_mismatch():
    rng = np.random.default_rng(38)
    t = tb.DenseTensor(rng.standard_normal((5, 4, 3)))
    bad = tb.TuckerModel(tb.DenseTensor(np.ones((2, 2, 2))), [orth(rng, 6, 2), orth(rng, 4, 2), orth(rng, 3, 2)],
                         (6, 4, 3))
    with pytest.raises(ValueError):
        tb.hooi_sweep(t, bad)


def test_fit_exact_zero_core_and_dual_formula():
    rng = np.random.default_rng(39)
    t, model = exact_tensor(rng, (6, 5, 4), (2, 3, 2))
    assert abs(tb.fit(t, model) - 1.0) < 1e-10
    zero = tb.TuckerModel(tb.DenseTensor(np.zeros(model.ranks)), model.factors, model.source_dims)
    assert abs(tb.fit(t, zero)) < 1e-14 and abs(tb.fit(t, zero, method="residual")) < 1e-14
    noisy = tb.DenseTensor(t.array + 0.1 * rng.standard_normal(t.dims))
    m = tb.t_hosvd(noisy, (2, 3, 2))
    assert abs(tb.fit(noisy, m) - tb.fit(noisy, m, method="residual")) < 1e-10


def test_reconstruct_rank1_identity_and_exhaustive_small():
    rng = np.random.default_rng(40)
    core = tb.DenseTensor(np.array([[[2.5]]]))
    fs = [rng.standard_normal((3, 1)), rng.standard_normal((4, 1)), rng.standard_normal((2, 1))]
    got = tb.reconstruct(tb.TuckerModel(core, fs, (3, 4, 2))).array
    assert np.abs(got - 2.5 * np.einsum("i,j,k->ijk", fs[0][:, 0], fs[1][:, 0], fs[2][:, 0])).max() < 1e-13
    c = rng.standard_normal((3, 2, 4))
    assert np.array_equal(tb.reconstruct(tb.TuckerModel(tb.DenseTensor(c), [np.eye(3), np.eye(2), np.eye(4)],
                                                         (3, 2, 4))).array, c)
    for dims in itertools.product((1, 2, 3), repeat=3):   # every tiny shape vs elementwise summation
        ranks = tuple(max(1, d - 1) for d in dims)
        core = rng.standard_normal(ranks)
        fs = [rng.standard_normal((d, r)) for d, r in zip(dims, ranks)]
        got = tb.reconstruct(tb.TuckerModel(tb.DenseTensor(core), fs, dims)).array
        want = np.zeros(dims)
        for idx in itertools.product(*[range(d) for d in dims]):
            want[idx] = sum(core[j] * fs[0][idx[0], j[0]] * fs[1][idx[1], j[1]] * fs[2][idx[2], j[2]]
                            for j in itertools.product(*[range(r) for r in ranks]))
        assert np.abs(got - want).max() < 1e-12


def test_tucker_als_exact_recovery_and_full_ranks():
    rng = np.random.default_rng(41)
    t, _ = exact_tensor(rng, (9, 8, 7), (3, 2, 3))
    model, trace = tb.tucker_als(t, tb.SolveConfig(ranks=(3, 2, 3)))
    assert trace.converged and rel(tb.reconstruct(model), t) < 1e-10
    full, ftrace = tb.tucker_als(t, tb.SolveConfig(ranks=t.dims, max_sweeps=0))
    assert len(ftrace.records) == 1 and rel(tb.reconstruct(full), t) < 1e-10


def rel(a, b):
    return float(np.linalg.norm(a.array - b.array) / np.linalg.norm(b.array))


def test_factors_orthonormal_at_every_sweep():
    rng = np.random.default_rng(42)
    t = tb.DenseTensor(rng.standard_normal((10, 9, 8)))
    model = tb.t_hosvd(t, (3, 3, 3))
    for _ in range(5):
        model = tb.hooi_sweep(t, model)
        model.validate()


# ---------------------------------------------------------------- PP (tucker.py:199-311)
def test_pp_singles_bit_identical_to_ascending_ttmc():
    rng = np.random.default_rng(43)
    t = tb.DenseTensor(rng.standard_normal((6, 5, 4, 3)))
    anchors = [orth(rng, s, r) for s, r in zip(t.dims, (3, 2, 2, 2))]
    state = tb.pp_operators(t, anchors)
    for n in range(4):  # the tree's single-mode operators are the ascending ttmc (tucker.py:222-265)
        want = tb.ttmc(t, anchors, skip=n)
        assert np.array_equal(state.op_single[n].array, want.array)
    # pair operators equal the naive two-skip contraction (order 3 pair definition)
    t3 = tb.DenseTensor(rng.standard_normal((5, 4, 3)))
    a3 = [orth(rng, s, 2) for s in t3.dims]
    st3 = tb.pp_operators(t3, a3)
    for (i, j), op in st3.op_pair.items():
        k = 3 - i - j
        want = tb.ttm(t3, a3[k].T, k)
        assert np.abs(op.array - want.array).max() < 1e-12


def test_pp_zero_delta_equals_frozen_sweep_and_quadratic_error():
    rng = np.random.default_rng(44)
    t = tb.DenseTensor(rng.standard_normal((7, 6, 5, 4)))
    model = tb.t_hosvd(t, (3, 3, 2, 2))
    for _ in range(2):
        model = tb.hooi_sweep(t, model)
    state = tb.pp_operators(t, model.factors)
    a = tb.pp_sweep(state, model)
    b = tb.pp_sweep(state, model)
    for fa, fb in zip(a.factors, b.factors):
        assert np.array_equal(fa, fb)                       # deterministic
    # zero entry deltas: every operand is the anchor contraction, i.e. a
    # frozen (Jacobi-style) sweep: S_n <- leading_eigvecs(gram(ttmc(t, anchors, skip=n)))
    for n in range(4):
        y = tb.ttmc(t, model.factors, skip=n)
        want, _ = tb.leading_eigvecs(tb.gram(tb.unfold(y, n)), model.ranks[n])
        assert np.array_equal(a.factors[n], want)
    # first-order operators (the state's entry deltas, tucker.py:268-282): the
    # operand error against the exact contraction at the perturbed factors is O(eps^2)
    dirs = [rng.standard_normal(f.shape) for f in model.factors]
    errs = []
    for eps in (1e-2, 1e-3):
        state.deltas = [eps * d for d in dirs]
        pert = [f + eps * d for f, d in zip(model.factors, dirs)]
        _, ops = tb.pp_sweep(state, model, return_operands=True)
        exact = tb.ttmc(t, pert, skip=0)
        errs.append(float(np.linalg.norm(ops[0].array - exact.array)))
    assert 50.0 < errs[0] / errs[1] < 200.0                 # ~100x per decade


def test_pp_solve_fit_matches_standard():
    rng = np.random.default_rng(45)
    t0, _ = exact_tensor(rng, (12, 11, 10), (4, 4, 4))
    t = tb.DenseTensor(t0.array + 0.05 * np.linalg.norm(t0.array) / math.sqrt(t0.array.size)
                       * rng.standard_normal(t0.dims))
    _, tr_pp = tb.tucker_als(t, tb.SolveConfig(ranks=(4, 4, 4), max_sweeps=25, fit_tol=1e-10, pp_enter_tol=0.1))
    _, tr_std = tb.tucker_als(t, tb.SolveConfig(ranks=(4, 4, 4), max_sweeps=25, fit_tol=1e-10, pp_enter_tol=0.0))
    assert abs(tr_pp.records[-1].fit - tr_std.records[-1].fit) < 1e-4
    pp_fits = [r.fit for r in tr_pp.records]
    assert all(b >= a - 1e-6 for a, b in zip(pp_fits, pp_fits[1:]))   # dips bounded by PP_DIP_TOL


# ---------------------------------------------------------------- colour (color.py)
def px(rgb):
    return tb.ColorImage(np.asarray(rgb, dtype=np.float64).reshape(1, -1, 3))


def test_ycbcr_kats_and_wrong_space():
    out = tb.rgb_to_ycbcr(px([[1, 1, 1], [0, 0, 0], [1, 0, 0]])).pixels[0]
    assert np.allclose(out[0], [1, 0.5, 0.5], atol=1e-15) and np.allclose(out[1], [0, 0.5, 0.5], atol=1e-15)
    assert np.allclose(out[2], [0.299, 0.5 - 0.299 / 1.772, 1.0], atol=1e-12)
    with pytest.raises(ValueError):
        tb.ycbcr_to_rgb(px([[0.5, 0.5, 0.5]]))           # an RGB-tagged image


def test_ycbcr_roundtrip_random_and_mid_gray():
    rng = np.random.default_rng(46)
    p = rng.uniform(0, 1, (50, 3))
    back = tb.ycbcr_to_rgb(tb.rgb_to_ycbcr(px(p))).pixels[0]
    # the forward transform clips chroma at [0, 1]; interior colours round-trip
    assert np.abs(back - p).max() < 1e-12
    g = tb.ycbcr_to_rgb(tb.rgb_to_ycbcr(px([[0.5, 0.5, 0.5]]))).pixels[0, 0]
    assert np.abs(g - 0.5).max() < 1e-15


def test_ipt_white_black_gray_and_scalar_oracle():
    out = tb.rgb_to_ipt(px([[1, 1, 1], [0, 0, 0]])).pixels[0]
    assert np.abs(out[0] - [1, 0.5, 0.5]).max() < 1e-9 and np.abs(out[1] - [0, 0.5, 0.5]).max() < 1e-15
    grays = np.linspace(0, 1, 11)[:, None].repeat(3, axis=1)
    o = tb.rgb_to_ipt(px(grays)).pixels[0]
    assert np.abs(o[:, 1:] - 0.5).max() < 1e-6
    p = np.random.default_rng(47).uniform(0, 1, (20, 3))
    assert np.abs(tb.rgb_to_ipt(px(p)).pixels[0] - oracle.rgb_to_ipt(p)).max() < 1e-12


def test_ipt_roundtrips_and_clamp_count():
    rng = np.random.default_rng(48)
    p = rng.uniform(0.05, 0.95, (40, 3))
    assert np.abs(tb.ipt_to_rgb(tb.rgb_to_ipt(px(p))).pixels[0] - p).max() < 1e-10
    for c in ([1, 0, 0], [1, 1, 1], [0, 0, 0]):
        assert np.abs(tb.ipt_to_rgb(tb.rgb_to_ipt(px([c]))).pixels[0, 0] - c).max() < 1e-9
    ipt = tb.ColorImage(np.array([[[1.5, 0.5, 0.5], [0.5, 0.5, 0.5], [0.2, 1.2, -0.3]]]), tb.SPACE_IPT)  # 2 out of gamut
    img, n = tb.ipt_to_rgb(ipt, count_clamped=True)
    assert n == 2 and img.pixels.min() >= 0.0 and img.pixels.max() <= 1.0
