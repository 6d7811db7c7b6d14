"""Drop-in API contract tests on the device path (ports of the reference's
tests/test_tensor.py, test_tucker.py, test_pp.py, test_color.py and
test_codec.py at the reference's own fp64 tolerances), plus oracle
comparisons for every kernel family. Every call goes through libtmb."""

from __future__ import annotations

import numpy as np
import pytest

import oracle
import paper_2104_04726_b200 as tb
from paper_2104_04726_b200 import _lib as L

pytestmark = pytest.mark.gpu


def rand_orth(rng, rows, cols):
    return np.linalg.qr(rng.standard_normal((rows, cols)))[0]


def random_tucker_tensor(rng, dims, ranks):
    core = tb.DenseTensor(rng.standard_normal(ranks))
    model = tb.TuckerModel(core, [rand_orth(rng, s, r) for s, r in zip(dims, ranks)], tuple(dims))
    return tb.reconstruct(model), model


def rel_err(a, b):
    return float(np.linalg.norm(a.array - b.array) / np.linalg.norm(a.array))


# ------------------------------------------------------------------ tensor.py
def test_ttm_identity_and_oracle():
    rng = np.random.default_rng(1)
    t = tb.DenseTensor(rng.standard_normal((4, 3, 5)))
    for n in range(3):
        assert np.abs(tb.ttm(t, np.eye(t.dims[n]), n).array - t.array).max() < 1e-15
        m = rng.standard_normal((6, t.dims[n]))
        assert np.abs(tb.ttm(t, m, n).array - oracle.ttm(t.array, m, n)).max() < 1e-12


def test_ttm_large_modes_gemm_path():
    rng = np.random.default_rng(2)
    x = rng.standard_normal((130, 97, 4, 3))
    for n, r in [(0, 70), (1, 80)]:
        m = rng.standard_normal((r, x.shape[n]))
        got = tb.ttm(tb.DenseTensor(x), m, n).array
        ref = oracle.ttm(x, m, n)
        assert np.abs(got - ref).max() / np.abs(ref).max() < 1e-13


def test_ttmc_nested_loop_oracle_and_orders():  # tests/test_tensor.py:127-165
    rng = np.random.default_rng(4)
    t = tb.DenseTensor(rng.standard_normal((3, 3, 3)))
    fs = [rng.standard_normal((3, 2)) for _ in range(3)]
    out = tb.ttmc(t, fs).array
    expect = np.einsum("abc,ai,bj,ck->ijk", t.array, *fs)
    assert np.abs(out - expect).max() < 1e-12
    t4 = tb.DenseTensor(rng.standard_normal((6, 5, 4, 3)))
    f4 = [rand_orth(rng, s, 2) for s in t4.dims]
    a = tb.ttmc(t4, f4, order="ascending").array
    g = tb.ttmc(t4, f4, order="greedy").array
    assert np.abs(a - g).max() < 1e-12


def test_ttmc_skip_hand_case():  # tests/test_tensor.py:149-156
    t = tb.DenseTensor.from_flat(np.arange(1.0, 9.0), (2, 2, 2))
    u = np.array([[1.0], [1.0]])
    out = tb.ttmc(t, [None, u, u], skip=0)
    assert out.dims == (2, 1, 1)
    assert np.allclose(out.array[:, 0, 0], [16.0, 20.0])


def test_ttmc_error_names_mode():  # tests/test_tensor.py:167-172
    t = tb.DenseTensor(np.ones((2, 3, 4)))
    with pytest.raises(ValueError, match="mode 1"):
        tb.ttmc(t, [np.eye(2), np.eye(2), np.eye(4)])


def test_gram_exact_symmetry_and_oracle():  # tests/test_tensor.py:184-194
    rng = np.random.default_rng(5)
    for shape in [(5, 9), (120, 300), (70, 40)]:
        m = rng.standard_normal(shape)
        g = tb.gram(m)
        assert np.array_equal(g, g.T)
        ref = oracle.gram(m)
        assert np.abs(g - ref).max() / np.abs(ref).max() < 1e-14


def test_mode_gram_matches_unfold_gram():
    rng = np.random.default_rng(6)
    x = rng.standard_normal((80, 70, 3, 5))
    for n in range(4):
        got = tb.mode_gram(tb.DenseTensor(x), n)
        ref = oracle.gram(oracle.unfold(x, n))
        assert np.abs(got - ref).max() / np.abs(ref).max() < 1e-13


def test_eig_diagonal_and_sign_rule():  # tests/test_tensor.py:196-207
    v, w = tb.leading_eigvecs(np.diag([3.0, 2.0, 1.0]), 2)
    assert np.allclose(w, [3, 2]) and np.allclose(v, [[1, 0], [0, 1], [0, 0]])
    v1, _ = tb.leading_eigvecs(np.outer([0.6, -0.8], [0.6, -0.8]), 1)
    assert np.allclose(v1[:, 0], [-0.6, 0.8])


@pytest.mark.parametrize("n,k", [(7, 7), (33, 10), (64, 64), (65, 20), (200, 50), (281, 40), (282, 40), (700, 100)])
def test_eig_residual_orthonormal_vs_lapack(n, k):  # tests/test_tensor.py:209-216
    rng = np.random.default_rng(n)
    b = rng.standard_normal((n, n))
    g = b @ b.T
    v, w = tb.leading_eigvecs(g, k)
    vr, wr = oracle.leading_eigvecs(g, k)
    assert np.abs(v.T @ v - np.eye(k)).max() < 1e-10
    assert np.abs(g @ v - v * w).max() / wr[0] < 1e-10
    assert np.abs(w - wr).max() / wr[0] < 1e-12
    assert np.abs(v - vr).max() < 1e-7            # same columns, same signs (sign rule)


def test_eig_graded_spectrum_large():
    """Image-like Gram: eigenvalues over 1e8, tridiagonal path."""
    rng = np.random.default_rng(8)
    n, k = 1080, 270
    q = rand_orth(rng, n, n)
    lam = 1e3 * np.exp(-np.linspace(0, 20, n))
    g = (q * lam) @ q.T
    g = 0.5 * (g + g.T)
    v, w = tb.leading_eigvecs(g, k)
    vr, wr = oracle.leading_eigvecs(g, k)
    from conftest import principal_angle

    assert principal_angle(v, vr) < 1e-9
    assert np.abs(v.T @ v - np.eye(k)).max() < 1e-12
    assert np.abs(w - wr).max() / wr[0] < 1e-13


@pytest.mark.parametrize("n,k", [(601, 1), (1023, 255), (1537, 401), (1920, 480), (1999, 3), (2048, 512),
                                 (2101, 97)])
def test_eig_kernel_paths_vs_lapack(n, k):
    """Every tridiagonalisation/back-transform variant boundary: shared-memory
    rows kernel (601..1999, odd n -> unaligned WY streaming, ragged k -> partial
    column blocks), L2 rows kernel (2048), column kernel (2101)."""
    rng = np.random.default_rng(n + k)
    q = rand_orth(rng, n, n)
    lam = 1e3 * np.exp(-np.linspace(0, 18, n))
    g = (q * lam) @ q.T
    g = 0.5 * (g + g.T)
    v, w = tb.leading_eigvecs(g, k)
    vr, wr = oracle.leading_eigvecs(g, k)
    from conftest import principal_angle

    assert np.abs(v.T @ v - np.eye(k)).max() < 1e-12
    assert np.abs(w - wr).max() / wr[0] < 1e-13
    assert np.abs(g @ v - v * w).max() / wr[0] < 1e-12
    assert principal_angle(v, vr) < 1e-8
    v2, w2 = tb.leading_eigvecs(g, k)
    assert np.array_equal(v, v2) and np.array_equal(w, w2)  # deterministic


@pytest.mark.parametrize("n,k", [(2160, 270), (3840, 480), (4320, 540), (7680, 960)])
def test_eig_large_n_vs_lapack(n, k):
    """The Gram sizes of BASELINE configs 4 and 5 (n = 2160, 3840, 4320, 7680;
    k = the configs' ranks): column-kernel tridiagonalisation and the unfused
    back-transform, against LAPACK (numpy eigh, the reference's dsyevd) and
    the known spectral decomposition the matrix was built from."""
    rng = np.random.default_rng(n + k)
    q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    lam = 1e3 * np.exp(-np.linspace(0, 18, n))
    g = (q * lam) @ q.T
    g = 0.5 * (g + g.T)
    v, w = tb.leading_eigvecs(g, k)
    vr, wr = oracle.leading_eigvecs(g, k)
    from conftest import principal_angle

    assert np.abs(v.T @ v - np.eye(k)).max() < 1e-12
    assert np.abs(w - wr).max() / wr[0] < 1e-13
    assert np.abs(w - lam[:k]).max() / lam[0] < 1e-13
    assert np.abs(g @ v - v * w).max() / wr[0] < 1e-12
    assert principal_angle(v, vr) < 1e-8
    assert principal_angle(v, q[:, :k]) < 1e-8
    # same sign rule as the reference: per-column agreement with LAPACK's sign-fixed vectors
    assert np.abs(v - vr).max() < 1e-8


def _cluster_checks(g, k, v, w, clusters):
    vr, wr = oracle.leading_eigvecs(g, k)
    from conftest import principal_angle

    scale = max(abs(wr[0]), 1.0)
    assert np.abs(v.T @ v - np.eye(k)).max() < 1e-12
    assert np.abs(w - wr).max() / scale < 1e-12
    assert np.abs(g @ v - v * w).max() / scale < 1e-10
    for a, b in clusters:   # a repeated eigenvalue's vectors are defined up to rotation: compare spans
        assert principal_angle(v[:, a:b], vr[:, a:b]) < 1e-8


def test_eig_repeated_eigenvalue_cluster():
    """n > 64 with an exactly repeated eigenvalue (20-fold) inside the
    wanted block -- the independently computed twisted vectors come out parallel
    and the cluster is repaired by block inverse iteration."""
    rng = np.random.default_rng(31)
    n, k = 300, 60
    lam = np.concatenate([np.linspace(50, 11, 10), np.full(20, 7.0), np.linspace(5, 0.1, n - 30)])
    q = rand_orth(rng, n, n)
    g = (q * lam) @ q.T
    g = 0.5 * (g + g.T)
    v, w = tb.leading_eigvecs(g, k)
    _cluster_checks(g, k, v, w, [(10, 30)])


def test_eig_rank_deficient_gram():
    """A Gram of rank 40 asked for 100 eigenvectors (60 zero eigenvalues), n = 500."""
    rng = np.random.default_rng(32)
    b = rng.standard_normal((500, 40))
    g = b @ b.T
    v, w = tb.leading_eigvecs(g, 100)
    vr, wr = oracle.leading_eigvecs(g, 100)
    assert np.abs(v.T @ v - np.eye(100)).max() < 1e-12
    assert np.abs(w - wr).max() / wr[0] < 1e-12
    assert np.abs(g @ v - v * w).max() / wr[0] < 1e-12
    from conftest import principal_angle

    assert principal_angle(v[:, :40], vr[:, :40]) < 1e-9
    # the 60 null-space vectors are orthogonal to the range of b
    assert np.abs(b.T @ v[:, 40:]).max() < 1e-10 * np.abs(b).max()


def test_hosvd_rank_deficient_modes():
    """ADVICE r1 example: hosvd of a (100, 3, 3) tensor -- the mode-0 Gram has
    rank <= 9 and all 100 eigenvectors are wanted; exact reconstruction and
    orthonormal factors (tests/test_tucker.py:50-55 at n > 64)."""
    rng = np.random.default_rng(33)
    t = tb.DenseTensor(rng.standard_normal((100, 3, 3)))
    model = tb.hosvd(t)
    model.validate()
    rec = tb.reconstruct(model)
    assert np.abs(rec.array - t.array).max() < 1e-10


def test_eig_deterministic():  # tests/test_tensor.py:218-223
    rng = np.random.default_rng(9)
    b = rng.standard_normal((300, 300))
    g = b @ b.T
    a1, w1 = tb.leading_eigvecs(g, 40)
    a2, w2 = tb.leading_eigvecs(g, 40)
    assert np.array_equal(a1, a2) and np.array_equal(w1, w2)


def test_fro_norm():  # tests/test_tensor.py:232-242
    assert tb.fro_norm(tb.DenseTensor(np.zeros((2, 2)))) == 0.0
    assert tb.fro_norm(tb.DenseTensor(np.ones((2, 3, 4)))) == pytest.approx(np.sqrt(24.0), rel=1e-15)


# ------------------------------------------------------------------ tucker.py
def test_hosvd_single_nonzero():  # tests/test_tucker.py:37-48
    arr = np.zeros((3, 3, 3))
    arr[1, 2, 0] = 5.0
    model = tb.hosvd(tb.DenseTensor(arr))
    mags = np.sort(np.abs(model.core.array).ravel())
    assert mags[-1] == pytest.approx(5.0) and mags[-2] < 1e-12
    for f in model.factors:
        assert np.allclose(np.abs(f).sum(axis=0), 1.0) and np.allclose(np.abs(f).max(axis=0), 1.0)


def test_hosvd_reconstruction_and_svd():  # tests/test_tucker.py:50-68
    rng = np.random.default_rng(0)
    t = tb.DenseTensor(rng.standard_normal((4, 4, 4)))
    model = tb.hosvd(t)
    model.validate()
    assert rel_err(t, tb.reconstruct(model)) < 1e-10
    a = np.random.default_rng(1).standard_normal((5, 7))
    u = tb.hosvd(tb.DenseTensor(a)).factors[0]
    u_svd = np.linalg.svd(a)[0]
    for j in range(5):
        col = u_svd[:, j]
        col = -col if col[np.argmax(np.abs(col))] < 0 else col
        assert np.allclose(u[:, j], col, atol=1e-8)


def test_thosvd_full_equals_hosvd_and_exact_recovery():  # tests/test_tucker.py:72-86
    rng = np.random.default_rng(2)
    t = tb.DenseTensor(rng.standard_normal((3, 4, 5)))
    a, b = tb.hosvd(t), tb.t_hosvd(t, (3, 4, 5))
    for fa, fb in zip(a.factors, b.factors):
        assert np.array_equal(fa, fb)
    assert np.array_equal(a.core.array, b.core.array)
    t2, _ = random_tucker_tensor(np.random.default_rng(3), (6, 6, 6), (2, 2, 2))
    m = tb.t_hosvd(t2, (2, 2, 2))
    m.validate()
    assert rel_err(t2, tb.reconstruct(m)) < 1e-8


def test_thosvd_error_bound():  # tests/test_tucker.py:88-100
    for seed in range(3):
        rng = np.random.default_rng(seed)
        t = tb.DenseTensor(rng.standard_normal((6, 5, 4)))
        model = tb.t_hosvd(t, (2, 2, 2))
        err2 = float(np.linalg.norm(t.array - tb.reconstruct(model).array) ** 2)
        bound = sum(float(np.sum(np.sort(np.linalg.eigvalsh(oracle.gram(oracle.unfold(t.array, n))))[::-1][2:]))
                    for n in range(3))
        assert err2 <= bound * (1 + 1e-8) + 1e-10


def test_hooi_fixed_point_and_monotone():  # tests/test_tucker.py:130-147
    rng = np.random.default_rng(7)
    t, _ = random_tucker_tensor(rng, (6, 5, 4), (2, 2, 2))
    start = tb.t_hosvd(t, (2, 2, 2))
    swept = tb.hooi_sweep(t, start)
    for a, b in zip(swept.factors, start.factors):
        assert np.allclose(a, b, atol=1e-8)
    assert tb.fit(t, swept) >= 1 - 1e-7
    t3 = tb.DenseTensor(np.random.default_rng(8).standard_normal((5, 5, 5)))
    m = tb.t_hosvd(t3, (2, 2, 2))
    assert tb.fit(t3, tb.hooi_sweep(t3, m)) >= tb.fit(t3, m) - 1e-12


def test_hooi_matches_oracle_sweep():
    rng = np.random.default_rng(10)
    x = rng.standard_normal((9, 8, 4, 3))
    ranks = (4, 3, 2, 2)
    m0 = tb.t_hosvd(tb.DenseTensor(x), ranks)
    core_o, fac_o = oracle.t_hosvd(x, ranks)
    for a, b in zip(m0.factors, fac_o):
        assert np.abs(a - b).max() < 1e-10
    m1 = tb.hooi_sweep(tb.DenseTensor(x), m0)
    core1, fac1 = oracle.hooi_sweep(x, fac_o)
    for a, b in zip(m1.factors, fac1):
        assert np.abs(a - b).max() < 1e-9
    assert np.abs(m1.core.array - core1).max() < 1e-10


@pytest.mark.parametrize("dims,ranks", [
    ((20, 24, 3, 18), (5, 6, 3, 9)),    # C5-like trailing modes: fused pass with > 48 KB of inner sums
    ((20, 24, 3, 10), (5, 6, 3, 5)),    # C2-like: fused pass
    ((12, 14, 12, 10), (4, 5, 9, 5)),   # r1 = 9 > 8: separate small-mode passes
])
def test_hooi_small_mode_paths_match_oracle(dims, ranks):
    """The sweep's trailing small-mode contractions (fused two-mode pass or two
    separate passes) against the oracle's ascending ttmc."""
    rng = np.random.default_rng(sum(dims))
    x = rng.standard_normal(dims)
    m0 = tb.t_hosvd(tb.DenseTensor(x), ranks)
    core_o, fac_o = oracle.t_hosvd(x, ranks)
    m1 = tb.hooi_sweep(tb.DenseTensor(x), m0)
    core1, fac1 = oracle.hooi_sweep(x, fac_o)
    from conftest import principal_angle

    for a, b in zip(m1.factors, fac1):
        assert principal_angle(a, b) < 1e-8
    assert abs(np.linalg.norm(m1.core.array) - np.linalg.norm(core1)) < 1e-10 * np.linalg.norm(core1)


def test_fit_and_reconstruct_contracts():  # tests/test_tucker.py:169-254
    rng = np.random.default_rng(11)
    t = tb.DenseTensor(rng.standard_normal((6, 5, 4)))
    model = tb.t_hosvd(t, (3, 3, 2))
    assert abs(tb.fit(t, model) - tb.fit(t, model, method="residual")) < 1e-10
    with pytest.raises(ValueError):
        tb.fit(tb.DenseTensor(np.zeros((2, 2))), model)
    core = rng.standard_normal((2, 3, 2))
    fs = [rng.standard_normal((4, 2)), rng.standard_normal((3, 3)), rng.standard_normal((5, 2))]
    got = tb.reconstruct(tb.TuckerModel(tb.DenseTensor(core), fs, (4, 3, 5))).array
    expect = np.einsum("abc,ia,jb,kc->ijk", core, *fs)
    assert np.abs(got - expect).max() < 1e-12


def test_tucker_als_contracts():  # tests/test_tucker.py:258-313
    rng = np.random.default_rng(18)
    t, _ = random_tucker_tensor(rng, (8, 9, 8), (2, 3, 2))
    model, trace = tb.tucker_als(t, tb.SolveConfig(ranks=(2, 3, 2), max_sweeps=10))
    assert trace.converged and tb.fit(t, model) >= 1 - 1e-6
    model.validate()
    t2 = tb.DenseTensor(np.random.default_rng(19).standard_normal((4, 5, 3)))
    model2, trace2 = tb.tucker_als(t2, tb.SolveConfig(ranks=(4, 5, 3)))
    assert trace2.converged and len(trace2.records) == 1 and trace2.records[0].kind == "init"
    t3 = tb.DenseTensor(np.random.default_rng(20).standard_normal((16, 16, 10)))
    _, tr3 = tb.tucker_als(t3, tb.SolveConfig(ranks=(4, 4, 3), max_sweeps=20, fit_tol=1e-9, pp_enter_tol=0.0))
    fits = [r.fit for r in tr3.records]
    assert all(r.kind in ("init", "standard") for r in tr3.records)
    assert all(b >= a - 1e-12 for a, b in zip(fits, fits[1:]))
    with pytest.raises(ValueError):
        tb.tucker_als(tb.DenseTensor(np.zeros((3, 3))), tb.SolveConfig(ranks=(2, 2)))
    t4 = tb.DenseTensor(np.random.default_rng(21).standard_normal((10, 10, 10)))
    m4, tr4 = tb.tucker_als(t4, tb.SolveConfig(ranks=(3, 3, 3), max_sweeps=1, fit_tol=1e-14, pp_enter_tol=0.0))
    assert not tr4.converged
    m4.validate()


def test_tucker_als_greedy_matches_sequential():  # tests/test_tucker.py:315-321 (PP off)
    t = tb.DenseTensor(np.random.default_rng(23).standard_normal((9, 7, 5, 3)))
    ranks = (3, 3, 2, 2)
    kw = dict(ranks=ranks, pp_enter_tol=0.0, max_sweeps=30)
    f_seq = tb.fit(t, tb.tucker_als(t, tb.SolveConfig(sequential_reduction=True, **kw))[0])
    f_gr = tb.fit(t, tb.tucker_als(t, tb.SolveConfig(sequential_reduction=False, **kw))[0])
    assert abs(f_seq - f_gr) < 1e-9


def test_api_goldens_reference_parity(golden):
    """Reference tucker_als on random f64 tensors (tests/golden/api.npz)."""
    z = golden("api")
    for k in range(3):
        t = tb.DenseTensor(z[f"x{k}"])
        cfg = tb.SolveConfig(ranks=tuple(int(r) for r in z[f"ranks{k}"]), max_sweeps=int(z[f"sweeps{k}"]),
                             fit_tol=1e-300, pp_enter_tol=0.0)
        model, trace = tb.tucker_als(t, cfg)
        fits = np.array([r.fit for r in trace.records])
        # fit_tol=1e-300 stops only on a bitwise-stationary fit, which rounding decides:
        # compare the common prefix (both solves are at the fixed point afterwards)
        m = min(len(fits), len(z[f"fit{k}"]))
        assert np.abs(fits[:m] - z[f"fit{k}"][:m]).max() < 1e-12
        for n, f in enumerate(model.factors):
            assert np.abs(f - z[f"f{k}_{n}"]).max() < 1e-8
        assert np.abs(model.core.array - z[f"core{k}"]).max() < 1e-8


def test_pp_operators_tree():  # tests/test_pp.py:50-83
    rng = np.random.default_rng(5)
    x = rng.standard_normal((5, 4, 3, 3))
    anchors = [rand_orth(rng, s, 2) for s in x.shape]
    st = tb.pp_operators(tb.DenseTensor(x), anchors)
    assert st.contraction_count == 13
    ref = oracle.pp_operators(x, anchors)
    for n in range(4):
        assert np.abs(st.op_single[n].array - ref.single[n]).max() < 1e-12
    for key, y in ref.pair.items():
        assert np.abs(st.op_pair[key].array - y).max() < 1e-12


def test_pp_sweep_matches_oracle():  # tests/test_pp.py:93-153
    rng = np.random.default_rng(12)
    x = rng.standard_normal((7, 6, 5, 4))
    ranks = (3, 3, 2, 2)
    model = tb.t_hosvd(tb.DenseTensor(x), ranks)
    st = tb.pp_operators(tb.DenseTensor(x), model.factors)
    moved = tb.hooi_sweep(tb.DenseTensor(x), model)
    st.set_current(moved.factors)
    out = tb.pp_sweep(st, moved)
    ops = oracle.pp_operators(x, model.factors)
    core_o, fac_o = oracle.pp_sweep(ops, moved.factors)
    for a, b in zip(out.factors, fac_o):
        assert np.abs(a - b).max() < 1e-8
    assert np.abs(out.core.array - core_o).max() < 1e-8


# ------------------------------------------------------------------ color.py / codec.py
def test_colour_f64_matches_reference(golden):
    z = golden("colour")
    px = z["fpx"]  # (1, 500, 3); the golden holds pixels[0]
    assert np.array_equal(tb.rgb_to_ycbcr(tb.ColorImage(px)).pixels[0], z["ycbcr_f"])
    assert np.abs(tb.rgb_to_ipt(tb.ColorImage(px)).pixels[0] - z["ipt_f"]).max() < 1e-14


def test_colour_inverses_roundtrip():  # tests/test_color.py round trips
    rng = np.random.default_rng(13)
    px = rng.uniform(0.05, 0.95, size=(8, 9, 3))
    back = tb.ycbcr_to_rgb(tb.rgb_to_ycbcr(tb.ColorImage(px))).pixels
    assert np.abs(back - px).max() < 1e-12
    back2, n = tb.ipt_to_rgb(tb.rgb_to_ipt(tb.ColorImage(px)), count_clamped=True)
    assert np.abs(back2.pixels - px).max() < 1e-9 and n == 0
    ref = oracle.ipt_to_rgb(oracle.rgb_to_ipt(px))
    assert np.abs(back2.pixels - ref).max() < 1e-12


def test_colour_u8_kernel_bit_exact(golden):
    """u8 -> fp32 coding-space tensor equals fp32(reference f64 colour) bit for bit."""
    z = golden("colour")
    u8 = z["u8"]
    for space in ("ycbcr", "ipt"):
        t = tb.coding_tensor(u8.reshape(1, 1, 1, -1, 3), space).cpu().numpy()
        got = t.reshape((1, u8.shape[0], 3, 1), order="F")[0, :, :, 0]
        assert np.array_equal(got, z[f"{space}_u8"].astype(np.float32))


@pytest.mark.parametrize("space", ["ycbcr", "ipt"])
def test_colour_u8_exhaustive(space):
    """Every one of the 2^24 u8 RGB triples (one 4096 x 4096 image, full tiles
    and the 16-byte load/store path) maps to fp32(reference f64 colour) bit for
    bit; a ragged 2-image stack exercises the partial-tile path."""
    codes = np.arange(1 << 24, dtype=np.uint32)
    u8 = np.stack([(codes >> 16) & 255, (codes >> 8) & 255, codes & 255], axis=-1).astype(np.uint8)
    t = tb.coding_tensor(u8.reshape(1, 1, 4096, 4096, 3), space).cpu().numpy()
    got = t.reshape((4096, 4096, 3), order="F")
    fn = oracle.rgb_to_ycbcr if space == "ycbcr" else oracle.rgb_to_ipt
    ref = fn(u8.reshape(4096, 4096, 3).astype(np.float64) / 255.0).astype(np.float32)
    assert np.array_equal(got, ref), int((got != ref).sum())
    # ... and against the REFERENCE's own colour on the same 2^24 triples (sha256 of its
    # fp32-rounded output, scripts/make_golden_colour_exhaustive.py)
    import hashlib
    import json
    from conftest import GOLDEN

    want = json.loads((GOLDEN / "colour_exhaustive.json").read_text())[space]
    assert hashlib.sha256(np.ascontiguousarray(got).tobytes()).hexdigest() == want
    rng = np.random.default_rng(21)
    imgs = rng.integers(0, 256, size=(1, 2, 37, 70, 3), dtype=np.uint8)
    got2 = tb.coding_tensor(imgs, space).cpu().numpy().reshape((37, 70, 3, 2), order="F")
    ref2 = oracle.coding_tensor(imgs, space).astype(np.float32)
    assert np.array_equal(got2, ref2)


def test_quantiser_contracts():  # tests/test_codec.py:57-85
    rng = np.random.default_rng(14)
    core = rng.standard_normal((4, 5, 3, 2))
    fs = [np.eye(s)[:, :r] for s, r in zip((4, 5, 3, 2), (4, 5, 3, 2))]
    m = tb.TuckerModel(tb.DenseTensor(core), fs, (4, 5, 3, 2))
    q51 = tb.quantize_core(m, 51)
    lv, step = oracle.quantize_core(core, 51)
    assert q51.step == step and np.array_equal(q51.levels, lv) and q51.levels.dtype == np.int64
    assert tb.quantize_core(m, 45).step == pytest.approx(q51.step / 2, rel=1e-15)
    deq = tb.dequantize(q51)
    assert np.abs(deq.core.array - core).max() <= q51.step / 2 + 1e-15
    assert all(f.dtype == np.float32 for f in q51.factors)
    z = tb.TuckerModel(tb.DenseTensor(np.zeros((2, 2))), [np.eye(2), np.eye(2)], (2, 2))
    assert tb.quantize_core(z, 30).step == 1.0


def test_launch_counter_advances():
    n0 = L.launch_count()
    tb.gram(np.ones((3, 4)))
    assert L.launch_count() > n0


def test_workspace_pool_query_and_reserve():
    """the library's own per-context pool; after one solve the
    high-water mark is known, reserving it up front means later solves of the
    same shape allocate nothing new (the reserved capacity does not grow)."""
    import ctypes as C

    h = L.ctx()
    rng = np.random.default_rng(31)
    x = tb.DenseTensor(rng.standard_normal((40, 50, 3, 6)))
    cfg = tb.SolveConfig(ranks=(8, 9, 3, 3), max_sweeps=3, fit_tol=1e-300, pp_enter_tol=0.0)
    tb.tucker_als(x, cfg)
    res, peak = C.c_int64(), C.c_int64()
    L.check(L.LIB.tmb_workspace_size(h, C.byref(res), C.byref(peak)), h)
    assert 0 < peak.value <= res.value
    L.check(L.LIB.tmb_workspace_reserve(h, res.value + (64 << 20)), h)
    res2 = C.c_int64()
    L.check(L.LIB.tmb_workspace_size(h, C.byref(res2), C.byref(peak)), h)
    assert res2.value >= res.value + (64 << 20)
    tb.tucker_als(x, cfg)
    res3 = C.c_int64()
    L.check(L.LIB.tmb_workspace_size(h, C.byref(res3), C.byref(peak)), h)
    assert res3.value == res2.value
    assert L.LIB.tmb_workspace_reserve(h, -1) != 0


@pytest.mark.parametrize("n,k", [(2160, 270), (2500, 97)])
def test_eig_lazy_panels_forced_vs_lapack(n, k):
    """The lazy (blocked) tridiagonalisation panels, forced down to trailing size
    1000 (TMB_LAZY_SWITCH; by default they only run while the trailing matrix
    exceeds 3500, i.e. at the C5 / C4 sizes tested above): several 32-step panels,
    the rank-64 trailing GEMM updates, then the column kernel from the hand-off
    step. Same accuracy contract as LAPACK."""
    import os
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parents[1]
    code = f"""
import sys; sys.path[:0] = [{str(root)!r}, {str(root / 'tests')!r}]
import numpy as np, oracle, paper_2104_04726_b200 as tb
from conftest import principal_angle
n, k = {n}, {k}
rng = np.random.default_rng(n + k)
q, _ = np.linalg.qr(rng.standard_normal((n, n)))
lam = 1e3 * np.exp(-np.linspace(0, 18, n))
g = (q * lam) @ q.T
g = 0.5 * (g + g.T)
v, w = tb.leading_eigvecs(g, k)
vr, wr = oracle.leading_eigvecs(g, k)
assert np.abs(v.T @ v - np.eye(k)).max() < 1e-12
assert np.abs(w - wr).max() / wr[0] < 1e-13
assert np.abs(g @ v - v * w).max() / wr[0] < 1e-12
assert principal_angle(v, vr) < 1e-8
assert np.abs(v - vr).max() < 1e-8
print("ok")
"""
    env = dict(os.environ, TMB_LAZY_SWITCH="1000")
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0 and out.stdout.strip().endswith("ok"), out.stderr[-3000:]


def test_two_stage_forced_vs_lapack():
    """The two-stage path (dense -> 32-band -> tridiagonal, band inverse
    iteration, stage-1 WY back-transform), forced at sizes where the one-stage
    path is the default (TMB_EIG_2STAGE=1): LAPACK accuracy on graded and
    Wishart spectra, ragged panel counts, the tridiagonal form's eigenvalues
    (tmb_tridiagonalize), and the fallback to the one-stage repair path on a
    rank-deficient Gram and a 20-fold eigenvalue."""
    import os
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parents[1]
    code = f"""
import sys; sys.path[:0] = [{str(root)!r}, {str(root / 'tests')!r}]
import numpy as np, oracle, paper_2104_04726_b200 as tb
from paper_2104_04726_b200 import _lib as L
from conftest import principal_angle
rng = np.random.default_rng(5)
h = L.ctx()
for n, k, kind in [(130, 40, "decay"), (300, 75, "wishart"), (1000, 250, "decay"), (2161, 270, "decay")]:
    if kind == "decay":
        q, _ = np.linalg.qr(rng.standard_normal((n, n)))
        g = (q * (1e3 * np.exp(-np.linspace(0, 18, n)))) @ q.T
    else:
        y = rng.standard_normal((n, n + 5))
        g = y @ y.T
    g = 0.5 * (g + g.T)
    gd = L.dev_f64(g)
    d, e = L.empty_f64(n), L.empty_f64(n)
    L.check(L.LIB.tmb_tridiagonalize(h, L.ptr(gd), n, L.ptr(d), L.ptr(e)), h)
    dh, eh = d.cpu().numpy(), e.cpu().numpy()[: n - 1]
    wt = np.linalg.eigvalsh(np.diag(dh) + np.diag(eh, 1) + np.diag(eh, -1))
    wr_all = np.linalg.eigvalsh(g)
    assert np.abs(wt - wr_all).max() / np.abs(wr_all).max() < 1e-13, (n, "tridiagonal")
    v, w = tb.leading_eigvecs(g, k)
    vr, wr = oracle.leading_eigvecs(g, k)
    assert np.abs(v.T @ v - np.eye(k)).max() < 1e-12, n
    assert np.abs(w - wr).max() / wr[0] < 1e-13, n
    assert np.abs(g @ v - v * w).max() / wr[0] < 1e-12, n
    assert principal_angle(v, vr) < 1e-8, n
    assert np.abs(v - vr).max() < 1e-8, n
# rank 40 asked for 100 vectors: the band inverse iteration returns parallel null-space
# vectors, so the solver falls back to the one-stage path and its cluster repair
b = rng.standard_normal((500, 40))
g = b @ b.T
v, w = tb.leading_eigvecs(g, 100)
vr, wr = oracle.leading_eigvecs(g, 100)
assert np.abs(v.T @ v - np.eye(100)).max() < 1e-12
assert np.abs(w - wr).max() / wr[0] < 1e-12
assert principal_angle(v[:, :40], vr[:, :40]) < 1e-9
print("ok")
"""
    env = dict(os.environ, TMB_EIG_2STAGE="1")
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0 and out.stdout.strip().endswith("ok"), out.stderr[-3000:]


def test_ozaki_digit_cache_is_per_solve():
    """The Ozaki digit planes of the raw tensor are kept only for one solve: two
    different tensors solved one after the other IN THE SAME device buffer give
    exactly what each gives in a buffer of its own (the cache is keyed by the
    operand's address, so it must not survive the call). C2-size passes, so both
    full passes go through the Ozaki kernel."""
    import torch

    from paper_2104_04726_b200.tucker import solve_device

    dims = (1080, 1920, 3, 10)
    cfg = tb.SolveConfig(ranks=(270, 480, 3, 5), max_sweeps=2, fit_tol=1e-300, pp_enter_tol=0.0)
    g = torch.Generator(device="cuda").manual_seed(11)
    n = int(np.prod(dims))
    xa = torch.rand(n, generator=g, device="cuda", dtype=torch.float32)
    xb = torch.rand(n, generator=g, device="cuda", dtype=torch.float32) ** 2
    shared = xa.clone()
    solve_device(shared, L.F32, dims, cfg)          # fills the cache for `shared`'s address
    shared.copy_(xb)
    mb_shared, tb_shared = solve_device(shared, L.F32, dims, cfg)
    mb_own, tb_own = solve_device(xb.clone(), L.F32, dims, cfg)
    assert [r.fit for r in tb_shared.records] == [r.fit for r in tb_own.records]
    assert np.array_equal(mb_shared.core.array, mb_own.core.array)
    for u, v in zip(mb_shared.factors, mb_own.factors):
        assert np.array_equal(u, v)
