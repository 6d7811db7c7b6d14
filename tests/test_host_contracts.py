"""Host-side API contracts that need no device arithmetic: DenseTensor,
unfold/fold layout views and the argument validation that the reference
raises before computing (tensor.py:33-108, 111-123, 138-173, 183-209;
tucker.py:74-95, 130-148; codec.py:114-148). These run on the CPU."""

from __future__ import annotations

import numpy as np
import pytest

import paper_2104_04726_b200 as tb


def test_from_flat_linearisation_and_length():  # DenseTensor.from_flat, tensor.py:52-61
    t = tb.DenseTensor.from_flat(np.arange(1.0, 25.0), (2, 3, 4))
    assert t.array[1, 0, 0] == 2 and t.array[0, 1, 0] == 3 and t.array[0, 0, 1] == 7
    assert np.array_equal(t.data, np.arange(1.0, 25.0))
    with pytest.raises(ValueError):
        tb.DenseTensor.from_flat(np.arange(5.0), (2, 3))


def test_dense_tensor_rejects_bad_input():  # tensor.py:42-50
    with pytest.raises(ValueError):
        tb.DenseTensor(np.array([[1.0, np.nan]]), check_finite=True)
    tb.DenseTensor(np.array([[1.0, np.nan]]))  # only checked on request
    with pytest.raises(ValueError):
        tb.DenseTensor(np.zeros((3, 0, 2)))


def test_unfold_layouts():  # tensor.py:89-108
    x = np.random.default_rng(0).standard_normal((3, 4, 5))
    t = tb.DenseTensor(x)
    assert np.array_equal(tb.unfold(t, 0)[:, 0], x[:, 0, 0])           # mode-0 columns are fibers
    assert np.array_equal(tb.unfold(t, 0)[:, 1], x[:, 1, 0])           # lowest remaining mode fastest
    assert tb.unfold(tb.DenseTensor(np.arange(4.0)), 0).shape == (4, 1)  # order 1: one column
    m = np.random.default_rng(1).standard_normal((3, 5))
    assert np.array_equal(tb.unfold(tb.DenseTensor(m), 1), m.T)         # order 2, mode 1 = transpose
    with pytest.raises(ValueError, match="mode 3"):
        tb.unfold(t, 3)


def test_fold_roundtrip_every_mode_and_shape_check():
    x = np.random.default_rng(2).standard_normal((2, 3, 4, 5))
    t = tb.DenseTensor(x)
    for n in range(4):
        assert np.array_equal(tb.fold(tb.unfold(t, n), n, x.shape).array, x)
    m = np.random.default_rng(3).standard_normal((4, 6))
    assert np.array_equal(tb.fold(m, 0, (4, 6)).array, m)
    with pytest.raises(ValueError):
        tb.fold(np.zeros((3, 7)), 0, (3, 4, 2))


def test_validation_raises_before_compute():
    t = tb.DenseTensor(np.ones((3, 4, 5)))
    with pytest.raises(ValueError, match="mode 1"):                     # ttm dimension mismatch
        tb.ttm(t, np.ones((2, 5)), 1)
    with pytest.raises(ValueError):
        tb.ttmc(t, [np.eye(3), np.eye(4)])                             # wrong factor count
    with pytest.raises(ValueError, match="mode 2"):
        tb.ttmc(t, [np.eye(3), np.eye(4), np.eye(4)])
    with pytest.raises(ValueError):
        tb.ttmc(t, [np.eye(3), np.eye(4), np.eye(5)], order="random")
    with pytest.raises(ValueError):
        tb.leading_eigvecs(np.eye(3), 4)                               # k out of range
    with pytest.raises(ValueError):
        tb.leading_eigvecs(np.eye(3), 0)
    with pytest.raises(ValueError):
        tb.leading_eigvecs(np.ones((2, 3)), 1)
    with pytest.raises(ValueError, match="mode 0"):
        tb.t_hosvd(t, (4, 2, 2))                                        # rank > dim
    with pytest.raises(ValueError):
        tb.t_hosvd(t, (2, 2))                                           # rank count


@pytest.mark.parametrize("kw", [dict(fit_tol=0.0), dict(pp_exit_tol=0.0), dict(max_sweeps=-1)])
def test_solve_config_validation(kw):  # tucker.py:84-95
    with pytest.raises(ValueError):
        tb.SolveConfig(ranks=(2, 2, 2), **kw).validate((3, 3, 3))
    with pytest.raises(ValueError, match="mode 1"):
        tb.SolveConfig(ranks=(2, 0, 2)).validate((3, 3, 3))


def test_quantiser_and_dequantiser_validation():  # codec.py:121-122, 140-144
    core = tb.DenseTensor(np.ones((2, 2, 1)))
    model = tb.TuckerModel(core, [np.eye(3)[:, :2], np.eye(2), np.eye(1)], (3, 2, 1))
    for qp in (-1, 52):
        with pytest.raises(ValueError):
            tb.quantize_core(model, qp)
    q = tb.QuantizedModel((3, 2, 1), (2, 2, 1), 1.0, 51, np.zeros((2, 2)), [np.zeros((3, 2), np.float32)] * 3)
    with pytest.raises(tb.CodecError):
        tb.dequantize(q)


def test_preset_ranks_rule():  # codec.py:86-95, against the oracle restatement
    import oracle

    for k in range(1, 6):
        for dims in [(1080, 1920, 5, 2), (36, 64, 3, 2), (7, 5, 9, 1)]:
            assert tuple(tb.preset_ranks(k, dims)) == tuple(oracle.preset_ranks(k, dims))
