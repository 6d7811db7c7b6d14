"""Pin the CPU oracle (oracle/) before trusting it (CPU only).

(1) the reference's own known-answer values (taken from
    the reference test files cited per test);
(2) golden vectors produced by running the reference implementation itself
    (scripts/make_golden.py -> tests/golden/*.npz).
"""

from __future__ import annotations

import hashlib
import math

import numpy as np
import pytest

import oracle
from conftest import principal_angle


# ------------------------------------------------------------ known answers
def test_unfold_kat():  # reference tests/test_tensor.py:44-48
    x = np.reshape(np.arange(1.0, 9.0), (2, 2, 2), order="F")
    assert np.array_equal(oracle.unfold(x, 0), [[1, 3, 5, 7], [2, 4, 6, 8]])


def test_linearisation_kat():  # tests/test_tensor.py:23-28
    x = np.reshape(np.arange(1.0, 9.0), (2, 2, 2), order="F")
    assert x[1, 0, 0] == 2 and x[0, 1, 0] == 3 and x[0, 0, 1] == 5


def test_fold_roundtrip():
    rng = np.random.default_rng(0)
    x = rng.standard_normal((3, 4, 2, 5))
    for n in range(4):
        assert np.array_equal(oracle.fold(oracle.unfold(x, n), n, x.shape), x)


def test_skip_mode_ttmc_kat():  # tests/test_tensor.py:149-156
    x = np.reshape(np.arange(1.0, 9.0), (2, 2, 2), order="F")
    u = np.array([[1.0], [1.0]])
    y = oracle.ttmc(x, [None, u, u], skip=0)
    assert y.shape == (2, 1, 1)
    assert np.allclose(y[:, 0, 0], [16.0, 20.0])


def test_eig_diag_kat():  # tests/test_tensor.py:196-200
    v, w = oracle.leading_eigvecs(np.diag([3.0, 2.0, 1.0]), 2)
    assert np.allclose(w, [3, 2])
    assert np.allclose(v, [[1, 0], [0, 1], [0, 0]])


def test_sign_rule_kat():  # tests/test_tensor.py:202-207
    assert np.allclose(oracle.sign_fix(np.array([[0.6], [-0.8]])), [[-0.6], [0.8]])


def test_hosvd_single_nonzero_kat():  # tests/test_tucker.py:37-48
    x = np.zeros((3, 3, 3))
    x[1, 2, 0] = 5.0
    core, factors = oracle.hosvd(x)
    mags = np.sort(np.abs(core).ravel())
    assert mags[-1] == pytest.approx(5.0) and mags[-2] < 1e-12
    for f in factors:
        assert np.allclose(np.abs(f).sum(axis=0), 1.0)


def test_pp_contraction_count_kat():  # tests/test_pp.py:74-83
    rng = np.random.default_rng(3)
    x = rng.standard_normal((4, 5, 3, 2))
    anchors = [np.linalg.qr(rng.standard_normal((s, 2)))[0] for s in x.shape]
    assert oracle.pp_operators(x, anchors).count == 13


@pytest.mark.parametrize("rgb,expect", [((1, 1, 1), (1, .5, .5)), ((0, 0, 0), (0, .5, .5)),
                                        ((1, 0, 0), (0.299, 0.5 - 0.299 / 1.772, 1.0))])
def test_ycbcr_kat(rgb, expect):  # tests/test_color.py:27-39
    assert np.allclose(oracle.rgb_to_ycbcr(np.array(rgb, float)), expect, atol=1e-12)


def test_ipt_kat():  # tests/test_color.py:93-107
    assert np.allclose(oracle.rgb_to_ipt(np.ones(3)), (1, .5, .5), atol=1e-9)
    assert np.allclose(oracle.rgb_to_ipt(np.zeros(3)), (0, .5, .5), atol=1e-12)
    for g in np.linspace(0, 1, 11):
        o = oracle.rgb_to_ipt(np.full(3, g))
        assert abs(o[1] - .5) < 1e-6 and abs(o[2] - .5) < 1e-6


def test_quantiser_kat():  # tests/test_codec.py:57-85
    rng = np.random.default_rng(4)
    core = rng.standard_normal((4, 5, 3, 2))
    lv, step = oracle.quantize_core(core, 51)
    assert step == pytest.approx(np.abs(core).max() * 2.0 ** -8, rel=1e-15)
    _, step45 = oracle.quantize_core(core, 45)
    assert step45 == pytest.approx(step / 2, rel=1e-15)
    assert np.abs(core - lv * step).max() <= step / 2 + 1e-15
    assert oracle.quantize_core(np.zeros((2, 2)), 30)[1] == 1.0


def test_preset_ranks_kat():  # codec.py:86-95 on the SPEC example shape
    assert oracle.preset_ranks(1, (36, 64, 5, 2)) == (2, 4, 1, 1)
    assert oracle.preset_ranks(5, (36, 64, 5, 2)) == (9, 16, 5, 2)


# ------------------------------------------------------------ reference goldens
def test_colour_matches_reference(golden):
    z = golden("colour")
    px = (z["u8"].astype(np.float64) / 255.0)
    assert np.array_equal(oracle.rgb_to_ycbcr(px), z["ycbcr_u8"])
    assert np.abs(oracle.rgb_to_ipt(px) - z["ipt_u8"]).max() < 1e-14
    assert np.array_equal(oracle.rgb_to_ycbcr(z["fpx"][0]), z["ycbcr_f"])
    assert np.abs(oracle.rgb_to_ipt(z["fpx"][0]) - z["ipt_f"]).max() < 1e-14


@pytest.mark.parametrize("name", ["c1", "c2q", "c3q"])
def test_coding_tensor_matches_reference(golden, name):
    z = golden(name)
    t = oracle.coding_tensor(z["images"], str(z["space"]))
    flat = t.ravel(order="F")
    assert np.abs(flat[z["tensor_sample_idx"]] - z["tensor_sample_f64"]).max() < 1e-14
    t32 = np.asfortranarray(t.astype(np.float32))
    assert hashlib.sha256(t32.tobytes(order="F")).hexdigest() == str(z["tensor_f32_sha"])


@pytest.mark.parametrize("name", ["c1", "c2q", "c3q"])
def test_tucker_als_matches_reference(golden, name):
    """Oracle restatement vs the reference run on the same fp32-rounded tensor."""
    z = golden(name)
    x = oracle.coding_tensor(z["images"], str(z["space"])).astype(np.float32).astype(np.float64)
    x = np.asfortranarray(x)
    core, factors, trace = oracle.tucker_als(x, tuple(z["ranks"]), max_sweeps=int(z["sweeps"]), fit_tol=1e-300,
                                             pp_enter_tol=0.0)
    for n in range(4):
        assert principal_angle(factors[n], z[f"factor{n}"]) < 1e-6
    fits = np.array([r[2] for r in trace.rows])
    m = min(len(fits), len(z["trace_fit"]))
    assert np.abs(fits[:m] - z["trace_fit"][:m]).max() < 1e-9
    lv, step = oracle.quantize_core(core, int(z["qp"]))
    assert step == pytest.approx(float(z["step"]), rel=1e-9)
    assert int((lv != z["levels"]).sum()) == 0


def test_api_cases_match_reference(golden):
    z = golden("api")
    k = 0
    while f"x{k}" in z:
        x = z[f"x{k}"]
        core, factors, trace = oracle.tucker_als(x, tuple(z[f"ranks{k}"]), max_sweeps=int(z[f"sweeps{k}"]),
                                                 fit_tol=1e-300, pp_enter_tol=0.0)
        assert np.abs(np.array([r[2] for r in trace.rows]) - z[f"fit{k}"]).max() < 1e-12
        for n, f in enumerate(factors):
            assert np.abs(f - z[f"f{k}_{n}"]).max() < 1e-8
        k += 1
    assert k == 3


def test_oracle_pp_tree_matches_naive():  # tests/test_pp.py:40-62 (dimension tree == sequential ttmc)
    rng = np.random.default_rng(5)
    x = rng.standard_normal((5, 4, 3, 3))
    anchors = [np.linalg.qr(rng.standard_normal((s, 2)))[0] for s in x.shape]
    ops = oracle.pp_operators(x, anchors)
    for n in range(4):
        assert np.abs(ops.single[n] - oracle.ttmc(x, anchors, skip=n)).max() < 1e-12
    for (i, n), y in ops.pair.items():
        naive = x
        for m in range(4):
            if m not in (i, n):
                naive = oracle.ttm(naive, anchors[m].T, m)
        assert np.abs(y - naive).max() < 1e-12


def test_oracle_fit_dual_formula():  # tests/test_tucker.py:193
    rng = np.random.default_rng(6)
    x = rng.standard_normal((6, 5, 4))
    core, factors = oracle.t_hosvd(x, (3, 3, 2))
    assert abs(oracle.fit(x, core) - oracle.fit(x, core, factors, method="residual")) < 1e-10
    assert math.isfinite(oracle.fit(x, core))


@pytest.mark.parametrize("name", ["c1", "c2q"])
def test_decode_matches_reference(name):
    """Decode side (dequantize -> reconstruct -> to_rgb -> scene_psnr) vs the
    reference run in this container (scripts/make_golden.py decode)."""
    from conftest import GOLDEN

    z = np.load(GOLDEN / f"{name}.npz")
    d = np.load(GOLDEN / f"decode_{name}.npz")
    images = z["images"]
    v_, e_ = images.shape[:2]
    levels, step = oracle.quantize_core(z["core"], int(z["qp"]))
    core, facs = oracle.dequantize_model(levels, step, [z[f"factor{n}"] for n in range(4)])
    rgb = oracle.decode_stack(core, facs, str(z["space"]), v_, e_)
    assert np.abs(rgb[0, 0].ravel()[d["rgb00_sample_idx"]] - d["rgb00_sample"]).max() < 1e-12
    mse = oracle.scene_mse(images, rgb)
    assert np.abs(mse - d["mse"]).max() / d["mse"].max() < 1e-12
    left = 10 * math.log10(255.0 ** 2 / float(np.mean(mse[0])))
    assert abs(left - float(d["psnr_left"])) < 1e-9


def test_latent_block_bytes_match_reference():
    """Latent block serialisation (codec.py:285-291, entropy.py:55-111) vs the
    reference's own bytes (scripts/make_golden.py latent)."""
    from conftest import GOLDEN

    z = np.load(GOLDEN / "latent.npz")
    block = oracle.serialize_latent_channel(z["levels"], float(z["step"]), [z[f"qfactor{n}"] for n in range(4)])
    assert block == z["block"].tobytes()
    assert oracle.varint_encode_ints(z["edge"]) == z["edge_bytes"].tobytes()
    vals, used = oracle.varint_decode_ints(z["edge_bytes"].tobytes(), z["edge"].size)
    assert np.array_equal(vals, z["edge"]) and used == z["edge_bytes"].size
