"""Host-side checks that need no GPU: the C-ABI library loads and exports every
symbol include/tmb.h declares, the Python drop-in validates arguments with the
reference's wording before any device work, and the product refuses to run
without its CUDA library (no CPU fallback)."""

from __future__ import annotations

import re
import shutil
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]

import paper_2104_04726_b200 as tb  # noqa: E402
from paper_2104_04726_b200 import _lib as L  # noqa: E402
from paper_2104_04726_b200.synth import CONFIGS, make_stack, qp_for_bits  # noqa: E402


def header_symbols() -> set[str]:
    text = (ROOT / "include" / "tmb.h").read_text()
    return set(re.findall(r"^\s*(?:int|int64_t|const char\*)\s+(tmb_\w+)\s*\(", text, flags=re.M))


def test_library_exports_every_header_symbol():
    declared = header_symbols()
    assert len(declared) >= 20
    out = subprocess.run(["nm", "-D", "--defined-only", str(L._PATH)], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (tmb_\w+)", out))
    assert declared <= exported, declared - exported
    for name in declared:  # and ctypes resolves each
        assert getattr(L.LIB, name) is not None
    assert declared == set(L.EXPORTS)


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", str(L._PATH)], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_version():
    assert L.LIB.tmb_version() == 1


def test_no_cpu_fallback_without_library(tmp_path):
    pkg = tmp_path / "paper_2104_04726_b200"
    shutil.copytree(ROOT / "paper_2104_04726_b200", pkg, ignore=shutil.ignore_patterns("*.so", "build", "csrc"))
    res = subprocess.run([sys.executable, "-c", "import paper_2104_04726_b200"], cwd=tmp_path,
                         capture_output=True, text=True)
    assert res.returncode != 0 and "no CPU fallback" in res.stderr


def test_compute_requires_cuda_device():
    import torch

    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    with pytest.raises(RuntimeError, match="CUDA device"):
        tb.fro_norm(tb.DenseTensor(np.ones(3)))


# ---------------------------------------------------------------- validation wording
def test_dense_tensor_validation():
    with pytest.raises(ValueError, match="dimensions must be >= 1"):
        tb.DenseTensor(np.zeros((2, 0)))
    with pytest.raises(ValueError, match="finite"):
        tb.DenseTensor(np.array([1.0, np.nan]), check_finite=True)
    with pytest.raises(ValueError, match="need"):
        tb.DenseTensor.from_flat(np.arange(5.0), (2, 2))


def test_unfold_fold_kat():
    t = tb.DenseTensor.from_flat(np.arange(1.0, 9.0), (2, 2, 2))
    assert np.array_equal(tb.unfold(t, 0), [[1, 3, 5, 7], [2, 4, 6, 8]])
    rng = np.random.default_rng(0)
    x = tb.DenseTensor(rng.standard_normal((3, 4, 2)))
    for n in range(3):
        assert np.array_equal(tb.fold(tb.unfold(x, n), n, x.dims).array, x.array)
    with pytest.raises(ValueError, match="mode 3"):
        tb.unfold(x, 3)


def test_mode_errors_before_device():
    t = tb.DenseTensor(np.ones((2, 3, 4)))
    with pytest.raises(ValueError, match="mode 1"):  # reference tests/test_tensor.py:171
        tb.ttm(t, np.ones((2, 2)), 1)
    with pytest.raises(ValueError, match="expected 3 factors"):
        tb.ttmc(t, [np.eye(2)])
    with pytest.raises(ValueError, match="out of range"):
        tb.leading_eigvecs(np.eye(3), 4)
    with pytest.raises(ValueError, match="square"):
        tb.leading_eigvecs(np.ones((2, 3)), 1)


def test_solve_config_validation():
    cfg = tb.SolveConfig(ranks=(2, 5))
    with pytest.raises(ValueError, match="mode 1: rank 5 not in"):
        cfg.validate((3, 4))
    with pytest.raises(ValueError, match="ranks for an order-3"):
        cfg.validate((3, 4, 5))
    with pytest.raises(ValueError, match="positive"):
        tb.SolveConfig(ranks=(1,), fit_tol=0.0).validate((2,))
    with pytest.raises(ValueError, match="max_sweeps"):
        tb.SolveConfig(ranks=(1,), max_sweeps=-1).validate((2,))


def test_quantiser_qp_range():
    m = tb.TuckerModel(tb.DenseTensor(np.ones((1, 1))), [np.ones((1, 1)), np.ones((1, 1))], (1, 1))
    with pytest.raises(ValueError, match="qp 52 out of range"):
        tb.quantize_core(m, 52)


def test_preset_ranks_matches_oracle():
    import oracle

    for dims in [(36, 64, 5, 2), (1080, 1920, 5, 2), (3, 3, 2, 1)]:
        for k in (1, 2, 3, 4, 5):
            assert tb.preset_ranks(k, dims) == oracle.preset_ranks(k, dims)
    with pytest.raises(ValueError, match="preset"):
        tb.preset_ranks(0, (4, 4, 2, 2))


def test_color_space_validation():
    img = tb.ColorImage(np.zeros((2, 2, 3)), "ycbcr")
    with pytest.raises(ValueError, match="expects a rgb image"):
        tb.rgb_to_ipt(img)
    with pytest.raises(ValueError, match="HxWx3"):
        tb.ColorImage(np.zeros((2, 2)))


# ---------------------------------------------------------------- synthetic inputs
def test_synth_deterministic_and_shaped():
    cfg = CONFIGS["c1"]
    a = make_stack(cfg, seed=3, height=48, width=64)
    b = make_stack(cfg, seed=3, height=48, width=64)
    c = make_stack(cfg, seed=4, height=48, width=64)
    assert a.shape == (2, 3, 48, 64, 3) and a.dtype == np.uint8
    assert np.array_equal(a, b) and not np.array_equal(a, c)
    # brackets ordered by exposure (brighter with longer t)
    assert a[0, 0].mean() < a[0, 1].mean() < a[0, 2].mean()


def test_config_table_matches_baseline():
    import json

    base = json.loads((ROOT / "BASELINE.json").read_text())
    assert len(base["configs"]) == 5
    assert CONFIGS["c1"].dims == (384, 512, 3, 6) and CONFIGS["c1"].ranks == (48, 64, 3, 3)
    assert CONFIGS["c2"].dims == (1080, 1920, 3, 10) and CONFIGS["c2"].ranks == (270, 480, 3, 5)
    assert CONFIGS["c5"].dims == (4320, 7680, 3, 18)
    assert qp_for_bits(8) == 51 and qp_for_bits(10) == 39
