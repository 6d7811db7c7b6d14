"""Full-size BASELINE config-2 golden from the REFERENCE implementation itself
(build container only; imports /root/reference/pkg/src):

    PYTHONDONTWRITEBYTECODE=1 OPENBLAS_NUM_THREADS=8 python scripts/make_golden_c2_full.py

The 1080x1920x3x10 IPT stack of bench.py (synth generator, seed 0), ranks
(270,480,3,5), 20 HOOI sweeps, qp 39. The fixture stays small: no images (the
seeded generator reproduces them; the fp32 tensor's sha256 pins that), the
trace, relative error, quantiser step and levels (int16), and per mode a
rotation- and sign-invariant sketch of the factor subspace, S = W^T U U^T W for
a fixed Gaussian W (s_n x 16), plus the factors' first 8 columns (sign-fixed
eigenvectors) for per-vector comparison.
"""
from __future__ import annotations

import hashlib
import os
import platform
import sys
import time
from pathlib import Path

import numpy as np

REF = "/root/reference/pkg/src"
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, REF)
sys.path.insert(0, str(ROOT))

from tmcodec.codec import quantize_core  # noqa: E402
from tmcodec.tensor import DenseTensor  # noqa: E402
from tmcodec.tucker import SolveConfig, reconstruct, tucker_als  # noqa: E402

from paper_2104_04726_b200.synth import CONFIGS, make_stack  # noqa: E402
sys.path.insert(0, str(ROOT / "scripts"))
from make_golden import ref_tensor  # noqa: E402


def sketch_basis(s: int) -> np.ndarray:
    return np.random.default_rng(1000 + s).standard_normal((s, 16)) / np.sqrt(s)


def main() -> None:
    cfg = CONFIGS["c2"]
    images = make_stack(cfg, seed=0)
    t32 = ref_tensor(images, cfg.space).astype(np.float32)
    x = np.asfortranarray(t32.astype(np.float64))
    t0 = time.time()
    model, trace = tucker_als(DenseTensor(x), SolveConfig(ranks=cfg.ranks, max_sweeps=cfg.sweeps, fit_tol=1e-300,
                                                          pp_enter_tol=0.0))
    dt = time.time() - t0
    q = quantize_core(model, cfg.qp)
    rec = reconstruct(model).array
    rel = float(np.linalg.norm((x - rec).ravel()) / np.linalg.norm(x.ravel()))
    rows = trace.rows()
    out = {}
    for n, u in enumerate(model.factors):
        w = sketch_basis(u.shape[0])
        p = w.T @ u
        out[f"sketch{n}"] = p @ p.T
        out[f"head{n}"] = u[:, :8]
    assert np.abs(q.levels).max() < 32767
    np.savez_compressed(
        ROOT / "tests" / "golden" / "c2_full.npz",
        tensor_f32_sha=np.array(hashlib.sha256(np.asfortranarray(t32).tobytes(order="F")).hexdigest()),
        ranks=np.array(cfg.ranks), sweeps=np.array(cfg.sweeps), qp=np.array(cfg.qp),
        levels=q.levels.astype(np.int16), step=np.array(q.step),
        trace_fit=np.array([r[2] for r in rows]), trace_kind=np.array([r[1] for r in rows]),
        rel_err=np.array(rel), core_norm=np.array(np.linalg.norm(model.core.array)),
        env=np.array(f"numpy {np.__version__}; OPENBLAS_NUM_THREADS={os.environ.get('OPENBLAS_NUM_THREADS')}; "
                     f"{platform.processor() or platform.machine()}; solve {dt:.1f}s"),
        **out,
    )
    print("c2_full fit", rows[-1][2], "rel", rel, f"{dt:.1f}s")


if __name__ == "__main__":
    main()
