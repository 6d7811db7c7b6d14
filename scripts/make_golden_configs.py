"""Compact goldens for BASELINE configs 3, 4 and 5 at FULL size, produced by
running the REFERENCE implementation itself (build container only; imports
/root/reference/pkg/src):

    PYTHONDONTWRITEBYTECODE=1 OPENBLAS_NUM_THREADS=8 python scripts/make_golden_configs.py [c3 c4 c5]

* c3  -- stack 0 of the 64-stack batch (seed 0, frame 0), 1080x1920x3x10 Y'CbCr,
         ranks (135,240,3,5), the full 10 sweeps, qp 51. Solved twice: on the
         fp32-rounded colour tensor (the device input format)
         and on the reference's own float64 colour tensor (App. B.1(ii): the
         product chain from u8 against the reference chain from u8).
* c4  -- the 2160x3840x3x14 IPT stack at spatial ranks 1/8, 1/4, 1/2 (+ (3,7)):
         the unquantised error-vs-rank curve. T-HOSVD + 2 HOOI sweeps per rank
         (at 4K the oracle takes minutes; the GPU runs the same
         exact-K solve and is compared sweep by sweep).
* c5  -- the 4320x7680x3x18 Y'CbCr stack, ranks (540,960,3,9): T-HOSVD + 2 HOOI
         sweeps, qp 51 (about 29 GB of RAM for the reference).

Each fixture holds no images (the seeded generator reproduces them; the fp32
tensor's sha256 pins that): the full trace (fits, kinds, changes, converged,
the index of the returned model), the relative reconstruction error, the core
norm, per mode a rotation/sign-invariant subspace sketch W^T U U^T W (fixed
Gaussian W, s_n x 16) and the first 8 factor columns, and the quantised levels
(all of them for c3; for c5 a seeded sample of 262144 positions plus the
sha256 of every level and a histogram).
"""
from __future__ import annotations

import gc
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

OUT = ROOT / "tests" / "golden"


def sketch_basis(s: int) -> np.ndarray:
    return np.random.default_rng(1000 + s).standard_normal((s, 16)) / np.sqrt(s)


def best_index(fits) -> int:
    """tucker.py:379-383: best = first strictly-greatest fit (init included)."""
    b = 0
    for i, f in enumerate(fits):
        if f > fits[b]:
            b = i
    return b


def solve(x: np.ndarray, ranks, sweeps: int, qp: int | None, tag: str) -> dict:
    t0 = time.time()
    model, trace = tucker_als(DenseTensor(x), SolveConfig(ranks=ranks, max_sweeps=sweeps, fit_tol=1e-300,
                                                          pp_enter_tol=0.0))
    dt = time.time() - t0
    rec = reconstruct(model).array
    rel = float(np.linalg.norm((x - rec).ravel()) / np.linalg.norm(x.ravel()))
    del rec
    gc.collect()
    rows = trace.rows()
    fits = [r[2] for r in rows]
    out = {
        f"{tag}trace_fit": np.array(fits), f"{tag}trace_kind": np.array([r[1] for r in rows]),
        f"{tag}trace_change": np.array([r[3] for r in rows]), f"{tag}converged": np.array(trace.converged),
        f"{tag}best_index": np.array(best_index(fits)), f"{tag}rel_err": np.array(rel),
        f"{tag}core_norm": np.array(np.linalg.norm(model.core.array)), f"{tag}solve_s": np.array(dt),
    }
    for n, u in enumerate(model.factors):
        w = sketch_basis(u.shape[0])
        p = w.T @ u
        out[f"{tag}sketch{n}"] = p @ p.T
        out[f"{tag}head{n}"] = u[:, :8]
    if qp is not None:
        q = quantize_core(model, qp)
        lv = q.levels.ravel(order="F")
        out[f"{tag}step"] = np.array(q.step)
        out[f"{tag}levels_sha"] = np.array(hashlib.sha256(np.ascontiguousarray(lv.astype(np.int64)).tobytes()).hexdigest())
        out[f"{tag}levels_hist"] = np.bincount(np.abs(lv).astype(np.int64))
        if lv.size <= 2_000_000:
            out[f"{tag}levels"] = lv.astype(np.int16)
        else:
            idx = np.sort(np.random.default_rng(77).choice(lv.size, 262144, replace=False))
            out[f"{tag}levels_idx"] = idx.astype(np.int64)
            out[f"{tag}levels_sample"] = lv[idx].astype(np.int16)
    print(tag or "main", "fit", fits[-1], "rel", rel, f"{dt:.1f}s", flush=True)
    return out


def env(dt: float) -> np.ndarray:
    return np.array(f"numpy {np.__version__}; OPENBLAS_NUM_THREADS={os.environ.get('OPENBLAS_NUM_THREADS')}; "
                    f"{platform.processor() or platform.machine()}; {dt:.1f}s")


def tensor_pair(cfg, seed: int, frame: int = 0):
    images = make_stack(cfg, seed=seed, frame=frame)
    t64 = ref_tensor(images, cfg.space)
    t32 = t64.astype(np.float32)
    sha = hashlib.sha256(np.asfortranarray(t32).tobytes(order="F")).hexdigest()
    return t64, t32, sha


def case_c3() -> None:
    cfg = CONFIGS["c3"]
    t0 = time.time()
    t64, t32, sha = tensor_pair(cfg, 0, 0)
    x = np.asfortranarray(t32.astype(np.float64))
    out = solve(x, cfg.ranks, cfg.sweeps, cfg.qp, "")
    del x
    out.update(solve(np.asfortranarray(t64), cfg.ranks, cfg.sweeps, cfg.qp, "f64in_"))
    np.savez_compressed(OUT / "c3_full.npz", tensor_f32_sha=np.array(sha), ranks=np.array(cfg.ranks),
                        sweeps=np.array(cfg.sweeps), qp=np.array(cfg.qp), seed=np.array(0), frame=np.array(0),
                        env=env(time.time() - t0), **out)


def case_c4() -> None:
    cfg = CONFIGS["c4_8"]
    t0 = time.time()
    t64, t32, sha = tensor_pair(cfg, 0, 0)
    del t64
    x = np.asfortranarray(t32.astype(np.float64))
    del t32
    out = {}
    for name in ("c4_8", "c4_4", "c4_2"):
        c = CONFIGS[name]
        out.update(solve(x, c.ranks, 2, None, f"{name}_"))
        out[f"{name}_ranks"] = np.array(c.ranks)
    np.savez_compressed(OUT / "c4_curve.npz", tensor_f32_sha=np.array(sha), sweeps=np.array(2), seed=np.array(0),
                        env=env(time.time() - t0), **out)


def case_c5() -> None:
    cfg = CONFIGS["c5"]
    t0 = time.time()
    t64, t32, sha = tensor_pair(cfg, 0, 0)
    del t64
    x = np.asfortranarray(t32.astype(np.float64))
    del t32
    gc.collect()
    out = solve(x, cfg.ranks, 2, cfg.qp, "")
    np.savez_compressed(OUT / "c5_2sweeps.npz", tensor_f32_sha=np.array(sha), ranks=np.array(cfg.ranks),
                        sweeps=np.array(2), qp=np.array(cfg.qp), seed=np.array(0), env=env(time.time() - t0), **out)


if __name__ == "__main__":
    OUT.mkdir(parents=True, exist_ok=True)
    for nm in sys.argv[1:] or ["c3", "c4", "c5"]:
        {"c3": case_c3, "c4": case_c4, "c5": case_c5}[nm]()
