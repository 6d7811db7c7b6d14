"""Generate tests/golden/*.npz by running the REFERENCE implementation itself.

Run in the build container only (it imports /root/reference/pkg/src):

    PYTHONDONTWRITEBYTECODE=1 OPENBLAS_NUM_THREADS=8 python scripts/make_golden.py

The fixtures pin both the CPU oracle (oracle/) and the CUDA path. Each case
stores the synthetic uint8 input stack, the solve configuration, and the
reference's factors, core, trace, quantised levels/step and relative error.
Inputs follow SURVEY.md Appendix B 1(i): the reference colour transform in
float64, rounded to float32 (the device tensor format), upcast to float64 and
handed to ``tucker_als`` with ``SolveConfig(max_sweeps=K, fit_tol=1e-300,
pp_enter_tol=0.0)`` for exactly K sweeps.
"""

from __future__ import annotations

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

from tmcodec.codec import _serialize_latent_channel, dequantize, quantize_core  # noqa: E402
from tmcodec.entropy import encode_ints  # noqa: E402
from tmcodec.metrics import mse as ref_mse, scene_psnr  # noqa: E402
from tmcodec.sceneio import SceneStack  # noqa: E402
from tmcodec.color import ColorImage, to_coding_space, to_rgb  # noqa: E402
from tmcodec.tensor import DenseTensor  # noqa: E402
from tmcodec.tucker import SolveConfig, TuckerModel, reconstruct, tucker_als  # noqa: E402

from paper_2104_04726_b200.synth import CONFIGS, make_stack, qp_for_bits  # noqa: E402

OUT = ROOT / "tests" / "golden"

# name -> (base config, seed, height, width, ranks, sweeps, bits)
CASES = {
    "c1": ("c1", 0, 384, 512, (48, 64, 3, 3), 10, 8),
    "c2q": ("c2", 1, 270, 480, (68, 120, 3, 5), 20, 10),
    "c3q": ("c3", 2, 270, 480, (34, 60, 3, 5), 10, 8),
}


def ref_tensor(images: np.ndarray, space: str) -> np.ndarray:
    v_, e_, h, w, _ = images.shape
    t = np.empty((h, w, 3, v_ * e_), order="F")
    for v in range(v_):
        for e in range(e_):
            img = ColorImage(images[v, e].astype(np.float64) / 255.0)
            t[:, :, :, v * e_ + e] = to_coding_space(img, space).pixels
    return t


def run_case(name: str) -> None:
    base, seed, h, w, ranks, sweeps, bits = CASES[name]
    cfg = CONFIGS[base]
    images = make_stack(cfg, seed=seed, height=h, width=w)
    t64 = ref_tensor(images, cfg.space)
    t32 = t64.astype(np.float32)
    x = np.asfortranarray(t32.astype(np.float64))
    t0 = time.time()
    model, trace = tucker_als(
        DenseTensor(x), SolveConfig(ranks=ranks, max_sweeps=sweeps, fit_tol=1e-300, pp_enter_tol=0.0)
    )
    dt = time.time() - t0
    q = quantize_core(model, qp_for_bits(bits))
    rec = reconstruct(model).array
    rel = float(np.linalg.norm((x - rec).ravel()) / np.linalg.norm(x.ravel()))
    rows = trace.rows()
    sample = np.random.default_rng(123).integers(0, x.size, 4096)
    np.savez_compressed(
        OUT / f"{name}.npz",
        images=images,
        space=np.array(cfg.space),
        ranks=np.array(ranks),
        sweeps=np.array(sweeps),
        qp=np.array(qp_for_bits(bits)),
        tensor_sample_idx=sample,
        tensor_sample_f64=t64.ravel(order="F")[sample],
        tensor_f32_sha=np.array(__import__("hashlib").sha256(np.asfortranarray(t32).tobytes(order="F")).hexdigest()),
        core=model.core.array,
        **{f"factor{n}": f for n, f in enumerate(model.factors)},
        levels=q.levels,
        step=np.array(q.step),
        trace_fit=np.array([r[2] for r in rows]),
        trace_change=np.array([r[3] for r in rows]),
        trace_kind=np.array([r[1] for r in rows]),
        converged=np.array(trace.converged),
        rel_err=np.array(rel),
        env=np.array(f"numpy {np.__version__}; OPENBLAS_NUM_THREADS={os.environ.get('OPENBLAS_NUM_THREADS')}; "
                     f"{platform.processor() or platform.machine()}; solve {dt:.2f}s"),
    )
    print(name, "fit", rows[-1][2], "rel", rel, f"{dt:.1f}s")


def decode_case(name: str) -> None:
    """Decode side through the reference: dequantize(quantize_core(model)) ->
    reconstruct -> to_rgb per image -> scene_psnr / mse vs the original images,
    for the model stored in tests/golden/<name>.npz."""
    z = np.load(OUT / f"{name}.npz")
    images = z["images"]
    space = str(z["space"])
    v_, e_, h, w, _ = images.shape
    factors = [z[f"factor{n}"] for n in range(4)]
    model = TuckerModel(DenseTensor(z["core"]), factors, (h, w, 3, v_ * e_))
    q = quantize_core(model, int(z["qp"]))
    t = reconstruct(dequantize(q)).array
    mses = np.zeros((v_, e_))
    ref_imgs, dec_imgs = {}, {}
    for v in range(v_):
        for e in range(e_):
            ref_imgs[(v, e)] = ColorImage(images[v, e].astype(np.float64) / 255.0)
            dec_imgs[(v, e)] = to_rgb(ColorImage(np.ascontiguousarray(t[:, :, :, v * e_ + e]), space))
            mses[v, e] = ref_mse(ref_imgs[(v, e)].pixels * 255.0, dec_imgs[(v, e)].pixels * 255.0)
    ref_scene = SceneStack(name, v_, e_, w, h, "rgb", ref_imgs)
    dec_scene = SceneStack(name, v_, e_, w, h, "rgb", dec_imgs)
    ps = scene_psnr(ref_scene, dec_scene)
    rgb0 = dec_imgs[(0, 0)].pixels
    sample = np.random.default_rng(7).integers(0, rgb0.size, 4096)
    np.savez_compressed(OUT / f"decode_{name}.npz", mse=mses, psnr_left=np.array(ps.left),
                        psnr_right=np.array(ps.right), per_exposure=np.array(ps.per_exposure),
                        rgb00_sample_idx=sample, rgb00_sample=rgb0.ravel()[sample])
    print("decode", name, ps.left, ps.right)


def latent_case() -> None:
    """Latent block bytes through the reference: quantize_core of the c1 golden
    model, _serialize_latent_channel, and encode_ints on edge-case integers."""
    z = np.load(OUT / "c1.npz")
    v_, e_, h, w, _ = z["images"].shape
    model = TuckerModel(DenseTensor(z["core"]), [z[f"factor{n}"] for n in range(4)], (h, w, 3, v_ * e_))
    q = quantize_core(model, int(z["qp"]))
    block = _serialize_latent_channel(q)
    edge = np.array([0, 1, -1, 63, -64, 64, -65, 8191, -8192, 2**31, -(2**31), 2**62, -(2**62),
                     2**63 - 1, -(2**63)], dtype=np.int64)
    np.savez_compressed(OUT / "latent.npz", block=np.frombuffer(block, dtype=np.uint8), levels=q.levels,
                        step=np.array(q.step), **{f"qfactor{n}": f for n, f in enumerate(q.factors)},
                        dims=np.array((h, w, 3, v_ * e_)), ranks=np.array(q.ranks), qp=np.array(q.qp),
                        edge=edge, edge_bytes=np.frombuffer(encode_ints(edge), dtype=np.uint8))
    print("latent block", len(block), "bytes")


def colour_kat() -> None:
    """Reference colour transforms on every gray level and 2000 random u8 triples."""
    rng = np.random.default_rng(5)
    g = np.arange(256, dtype=np.float64)[:, None].repeat(3, axis=1)
    rnd = rng.integers(0, 256, size=(2000, 3)).astype(np.float64)
    u8 = np.concatenate([g, rnd]).astype(np.uint8)
    px = (u8.astype(np.float64) / 255.0)[None]
    fpx = rng.uniform(0.0, 1.0, size=(1, 500, 3))
    out = {"u8": u8, "fpx": fpx}
    for space in ("ycbcr", "ipt"):
        out[f"{space}_u8"] = to_coding_space(ColorImage(px), space).pixels[0]
        out[f"{space}_f"] = to_coding_space(ColorImage(fpx), space).pixels[0]
    np.savez_compressed(OUT / "colour.npz", **out)
    print("colour KAT written")


def api_cases() -> None:
    """Small f64 solves with the reference defaults (PP-capable config) and
    exact-K solves, for drop-in API parity at fp64 tolerances."""
    rng = np.random.default_rng(11)
    out = {}
    specs = [((6, 7, 5), (3, 4, 2), 8), ((9, 8, 4, 3), (4, 3, 2, 2), 6), ((12, 10), (3, 3), 5)]
    for k, (dims, ranks, sweeps) in enumerate(specs):
        x = rng.standard_normal(dims)
        model, trace = tucker_als(DenseTensor(x), SolveConfig(ranks=ranks, max_sweeps=sweeps,
                                                               fit_tol=1e-300, pp_enter_tol=0.0))
        out[f"x{k}"] = x
        out[f"ranks{k}"] = np.array(ranks)
        out[f"sweeps{k}"] = np.array(sweeps)
        out[f"core{k}"] = model.core.array
        for n, f in enumerate(model.factors):
            out[f"f{k}_{n}"] = f
        out[f"fit{k}"] = np.array([r[2] for r in trace.rows()])
    np.savez_compressed(OUT / "api.npz", **out)
    print("api cases written")


def pp_cases() -> None:
    """Solves whose traces enter the pairwise-perturbation phase: the reference's
    DEFAULT SolveConfig on random tensors, and config 1 forced past convergence."""
    out = {}
    specs = [(23, (9, 7, 5, 3), (3, 3, 2, 2), {}), (1, (12, 10, 6, 4), (4, 3, 2, 2), {}),
             (2, (20, 16, 3, 6), (6, 5, 3, 3), {}), (3, (10, 9, 8), (3, 3, 3), {}),
             (1, (12, 10, 6, 4), (4, 3, 2, 2), {"fit_tol": 1e-9, "max_sweeps": 40})]
    for k, (seed, dims, ranks, kw) in enumerate(specs):
        x = np.random.default_rng(seed).standard_normal(dims)
        model, trace = tucker_als(DenseTensor(x), SolveConfig(ranks=ranks, **kw))
        out[f"x{k}"] = x
        out[f"ranks{k}"] = np.array(ranks)
        out[f"max_sweeps{k}"] = np.array(kw.get("max_sweeps", 50))
        out[f"fit_tol{k}"] = np.array(kw.get("fit_tol", 1e-5))
        out[f"kinds{k}"] = np.array("".join(r.kind[0] for r in trace.records))
        out[f"fit{k}"] = np.array([r.fit for r in trace.records])
        out[f"converged{k}"] = np.array(trace.converged)
        out[f"core{k}"] = model.core.array
        for n, f in enumerate(model.factors):
            out[f"f{k}_{n}"] = f
    # config 1, 25 sweeps, fit_tol 1e-12: PP enters around sweep 7
    z = np.load(OUT / "c1.npz")
    x = np.asfortranarray(ref_tensor(z["images"], "ycbcr").astype(np.float32).astype(np.float64))
    model, trace = tucker_als(DenseTensor(x), SolveConfig(ranks=(48, 64, 3, 3), max_sweeps=25, fit_tol=1e-12))
    out["c1_kinds"] = np.array("".join(r.kind[0] for r in trace.records))
    out["c1_fit"] = np.array([r.fit for r in trace.records])
    out["c1_core"] = model.core.array
    for n, f in enumerate(model.factors):
        out[f"c1_f{n}"] = f
    np.savez_compressed(OUT / "pp.npz", **out)
    print("pp cases written:", [str(out[f"kinds{k}"]) for k in range(len(specs))], str(out["c1_kinds"]))


if __name__ == "__main__":
    OUT.mkdir(parents=True, exist_ok=True)
    names = sys.argv[1:] or (list(CASES) + ["colour", "api", "pp", "decode", "latent"])
    for nm in names:
        if nm == "colour":
            colour_kat()
        elif nm == "latent":
            latent_case()
        elif nm == "decode":
            for name in ("c1", "c2q"):
                decode_case(name)
        elif nm == "api":
            api_cases()
        elif nm == "pp":
            pp_cases()
        else:
            run_case(nm)
