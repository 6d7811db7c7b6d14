"""Goldens for the drop-in stream API, produced by running the REFERENCE
(build container only; imports /root/reference/pkg/src):

    PYTHONDONTWRITEBYTECODE=1 OPENBLAS_NUM_THREADS=8 python scripts/make_golden_stream.py

* ``stream.npz``: small synthetic scenes encoded by the reference's
  ``encode_stream`` (codec.py:377-430) under a default-knob config (PP on,
  fit_tol 1e-5, rank preset, range coder) and an exact-K config (explicit
  ranks, stored entropy stage, IPT): the u8 images, the serialized stream, the
  per-channel quantised levels and steps it carries, and the reference's own
  decode (``decode_stream``) PSNR against the source scene.
* ``rc.npz``: range-coder known-answer vectors (``kernels.rc_encode``,
  _kernels_py.py:24-58) on uniform and skewed byte strings, incl. lengths that
  cross the 2^16 count-halving point.
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

REF = "/root/reference/pkg/src"
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, REF)
sys.path.insert(0, str(ROOT))

from tmcodec import _kernels_py as kp  # noqa: E402
from tmcodec.codec import (EncodeConfig, _deserialize_latent_channel, decode_stream, encode_stream,  # noqa: E402
                           parse_stream, serialize_stream)
from tmcodec.color import ColorImage  # noqa: E402
from tmcodec.entropy import entropy_stage  # noqa: E402
from tmcodec.metrics import scene_psnr  # noqa: E402
from tmcodec.sceneio import SceneStack  # noqa: E402

from paper_2104_04726_b200.synth import CONFIGS, make_stack  # noqa: E402

OUT = ROOT / "tests" / "golden"

CASES = [
    # (name, base cfg, seed, h, w, EncodeConfig kwargs)
    ("default_ycbcr", "c1", 3, 48, 64, dict(space="ycbcr", preset=2, qp=30)),
    ("exact_ipt", "c2", 4, 40, 56, dict(space="ipt", ranks=(12, 16, 3, 2), qp=20, entropy_tag=0, max_sweeps=6,
                                        fit_tol=1e-300, pp_enter_tol=0.0)),
    ("pp_ycbcr", "c1", 5, 32, 48, dict(space="ycbcr", ranks=(10, 12, 2, 2), qp=36, fit_tol=1e-9, max_sweeps=30)),
]


def scene_from(images: np.ndarray) -> SceneStack:
    v_, e_, h, w, _ = images.shape
    imgs = {(v, e): ColorImage(images[v, e].astype(np.float64) / 255.0) for v in range(v_) for e in range(e_)}
    return SceneStack("golden", v_, e_, w, h, "rgb", imgs)


def main() -> None:
    out = {}
    for name, base, seed, h, w, kw in CASES:
        images = make_stack(CONFIGS[base], seed=seed, height=h, width=w)
        scene = scene_from(images)
        cfg = EncodeConfig(**kw)
        stream = encode_stream(scene, cfg)
        data = serialize_stream(stream)
        back = parse_stream(data)
        hd = back.header
        dec = decode_stream(back)
        ps = scene_psnr(scene, dec)
        out[f"{name}_images"] = images
        out[f"{name}_stream"] = np.frombuffer(data, dtype=np.uint8)
        out[f"{name}_ranks"] = np.array(hd.ranks)
        out[f"{name}_psnr"] = np.array([ps.left, ps.right])
        for c, block in enumerate(back.blocks):
            q = _deserialize_latent_channel(entropy_stage(block, hd.entropy_tag, "decode"), hd.dims, hd.ranks, hd.qp)
            out[f"{name}_levels{c}"] = q.levels
            out[f"{name}_step{c}"] = np.array(q.step)
            for n, f in enumerate(q.factors):
                out[f"{name}_f{c}_{n}"] = f
        print(name, "ranks", hd.ranks, "bytes", len(data), "psnr", ps.left, ps.right)
    np.savez_compressed(OUT / "stream.npz", cases=np.array([c[0] for c in CASES]), **out)

    rng = np.random.default_rng(21)
    rc = {}
    vecs = [b"", b"\x00", bytes(range(256)), bytes(rng.integers(0, 256, 4000, dtype=np.uint8)),
            bytes(np.minimum(rng.geometric(0.08, 9000), 255).astype(np.uint8)),   # skewed, crosses 2^16 halving
            bytes(np.zeros(5000, dtype=np.uint8))]
    for i, v in enumerate(vecs):
        rc[f"in{i}"] = np.frombuffer(v, dtype=np.uint8)
        rc[f"out{i}"] = np.frombuffer(kp.rc_encode(v) if v else b"", dtype=np.uint8)
    np.savez_compressed(OUT / "rc.npz", n=np.array(len(vecs)), **rc)
    print("rc vectors", [len(v) for v in vecs])


if __name__ == "__main__":
    main()
