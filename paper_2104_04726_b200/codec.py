"""Core quantiser of the latent path on the B200 (codec.py:78-148 of the reference).

``quantize_core`` / ``dequantize`` / ``QuantizedModel`` / ``preset_ranks`` /
``CodecError``, plus the latent path's callers and data format either side of
the solve: ``solve_channels`` (the three per-channel
solves of ``_solve_channels``, codec.py:366-374, on the device) and the latent
block bytes (``_serialize_latent_channel`` / ``_deserialize_latent_channel``,
codec.py:285-318, with the level varints encoded and decoded on the device).
The container, range coder and frames codec are outside the hot path
 and are not part of this package.
"""

from __future__ import annotations

import math
import struct
from dataclasses import dataclass
from typing import Sequence

import numpy as np

from . import _lib as L
from .tensor import DenseTensor
from .tucker import TuckerModel

__all__ = ["CodecError", "QuantizedModel", "quantize_core", "dequantize", "preset_ranks", "PRESETS", "PRESET_RHO",
           "serialize_latent_channel", "deserialize_latent_channel", "solve_channels"]

PRESET_RHO = 0.25
PRESETS = (1, 2, 3, 4, 5)


class CodecError(ValueError):
    """Malformed stream or invalid codec configuration."""


def preset_ranks(preset: int, dims: tuple[int, int, int, int]) -> tuple[int, int, int, int]:
    """RANK k -> (H, W, E, V) multilinear ranks (codec.py:86-95)."""
    if preset not in PRESETS:
        raise ValueError(f"rank preset {preset} not in {PRESETS}")
    h, w, exposures, views = dims

    def spatial(s: int) -> int:
        return min(s, max(1, math.ceil(math.ceil(preset * s / 5) * PRESET_RHO)))

    return (spatial(h), spatial(w), min(preset, exposures), min(preset, views))


@dataclass
class QuantizedModel:
    """Uniformly quantised core (int64 levels) + float32 factors (codec.py:102-111)."""

    source_dims: tuple[int, ...]
    ranks: tuple[int, ...]
    step: float
    qp: int
    levels: np.ndarray
    factors: list[np.ndarray]


def quantize_levels_device(core_dev, n: int, qp: int):
    """Device core -> (device int64 levels, step): amax reduce + round-half-away."""
    torch = L._torch()
    if not 0 <= qp <= 51:
        raise ValueError(f"qp {qp} out of range [0, 51]")
    h = L.ctx()
    lv = torch.empty(max(n, 1), dtype=torch.int64, device="cuda")
    step = L.C.c_double()
    L.check(L.LIB.tmb_quantize_core(h, L.ptr(core_dev), n, int(qp), L.ptr(lv), L.C.byref(step)), h)
    return lv, float(step.value)


def quantize_core(model: TuckerModel, qp: int) -> QuantizedModel:
    """step = max|core| 2^((qp-51)/6) 2^-8 (1.0 for a zero core); levels round
    half away from zero (codec.py:114-134)."""
    if not 0 <= qp <= 51:
        raise ValueError(f"qp {qp} out of range [0, 51]")
    core = model.core
    lv, step = quantize_levels_device(L.dev_f64(core.array), core.size, qp)
    levels = np.reshape(lv[: core.size].cpu().numpy(), core.dims, order="F")
    return QuantizedModel(tuple(model.source_dims), tuple(model.ranks), step, qp, levels,
                          [np.asarray(f, dtype=np.float32) for f in model.factors])


def dequantize(q: QuantizedModel) -> TuckerModel:
    """levels * step, float32 factors upcast, orthonormality re-validated at
    1e-3 (codec.py:137-148)."""
    if q.levels.shape != tuple(q.ranks):
        raise CodecError(f"core payload shape {q.levels.shape} != ranks {q.ranks}")
    for n, f in enumerate(q.factors):
        if f.shape != (q.source_dims[n], q.ranks[n]):
            raise CodecError(f"mode {n}: factor payload shape {f.shape} is corrupt")
    torch = L._torch()
    h = L.ctx()
    flat = np.ascontiguousarray(np.asarray(q.levels, dtype=np.int64).ravel(order="F"))
    lv = torch.from_numpy(flat).to("cuda")
    out = L.empty_f64(flat.size)
    L.check(L.LIB.tmb_dequantize(h, L.ptr(lv), flat.size, float(q.step), L.ptr(out)), h)
    core = DenseTensor(L.host_f(out, tuple(q.ranks)))
    model = TuckerModel(core, [np.asarray(f, dtype=np.float64) for f in q.factors], tuple(q.source_dims))
    model.validate(ortho_tol=1e-3)
    return model


# ---------------------------------------------------------------------------
# latent path: per-channel solves and the latent block bytes
# ---------------------------------------------------------------------------


def _varint_encode_dev(levels_dev, n: int) -> bytes:
    torch = L._torch()
    cap = max(1, 10 * n)
    out = torch.empty(cap, dtype=torch.uint8, device="cuda")
    nb = L.C.c_int64()
    h = L.ctx()
    L.check(L.LIB.tmb_varint_encode(h, L.ptr(levels_dev), n, L.ptr(out), cap, L.C.byref(nb)), h)
    return bytes(out[: nb.value].cpu().numpy().tobytes())


def serialize_latent_channel(q: QuantizedModel) -> bytes:
    """One channel's latent block (codec.py:285-291): float32 little-endian
    column-major factors, the F-order levels as zigzag varints (encoded on the
    device, entropy.py:55-111), then the float64 step."""
    torch = L._torch()
    out = bytearray()
    for f in q.factors:
        out += np.asarray(f, dtype="<f4").tobytes(order="F")
    flat = np.ascontiguousarray(np.asarray(q.levels, dtype=np.int64).ravel(order="F"))
    out += _varint_encode_dev(torch.from_numpy(flat).to("cuda"), flat.size)
    out += struct.pack("<d", q.step)
    return bytes(out)


def deserialize_latent_channel(data: bytes, dims: Sequence[int], ranks: Sequence[int], qp: int) -> QuantizedModel:
    """Inverse of serialize_latent_channel (codec.py:294-318), with the
    reference's CodecError conditions; the varints are decoded on the device."""
    torch = L._torch()
    dims = tuple(int(d) for d in dims)
    ranks = tuple(int(r) for r in ranks)
    factor_bytes = sum(s * r * 4 for s, r in zip(dims, ranks))
    if len(data) < factor_bytes + 8:
        raise CodecError("latent block truncated")
    factors, pos = [], 0
    for s, r in zip(dims, ranks):
        f = np.frombuffer(data, dtype="<f4", count=s * r, offset=pos)
        factors.append(np.reshape(f, (s, r), order="F"))
        pos += s * r * 4
    (step,) = struct.unpack_from("<d", data, len(data) - 8)
    count = int(np.prod(ranks))
    body = np.frombuffer(data, dtype=np.uint8, count=len(data) - 8 - pos, offset=pos)
    levels = torch.empty(max(count, 1), dtype=torch.int64, device="cuda")
    src = torch.from_numpy(body.copy()).to("cuda") if body.size else torch.empty(1, dtype=torch.uint8, device="cuda")
    used = L.C.c_int64()
    h = L.ctx()
    rc = L.LIB.tmb_varint_decode(h, L.ptr(src), int(body.size), count, L.ptr(levels), L.C.byref(used))
    if rc != 0:
        try:
            L.check(rc, h)
        except ValueError as exc:
            raise CodecError(f"latent block corrupt: {exc}") from exc
    if used.value != body.size:
        raise CodecError(f"latent block has {body.size - used.value} trailing bytes")
    lv = np.reshape(levels[:count].cpu().numpy(), ranks, order="F")
    return QuantizedModel(dims, ranks, step, qp, lv, factors)


def solve_channels(images_u8, space: str, ranks: Sequence[int], cfg, qp: int | None = None):
    """The latent path's three per-channel solves on the device (codec.py:366-374
    after the colour conversion of codec.py:389): the (V, E, H, W, 3) uint8 stack
    is converted straight into three (H, W, E, V) float32 tensors
    (stack_to_tensor, sceneio.py:191-199) and each is solved with ``cfg``
    (a SolveConfig whose ranks are the (H, W, E, V) ranks). Returns a list of
    (TuckerModel, SolveTrace), or of QuantizedModel when ``qp`` is given."""
    from .tucker import solve_device

    torch = L._torch()
    if isinstance(images_u8, np.ndarray):
        images_u8 = torch.from_numpy(np.ascontiguousarray(images_u8))
    if images_u8.dtype != torch.uint8 or images_u8.dim() != 5 or images_u8.shape[-1] != 3:
        raise ValueError("expected a (V, E, H, W, 3) uint8 image stack")
    v, e, h, w, _ = images_u8.shape
    dims = (h, w, e, v)
    cfg.validate(dims)
    src = images_u8.to("cuda").contiguous()
    planes = torch.empty(3 * h * w * e * v, dtype=torch.float32, device="cuda")
    hc = L.ctx()
    L.check(L.LIB.tmb_color_u8_channels(hc, L.ptr(src), v * e, h, w, L.SPACES[space], L.ptr(planes)), hc)
    per = h * w * e * v
    out = []
    for c in range(3):
        model, trace = solve_device(planes[c * per:(c + 1) * per], L.F32, dims, cfg)
        out.append(quantize_core(model, qp) if qp is not None else (model, trace))
    return out
