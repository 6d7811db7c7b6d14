"""Core quantiser of the latent path on the B200 (codec.py:78-148 of the reference).

``quantize_core`` / ``dequantize`` / ``QuantizedModel`` / ``preset_ranks`` /
``CodecError``. The container, entropy stage and frames codec are outside the
hot path and are not part of this package.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import _lib as L
from .tensor import DenseTensor
from .tucker import TuckerModel

__all__ = ["CodecError", "QuantizedModel", "quantize_core", "dequantize", "preset_ranks", "PRESETS", "PRESET_RHO"]

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
