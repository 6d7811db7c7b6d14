"""Seeded synthetic multi-exposure stereo stacks for the BASELINE.json configs.

The paper measured on its own ZED-camera HDR stereo captures, which are not
available here; these stacks stand in for them. The generator
mirrors the capture's value distribution -- 8-bit gamma-encoded LDR brackets of
one HDR scene, a stereo pair with horizontal disparity, sensor noise on one
view -- at the sizes BASELINE.json names.

Pinned recipe (BASELINE.json configs):

1. ``rng = np.random.default_rng(seed)`` (PCG64).
2. HDR radiance L (H x W x 3) = 8 anisotropic Gaussian blobs (random centre,
   orientation, two axis sigmas, per-channel RGB amplitude) + 4-octave value
   noise per channel (bicubic-smoothstep interpolation of a random lattice,
   amplitude halved per octave).  E = 10**(4 (L - Lmin)/(Lmax - Lmin) - 4),
   i.e. a 1e4:1 range.
3. Exposure times t = 2**k for the config's exponent list.
4. Left LDR = round-half-up(255 clip((E t)**(1/2.2), 0, 1)) -- the
   ``quantize_8bit`` rule of the reference (``sceneio.py:104-107``).
5. Right view: E resampled at w + d(h, w) (linear interpolation along the row)
   for a smooth disparity field d in [0, D] px, rendered the same way, then
   N(0, 1 LSB) added to the u8 codes, re-rounded (half up) and clipped.
6. Images are returned as uint8 (V, E, H, W, 3); the coding-space tensor
   (H, W, 3, V*E) with index v*E + e is produced by the colour kernel.
7. Batch config: stack i uses seed ``seed0 + i`` and a disparity field whose
   phase drifts with i (``frame`` argument).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

__all__ = ["StackConfig", "CONFIGS", "make_stack", "qp_for_bits"]


@dataclass(frozen=True)
class StackConfig:
    name: str
    height: int
    width: int
    exposure_exps: tuple[int, ...]
    disparity: float
    space: str
    ranks: tuple[int, int, int, int]
    sweeps: int
    bits: int | None  # core quantisation bits (None = unquantised curve)
    views: int = 2

    @property
    def exposures(self) -> int:
        return len(self.exposure_exps)

    @property
    def dims(self) -> tuple[int, int, int, int]:
        return (self.height, self.width, 3, self.views * self.exposures)

    @property
    def qp(self) -> int | None:
        return None if self.bits is None else qp_for_bits(self.bits)


def qp_for_bits(bits: int) -> int:
    """b-bit core quantisation <-> qp (codec.py:117-125: step doubles every 6 QP,
    qp 51 puts max|level| at 2**8)."""
    return 51 - 6 * (bits - 8)


CONFIGS: dict[str, StackConfig] = {
    "c1": StackConfig("c1", 384, 512, (-2, 0, 2), 32.0, "ycbcr", (48, 64, 3, 3), 10, 8),
    "c2": StackConfig("c2", 1080, 1920, (-4, -2, 0, 2, 4), 64.0, "ipt", (270, 480, 3, 5), 20, 10),
    "c3": StackConfig("c3", 1080, 1920, (-4, -2, 0, 2, 4), 64.0, "ycbcr", (135, 240, 3, 5), 10, 8),
    "c4_8": StackConfig("c4_8", 2160, 3840, tuple(range(-3, 4)), 128.0, "ipt", (270, 480, 3, 7), 15, None),
    "c4_4": StackConfig("c4_4", 2160, 3840, tuple(range(-3, 4)), 128.0, "ipt", (540, 960, 3, 7), 15, None),
    "c4_2": StackConfig("c4_2", 2160, 3840, tuple(range(-3, 4)), 128.0, "ipt", (1080, 1920, 3, 7), 15, None),
    "c5": StackConfig("c5", 4320, 7680, tuple(range(-4, 5)), 256.0, "ycbcr", (540, 960, 3, 9), 10, 8),
}


def _smoothstep(x: np.ndarray) -> np.ndarray:
    return x * x * (3.0 - 2.0 * x)


def _value_noise(rng, height: int, width: int, cells: int) -> np.ndarray:
    """One octave: random lattice of (cells+1)^2 values, smoothstep-bilinear."""
    lat = rng.uniform(-1.0, 1.0, size=(cells + 1, cells + 1))
    y = np.linspace(0.0, cells, height, endpoint=False)
    x = np.linspace(0.0, cells, width, endpoint=False)
    iy = np.minimum(y.astype(np.int64), cells - 1)
    ix = np.minimum(x.astype(np.int64), cells - 1)
    fy = _smoothstep(y - iy)[:, None]
    fx = _smoothstep(x - ix)[None, :]
    a = lat[iy][:, ix]
    b = lat[iy][:, ix + 1]
    c = lat[iy + 1][:, ix]
    d = lat[iy + 1][:, ix + 1]
    top = a + (b - a) * fx
    bot = c + (d - c) * fx
    return top + (bot - top) * fy


def _radiance(rng, height: int, width: int) -> np.ndarray:
    yy = np.arange(height, dtype=np.float64)[:, None]
    xx = np.arange(width, dtype=np.float64)[None, :]
    scale = float(min(height, width))
    lum = np.zeros((height, width, 3))
    for _ in range(8):
        cy = rng.uniform(0.0, height)
        cx = rng.uniform(0.0, width)
        theta = rng.uniform(0.0, np.pi)
        s1, s2 = rng.uniform(0.04, 0.35, size=2) * scale
        amp = rng.uniform(0.1, 1.0, size=3)
        dy, dx = yy - cy, xx - cx
        u = dx * np.cos(theta) + dy * np.sin(theta)
        v = -dx * np.sin(theta) + dy * np.cos(theta)
        g = np.exp(-0.5 * ((u / s1) ** 2 + (v / s2) ** 2))
        lum += g[:, :, None] * amp[None, None, :]
    for c in range(3):
        amp = 0.5
        cells = 4
        for _ in range(4):
            lum[:, :, c] += amp * _value_noise(rng, height, width, cells)
            amp *= 0.5
            cells *= 2
    lo, hi = lum.min(), lum.max()
    return 10.0 ** (4.0 * (lum - lo) / (hi - lo) - 4.0)


def _disparity(rng, height: int, width: int, dmax: float, frame: int) -> np.ndarray:
    base = _value_noise(rng, height, width, 3) + 0.5 * _value_noise(rng, height, width, 6)
    phase = rng.uniform(0.0, 2.0 * np.pi)
    xx = np.arange(width, dtype=np.float64)[None, :] / width
    yy = np.arange(height, dtype=np.float64)[:, None] / height
    wave = np.sin(2.0 * np.pi * (0.7 * xx + 0.4 * yy) + phase + 0.05 * frame)
    f = base + 0.5 * wave
    lo, hi = f.min(), f.max()
    return dmax * (f - lo) / (hi - lo)


def _warp_rows(e: np.ndarray, d: np.ndarray) -> np.ndarray:
    """Sample every row of e (H x W x 3) at w + d(h, w), linear interpolation."""
    height, width = d.shape
    x = np.clip(np.arange(width, dtype=np.float64)[None, :] + d, 0.0, width - 1.0)
    x0 = np.minimum(np.floor(x).astype(np.int64), width - 2) if width > 1 else np.zeros_like(x, np.int64)
    f = (x - x0)[:, :, None]
    rows = np.arange(height)[:, None]
    x1 = np.minimum(x0 + 1, width - 1)
    return e[rows, x0] * (1.0 - f) + e[rows, x1] * f


def _render(e: np.ndarray, t: float) -> np.ndarray:
    v = np.clip((e * t) ** (1.0 / 2.2), 0.0, 1.0) * 255.0
    return np.floor(v + 0.5).astype(np.uint8)


def make_stack(cfg: StackConfig | str, seed: int = 0, frame: int = 0,
               height: int | None = None, width: int | None = None) -> np.ndarray:
    """uint8 array (V, E, H, W, 3) of sRGB codes for one synthetic stack."""
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    h = cfg.height if height is None else height
    w = cfg.width if width is None else width
    rng = np.random.default_rng(seed)
    e_left = _radiance(rng, h, w)
    d = _disparity(rng, h, w, cfg.disparity * w / cfg.width, frame)
    e_right = _warp_rows(e_left, d)
    out = np.empty((cfg.views, cfg.exposures, h, w, 3), dtype=np.uint8)
    for k, ex in enumerate(cfg.exposure_exps):
        t = 2.0 ** ex
        out[0, k] = _render(e_left, t)
        right = _render(e_right, t).astype(np.float64) + rng.standard_normal((h, w, 3))
        out[1, k] = np.clip(np.floor(right + 0.5), 0, 255).astype(np.uint8)
    return out
