"""Colour transforms on the B200 (drop-in for the reference's ``color.py``).

Y'CbCr (full-range BT.601) and IPT (Ebner & Fairchild) with the reference's
constants and operation order (color.py:40-205). Pixelwise fp64 kernels in
libtmb; the hot path converts u8 stacks straight into the solver tensor
(``pipeline.coding_tensor``).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib as L

__all__ = ["ColorImage", "SPACE_RGB", "SPACE_YCBCR", "SPACE_IPT", "rgb_to_ycbcr", "ycbcr_to_rgb", "rgb_to_ipt",
           "ipt_to_rgb", "to_coding_space", "to_rgb"]

SPACE_RGB = "rgb"
SPACE_YCBCR = "ycbcr"
SPACE_IPT = "ipt"
RGB_ENCODINGS = ("srgb",)


def _check_encoding(encoding: str) -> None:
    if encoding not in RGB_ENCODINGS:
        raise ValueError(f"unsupported RGB encoding {encoding!r}; supported: {RGB_ENCODINGS}")


@dataclass
class ColorImage:
    """H x W x 3 float64 pixels with a space tag (color.py:82-103)."""

    pixels: np.ndarray
    space: str = SPACE_RGB

    def __post_init__(self):
        self.pixels = np.asarray(self.pixels, dtype=np.float64)
        if self.pixels.ndim != 3 or self.pixels.shape[2] != 3:
            raise ValueError(f"expected HxWx3 pixels, got shape {self.pixels.shape}")

    @property
    def height(self) -> int:
        return self.pixels.shape[0]

    @property
    def width(self) -> int:
        return self.pixels.shape[1]

    def plane(self, c: int) -> np.ndarray:
        return self.pixels[:, :, c]


def _require_space(img: ColorImage, space: str, op: str) -> None:
    if img.space != space:
        raise ValueError(f"{op} expects a {space} image, got {img.space}")


def _run(px: np.ndarray, space: str, inverse: bool):
    torch = L._torch()
    flat = np.ascontiguousarray(px, dtype=np.float64).reshape(-1, 3)
    h = L.ctx()
    src = torch.from_numpy(flat).to("cuda")
    out = torch.empty_like(src)
    npx = flat.shape[0]
    if inverse:
        ncl = L.C.c_int64(0)
        L.check(L.LIB.tmb_color_inv_f64(h, L.ptr(src), npx, L.SPACES[space], L.ptr(out), L.C.byref(ncl)), h)
        return out.cpu().numpy().reshape(px.shape), int(ncl.value)
    L.check(L.LIB.tmb_color_f64(h, L.ptr(src), npx, L.SPACES[space], L.ptr(out)), h)
    return out.cpu().numpy().reshape(px.shape), 0


def rgb_to_ycbcr(img: ColorImage) -> ColorImage:
    _require_space(img, SPACE_RGB, "rgb_to_ycbcr")
    return ColorImage(_run(img.pixels, SPACE_YCBCR, False)[0], SPACE_YCBCR)


def ycbcr_to_rgb(img: ColorImage) -> ColorImage:
    _require_space(img, SPACE_YCBCR, "ycbcr_to_rgb")
    return ColorImage(_run(img.pixels, SPACE_YCBCR, True)[0], SPACE_RGB)


def rgb_to_ipt(img: ColorImage, encoding: str = "srgb") -> ColorImage:
    _require_space(img, SPACE_RGB, "rgb_to_ipt")
    _check_encoding(encoding)
    return ColorImage(_run(img.pixels, SPACE_IPT, False)[0], SPACE_IPT)


def ipt_to_rgb(img: ColorImage, count_clamped: bool = False, encoding: str = "srgb"):
    _require_space(img, SPACE_IPT, "ipt_to_rgb")
    _check_encoding(encoding)
    px, n = _run(img.pixels, SPACE_IPT, True)
    out = ColorImage(px, SPACE_RGB)
    return (out, n) if count_clamped else out


def to_coding_space(img: ColorImage, space: str) -> ColorImage:
    if space == SPACE_RGB:
        _require_space(img, SPACE_RGB, "to_coding_space")
        return img
    if space == SPACE_YCBCR:
        return rgb_to_ycbcr(img)
    if space == SPACE_IPT:
        return rgb_to_ipt(img)
    raise ValueError(f"unknown color space {space!r}")


def to_rgb(img: ColorImage) -> ColorImage:
    if img.space == SPACE_RGB:
        return img
    if img.space == SPACE_YCBCR:
        return ycbcr_to_rgb(img)
    if img.space == SPACE_IPT:
        return ipt_to_rgb(img)
    raise ValueError(f"unknown color space {img.space!r}")
