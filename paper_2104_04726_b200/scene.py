"""Scene stacks (drop-in for the reference's ``sceneio.py`` surface).

``SceneStack`` is the input of ``encode_stream`` and the output of
``decode_stream`` (codec.py:377-468), so a drop-in must accept and return the
same type: views x exposures ``ColorImage``s keyed (view, exposure)
(sceneio.py:41-76). Scene files are decoded by ``ingest`` (the reference's
directory conventions, sceneio.py:79-188). ``stack_to_tensor`` /
``tensor_to_stack`` are the per-channel (H, W, E, V) layout maps
(sceneio.py:38, 191-226) -- on the device path the colour kernels write that
layout directly (``tmb_color_f64_channels``); these host versions exist for
callers that use them on their own. File I/O and these layout maps are host
work outside the hot path.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

from .color import SPACE_RGB, ColorImage
from .ingest import DEFAULT_PATTERN, VIEW_NAMES, find_scene_files, read_image_u8
from .tensor import DenseTensor

__all__ = ["SceneStack", "VIEW_NAMES", "DEFAULT_PATTERN", "TENSOR_LAYOUT", "load_scene", "read_image",
           "write_image", "write_scene", "quantize_8bit", "stack_to_tensor", "tensor_to_stack"]

TENSOR_LAYOUT = ("height", "width", "exposure", "view")   # sceneio.py:38; header layout id 1


@dataclass
class SceneStack:
    """Views x exposures colour images of one scene (sceneio.py:41-76)."""

    name: str
    views: int
    exposures: int
    width: int
    height: int
    space: str
    images: dict[tuple[int, int], ColorImage] = field(default_factory=dict)

    def image(self, view: int, exposure: int) -> ColorImage:
        return self.images[(view, exposure)]

    def validate(self) -> None:
        if len(self.images) != self.views * self.exposures:
            raise ValueError(f"scene table incomplete: {len(self.images)} of {self.views * self.exposures}")
        for (v, e), img in self.images.items():
            if img.space != self.space:
                raise ValueError(f"image ({v},{e}) space {img.space} != scene space {self.space}")
            if (img.height, img.width) != (self.height, self.width):
                raise ValueError(f"image ({v},{e}) is {img.width}x{img.height}, scene is {self.width}x{self.height}")

    def map_images(self, fn) -> "SceneStack":
        images = {k: fn(img) for k, img in self.images.items()}
        space = next(iter(images.values())).space
        return SceneStack(self.name, self.views, self.exposures, self.width, self.height, space, images)

    def pixel_stack(self) -> np.ndarray:
        """(V*E, H, W, 3) float64 pixels in (view, exposure) order: image
        v*E + e, i.e. the (H, W, E, V) F-order plane index of every channel."""
        out = np.empty((self.views * self.exposures, self.height, self.width, 3), dtype=np.float64)
        for v in range(self.views):
            for e in range(self.exposures):
                out[v * self.exposures + e] = self.image(v, e).pixels
        return out


def read_image(path: str | Path) -> ColorImage:
    """8-bit RGB PNG or binary PPM -> [0, 1] RGB ColorImage (sceneio.py:79-87)."""
    return ColorImage(read_image_u8(path).astype(np.float64) / 255.0, SPACE_RGB)


def quantize_8bit(values: np.ndarray) -> np.ndarray:
    """[0, 1] floats -> uint8: clamp, x255, round half up (sceneio.py:104-107)."""
    v = np.clip(values, 0.0, 1.0) * 255.0
    return np.floor(v + 0.5).astype(np.uint8)


def write_image(img: ColorImage, path: str | Path, fmt: str | None = None) -> None:
    """8-bit PNG or binary PPM (sceneio.py:90-101)."""
    path = Path(path)
    if fmt is None:
        fmt = "ppm" if path.suffix.lower() == ".ppm" else "png"
    samples = quantize_8bit(img.pixels)
    if fmt == "ppm":
        h, w = samples.shape[:2]
        with open(path, "wb") as f:
            f.write(f"P6\n{w} {h}\n255\n".encode("ascii"))
            f.write(np.ascontiguousarray(samples, dtype=np.uint8).tobytes())
    elif fmt == "png":
        from PIL import Image

        Image.fromarray(samples, mode="RGB").save(path, format="PNG")
    else:
        raise ValueError(f"unsupported image format {fmt!r}")


def load_scene(path: str | Path, pattern: str = DEFAULT_PATTERN) -> SceneStack:
    """Scene directory -> RGB SceneStack (sceneio.py:152-188)."""
    root = Path(path)
    files = find_scene_files(root, pattern)
    images = {(v, e): read_image(p) for v, row in enumerate(files) for e, p in enumerate(row)}
    first = images[(0, 0)]
    for (v, e), img in images.items():
        if (img.height, img.width) != (first.height, first.width):
            raise ValueError(f"mixed resolutions: ({VIEW_NAMES[v]},{e}) is {img.width}x{img.height}, "
                             f"expected {first.width}x{first.height}")
    stack = SceneStack(root.name, len(VIEW_NAMES), len(files[0]), first.width, first.height, SPACE_RGB, images)
    stack.validate()
    return stack


def write_scene(stack: SceneStack, outdir: str | Path, fmt: str = "png") -> list[Path]:
    """Every image as {view}_{exposure}.{fmt} (sceneio.py:229-239)."""
    outdir = Path(outdir)
    outdir.mkdir(parents=True, exist_ok=True)
    paths = []
    for v in range(stack.views):
        for e in range(stack.exposures):
            p = outdir / f"{VIEW_NAMES[v]}_{e}.{fmt}"
            write_image(stack.image(v, e), p, fmt=fmt)
            paths.append(p)
    return paths


def stack_to_tensor(stack: SceneStack, channel: int) -> DenseTensor:
    """One channel as an order-4 (H, W, E, V) tensor (sceneio.py:191-199)."""
    if not 0 <= channel <= 2:
        raise ValueError(f"channel {channel} out of range [0, 2]")
    arr = np.empty((stack.height, stack.width, stack.exposures, stack.views), dtype=np.float64)
    for v in range(stack.views):
        for e in range(stack.exposures):
            arr[:, :, e, v] = stack.image(v, e).plane(channel)
    return DenseTensor(arr, check_finite=True)


def tensor_to_stack(channels: list[DenseTensor], space: str, name: str = "scene") -> SceneStack:
    """Inverse of stack_to_tensor over the three channel tensors (sceneio.py:202-226)."""
    if len(channels) != 3:
        raise ValueError(f"expected 3 channel tensors, got {len(channels)}")
    dims = channels[0].dims
    if len(dims) != 4:
        raise ValueError(f"expected order-4 tensors, got dims {dims}")
    for c, t in enumerate(channels):
        if t.dims != dims:
            raise ValueError(f"channel {c} dims {t.dims} != channel 0 dims {dims}")
        if not np.isfinite(t.array).all():
            raise ValueError(f"channel {c} contains non-finite entries")
    h, w, exposures, views = dims
    images = {}
    for v in range(views):
        for e in range(exposures):
            images[(v, e)] = ColorImage(np.stack([channels[c].array[:, :, e, v] for c in range(3)], axis=2), space)
    return SceneStack(name, views, exposures, w, h, space, images)
