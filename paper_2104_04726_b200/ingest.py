"""Scene ingestion for the hot path.

The reference loads a scene directory image by image into float64 ColorImages
(sceneio.load_scene / read_image, sceneio.py:79-188) before the codec converts
each to the coding space. Here the same directory convention (files
``{view}_{exposure}`` + .png/.ppm, views left/right, E inferred from the
consecutive left exposures, equal resolutions required) is decoded straight
into one pinned (V, E, H, W, 3) uint8 stack -- the input of the colour kernel
-- with the files decoded on host threads, and ``encode_scene_dirs`` overlaps
decoding + the pinned host->device copy of scene i+1 with the device solve of
scene i.
"""

from __future__ import annotations

import re
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path
from typing import Iterable, Sequence

import numpy as np

__all__ = ["VIEW_NAMES", "DEFAULT_PATTERN", "find_scene_files", "read_image_u8", "load_scene_u8",
           "encode_scene_dirs"]

VIEW_NAMES = ("left", "right")          # sceneio.py:32
DEFAULT_PATTERN = "{view}_{exposure}"   # sceneio.py:33
EXTENSIONS = (".png", ".ppm")  # sceneio.py:34


def _find_file(root: Path, pattern: str, view: str, exposure: int) -> Path | None:
    stem = pattern.format(view=view, exposure=exposure)  # sceneio.py:141-150
    if "." in Path(stem).name:
        p = root / stem
        return p if p.exists() else None
    for ext in EXTENSIONS:
        p = root / (stem + ext)
        if p.exists():
            return p
    return None


def find_scene_files(path: str | Path, pattern: str = DEFAULT_PATTERN) -> list[list[Path]]:
    """[view][exposure] file paths with the reference's discovery rules
    (sceneio.py:153-168): E = number of consecutive left exposures."""
    root = Path(path)
    if not root.is_dir():
        raise FileNotFoundError(f"scene directory not found: {root}")
    exposures = 0
    while _find_file(root, pattern, "left", exposures) is not None:
        exposures += 1
    if exposures == 0:
        raise FileNotFoundError(f"no images matching {pattern!r} for view 'left' in {root}")
    files = []
    for view in VIEW_NAMES:
        row = []
        for e in range(exposures):
            p = _find_file(root, pattern, view, e)
            if p is None:
                raise FileNotFoundError(f"missing scene file for (view={view}, exposure={e})")
            row.append(p)
        files.append(row)
    return files


_PPM_TOKEN = re.compile(rb"\s*(?:#[^\n]*\n\s*)*(\S+)")


def _read_ppm(path: Path) -> np.ndarray:
    """Binary P6, maxval 255 (sceneio.py:109-130)."""
    data = path.read_bytes()
    tokens, pos = [], 0
    while len(tokens) < 4:
        m = _PPM_TOKEN.match(data, pos)
        if not m:
            raise ValueError(f"{path}: truncated PPM header")
        tokens.append(m.group(1))
        pos = m.end()
    if tokens[0] != b"P6":
        raise ValueError(f"{path}: not a binary PPM (P6) file")
    width, height, maxval = int(tokens[1]), int(tokens[2]), int(tokens[3])
    if maxval != 255:
        raise ValueError(f"{path}: only maxval 255 supported, got {maxval}")
    raster = data[pos + 1: pos + 1 + width * height * 3]
    if len(raster) != width * height * 3:
        raise ValueError(f"{path}: truncated PPM raster")
    return np.frombuffer(raster, dtype=np.uint8).reshape(height, width, 3)


def read_image_u8(path: str | Path) -> np.ndarray:
    """8-bit RGB PNG or binary PPM -> (H, W, 3) uint8 (the samples behind
    read_image's u8/255, sceneio.py:79-87)."""
    path = Path(path)
    if path.suffix.lower() == ".ppm":
        return _read_ppm(path)
    from PIL import Image

    with Image.open(path) as im:
        return np.asarray(im.convert("RGB"), dtype=np.uint8)


def load_scene_u8(path: str | Path, pattern: str = DEFAULT_PATTERN, threads: int = 8, pinned: bool = True):
    """One scene directory -> (V, E, H, W, 3) uint8 stack (pinned torch tensor
    when ``pinned``), files decoded on ``threads`` host threads, with the
    reference's mixed-resolution check (sceneio.py:170-177)."""
    import torch

    files = find_scene_files(path, pattern)
    flat = [p for row in files for p in row]
    with ThreadPoolExecutor(max_workers=max(1, threads)) as pool:
        imgs = list(pool.map(read_image_u8, flat))
    h, w = imgs[0].shape[:2]
    for i, img in enumerate(imgs):
        if img.shape[:2] != (h, w):
            v, e = divmod(i, len(files[0]))
            raise ValueError(f"mixed resolutions: ({VIEW_NAMES[v]},{e}) is {img.shape[1]}x{img.shape[0]}, "
                             f"expected {w}x{h}")
    v_, e_ = len(files), len(files[0])
    out = torch.empty((v_, e_, h, w, 3), dtype=torch.uint8, pin_memory=pinned and torch.cuda.is_available())
    arr = out.numpy()
    for i, img in enumerate(imgs):
        arr[i // e_, i % e_] = img
    return out


def encode_scene_dirs(paths: Iterable[str | Path], space: str, ranks: Sequence[int], sweeps: int, qp: int,
                      pattern: str = DEFAULT_PATTERN, threads: int = 8):
    """Encode a sequence of scene directories: scene i+1 is decoded into pinned
    memory on host threads while the device encodes scene i (encode_stack).
    Yields (path, StackResult)."""
    from .pipeline import encode_stack

    paths = list(paths)
    if not paths:
        return
    with ThreadPoolExecutor(max_workers=1) as pre:
        nxt = pre.submit(load_scene_u8, paths[0], pattern, threads)
        for i, p in enumerate(paths):
            images = nxt.result()
            if i + 1 < len(paths):
                nxt = pre.submit(load_scene_u8, paths[i + 1], pattern, threads)
            yield p, encode_stack(images, space, ranks, sweeps, qp)
