"""sha256 of the REFERENCE's colour transforms over all 2^24 u8 RGB triples
(build container only; imports /root/reference/pkg/src):

    PYTHONDONTWRITEBYTECODE=1 python scripts/make_golden_colour_exhaustive.py

One 4096 x 4096 image holds every triple (code = r<<16 | g<<8 | b, row-major);
``to_coding_space(ColorImage(u8 / 255), space)`` -- the reference's own colour
(color.py:185-194 as codec.py:389 calls it on sceneio.read_image's u8/255) --
rounded to float32 (the device tensor format). The (4096, 4096, 3) C-order
float32 bytes are hashed; tests/test_gpu_api.py::test_colour_u8_exhaustive
compares the device kernel's output to these hashes, so the fp32 tensor is
pinned bit for bit against the reference itself, not only the oracle.
"""
from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from tmcodec.color import ColorImage, to_coding_space  # noqa: E402

ROOT = Path(__file__).resolve().parents[1]

codes = np.arange(1 << 24, dtype=np.uint32)
u8 = np.stack([(codes >> 16) & 255, (codes >> 8) & 255, codes & 255], axis=-1).astype(np.uint8)
img = ColorImage(u8.reshape(4096, 4096, 3).astype(np.float64) / 255.0)
out = {}
for space in ("ycbcr", "ipt"):
    f32 = np.ascontiguousarray(to_coding_space(img, space).pixels.astype(np.float32))
    out[space] = hashlib.sha256(f32.tobytes()).hexdigest()
    print(space, out[space])
(ROOT / "tests" / "golden" / "colour_exhaustive.json").write_text(json.dumps(out, indent=1) + "\n")
