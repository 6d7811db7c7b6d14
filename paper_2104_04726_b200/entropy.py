"""Entropy stage and integer serialisation of the latent stream (drop-in for the
reference's ``entropy.py``).

Stage tags (entropy.py:37-52): 0 = stored, 1 = adaptive range coder with a u32
little-endian raw-length marker. The range coder is libtmb's host-side C++
coder (``tmb_rc_encode`` / ``tmb_rc_decode``, csrc/h_entropy.cu), byte-identical
to the reference's (_kernels_py.py:24-109); zigzag/LEB128 varints of the core
levels are encoded and decoded on the device (``tmb_varint_*``, k_latent.cu).
This is serial byte work after the hot path: it is here
so ``encode_stream`` / ``decode_stream`` read and write the reference's format.
"""

from __future__ import annotations

import ctypes as C
import struct

import numpy as np

from . import _lib as L

__all__ = ["TAG_STORED", "TAG_RANGE", "entropy_stage", "zigzag_encode", "zigzag_decode", "varint_encode",
           "varint_decode", "encode_ints", "decode_ints", "rc_encode", "rc_decode"]

TAG_STORED = 0
TAG_RANGE = 1


def _u8p(buf) -> C.POINTER(C.c_uint8):
    return C.cast(buf, C.POINTER(C.c_uint8))


def rc_encode(data: bytes) -> bytes:
    """Range-code a byte string (kernels.rc_encode, _kernels_py.py:24-58)."""
    data = bytes(data)
    cap = C.c_int64()
    L.LIB.tmb_rc_bound(len(data), C.byref(cap))
    src = (C.c_uint8 * max(len(data), 1)).from_buffer_copy(data or b"\0")
    out = (C.c_uint8 * cap.value)()
    n = C.c_int64()
    rc = L.LIB.tmb_rc_encode(_u8p(src), len(data), _u8p(out), cap.value, C.byref(n))
    if rc != L.TMB_OK:
        raise RuntimeError(f"tmb_rc_encode failed ({rc})")
    return bytes(out[: n.value])


def rc_decode(data: bytes, n: int) -> bytes:
    """Decode n symbols produced by rc_encode (_kernels_py.py:61-109)."""
    data = bytes(data)
    src = (C.c_uint8 * max(len(data), 1)).from_buffer_copy(data or b"\0")
    out = (C.c_uint8 * max(n, 1))()
    rc = L.LIB.tmb_rc_decode(_u8p(src), len(data), int(n), _u8p(out))
    if rc != L.TMB_OK:
        raise ValueError(f"range-coded payload corrupt ({rc})")
    return bytes(out[:n])


def entropy_stage(data: bytes, tag: int, direction: str) -> bytes:
    """Apply or invert the entropy stage named by ``tag`` (entropy.py:37-52)."""
    if direction not in ("encode", "decode"):
        raise ValueError(f"direction must be 'encode' or 'decode', got {direction!r}")
    if tag == TAG_STORED:
        return bytes(data)
    if tag == TAG_RANGE:
        if direction == "encode":
            return struct.pack("<I", len(data)) + (rc_encode(data) if data else b"")
        if len(data) < 4:
            raise ValueError("range-coded payload truncated: missing length marker")
        (n,) = struct.unpack_from("<I", data, 0)
        if n == 0:
            return b""
        return rc_decode(data[4:], n)
    raise ValueError(f"unknown entropy stage tag {tag}")


def zigzag_encode(values: np.ndarray) -> np.ndarray:
    """int64 -> uint64 zigzag (entropy.py:55-58)."""
    v = np.asarray(values, dtype=np.int64)
    return ((v << 1) ^ (v >> 63)).astype(np.uint64)


def zigzag_decode(values: np.ndarray) -> np.ndarray:
    u = np.asarray(values, dtype=np.uint64)
    return ((u >> np.uint64(1)).astype(np.int64)) ^ -((u & np.uint64(1)).astype(np.int64))


def encode_ints(values: np.ndarray) -> bytes:
    """Signed int64 array -> zigzag LEB128 varint bytes, on the device
    (entropy.py:109-111)."""
    torch = L._torch()
    flat = np.ascontiguousarray(np.asarray(values, dtype=np.int64).ravel())
    if flat.size == 0:
        return b""
    src = torch.from_numpy(flat).to("cuda")
    cap = 10 * flat.size
    out = torch.empty(cap, dtype=torch.uint8, device="cuda")
    nb = C.c_int64()
    h = L.ctx()
    L.check(L.LIB.tmb_varint_encode(h, L.ptr(src), flat.size, L.ptr(out), cap, C.byref(nb)), h)
    return bytes(out[: nb.value].cpu().numpy().tobytes())


def decode_ints(data: bytes, count: int) -> tuple[np.ndarray, int]:
    """Inverse of encode_ints (entropy.py:114-117); returns (int64 array, bytes
    consumed). ValueError on truncated / over-long varints."""
    torch = L._torch()
    if count == 0:
        return np.zeros(0, dtype=np.int64), 0
    body = np.frombuffer(bytes(data), dtype=np.uint8)
    src = torch.from_numpy(body.copy()).to("cuda") if body.size else torch.empty(1, dtype=torch.uint8, device="cuda")
    lv = torch.empty(count, dtype=torch.int64, device="cuda")
    used = C.c_int64()
    h = L.ctx()
    L.check(L.LIB.tmb_varint_decode(h, L.ptr(src), int(body.size), int(count), L.ptr(lv), C.byref(used)), h)
    return lv.cpu().numpy(), int(used.value)


def varint_encode(values: np.ndarray) -> bytes:
    """LEB128 varints of a uint64 array (entropy.py:66-85): the device encoder
    applied to the zigzag pre-image, so the bytes are those of the values."""
    return encode_ints(zigzag_decode(np.asarray(values, dtype=np.uint64)))


def varint_decode(data: bytes, count: int) -> tuple[np.ndarray, int]:
    vals, used = decode_ints(data, count)
    return zigzag_encode(vals), used
