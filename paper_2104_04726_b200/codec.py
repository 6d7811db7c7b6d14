"""Core quantiser of the latent path on the B200 (codec.py:78-148 of the reference).

``quantize_core`` / ``dequantize`` / ``QuantizedModel`` / ``preset_ranks`` /
``CodecError``, plus the latent path's callers and data format either side of
the solve: ``solve_channels`` (the three per-channel
solves of ``_solve_channels``, codec.py:366-374, on the device) and the latent
block bytes (``_serialize_latent_channel`` / ``_deserialize_latent_channel``,
codec.py:285-318, with the level varints encoded and decoded on the device).
The drop-in stream entry points (``EncodeConfig``, ``encode_stream``,
``decode_stream``, ``CompressedStream``, ``serialize_stream``/``parse_stream``,
codec.py:150-468) run the latent path: colour, the three channel solves
(one native ``tmb_solve_channels`` call), quantiser and level varints on the
device; the range coder (libtmb host C++) and the container bytes on the host.
The frames path (3D-HEVC stand-in) raises NotImplementedError.
"""

from __future__ import annotations

import math
import struct
from dataclasses import dataclass, field
from typing import Sequence

import numpy as np

from . import _lib as L
from .tensor import DenseTensor
from .tucker import TuckerModel

__all__ = ["CodecError", "QuantizedModel", "quantize_core", "dequantize", "preset_ranks", "PRESETS", "PRESET_RHO",
           "serialize_latent_channel", "deserialize_latent_channel", "solve_channels", "solve_channels_f64",
           "BackendConfig", "BackendConfigRequired", "PATH_LATENT", "PATH_FRAMES", "StreamHeader",
           "CompressedStream", "serialize_stream", "parse_stream", "stream_bits", "EncodeConfig", "encode_stream",
           "decode_stream"]

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
    (TuckerModel, SolveTrace), or of QuantizedModel when ``qp`` is given.

    Precision note: this is the BASELINE harness's format -- the u8 colour
    kernel writes fp32(reference float64 colour), bit for bit, and the solve
    accumulates in fp64 from those fp32 values. The reference codec solves the
    float64 colour values themselves; the float64 drop-in for that is
    ``encode_stream`` / ``solve_channels_f64`` (App. B.1(ii) measures the
    difference: angles ~1e-4 rad, levels equal except ties)."""
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


# ---------------------------------------------------------------------------
# drop-in stream API: EncodeConfig / encode_stream / decode_stream and the
# container (codec.py:150-468 of the reference)
# ---------------------------------------------------------------------------

PATH_LATENT = "latent"
PATH_FRAMES = "frames"
MAGIC = b"TMC1"
VERSION = 1
LAYOUT_HWEV = 1
_HEADER_FMT = "<4sBBBBBHHB4HBBB6s"      # codec.py:1-14: 31 bytes, little-endian
_HEADER_SIZE = struct.calcsize(_HEADER_FMT)
_PATH_TAGS = {PATH_LATENT: 0, PATH_FRAMES: 1}
_SPACE_TAGS = {"rgb": 0, "ycbcr": 1, "ipt": 2}
_BACKEND_TAGS = {"builtin": 0, "external": 1}
_PATH_NAMES = {v: k for k, v in _PATH_TAGS.items()}
_SPACE_NAMES = {v: k for k, v in _SPACE_TAGS.items()}
_BACKEND_NAMES = {v: k for k, v in _BACKEND_TAGS.items()}
_FRAMES_OUT = ("the frames path (the 3D-HEVC stand-in frames codec and its external-encoder adapter, "
               "frames.py) is outside this package's scope (SURVEY.md §2 row 8; the north star keeps 3D-HEVC "
               "encode outside); use path='latent'")


class BackendConfigRequired(CodecError):
    """An external frames stream needs a BackendConfig to decode (codec.py)."""


@dataclass
class BackendConfig:
    """Frame-coding backend selection (frames.py:47-69); validated like the
    reference's, but only the latent path is implemented here."""

    kind: str = "builtin"
    qp: int = 0
    template: str | None = None
    decode_template: str | None = None
    timeout: float = 600.0
    scratch: str | None = None

    def validate(self) -> None:
        if self.kind not in ("builtin", "external"):
            raise ValueError(f"unknown backend kind {self.kind!r}")
        if not 0 <= self.qp <= 51:
            raise ValueError(f"qp {self.qp} out of range [0, 51]")
        if (self.template is not None) != (self.kind == "external"):
            raise ValueError("command template must be given exactly for external backends")


@dataclass
class StreamHeader:
    """Container header fields (codec.py:156-172)."""

    path: str
    space: str
    views: int
    exposures: int
    height: int
    width: int
    ranks: tuple[int, int, int, int]
    qp: int
    entropy_tag: int
    layout: int = LAYOUT_HWEV
    backend_kind: str = "builtin"

    @property
    def dims(self) -> tuple[int, int, int, int]:
        return (self.height, self.width, self.exposures, self.views)


@dataclass
class CompressedStream:
    header: StreamHeader
    blocks: list[bytes]
    command: str | None = None


def serialize_stream(stream: CompressedStream) -> bytes:
    """Header + optional command block + three u32-prefixed channel blocks
    (codec.py:182-211)."""
    h = stream.header
    reserved = bytes([_BACKEND_TAGS[h.backend_kind]]) + b"\x00" * 5
    out = bytearray(struct.pack(_HEADER_FMT, MAGIC, VERSION, _PATH_TAGS[h.path], _SPACE_TAGS[h.space], h.views,
                                h.exposures, h.height, h.width, len(h.ranks), *h.ranks, h.qp, h.entropy_tag,
                                h.layout, reserved))
    if h.backend_kind == "external":
        cmd = (stream.command or "").encode("utf-8")
        out += struct.pack("<I", len(cmd)) + cmd
    if len(stream.blocks) != 3:
        raise CodecError(f"expected 3 channel blocks, got {len(stream.blocks)}")
    for block in stream.blocks:
        out += struct.pack("<I", len(block)) + block
    return bytes(out)


def parse_stream(data: bytes) -> CompressedStream:
    """Inverse of serialize_stream with the reference's CodecError checks
    (codec.py:214-270)."""
    from .entropy import TAG_RANGE, TAG_STORED

    if len(data) < _HEADER_SIZE:
        raise CodecError("truncated stream: header incomplete")
    fields = struct.unpack_from(_HEADER_FMT, data, 0)
    magic, version, path_tag, space_tag, views, exposures, height, width, order = fields[:9]
    ranks = fields[9:13]
    qp, entropy_tag, layout, reserved = fields[13:]
    if magic != MAGIC:
        raise CodecError(f"bad magic {magic!r}, expected {MAGIC!r}")
    if version != VERSION:
        raise CodecError(f"unsupported stream version {version}")
    if path_tag not in _PATH_NAMES:
        raise CodecError(f"unknown path tag {path_tag}")
    if space_tag not in _SPACE_NAMES:
        raise CodecError(f"unknown space tag {space_tag}")
    if order != 4 or layout != LAYOUT_HWEV:
        raise CodecError(f"unsupported tensor layout (order={order}, layout={layout})")
    if entropy_tag not in (TAG_STORED, TAG_RANGE):
        raise CodecError(f"unknown entropy stage tag {entropy_tag}")
    backend_kind = _BACKEND_NAMES.get(reserved[0])
    if backend_kind is None:
        raise CodecError(f"unknown backend kind {reserved[0]}")
    pos = _HEADER_SIZE

    def take_block() -> bytes:
        nonlocal pos
        if pos + 4 > len(data):
            raise CodecError("truncated stream: missing block length")
        (length,) = struct.unpack_from("<I", data, pos)
        pos += 4
        if pos + length > len(data):
            raise CodecError("truncated stream: block payload incomplete")
        block = data[pos:pos + length]
        pos += length
        return block

    command = take_block().decode("utf-8") if backend_kind == "external" else None
    blocks = [take_block() for _ in range(3)]
    if pos != len(data):
        raise CodecError(f"{len(data) - pos} trailing bytes after final block")
    header = StreamHeader(_PATH_NAMES[path_tag], _SPACE_NAMES[space_tag], views, exposures, height, width,
                          tuple(int(r) for r in ranks), qp, entropy_tag, layout, backend_kind)
    return CompressedStream(header, blocks, command)


def stream_bits(stream: CompressedStream) -> tuple[int, int, int]:
    """(bits_total, bits_payload, bits_overhead) (codec.py:273-277)."""
    total = len(serialize_stream(stream)) * 8
    payload = sum(len(b) for b in stream.blocks) * 8
    return total, payload, total - payload


@dataclass
class EncodeConfig:
    """Everything encode_stream needs besides the scene (codec.py:323-363);
    same fields and defaults."""

    space: str = "ycbcr"
    path: str = PATH_LATENT
    qp: int = 10
    preset: int | None = None
    ranks: tuple[int, int, int, int] | None = None
    entropy_tag: int = 1
    backend: BackendConfig = field(default_factory=BackendConfig)
    max_sweeps: int = 50
    fit_tol: float = 1e-5
    pp_enter_tol: float = 0.1
    pp_exit_tol: float = 0.3
    sequential_reduction: bool = True
    seed: int = 0

    def resolve_ranks(self, dims: tuple[int, int, int, int]) -> tuple[int, int, int, int]:
        if self.ranks is not None:
            ranks = tuple(int(r) for r in self.ranks)
            if len(ranks) != 4:
                raise ValueError(f"need 4 ranks, got {ranks}")
            for n, (r, s) in enumerate(zip(ranks, dims)):
                if not 1 <= r <= s:
                    raise ValueError(f"mode {n}: rank {r} not in [1, {s}]")
            return ranks
        if self.preset is not None:
            return preset_ranks(self.preset, dims)
        return tuple(dims)  # full rank

    def solve_config(self, ranks: tuple[int, ...]):
        from .tucker import SolveConfig

        return SolveConfig(ranks=ranks, max_sweeps=self.max_sweeps, fit_tol=self.fit_tol,
                           pp_enter_tol=self.pp_enter_tol, pp_exit_tol=self.pp_exit_tol,
                           sequential_reduction=self.sequential_reduction, seed=self.seed)


@dataclass
class ChannelSolve:
    """One channel's solve, resident on the device."""

    core: object          # device float64 core (F-order, ranks)
    factors: list         # device float64 factors (column-major s_n x r_n)
    trace: object         # SolveTrace


def solve_channels_f64(pixels: np.ndarray, space: str, dims: tuple[int, int, int, int], cfg) -> list[ChannelSolve]:
    """``_solve_channels`` (codec.py:366-374) after ``map_images(to_coding_space)``
    (codec.py:389), on the device in float64 like the reference: the (V*E, H, W,
    3) float64 pixels go through ``tmb_color_f64_channels`` straight into the
    three (H, W, E, V) channel tensors, and ``tmb_solve_channels`` runs the
    three tucker_als solves in one native call. Returns device-resident models."""
    from .tucker import _trace_buffers, _trace_from_c

    torch = L._torch()
    h, w, e, v = dims
    ranks = tuple(int(r) for r in cfg.ranks)
    cfg.validate(dims)
    px = torch.from_numpy(np.ascontiguousarray(pixels, dtype=np.float64)).to("cuda")
    per = h * w * e * v
    x = torch.empty(3 * per, dtype=torch.float64, device="cuda")
    hc = L.ctx()
    L.check(L.LIB.tmb_color_f64_channels(hc, L.ptr(px), v * e, h, w, L.SPACES[space], L.ptr(x)), hc)
    del px
    cores = [L.empty_f64(int(np.prod(ranks))) for _ in range(3)]
    facs = [L.empty_f64(s * r) for _ in range(3) for s, r in zip(dims, ranks)]
    bufs = [_trace_buffers(cfg.max_sweeps + 1) for _ in range(3)]
    traces = (L.Trace * 3)(*[b[0] for b in bufs])
    c = cfg.to_c()
    L.check(L.LIB.tmb_solve_channels(hc, L.ptr(x), L.F64, L.i64s(dims), L.i64s(ranks), L.C.byref(c), L.ptrs(cores),
                                     L.ptrs(facs), traces), hc)
    return [ChannelSolve(cores[ch], facs[4 * ch:4 * ch + 4], _trace_from_c(traces[ch])) for ch in range(3)]


def _latent_block(sol: ChannelSolve, dims, ranks, qp: int) -> bytes:
    """quantize_core + _serialize_latent_channel (codec.py:114-134, 285-291) of a
    device-resident channel model: levels quantised and varint-coded on the
    device, factors cast to float32 (the reference's np.asarray(f, float32))."""
    n = int(np.prod(ranks))
    lv, step = quantize_levels_device(sol.core, n, qp)
    out = bytearray()
    for f, s, r in zip(sol.factors, dims, ranks):
        out += np.asarray(f[: s * r].cpu().numpy(), dtype="<f4").tobytes()   # column-major already
    out += _varint_encode_dev(lv, n)
    out += struct.pack("<d", step)
    return bytes(out)


def encode_stream(scene, cfg: EncodeConfig) -> CompressedStream:
    """Compress a scene along the latent path (codec.py:377-430): colour,
    the three channel solves, quantiser and latent varints on the device; the
    range coder and container on the host (libtmb's C++ coder)."""
    from .entropy import entropy_stage

    if cfg.path not in _PATH_TAGS:
        raise ValueError(f"unknown path {cfg.path!r}")
    if cfg.space not in _SPACE_TAGS:
        raise ValueError(f"unknown color space {cfg.space!r}")
    if not 0 <= cfg.qp <= 51:
        raise ValueError(f"qp {cfg.qp} out of range [0, 51]")
    cfg.backend.validate()
    if scene.space != "rgb":
        raise ValueError("encode_stream expects an RGB scene")
    if cfg.path == PATH_FRAMES:
        raise NotImplementedError(_FRAMES_OUT)
    dims = (scene.height, scene.width, scene.exposures, scene.views)
    ranks = cfg.resolve_ranks(dims)
    pixels = scene.pixel_stack()
    if not np.isfinite(pixels).all():   # stack_to_tensor's check_finite (sceneio.py:199)
        raise ValueError("tensor entries must be finite")
    sols = solve_channels_f64(pixels, cfg.space, dims, cfg.solve_config(ranks))
    blocks = [entropy_stage(_latent_block(s, dims, ranks, cfg.qp), cfg.entropy_tag, "encode") for s in sols]
    header = StreamHeader(PATH_LATENT, cfg.space, scene.views, scene.exposures, scene.height, scene.width, ranks,
                          cfg.qp, cfg.entropy_tag, LAYOUT_HWEV, "builtin")
    return CompressedStream(header, blocks, None)


def decode_stream(stream: CompressedStream, backend: BackendConfig | None = None, name: str = "scene"):
    """Reconstruct the RGB scene a latent stream encodes (codec.py:433-468):
    entropy stage (host) -> latent block (varints decoded on the device) ->
    dequantize -> reconstruct -> tensor_to_stack -> to_rgb, the last three on
    the device (tmb_reconstruct per channel, tmb_channels_to_rgb)."""
    from .color import ColorImage
    from .entropy import entropy_stage
    from .scene import SceneStack

    h = stream.header
    if h.path != PATH_LATENT:
        raise NotImplementedError(_FRAMES_OUT)
    torch = L._torch()
    dims = h.dims
    ranks = tuple(h.ranks)
    per = int(np.prod(dims))
    planes = torch.empty(3 * per, dtype=torch.float64, device="cuda")
    hc = L.ctx()
    for c, block in enumerate(stream.blocks):
        raw = entropy_stage(block, h.entropy_tag, "decode")
        q = deserialize_latent_channel(raw, dims, ranks, h.qp)
        model = dequantize(q)
        core = L.dev_f64(model.core.array)
        facs = [L.dev_f64(f) for f in model.factors]
        L.check(L.LIB.tmb_reconstruct(hc, 4, L.i64s(ranks), L.i64s(dims), L.ptr(core), L.ptrs(facs),
                                      L.ptr(planes[c * per:(c + 1) * per])), hc)
    height, width, exposures, views = dims
    rgb = torch.empty(views * exposures * height * width * 3, dtype=torch.float64, device="cuda")
    L.check(L.LIB.tmb_channels_to_rgb(hc, L.ptr(planes), views * exposures, height, width, L.SPACES[h.space],
                                      L.ptr(rgb)), hc)
    arr = rgb.cpu().numpy().reshape(views * exposures, height, width, 3)
    images = {(v, e): ColorImage(arr[v * exposures + e], "rgb") for v in range(views) for e in range(exposures)}
    return SceneStack(name, views, exposures, width, height, "rgb", images)
