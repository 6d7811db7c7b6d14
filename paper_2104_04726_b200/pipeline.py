"""The fused hot path: one multi-exposure stereo stack, u8 images -> coding-space
tensor -> Tucker-ALS -> quantised core (+ reconstruction error), in one
libtmb call (``tmb_encode_stack_u8``) with every intermediate resident in HBM.

This is the device form of the reference's encode chain for the BASELINE
configs: ``to_coding_space`` per image (color.py:185-194, codec.py:389) ->
``tucker_als`` (tucker.py:331-397) -> ``quantize_core`` (codec.py:114-134) ->
``reconstruct`` (tucker.py:166-171), on the (H, W, 3, V*E) tensor of SURVEY §8.0.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Sequence

import numpy as np

from . import _lib as L
from .tensor import DenseTensor
from .tucker import SolveConfig, SolveTrace, TuckerModel, _trace_buffers, _trace_from_c

__all__ = ["StackResult", "encode_stack", "encode_stack_device", "encode_stacks", "encode_stacks_device", "stream_lanes", "coding_tensor", "ScenePSNR", "DecodedStack",
           "decode_stack"]


@dataclass
class StackResult:
    model: TuckerModel | None
    trace: SolveTrace
    levels: np.ndarray | None
    step: float
    rel_err: float | None
    device: dict | None = None  # device tensors when requested


def coding_tensor(images_u8, space: str):
    """(V, E, H, W, 3) uint8 (host ndarray or CUDA tensor) -> float32 CUDA
    tensor holding the F-order (H, W, 3, V*E) coding-space stack."""
    torch = L._torch()
    if isinstance(images_u8, np.ndarray):
        images_u8 = torch.from_numpy(np.ascontiguousarray(images_u8))
    if images_u8.dtype != torch.uint8 or images_u8.dim() != 5 or images_u8.shape[-1] != 3:
        raise ValueError("expected a (V, E, H, W, 3) uint8 image stack")
    v, e, h, w, _ = images_u8.shape
    src = images_u8.to("cuda").contiguous()
    out = torch.empty(h * w * 3 * v * e, dtype=torch.float32, device="cuda")
    hctx = L.ctx()
    L.check(L.LIB.tmb_color_u8(hctx, L.ptr(src), v * e, h, w, L.SPACES[space], L.ptr(out)), hctx)
    return out


def encode_stack_device(images_dev, space: str, ranks: Sequence[int], cfg: SolveConfig, qp: int,
                        rel_err: bool = True, bufs: dict | None = None) -> tuple[dict, L.Trace, float, float | None]:
    """Device-resident hot path. ``images_dev``: (V, E, H, W, 3) uint8 CUDA
    tensor. Returns the device buffers dict (tensor, core, factors, levels),
    the raw trace, the quantiser step and the relative error."""
    torch = L._torch()
    v, e, h, w, _ = images_dev.shape
    dims = (h, w, 3, v * e)
    ranks = tuple(int(r) for r in ranks)
    cfg.validate(dims)
    if bufs is None:
        bufs = {
            "tensor": torch.empty(h * w * 3 * v * e, dtype=torch.float32, device="cuda"),
            "core": L.empty_f64(int(np.prod(ranks))),
            "factors": [L.empty_f64(s * r) for s, r in zip(dims, ranks)],
            "levels": torch.empty(int(np.prod(ranks)), dtype=torch.int64, device="cuda"),
        }
    tr, _keep = _trace_buffers(cfg.max_sweeps + 1)
    c = cfg.to_c()
    step = L.C.c_double()
    rel = L.C.c_double()
    hctx = L.ctx()
    L.check(L.LIB.tmb_encode_stack_u8(hctx, L.ptr(images_dev), v * e, h, w, L.SPACES[space], L.i64s(ranks),
                                      L.C.byref(c), int(qp), L.ptr(bufs["tensor"]), L.ptr(bufs["core"]),
                                      L.ptrs(bufs["factors"]), L.ptr(bufs["levels"]), L.C.byref(step),
                                      L.C.byref(tr), L.C.byref(rel) if rel_err else None), hctx)
    bufs["_trace_keep"] = _keep
    return bufs, tr, float(step.value), (float(rel.value) if rel_err else None)


def encode_stack(images_u8: np.ndarray, space: str, ranks: Sequence[int], sweeps: int, qp: int,
                 fit_tol: float = 1e-300, pp_enter_tol: float = 0.0, rel_err: bool = True,
                 return_model: bool = True) -> StackResult:
    """Host API for one stack: H2D of the u8 images, the fused device path,
    D2H of the quantised levels (and optionally the model)."""
    torch = L._torch()
    if isinstance(images_u8, np.ndarray):
        images_u8 = torch.from_numpy(np.ascontiguousarray(images_u8))
    imgs = images_u8.to("cuda", non_blocking=True)  # async from pinned host memory
    v, e, h, w, _ = imgs.shape
    dims = (h, w, 3, v * e)
    cfg = SolveConfig(ranks=tuple(ranks), max_sweeps=sweeps, fit_tol=fit_tol, pp_enter_tol=pp_enter_tol)
    bufs, tr, step, rel = encode_stack_device(imgs, space, ranks, cfg, qp, rel_err=rel_err)
    ranks = tuple(int(r) for r in ranks)
    # D2H into pinned host tensors (torch's caching host allocator), one sync for all;
    # the returned arrays keep their pinned blocks alive
    ncore = int(np.prod(ranks))
    outs = [bufs["levels"][:ncore]]
    if return_model:
        outs += [bufs["core"][:ncore]] + [f[: dims[n] * ranks[n]] for n, f in enumerate(bufs["factors"])]
    host = [torch.empty(o.shape, dtype=o.dtype, pin_memory=True) for o in outs]
    for h_, o in zip(host, outs):
        h_.copy_(o, non_blocking=True)
    torch.cuda.current_stream().synchronize()
    levels = np.reshape(host[0].numpy(), ranks, order="F")
    model = None
    if return_model:
        core = DenseTensor(np.reshape(host[1].numpy(), ranks, order="F"))
        facs = [np.reshape(host[2 + n].numpy(), (dims[n], ranks[n]), order="F") for n in range(len(dims))]
        model = TuckerModel(core, facs, dims)
    return StackResult(model, _trace_from_c(tr), levels, step, rel, bufs)


class _Lane:
    """One host thread with its own CUDA stream and its own libtmb context
    (``L.ctx()`` is per thread). Independent stacks on different lanes run
    concurrently on the GPU: a stack's latency-bound phases (the
    one-grid-barrier-per-column tridiagonalisation holds every SM at ~1/3
    issue) leave room for the other lane's GEMMs, colour pass and quantiser,
    and each solve's host-side waits (convergence trace, eigen-solver checks)
    block only its own thread. Lanes persist for the process so their
    contexts, arenas and Ozaki caches are reused across calls."""

    def __init__(self, device: int):
        import queue
        import threading

        self.device = device
        self.q: "queue.Queue" = queue.Queue()
        self.state: dict = {}
        self.ready = threading.Event()
        self.thread = threading.Thread(target=self._run, name=f"tmb-lane-{device}", daemon=True)
        self.thread.start()
        self.ready.wait()

    def _run(self) -> None:
        torch = L._torch()
        torch.cuda.set_device(self.device)
        self.stream = torch.cuda.Stream()
        with torch.cuda.stream(self.stream):
            self.ctx = L.ctx()
        self.ready.set()
        while True:
            fn, fut = self.q.get()
            try:
                with torch.cuda.stream(self.stream):
                    fut.set_result(fn(self))
            except BaseException as exc:  # noqa: BLE001 -- re-raised by the caller's result()
                fut.set_exception(exc)

    def submit(self, fn):
        import concurrent.futures as cf

        fut = cf.Future()
        self.q.put((fn, fut))
        return fut


_LANES: dict[int, list[_Lane]] = {}


def stream_lanes(count: int) -> list[_Lane]:
    """The first ``count`` persistent lanes of the current device."""
    torch = L._torch()
    dev = torch.cuda.current_device()
    pool = _LANES.setdefault(dev, [])
    while len(pool) < count:
        pool.append(_Lane(dev))
    return pool[:count]


DEFAULT_LANES = 2


def _encode_seq(stacks, space, ranks, cfg, qp, rel_err, ncore):
    """The single-stream pipeline on the current stream: the u8 images go
    through two device slots on a copy stream (H2D of stack i+1 overlaps the
    solve of stack i); the solve, quantiser and the D2H of each stack's levels
    run on the current stream."""
    torch = L._torch()
    comp = torch.cuda.current_stream()
    copy = torch.cuda.Stream()
    shape = tuple(stacks[0].shape)
    slots = [torch.empty(shape, dtype=torch.uint8, device="cuda") for _ in range(min(2, len(stacks)))]
    loaded = [torch.cuda.Event() for _ in slots]
    freed = [torch.cuda.Event() for _ in slots]

    def issue(i: int) -> None:
        k = i % len(slots)
        with torch.cuda.stream(copy):
            copy.wait_event(freed[k])              # the solve of stack i-2 is done with this slot
            slots[k].copy_(stacks[i], non_blocking=True)
            loaded[k].record(copy)

    issue(0)
    bufs = None
    pending = []
    for i in range(len(stacks)):
        k = i % len(slots)
        if i + 1 < len(stacks):
            issue(i + 1)
        comp.wait_event(loaded[k])
        bufs, tr, step, rel = encode_stack_device(slots[k], space, ranks, cfg, qp, rel_err, bufs)
        freed[k].record(comp)
        host = torch.empty(ncore, dtype=torch.int64, pin_memory=True)
        host.copy_(bufs["levels"][:ncore], non_blocking=True)  # same stream: ordered before the next solve
        pending.append((host, _trace_from_c(tr), step, rel))
    comp.synchronize()
    return [StackResult(None, trace, np.reshape(host.numpy(), ranks, order="F"), step, rel)
            for host, trace, step, rel in pending]


def encode_stacks(stacks, space: str, ranks: Sequence[int], sweeps: int, qp: int, fit_tol: float = 1e-300,
                  pp_enter_tol: float = 0.0, rel_err: bool = True, lanes: int | None = None) -> list[StackResult]:
    """Encode a sequence of independent stacks on this rank's GPU (BASELINE
    config 3).

    ``stacks``: (V, E, H, W, 3) uint8 host tensors/arrays of one shape (pinned
    torch tensors give truly asynchronous copies). Stack i goes to lane
    ``i % lanes`` (``_Lane``: a host thread with its own stream and context;
    default ``DEFAULT_LANES``), so two solves share the GPU; on each lane the
    H2D of its next stack overlaps the solve of its current one ("H2D of stack
    i+1's u8 planes overlaps compute of stack i"). Results are bit-identical
    to per-stack ``encode_stack`` calls whatever the lane count (every kernel
    is deterministic and lanes share no device state). Returns one
    ``StackResult`` per stack, in input order (levels, step, trace, relative
    error; no model). This is the data-parallel unit of work:
    ``dist.assign_stacks`` gives each rank its stack ids and every rank calls
    this on its own share, with no inter-GPU traffic (the reference's analogue
    is its process pool over independent cells, cli.py:379-382).
    """
    torch = L._torch()
    stacks = [torch.from_numpy(np.ascontiguousarray(s)) if isinstance(s, np.ndarray) else s for s in stacks]
    if not stacks:
        return []
    shape = tuple(stacks[0].shape)
    for s in stacks:
        if tuple(s.shape) != shape or s.dtype != torch.uint8:
            raise ValueError("encode_stacks needs (V, E, H, W, 3) uint8 stacks of one shape")
    v, e, h, w, _ = shape
    dims = (h, w, 3, v * e)
    ranks = tuple(int(r) for r in ranks)
    cfg = SolveConfig(ranks=ranks, max_sweeps=sweeps, fit_tol=fit_tol, pp_enter_tol=pp_enter_tol)
    cfg.validate(dims)
    ncore = int(np.prod(ranks))
    nl = max(1, min(int(DEFAULT_LANES if lanes is None else lanes), len(stacks)))
    if nl == 1:
        return _encode_seq(stacks, space, ranks, cfg, qp, rel_err, ncore)
    futs = [lane.submit(lambda _l, j=j: _encode_seq(stacks[j::nl], space, ranks, cfg, qp, rel_err, ncore))
            for j, lane in enumerate(stream_lanes(nl))]
    parts = [f.result() for f in futs]
    out: list = [None] * len(stacks)
    for j, part in enumerate(parts):
        out[j::nl] = part
    return out


def encode_stacks_device(dev_stacks, space: str, ranks: Sequence[int], cfg: SolveConfig, qp: int,
                         rel_err: bool = True, lanes: int | None = None) -> list[tuple[SolveTrace, float, float | None]]:
    """Device-resident form of :func:`encode_stacks` (inputs already in HBM,
    results left on the device): stack i solves on lane ``i % lanes``, each
    lane reusing its own device buffers across calls. Ordered after the
    caller's stream on entry; the caller's stream waits for every lane on
    exit. Returns (trace, step, rel_err) per stack, in input order."""
    torch = L._torch()
    if not dev_stacks:
        return []
    ranks = tuple(int(r) for r in ranks)
    nl = max(1, min(int(DEFAULT_LANES if lanes is None else lanes), len(dev_stacks)))
    caller = torch.cuda.current_stream()
    start = torch.cuda.Event()
    start.record(caller)

    def run(lane, j):
        lane.stream.wait_event(start)
        res = []
        for d in dev_stacks[j::nl]:
            bufs, tr, step, rel = encode_stack_device(d, space, ranks, cfg, qp, rel_err, lane.state.get("bufs"))
            lane.state["bufs"] = bufs
            res.append((_trace_from_c(tr), step, rel))
        done = torch.cuda.Event()
        done.record(lane.stream)
        return res, done

    futs = [lane.submit(lambda ln, j=j: run(ln, j)) for j, lane in enumerate(stream_lanes(nl))]
    out: list = [None] * len(dev_stacks)
    for j, f in enumerate(futs):
        res, done = f.result()
        caller.wait_event(done)
        out[j::nl] = res
    return out


# ---------------------------------------------------------------------------
# decode side
# ---------------------------------------------------------------------------


@dataclass
class ScenePSNR:
    """metrics.ScenePSNR (metrics.py:33-38): per-view PSNR (8-bit units, MSE
    averaged over exposures and channels) and the per-exposure (left, right) pairs."""

    left: float
    right: float
    per_exposure: list[tuple[float, float]]


@dataclass
class DecodedStack:
    rgb: np.ndarray | None       # (V, E, H, W, 3) float64 RGB, when requested
    mse: np.ndarray | None       # (V, E) metrics.mse in 8-bit units vs the original images
    psnr: ScenePSNR | None


def _to_db(m: float) -> float:
    import math

    return math.inf if m == 0.0 else 10.0 * math.log10(255.0 * 255.0 / m)


def decode_stack(q, space: str, views: int, exposures: int, images_u8=None, return_rgb: bool = True
                 ) -> DecodedStack:
    """Decode one stack on the device: ``dequantize`` (codec.py:137-148) ->
    ``reconstruct`` (tucker.py:166-171) -> ``to_rgb`` per image (color.py:197-205),
    and with ``images_u8`` (V, E, H, W, 3) the reference's ``scene_psnr``
    (metrics.py:41-76) against them. ``q`` is a QuantizedModel of a (H, W, 3,
    V*E) stack (or a TuckerModel, decoded without quantisation)."""
    from .codec import QuantizedModel, dequantize

    torch = L._torch()
    model = dequantize(q) if isinstance(q, QuantizedModel) else q
    h, w, c3, ve = model.source_dims
    if c3 != 3 or ve != views * exposures:
        raise ValueError(f"model dims {model.source_dims} are not a ({views}x{exposures})-image stack")
    ranks = tuple(model.ranks)
    hc = L.ctx()
    core = L.dev_f64(model.core.array)
    facs = [L.dev_f64(f) for f in model.factors]
    rec = L.empty_f64(h * w * 3 * ve)
    L.check(L.LIB.tmb_reconstruct(hc, 4, L.i64s(ranks), L.i64s(model.source_dims), L.ptr(core), L.ptrs(facs),
                                  L.ptr(rec)), hc)
    out = torch.empty(ve * h * w * 3, dtype=torch.float64, device="cuda") if return_rgb else None
    src = None
    sse = None
    if images_u8 is not None:
        if isinstance(images_u8, np.ndarray):
            images_u8 = torch.from_numpy(np.ascontiguousarray(images_u8))
        if tuple(images_u8.shape) != (views, exposures, h, w, 3) or images_u8.dtype != torch.uint8:
            raise ValueError(f"reference images must be ({views}, {exposures}, {h}, {w}, 3) uint8")
        src = images_u8.to("cuda").contiguous()
        sse = np.zeros(ve, dtype=np.float64)
    L.check(L.LIB.tmb_decode_sse(hc, L.ptr(rec), ve, h, w, L.SPACES[space], L.ptr(src) if src is not None else None,
                                 L.ptr(out) if out is not None else None,
                                 sse.ctypes.data_as(L.C.POINTER(L.C.c_double)) if sse is not None else None), hc)
    rgb = out.cpu().numpy().reshape(views, exposures, h, w, 3) if out is not None else None
    mse = psnr = None
    if sse is not None:
        mse = (sse / (3.0 * h * w)).reshape(views, exposures)
        per_view = [_to_db(float(np.mean(mse[v]))) for v in range(views)]
        per_exp = [[_to_db(float(m)) for m in mse[v]] for v in range(views)]
        pairs = list(zip(per_exp[0], per_exp[1] if views > 1 else per_exp[0]))
        psnr = ScenePSNR(per_view[0], per_view[1] if views > 1 else per_view[0], pairs)
    return DecodedStack(rgb, mse, psnr)
