"""ctypes binding of libtmb.so (include/tmb.h) plus device-memory plumbing.

PyTorch provides device memory and the current CUDA stream; every computation
runs in libtmb's kernels. There is no CPU implementation behind this module:
if the library is missing the package import fails, and if no CUDA device is
present every compute call raises.
"""

from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

import numpy as np

_PATH = Path(os.environ.get("TMB_LIB", Path(__file__).resolve().parent / "libtmb.so"))
if not _PATH.exists():
    raise ImportError(
        f"{_PATH} is not built; run `python paper_2104_04726_b200/_build.py` "
        "(or __graft_entry__.build()). There is no CPU fallback."
    )
LIB = C.CDLL(str(_PATH))

TMB_OK, TMB_EINVAL, TMB_ENUMERIC, TMB_ECUDA, TMB_ENOTIMPL = 0, 1, 2, 3, 4
SPACES = {"rgb": 0, "ycbcr": 1, "ipt": 2}
F32, F64 = 0, 1
KINDS = {0: "init", 1: "standard", 2: "pp"}

_vp, _i64, _int, _dbl = C.c_void_p, C.c_int64, C.c_int, C.c_double
_pi64 = C.POINTER(C.c_int64)
_pvp = C.POINTER(C.c_void_p)


class SolveCfg(C.Structure):
    _fields_ = [("max_sweeps", C.c_int), ("fit_tol", C.c_double), ("pp_enter_tol", C.c_double),
                ("pp_exit_tol", C.c_double), ("sequential_reduction", C.c_int)]


class Trace(C.Structure):
    _fields_ = [("capacity", C.c_int), ("n_records", C.c_int), ("converged", C.c_int),
                ("best_index", C.c_int), ("kind", C.POINTER(C.c_int)), ("fit", C.POINTER(C.c_double)),
                ("max_change", C.POINTER(C.c_double))]


SIGNATURES = {
    "tmb_version": ([], _int),
    "tmb_ctx_create": ([_int, _vp, C.POINTER(_vp)], _int),
    "tmb_ctx_destroy": ([_vp], _int),
    "tmb_ctx_set_stream": ([_vp, _vp], _int),
    "tmb_last_error": ([_vp], C.c_char_p),
    "tmb_launch_count": ([_vp], _i64),
    "tmb_workspace_size": ([_vp, C.POINTER(C.c_int64), C.POINTER(C.c_int64)], C.c_int),
    "tmb_workspace_reserve": ([_vp, C.c_int64], C.c_int),
    "tmb_timing": ([_vp, _int], _int),
    "tmb_timing_read": ([_vp, _int, _pi64, C.POINTER(_dbl), C.POINTER(_dbl)], _int),
    "tmb_color_u8": ([_vp, _vp, _i64, _i64, _i64, _int, _vp], _int),
    "tmb_color_f64": ([_vp, _vp, _i64, _int, _vp], _int),
    "tmb_color_inv_f64": ([_vp, _vp, _i64, _int, _vp, _pi64], _int),
    "tmb_decode_sse": ([_vp, _vp, _i64, _i64, _i64, _int, _vp, _vp, C.POINTER(_dbl)], _int),
    "tmb_color_u8_channels": ([_vp, _vp, _i64, _i64, _i64, _int, _vp], _int),
    "tmb_varint_encode": ([_vp, _vp, _i64, _vp, _i64, _pi64], _int),
    "tmb_varint_decode": ([_vp, _vp, _i64, _i64, _vp, _pi64], _int),
    "tmb_ttm": ([_vp, _vp, _int, _int, _pi64, _int, _vp, _i64, _vp], _int),
    "tmb_ttmc": ([_vp, _vp, _int, _int, _pi64, _pvp, _pi64, _pi64, _int, _int, _int, _vp], _int),
    "tmb_gram": ([_vp, _vp, _i64, _i64, _vp], _int),
    "tmb_pp_operators": ([_vp, _vp, _int, _int, _pi64, _pi64, _pvp, C.POINTER(_vp)], _int),
    "tmb_pp_info": ([_vp, C.POINTER(_int), C.POINTER(_int)], _int),
    "tmb_pp_operator": ([_vp, C.c_uint, C.POINTER(_vp), _pi64], _int),
    "tmb_pp_operator_copy": ([_vp, _vp, C.c_uint, _vp], _int),
    "tmb_pp_set_deltas": ([_vp, _vp, _pvp, _int, C.POINTER(_dbl)], _int),
    "tmb_pp_sweep": ([_vp, _vp, _vp, _pvp, _pvp], _int),
    "tmb_pp_destroy": ([_vp], _int),
    "tmb_mirror_upper": ([_vp, _vp, _i64], _int),
    "tmb_mode_gram": ([_vp, _vp, _int, _int, _pi64, _int, _vp], _int),
    "tmb_leading_eigvecs": ([_vp, _vp, _i64, _i64, _vp, _vp], _int),
    "tmb_tridiagonalize": ([_vp, _vp, _i64, _vp, _vp], _int),
    "tmb_sumsq": ([_vp, _vp, _int, _i64, C.POINTER(_dbl)], _int),
    "tmb_resid_sumsq": ([_vp, _vp, _int, _vp, _i64, C.POINTER(_dbl)], _int),
    "tmb_axpy": ([_vp, _i64, _dbl, _vp, _vp], _int),
    "tmb_t_hosvd": ([_vp, _vp, _int, _int, _pi64, _pi64, _int, _vp, _pvp], _int),
    "tmb_hooi_sweep": ([_vp, _vp, _int, _int, _pi64, _pi64, _pvp, _int, _vp, _pvp], _int),
    "tmb_reconstruct": ([_vp, _int, _pi64, _pi64, _vp, _pvp, _vp], _int),
    "tmb_tucker_als": ([_vp, _vp, _int, _int, _pi64, _pi64, C.POINTER(SolveCfg), _vp, _pvp, C.POINTER(Trace)], _int),
    "tmb_quantize_core": ([_vp, _vp, _i64, _int, _vp, C.POINTER(_dbl)], _int),
    "tmb_dequantize": ([_vp, _vp, _i64, _dbl, _vp], _int),
    "tmb_color_f64_channels": ([_vp, _vp, _i64, _i64, _i64, _int, _vp], _int),
    "tmb_channels_to_rgb": ([_vp, _vp, _i64, _i64, _i64, _int, _vp], _int),
    "tmb_solve_channels": ([_vp, _vp, _int, _pi64, _pi64, C.POINTER(SolveCfg), _pvp, _pvp, C.POINTER(Trace)], _int),
    "tmb_rc_bound": ([_i64, _pi64], _int),
    "tmb_rc_encode": ([_vp, _i64, _vp, _i64, _pi64], _int),
    "tmb_rc_decode": ([_vp, _i64, _i64, _vp], _int),
    "tmb_encode_stack_u8": ([_vp, _vp, _i64, _i64, _i64, _int, _pi64, C.POINTER(SolveCfg), _int, _vp, _vp, _pvp,
                             _vp, C.POINTER(_dbl), C.POINTER(Trace), C.POINTER(_dbl)], _int),
}
for _name, (_args, _res) in SIGNATURES.items():
    _fn = getattr(LIB, _name)
    _fn.argtypes = _args
    _fn.restype = _res

EXPORTS = tuple(SIGNATURES)


class TmbNumericError(RuntimeError):
    """Device eigen-solver / numeric failure (TMB_ENUMERIC)."""


_tls = threading.local()


def _torch():
    import torch  # deferred: plumbing only

    if not torch.cuda.is_available():
        raise RuntimeError("paper_2104_04726_b200 needs a CUDA device (B200); there is no CPU fallback")
    return torch


def ctx():
    """Per-thread, per-device libtmb context bound to torch's current stream."""
    torch = _torch()
    dev = torch.cuda.current_device()
    cache = getattr(_tls, "ctx", None)
    if cache is None:
        cache = _tls.ctx = {}
    h = cache.get(dev)
    if h is None:
        h = C.c_void_p()
        rc = LIB.tmb_ctx_create(dev, None, C.byref(h))
        if rc != TMB_OK:
            raise RuntimeError(f"tmb_ctx_create failed (code {rc}) on device {dev}")
        cache[dev] = h
    LIB.tmb_ctx_set_stream(h, C.c_void_p(torch.cuda.current_stream().cuda_stream))
    return h


def check(rc: int, h) -> None:
    if rc == TMB_OK:
        return
    msg = LIB.tmb_last_error(h).decode()
    if rc == TMB_EINVAL:
        raise ValueError(msg)
    if rc == TMB_ENOTIMPL:
        raise NotImplementedError(msg)
    if rc == TMB_ENUMERIC:
        raise TmbNumericError(msg)
    raise RuntimeError(f"libtmb error {rc}: {msg}")


def launch_count() -> int:
    return int(LIB.tmb_launch_count(ctx()))


# ---------------------------------------------------------------- device helpers
def dev_f64(a: np.ndarray):
    """Host array -> device float64 tensor holding its F-order (mode-0-fastest) bytes."""
    torch = _torch()
    flat = np.ascontiguousarray(np.asarray(a, dtype=np.float64).ravel(order="F"))
    return torch.from_numpy(flat).to("cuda", non_blocking=False)


def empty_f64(n: int):
    torch = _torch()
    return torch.empty(max(int(n), 1), dtype=torch.float64, device="cuda")


def host_f(t, shape) -> np.ndarray:
    """Device tensor (F-order data) -> host ndarray of the given shape."""
    n = int(np.prod(shape)) if len(shape) else 1
    flat = t[:n].cpu().numpy()
    return np.reshape(flat, shape, order="F")


def ptr(t) -> C.c_void_p:
    return C.c_void_p(t.data_ptr())


def ptrs(ts) -> C.Array:
    return (C.c_void_p * len(ts))(*[t.data_ptr() for t in ts])


def i64s(vals) -> C.Array:
    vals = [int(v) for v in vals]
    return (C.c_int64 * max(len(vals), 1))(*vals)
