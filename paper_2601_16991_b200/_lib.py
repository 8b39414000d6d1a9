"""ctypes binding of the C ABI in ``include/salr_b200.h`` (libsalr_b200.so).

The library is built in-tree (``_build.py``).  There is no fallback: if the
shared object or a CUDA device is missing, every compute entry point raises
:class:`SalrError` instead of silently computing elsewhere.
"""

from __future__ import annotations

import ctypes
import os
import threading

import torch

from .errors import (BoundsError, ConfigError, CorruptionError, DomainError, FormatError,
                     SalrError, ShapeError)

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libsalr_b200.so")
# A/B comparison of library builds (tools/ab*.sh) is a debug-build feature:
# the release package always loads its own in-tree library.
if os.environ.get("SALR_B200_DEBUG") == "1" and os.environ.get("SALR_B200_LIB_AB"):
    LIB_PATH = os.environ["SALR_B200_LIB_AB"]

_DEFAULT_LIB = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libsalr_b200.so")
F32, BF16, F64 = 0, 1, 2
TILE_K, TILE_N = 64, 128

_STATUS = {1: ShapeError, 2: DomainError, 3: BoundsError, 4: ConfigError, 5: FormatError,
           6: CorruptionError, 7: SalrError}

_i64, _vp, _int = ctypes.c_int64, ctypes.c_void_p, ctypes.c_int
_SIGS = {
    "salr_version": ([], _int),
    "salr_last_error": ([], ctypes.c_char_p),
    "salr_tb_geometry": ([_i64, _i64, ctypes.POINTER(_i64), ctypes.POINTER(_i64), ctypes.POINTER(_i64)], _int),
    "salr_encode_count": ([_vp, _int, _i64, _i64, _i64, _int, _vp, _vp, _vp], _int),
    "salr_encode_write": ([_vp, _int, _i64, _i64, _i64, _int, _vp, _vp, _vp, _vp], _int),
    "salr_decode": ([_vp, _vp, _int, _i64, _i64, _i64, _i64, _i64, _i64, _vp, _int, _i64, _vp], _int),
    "salr_tb_nnz": ([_vp, _vp, _i64, _vp, _vp], _int),
    "salr_to_reference": ([_vp, _vp, _int, _i64, _i64, _vp, _vp, _vp, _int, _vp], _int),
    "salr_from_reference_count": ([_vp, _i64, _i64, _int, _vp, _vp, _vp, _vp], _int),
    "salr_from_reference_write": ([_vp, _vp, _int, _i64, _i64, _int, _vp, _vp, _vp, _vp, _vp], _int),
    "salr_tb2_count": ([_vp, _vp, _i64, _i64, _vp, _vp], _int),
    "salr_tb2_write": ([_vp, _vp, _i64, _i64, _vp, _vp, _vp], _int),
    "salr_tb_from_tb2_count": ([_vp, _vp, _i64, _i64, _vp, _vp], _int),
    "salr_tb_from_tb2_write": ([_vp, _vp, _i64, _i64, _vp, _vp, _vp], _int),
    "salr_tb2_decode": ([_vp, _vp, _i64, _i64, _vp, _i64, _vp], _int),
    "salr_nm24_write": ([_vp, _i64, _i64, _i64, _vp, _vp, _vp], _int),
    "salr_nm24_decode": ([_vp, _i64, _i64, _vp, _i64, _vp], _int),
    "salr_linear_workspace_bytes": ([_i64, _i64, _i64, _i64, _int], ctypes.c_size_t),
    "salr_linear_workspace_zero_bytes": ([], ctypes.c_size_t),
    "salr_topk_mask_workspace_bytes": ([_i64], ctypes.c_size_t),
    "salr_topk_mask": ([_vp, _int, _i64, _i64, _vp, _vp, ctypes.c_size_t, _vp], _int),
    "salr_nm_mask": ([_vp, _int, _i64, _i64, _int, _int, _vp, _vp], _int),
    "salr_debug_set_trace": ([_vp], _int),
    "salr_debug_last_launch": ([_vp], _int),
    "salr_debug_set_probe": ([_vp, ctypes.c_size_t, _int, ctypes.c_uint32], _int),
    "salr_linear_forward": ([_vp, _i64, _i64, _i64, _vp, _vp, _i64, _i64, _vp, _vp, _i64, _vp, _int, _i64,
                             _vp, ctypes.c_size_t, _int, _int, _int, _vp], _int),
    "salr_chain_workspace_bytes": ([_i64, _int], ctypes.c_size_t),
    "salr_chain_workspace_zero_bytes": ([], ctypes.c_size_t),
    "salr_chain_forward": ([_vp, _int, _vp, _i64, _i64, _vp, ctypes.c_size_t, _int, _vp], _int),
}


class ChainLinear(ctypes.Structure):
    """salr_chain_linear_t (include/salr_b200.h)."""
    _fields_ = [("records", _vp), ("tile_off", _vp), ("max_record_bytes", _i64), ("K", _i64), ("N", _i64),
                ("acat", _vp), ("bcat_t", _vp), ("r_pad", _i64), ("y", _vp), ("ldy", _i64)]
EXPORTS = tuple(_SIGS)

_lock = threading.Lock()
_lib = None


def load() -> ctypes.CDLL:
    """Load (once) and type the shared library; raise loudly if absent."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise SalrError(f"CUDA extension not built: {LIB_PATH} missing "
                                "(run `python -m paper_2601_16991_b200._build`)")
            lib = ctypes.CDLL(LIB_PATH)
            for name, (args, res) in _SIGS.items():
                if LIB_PATH != _DEFAULT_LIB and not hasattr(lib, name):
                    continue  # an older build under A/B comparison
                fn = getattr(lib, name)
                fn.argtypes, fn.restype = args, res
            _lib = lib
    return _lib


def check(rc: int) -> None:
    if rc != 0:
        msg = load().salr_last_error().decode(errors="replace")
        raise _STATUS.get(rc, SalrError)(msg)


def require_cuda() -> torch.device:
    if not torch.cuda.is_available():
        raise SalrError("the SALR B200 path needs a CUDA device; there is no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def ptr(t) -> ctypes.c_void_p:
    return ctypes.c_void_p(0 if t is None else t.data_ptr())


def stream_ptr(stream=None) -> ctypes.c_void_p:
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def dtype_code(dt: torch.dtype) -> int:
    if dt == torch.float32:
        return F32
    if dt == torch.bfloat16:
        return BF16
    if dt == torch.float64:
        return F64
    raise DomainError(f"unsupported dtype {dt}")


def geometry(rows: int, cols: int):
    a, b, c = _i64(), _i64(), _i64()
    check(load().salr_tb_geometry(rows, cols, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c)))
    return a.value, b.value, c.value
