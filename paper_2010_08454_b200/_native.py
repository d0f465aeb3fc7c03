"""ctypes binding of libcuppl_gpu.so (the C ABI in include/cuppl_gpu.h).

There is no fallback: if the library is missing or fails to load, every entry point raises
NativeLibraryError. Device buffers are torch CUDA tensors passed by data_ptr(); the stream
is torch's current CUDA stream.
"""

from __future__ import annotations

import ctypes as C
import threading
from pathlib import Path

from . import errors

LIB_PATH = Path(__file__).resolve().parent / "_lib" / "libcuppl_gpu.so"
ABI_VERSION = 1

OK, E_INVALID_PARAM, E_ALL_ZERO, E_CUDA, E_NCCL, E_CAPACITY, E_UNSUPPORTED, E_ARGUMENT = range(8)

TAG_IS, TAG_SMC_INIT, TAG_SMC_STEP, TAG_SMC_COMB, TAG_MH, TAG_MH_INIT, TAG_DIST = range(1, 8)

REC_STATS = 16
REC_BINS = 8


class IsRecord(C.Structure):
    """cuppl_is_record (include/cuppl_gpu.h)."""

    _fields_ = [
        ("max_lw", C.c_double),
        ("sum_w", C.c_double),
        ("sum_w2", C.c_double),
        ("argmax_lw", C.c_double),
        ("argmax_pid", C.c_uint64),
        ("n_finite", C.c_uint64),
        ("n_total", C.c_uint64),
        ("reserved", C.c_uint64),
        ("stat_w", C.c_double * REC_STATS),
        ("bin_w", C.c_double * REC_BINS),
    ]


REC_BYTES = C.sizeof(IsRecord)
assert REC_BYTES == 256


class Dist(C.Structure):
    """cuppl_dist (include/cuppl_gpu.h)."""

    _fields_ = [
        ("tag", C.c_int32),
        ("n_table", C.c_int32),
        ("p0", C.c_double),
        ("p1", C.c_double),
        ("p2", C.c_double),
        ("table", C.c_void_p),
    ]


class SmcModel(C.Structure):
    """cuppl_smc_model (include/cuppl_gpu.h)."""

    _fields_ = [
        ("n_states", C.c_int32),
        ("inv_sd", C.c_float),
        ("c", C.c_float),
        ("reserved", C.c_int32),
        ("alias_trans", C.c_void_p),
        ("alias_init", C.c_void_p),
        ("mu", C.c_void_p),
        ("key_dev", C.c_void_p),
    ]


class ResampleStats(C.Structure):
    """cuppl_resample_stats (include/cuppl_gpu.h)."""

    _fields_ = [("max_lw", C.c_double), ("total", C.c_uint64), ("sum_e", C.c_double), ("sum_e2", C.c_double)]


_lock = threading.Lock()
_lib: C.CDLL | None = None

_P = C.c_void_p
_U64 = C.c_uint64
_U32 = C.c_uint32
_I32 = C.c_int32
_F32 = C.c_float
_SIG = {
    "cuppl_abi_version": ([], C.c_int),
    "cuppl_last_error": ([], C.c_char_p),
    "cuppl_device_info": ([_P, _P, _P], C.c_int),
    "cuppl_philox_blocks": ([_U64, _U64, _U32, _U32, _U64, _P, _P], C.c_int),
    "cuppl_dist_sample": ([_P, _U64, _U32, _U64, _U64, _P, _P], C.c_int),
    "cuppl_dist_score": ([_P, _P, _U64, _P, _P], C.c_int),
    "cuppl_is_workspace_bytes": ([], C.c_size_t),
    "cuppl_is_workspace_bytes_n": ([C.c_int], C.c_size_t),
    "cuppl_is_poly": ([_P, _P, C.c_int, _U64, _U64, _U64, _P, _P, _P, _P, _P, _P, C.c_size_t, _P], C.c_int),
    "cuppl_is_linreg": ([_P, _P, C.c_int, _F32, _U64, _U64, _U64, _P, _P, _P, _P, _P, C.c_size_t, _P], C.c_int),
    "cuppl_is_record_merge": ([_P, C.c_int, _P], C.c_int),
    "cuppl_normalize_workspace_bytes": ([], C.c_size_t),
    "cuppl_normalize_f64": ([_P, _P, _U64, C.c_int, _P, _P, _P, _P, C.c_size_t, _P], C.c_int),
    "cuppl_normalize_f32": ([_P, _P, _U64, C.c_int, _P, _P, _P, _P, C.c_size_t, _P], C.c_int),
    "cuppl_mh_padded_points": ([C.c_int], C.c_int),
    "cuppl_mh_gmm": ([_P, C.c_int, C.c_int, _F32, _F32, _U32, _U32, _U32, _U32, _U32, _U64, _P, _P, _P, _P,
                      _U32, _P], C.c_int),
    "cuppl_arena_alloc": ([C.c_size_t, _P], C.c_int),
    "cuppl_arena_free": ([_P], C.c_int),
    "cuppl_ipc_handle": ([_P, _P], C.c_int),
    "cuppl_ipc_open": ([_P, _P], C.c_int),
    "cuppl_ipc_close": ([_P], C.c_int),
    "cuppl_calibrate": ([C.c_int, C.c_int, C.c_int, _P, _P], C.c_int),
    "cuppl_smc_workspace_bytes": ([_U64], C.c_size_t),
    "cuppl_smc_init": ([_P, _U64, _U64, _U64, _F32, _P, _P, _P, C.c_size_t, _P], C.c_int),
    "cuppl_smc_scan": ([_P, _U64, _F32, _P, _P, _P, _P, _P, C.c_size_t, _P], C.c_int),
    "cuppl_smc_log_weights": ([_P, _F32, _P, _U64, _P, _P], C.c_int),
    "cuppl_smc_fold": ([_U64, _P, _P, C.c_size_t, _P], C.c_int),
    "cuppl_smc_resample": ([_P, _U64, _U64, _U64, _U32, C.c_int, C.c_int, _F32, _F32, _P, _P, _P, _P,
                            _P, _P, _P, _P, _P, C.c_size_t, _P], C.c_int),
    "cuppl_resample_workspace_bytes": ([_U64], C.c_size_t),
    "cuppl_peer_exchange": ([_P, _U32, _P, _U64, _U64, C.c_int, C.c_int, _P, _P, _P, _P, _U64, _P], C.c_int),
    "cuppl_resample": ([_P, _U64, _P, _U64, _U64, _U32, _P, _P, _P, _P, C.c_size_t, _P], C.c_int),
}


def signatures() -> dict:
    return dict(_SIG)


def lib() -> C.CDLL:
    """Load libcuppl_gpu.so (once). Raises NativeLibraryError if it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not LIB_PATH.exists():
            raise errors.NativeLibraryError(
                f"{LIB_PATH} is not built (python -m paper_2010_08454_b200.build); "
                "there is no CPU fallback")
        try:
            L = C.CDLL(str(LIB_PATH))
        except OSError as e:  # pragma: no cover
            raise errors.NativeLibraryError(f"cannot load {LIB_PATH}: {e}") from e
        for name, (args, res) in _SIG.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = res
        if L.cuppl_abi_version() != ABI_VERSION:
            raise errors.NativeLibraryError("ABI version mismatch")
        _lib = L
        return L


def last_error() -> str:
    msg = lib().cuppl_last_error()
    return msg.decode() if msg else ""


def check(rc: int, what: str = "", seed=None, step=None) -> None:
    """Map a cuppl_status onto the reference exception classes."""
    if rc == OK:
        return
    msg = f"{what}: {last_error()}" if what else last_error()
    if rc == E_INVALID_PARAM:
        raise errors.InvalidDistParamError(msg)
    if rc == E_ALL_ZERO:
        raise errors.AllZeroWeightError(msg)
    if rc == E_UNSUPPORTED:
        raise errors.UnsupportedDistError(msg)
    if rc in (E_CUDA, E_NCCL):
        raise errors.InferRuntimeError(msg, cause=errors.NativeLibraryError(msg), seed=seed, step=step)
    raise errors.InferRuntimeError(msg, seed=seed, step=step)


def stream_ptr(device=None) -> int:
    import torch

    return torch.cuda.current_stream(device).cuda_stream


def ptr(t) -> int | None:
    """data_ptr of a CUDA tensor (None passes NULL)."""
    if t is None:
        return None
    if not t.is_cuda:
        raise errors.NativeLibraryError("expected a CUDA tensor")
    return t.data_ptr()
