"""ctypes binding of libls_eval.so (include/ls_eval.h).

The library is built in-tree by ``__graft_entry__.build()`` /
``make -C paper_2509_00217_b200/csrc``. There is no fallback: if the library
or a CUDA device is missing, every evaluator entry point raises
``NativeUnavailable``.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

from .workload import WorkloadDesc

__all__ = ["NativeUnavailable", "NativeError", "lib", "lib_path", "ResultSoA", "EliteRec", "check",
           "LS_OK", "REASON_DECODE_ERROR", "KEY_RAW", "KEY_REWARD"]

LS_OK = 0
REASON_DECODE_ERROR = 255
KEY_RAW = 0
KEY_REWARD = 1

_PKG = Path(__file__).resolve().parent


def lib_path() -> Path:
    return Path(os.environ.get("LS_EVAL_LIB", str(_PKG / "libls_eval.so")))


class NativeUnavailable(RuntimeError):
    """The CUDA evaluator library (or a GPU) is not available; there is no CPU fallback."""


class NativeError(RuntimeError):
    """A libls_eval.so call returned a non-zero status."""

    def __init__(self, status: int, message: str):
        super().__init__(f"libls_eval status {status}: {message}")
        self.status = status


class ResultSoA(ctypes.Structure):
    _fields_ = [
        ("reason", ctypes.c_void_p),
        ("throughput", ctypes.c_void_p),
        ("tpot_s", ctypes.c_void_p),
        ("memory_bytes", ctypes.c_void_p),
        ("compute_s", ctypes.c_void_p),
        ("comm_s", ctypes.c_void_p),
        ("pipeline_s", ctypes.c_void_p),
    ]


class SearchState(ctypes.Structure):
    """ls_search_state: device-resident environment + elite + eval-log state."""

    _fields_ = [
        ("best_raw", ctypes.c_void_p),
        ("elite_vec", ctypes.c_void_p),
        ("elite_reward", ctypes.c_void_p),
        ("elite_capacity", ctypes.c_int32),
        ("log_pos", ctypes.c_void_p),
        ("log_capacity", ctypes.c_int64),
        ("log_vec", ctypes.c_void_p),
        ("log_raw", ctypes.c_void_p),
        ("log_reward", ctypes.c_void_p),
        ("log_reason", ctypes.c_void_p),
        ("alpha", ctypes.c_double),
        ("beta", ctypes.c_double),
        ("penalty", ctypes.c_double),
    ]


class EliteRec(ctypes.Structure):
    _fields_ = [
        ("key", ctypes.c_double),
        ("raw", ctypes.c_double),
        ("index", ctypes.c_int64),
        ("code", ctypes.c_uint64),
    ]


_LIB = None

_SIGS = {
    "ls_last_error": (ctypes.c_char_p, []),
    "ls_abi_version": (ctypes.c_uint32, []),
    "ls_ctx_create": (ctypes.c_int, [ctypes.POINTER(WorkloadDesc), ctypes.c_int, ctypes.POINTER(ctypes.c_void_p)]),
    "ls_ctx_destroy": (ctypes.c_int, [ctypes.c_void_p]),
    "ls_space_size": (ctypes.c_uint64, [ctypes.c_void_p]),
    "ls_evaluate": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
                                   ctypes.POINTER(ResultSoA), ctypes.c_void_p]),
    "ls_evaluate_host": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
                                        ctypes.POINTER(ResultSoA)]),
    "ls_host_alloc": (ctypes.c_int, [ctypes.c_size_t, ctypes.POINTER(ctypes.c_void_p)]),
    "ls_host_free": (ctypes.c_int, [ctypes.c_void_p]),
    "ls_scan_scratch_bytes": (ctypes.c_size_t, [ctypes.c_int64]),
    "ls_reward_scan": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                                      ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                      ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]),
    "ls_topk_scratch_bytes": (ctypes.c_size_t, [ctypes.c_int64, ctypes.c_int]),
    "ls_topk": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
                               ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_int64,
                               ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]),
    "ls_evaluate_topk_scratch_bytes": (ctypes.c_size_t, [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int]),
    "ls_evaluate_topk": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
                                        ctypes.POINTER(ResultSoA), ctypes.c_int, ctypes.c_int64, ctypes.c_void_p,
                                        ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]),
    "ls_stream_size": (ctypes.c_uint64, [ctypes.c_void_p, ctypes.c_int]),
    "ls_generate": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_uint64, ctypes.c_int64, ctypes.c_int64,
                                   ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p]),
    "ls_sweep": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_uint64, ctypes.c_int64, ctypes.c_int64,
                                ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]),
    "ls_topk_merge": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                     ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]),
    "ls_env_step": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(SearchState), ctypes.c_void_p, ctypes.c_void_p,
                                   ctypes.c_void_p]),
}

EXPORTED_SYMBOLS = tuple(_SIGS)


def lib(require_gpu: bool = False):
    """Load libls_eval.so once; raise NativeUnavailable if it cannot be loaded."""
    global _LIB
    if _LIB is None:
        path = lib_path()
        if not path.exists():
            raise NativeUnavailable(
                f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
            )
        try:
            handle = ctypes.CDLL(str(path))
        except OSError as err:
            raise NativeUnavailable(f"cannot load {path}: {err}") from err
        for name, (res, args) in _SIGS.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _LIB = handle
    if require_gpu:
        import torch

        if not torch.cuda.is_available():
            raise NativeUnavailable("no CUDA device: the evaluator has no CPU fallback")
    return _LIB


def check(status: int) -> None:
    if status != LS_OK:
        msg = _LIB.ls_last_error().decode("utf-8", "replace") if _LIB is not None else ""
        raise NativeError(status, msg)
