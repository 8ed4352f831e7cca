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
           "LS_OK", "LS_ERR_UNSUPPORTED", "REASON_DECODE_ERROR", "KEY_RAW", "KEY_REWARD"]

LS_OK = 0
LS_ERR_UNSUPPORTED = 4
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


PSEG_COUNT = 20


class PolicyDims(ctypes.Structure):
    _fields_ = [("obs_dim", ctypes.c_int32), ("width", ctypes.c_int32), ("ffn_width", ctypes.c_int32),
                ("history_len", ctypes.c_int32), ("num_heads", ctypes.c_int32), ("kmax", ctypes.c_int32),
                ("n_steps", ctypes.c_int32)]


class PolicyLayout(ctypes.Structure):
    _fields_ = [("off", ctypes.c_int64 * PSEG_COUNT), ("total", ctypes.c_int64)]


class PpoPlan(ctypes.Structure):
    """ls_ppo_plan: every pointer is device memory."""

    _fields_ = [("dims", PolicyDims)] + [(n, ctypes.c_void_p) for n in (
        "params", "adam_m", "adam_v", "grad_out", "workspace", "blocked", "head_size", "obs_denom")] + [
        ("env", SearchState)] + [(n, ctypes.c_void_p) for n in (
            "uniforms", "lr_table", "spent", "adam_step", "status", "batch_obs", "batch_action", "batch_logp",
            "batch_value", "batch_reward")] + [(n, ctypes.c_double) for n in (
                "tau", "clip_eps", "value_coef", "entropy_coef", "beta1", "beta2", "adam_eps")] + [
        ("epochs", ctypes.c_int32)]


class SaPlan(ctypes.Structure):
    """ls_sa_plan: one simulated-annealing chain on the device."""

    _fields_ = [("steps", ctypes.c_int32), ("moves", ctypes.c_int32)] + [
        (n, ctypes.c_void_p) for n in ("init", "coords", "drawn", "u", "temperature")] + [("env", SearchState)]


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
    "ls_evaluate_host_compact": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_int64,
                                                ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                                                ctypes.POINTER(ctypes.c_int64)]),
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
    "ls_set_precision": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int]),
    "ls_reserve_sms": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int]),
    "ls_stream_size": (ctypes.c_uint64, [ctypes.c_void_p, ctypes.c_int]),
    "ls_generate": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_uint64, ctypes.c_int64, ctypes.c_int64,
                                   ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p]),
    "ls_sweep": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_uint64, ctypes.c_int64, ctypes.c_int64,
                                ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]),
    "ls_topk_merge": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                     ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]),
    "ls_topk_merge_steps": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
                                           ctypes.c_void_p, ctypes.c_void_p]),
    "ls_packed_layout": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int64)]),
    "ls_pack": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p,
                               ctypes.c_void_p]),
    "ls_evaluate_packed": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.POINTER(ResultSoA),
                                          ctypes.c_void_p]),
    "ls_evaluate_host_packed": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                                               ctypes.POINTER(ResultSoA)]),
    "ls_evaluate_packed_topk": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                                               ctypes.POINTER(ResultSoA), ctypes.c_int, ctypes.c_int64, ctypes.c_void_p,
                                               ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]),
    "ls_evaluate_packed_topk_signal": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                                                      ctypes.POINTER(ResultSoA), ctypes.c_int, ctypes.c_int64,
                                                      ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                                      ctypes.c_void_p, ctypes.c_uint32, ctypes.c_void_p]),
    "ls_stream_wait_signal": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint32]),
    "ls_evaluate_packed_topk_sinks": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                                                     ctypes.POINTER(ResultSoA), ctypes.c_int, ctypes.c_int64,
                                                     ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                                     ctypes.c_void_p, ctypes.c_int, ctypes.c_uint32, ctypes.c_void_p]),
    "ls_topk_merge_steps_wait": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                                ctypes.c_uint32, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                                ctypes.c_void_p]),
    "ls_ipc_alloc": (ctypes.c_int, [ctypes.c_size_t, ctypes.POINTER(ctypes.c_void_p)]),
    "ls_ipc_free": (ctypes.c_int, [ctypes.c_void_p]),
    "ls_ipc_handle": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p]),
    "ls_ipc_open": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(ctypes.c_void_p)]),
    "ls_ipc_close": (ctypes.c_int, [ctypes.c_void_p]),
    "ls_env_step": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(SearchState), ctypes.c_void_p, ctypes.c_void_p,
                                   ctypes.c_void_p]),
    "ls_evaluate_one": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_char_p, ctypes.c_void_p, ctypes.c_void_p]),
    "ls_sa_chain": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(SaPlan), ctypes.c_void_p]),
    "ls_policy_layout_of": (ctypes.c_int, [ctypes.POINTER(PolicyDims), ctypes.POINTER(PolicyLayout)]),
    "ls_ppo_workspace_bytes": (ctypes.c_size_t, [ctypes.POINTER(PolicyDims)]),
    "ls_ppo_prime": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(PpoPlan), ctypes.c_void_p]),
    "ls_ppo_round": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(PpoPlan), ctypes.c_int, ctypes.c_void_p]),
    "ls_ppo_forward": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(PpoPlan), ctypes.c_int, ctypes.c_void_p,
                                      ctypes.c_void_p, ctypes.c_void_p]),
    "ls_ppo_update": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(PpoPlan), ctypes.c_int, ctypes.c_void_p]),
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
        tolerant = "LS_EVAL_LIB" in os.environ  # A/B builds of other revisions may lack newer entry points
        for name, (res, args) in _SIGS.items():
            if tolerant and not hasattr(handle, name):
                continue
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
