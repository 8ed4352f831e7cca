"""ctypes front-end of oracle/liboracle.so (plain C restatement of
reference simulator.py:239-341 + layout.py:347-456 + strategy.py:245-263).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_LIB = None

FIELDS = ("throughput", "tpot_s", "memory_bytes", "compute_s", "comm_s", "pipeline_s")


def build() -> Path:
    """Compile liboracle.so in place (gcc, -ffp-contract=off)."""
    subprocess.run(["make", "-s", "-C", str(_HERE)], check=True)
    return _HERE / "liboracle.so"


def lib():
    global _LIB
    if _LIB is None:
        path = _HERE / "liboracle.so"
        if not path.exists():
            build()
        _LIB = ctypes.CDLL(str(path))
        dp = ctypes.POINTER(ctypes.c_double)
        _LIB.or_simulate_batch.restype = ctypes.c_int
        _LIB.or_simulate_batch.argtypes = [
            ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p,
            dp, dp, dp, dp, dp, dp, ctypes.c_int,
        ]
        _LIB.or_gen_uniform.restype = ctypes.c_int
        _LIB.or_gen_uniform.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int64, ctypes.c_int64,
                                        ctypes.c_void_p, ctypes.c_int64, ctypes.c_int]
        _LIB.or_layer_plan.restype = ctypes.c_int
        _LIB.or_layer_plan.argtypes = [
            ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
            ctypes.c_void_p, ctypes.c_int,
        ]
    return _LIB


def _dptr(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def simulate_planes(desc, planes: np.ndarray, threads: int | None = None, fields=FIELDS, out: dict | None = None) -> dict:
    """Score [A, N] uint8 SoA planes; returns reason + the requested float fields
    (default all six). ``out`` may supply preallocated arrays."""
    planes = np.ascontiguousarray(planes, dtype=np.uint8)
    A, n = planes.shape
    if A != desc.vector_length:
        raise ValueError(f"planes have {A} heads, workload expects {desc.vector_length}")
    if out is None:
        out = {"reason": np.zeros(n, dtype=np.uint8)}
        for f in fields:
            out[f] = np.zeros(n, dtype=np.float64)
    if threads is None:
        threads = min(os.cpu_count() or 1, max(1, n // 4096))
    null = ctypes.POINTER(ctypes.c_double)()
    lib().or_simulate_batch(
        ctypes.byref(desc), planes.ctypes.data, n, n, out["reason"].ctypes.data,
        *(_dptr(out[f]) if f in out else null for f in FIELDS), int(threads),
    )
    return out


def uniform_planes(desc, seed: int, start: int, n: int, threads: int | None = None) -> np.ndarray:
    """Host twin of the device uniform stream (ls_generate LS_GEN_UNIFORM):
    positions [start, start + n) as [A, n] uint8 planes (oracle/streams.c)."""
    planes = np.empty((desc.vector_length, n), dtype=np.uint8)
    if threads is None:
        threads = min(os.cpu_count() or 1, max(1, n // 65536))
    if lib().or_gen_uniform(ctypes.byref(desc), int(seed) & (2**64 - 1), int(start), int(n), planes.ctypes.data,
                            max(n, 1), int(threads)) != 0:
        raise ValueError("uniform stream: vectors of up to 16 heads")
    return planes


def layer_plan(desc, vector) -> list[tuple[int, int, float, int]] | None:
    """Layer plan collectives (kind, group, payload, intra) or None on layout error."""
    vec = np.ascontiguousarray(np.asarray(vector, dtype=np.uint8))
    cap = 32
    kinds = np.zeros(cap, dtype=np.int32)
    groups = np.zeros(cap, dtype=np.int64)
    payloads = np.zeros(cap, dtype=np.float64)
    intra = np.zeros(cap, dtype=np.int32)
    n = lib().or_layer_plan(ctypes.byref(desc), vec.ctypes.data, kinds.ctypes.data, groups.ctypes.data,
                            payloads.ctypes.data, intra.ctypes.data, cap)
    if n < 0:
        return None
    return [(int(kinds[i]), int(groups[i]), float(payloads[i]), int(intra[i])) for i in range(n)]
