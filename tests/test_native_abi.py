"""The drop-in boundary: libls_eval.so loads and exports every symbol
include/ls_eval.h declares (no compute calls: runs without a GPU)."""

import ctypes
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


def declared_symbols():
    text = (ROOT / "include" / "ls_eval.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:const char\*|int|uint32_t|uint64_t|size_t)\s+(ls_\w+)\(", text, re.M)))


def test_header_declares_the_abi():
    names = declared_symbols()
    for required in ("ls_ctx_create", "ls_ctx_destroy", "ls_evaluate", "ls_evaluate_host", "ls_reward_scan",
                     "ls_topk", "ls_topk_merge", "ls_last_error"):
        assert required in names


def test_library_exports_every_declared_symbol():
    from paper_2509_00217_b200 import _native

    path = _native.lib_path()
    if not path.exists():
        pytest.fail(f"{path} not built: run __graft_entry__.build()")
    handle = ctypes.CDLL(str(path))
    missing = [n for n in declared_symbols() if not hasattr(handle, n)]
    assert not missing, missing
    assert set(declared_symbols()) <= set(_native.EXPORTED_SYMBOLS)


def test_abi_version_and_struct_layout():
    from paper_2509_00217_b200 import _native
    from paper_2509_00217_b200.workload import WorkloadDesc

    lib = _native.lib()
    assert lib.ls_abi_version() == 1
    # ls_workload_desc layout: 2 u32 + 10 i64 + 2 i32 + 5 f64 + 2 i64 + 2 f64 + i64 + f64
    #                          + 4 i32 + 4*64 i64 + i32 + 24 i8 (+ padding)
    assert ctypes.sizeof(WorkloadDesc) == 8 + 80 + 8 + 40 + 16 + 16 + 16 + 16 + 2048 + 4 + 24 + 4
    assert ctypes.sizeof(_native.EliteRec) == 32


def test_ctx_create_without_gpu_fails_cleanly():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2509_00217_b200 import _native
    from paper_2509_00217_b200.evaluator import Evaluator, NativeUnavailable
    from golden_io import load_eval

    wl, _, _ = load_eval("tiny")
    with pytest.raises(NativeUnavailable):
        Evaluator(wl)
