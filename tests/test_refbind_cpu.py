"""The reference-side binding without a GPU: refbind builds a subclass of the
reference's own SearchEnv (baseline/_ref) that keeps the reference's step /
reward / budget code, and constructing it without a CUDA device fails loudly
(NativeUnavailable) — there is no CPU fallback behind the seam."""

import sys
from pathlib import Path

import pytest

REF = Path(__file__).resolve().parent.parent / "baseline" / "_ref"
pytestmark = pytest.mark.skipif(not (REF / "shardsearch").exists(), reason="reference not installed in baseline/_ref")


def _ref():
    if str(REF) not in sys.path:
        sys.path.insert(0, str(REF))
    import shardsearch

    return shardsearch


def test_subclass_keeps_the_reference_protocol():
    shardsearch = _ref()
    from shardsearch.env import SearchEnv

    from paper_2509_00217_b200.refbind import gpu_search_env

    cls = gpu_search_env(shardsearch)
    assert issubclass(cls, SearchEnv) and cls.__name__ == "GpuSearchEnv"
    for name in ("step", "final_selection", "close", "budget_left"):
        assert getattr(cls, name) is getattr(SearchEnv, name)  # only the seam is replaced
    assert cls.evaluate_raw is not SearchEnv.evaluate_raw


def test_no_cpu_fallback():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    shardsearch = _ref()
    from shardsearch.config import load_config, packaged_config_path

    from paper_2509_00217_b200.evaluator import NativeUnavailable
    from paper_2509_00217_b200.refbind import gpu_search_env

    cfg = load_config(packaged_config_path("tiny"))
    with pytest.raises(NativeUnavailable):
        gpu_search_env(shardsearch)(model=cfg.model, hw=cfg.hardware, space=cfg.space,
                                    context_len=cfg.simulation.context_len, budget=3,
                                    slo_tpot=cfg.simulation.slo_tpot)
