"""The reference-side binding: the reference's own ``SearchEnv`` with its
scoring seam routed through libls_eval.so.

A maintainer of the reference (``shardsearch``) adopts the GPU evaluator by
subclassing its ``SearchEnv`` and overriding ``evaluate_raw`` — the seam the
reference's ``step`` calls (pkg/src/shardsearch/env.py:140-158) and the one
its own tests stub per instance (pkg/tests/test_acceptance.py:430-463).
``gpu_search_env(shardsearch)`` builds that subclass from the reference
package object, so this module does not import the reference itself::

    import shardsearch
    from paper_2509_00217_b200.refbind import gpu_search_env

    GpuSearchEnv = gpu_search_env(shardsearch)
    env = GpuSearchEnv(model=cfg.model, hw=cfg.hardware, space=cfg.space,
                       context_len=cfg.simulation.context_len, budget=4000,
                       slo_tpot=cfg.simulation.slo_tpot)

Everything else (reward shaping, budget, eval log, ``final_selection``, the
reference's PPO / RW / SA drivers) is the reference's code, unchanged. The
verdicts come from ``ls_evaluate_one`` and are bit-identical to the
reference's ``simulate``; ``SimResult.detail`` is produced on the host.
"""

from __future__ import annotations

from .evaluator import Evaluator
from .simulator import SimRequest, result_from_verdict, simulate
from .workload import Workload

__all__ = ["gpu_search_env"]


def gpu_search_env(shardsearch):
    """Subclass of ``shardsearch.env.SearchEnv`` whose ``evaluate_raw`` runs on the GPU."""
    import importlib

    ref_env = importlib.import_module(shardsearch.__name__ + ".env")
    ref_sim = importlib.import_module(shardsearch.__name__ + ".simulator")
    ref_strategy = importlib.import_module(shardsearch.__name__ + ".strategy")

    class GpuSearchEnv(ref_env.SearchEnv):
        def __init__(self, *args, device=None, **kwargs):
            super().__init__(*args, **kwargs)
            # the reference's spec objects are read by field name
            self._gpu = Evaluator(Workload(self.model, self.hw, self.space, self.context_len, self.slo_tpot),
                                  device)

        def evaluate_raw(self, strategy):  # env.py:140-150
            try:
                vector = ref_strategy.encode_strategy(strategy, self.space)
            except ValueError:  # degrees outside the space's domains: the free-standing facade
                ours = simulate(SimRequest(self.model, self.hw, strategy, self.context_len, self.slo_tpot))
            else:
                code, fields = self._gpu.evaluate_one(vector)
                ours = result_from_verdict(code, fields, self.model, self.hw, strategy, self.slo_tpot)
            return ref_sim.SimResult(
                valid=ours.valid,
                invalid_reason=ref_sim.InvalidReason(ours.invalid_reason.value),
                throughput=ours.throughput,
                tpot_s=ours.tpot_s,
                memory_bytes=ours.memory_bytes,
                breakdown=ref_sim.TimeBreakdown(ours.breakdown.compute_s, ours.breakdown.comm_s,
                                                ours.breakdown.pipeline_s),
                detail=ours.detail,
            )

    GpuSearchEnv.__qualname__ = GpuSearchEnv.__name__ = "GpuSearchEnv"
    return GpuSearchEnv
