"""Load the golden fixtures of tests/golden/ (made by make_golden.py from the
reference itself) into this package's spec objects."""

from __future__ import annotations

import json
from pathlib import Path

import numpy as np

from paper_2509_00217_b200.spec import HardwareSpec, ModelSpec
from paper_2509_00217_b200.strategy import ActionSpaceSpec, AxisChoice
from paper_2509_00217_b200.workload import Workload

GOLDEN = Path(__file__).resolve().parent / "golden"
FIELDS = ("throughput", "tpot_s", "memory_bytes", "compute_s", "comm_s", "pipeline_s")


def eval_sets():
    return sorted(p.stem[len("eval_"):] for p in GOLDEN.glob("eval_*.npz"))


def search_sets():
    return sorted(p.stem[len("search_"):] for p in GOLDEN.glob("search_*.npz"))


def workload_from_meta(meta) -> Workload:
    sp = meta["space"]
    space = ActionSpaceSpec(
        tp_domain=tuple(sp["tp_domain"]), ep_domain=tuple(sp["ep_domain"]), pp_domain=tuple(sp["pp_domain"]),
        batch_domain=tuple(sp["batch_domain"]), op_names=tuple(sp["op_names"]),
        pinned=tuple((n, AxisChoice(a)) for n, a in sp["pinned"]),
    )
    return Workload(ModelSpec(**meta["model"]), HardwareSpec(**meta["hw"]), space, meta["context_len"],
                    meta["slo_tpot"], meta.get("sum_mode"))


def load_eval(name):
    z = np.load(GOLDEN / f"eval_{name}.npz")
    meta = json.loads(str(z["meta"]))
    data = {k: z[k] for k in z.files if k != "meta"}
    return workload_from_meta(meta), meta, data


def load_search(name):
    z = np.load(GOLDEN / f"search_{name}.npz")
    meta = json.loads(str(z["meta"]))
    data = {k: z[k] for k in z.files if k != "meta"}
    return workload_from_meta(meta), meta, data


def mismatches(got: dict, want: dict) -> np.ndarray:
    """Boolean mask of candidates whose reason or any float64 BIT PATTERN differs."""
    bad = np.asarray(got["reason"]) != np.asarray(want["reason"])
    for f in FIELDS:
        if f in got:
            bad |= np.asarray(got[f], dtype=np.float64).view(np.uint64) != np.asarray(want[f]).view(np.uint64)
    return bad
