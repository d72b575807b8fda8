"""The exact (branch-and-bound) path on the device at its abort boundary:
for each instance the reference's node count N is known, and the reference's
own result at budgets N-1 (aborts -> heuristic fallthrough), N (exact) and
N/2 must be reproduced (tests/golden/exact_budget.json).  Exercises the
frontier-parallel node accounting (k_exact_plan / k_exact_task)."""
import json
import os

import numpy as np
import pytest

from paper_2602_12151_b200 import core
from paper_2602_12151_b200._native import GpuContext

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CASES = json.load(open(os.path.join(ROOT, "tests", "golden", "exact_budget.json")))
# values that need the 64-bit DFS table: row LCMs past 2^30, demands past 2^20
WIDE = json.load(open(os.path.join(ROOT, "tests", "golden", "exact_budget_wide.json")))


@pytest.fixture(scope="module")
def gctx(cuda):
    return GpuContext(core.cluster(1, 1), core.ModelSpec("none", 1, 1, 1, 1, 1))


@pytest.mark.parametrize("which", [0, 1, 2])
def test_exact_budget_boundary(gctx, which):
    for c in CASES:
        b = c["budgets"][which]
        gctx.set_solve_options(core.SolveOptions(400, 20, b["budget"]))
        x, obj, *_ = gctx.solve_batch(np.asarray([c["n"]]), np.asarray([c["e"]]), np.asarray([c["lambda"]]))
        assert int(obj[0]) == b["objective"] and x[0].tolist() == b["x"], (c["nodes"], b["budget"])
    gctx.set_solve_options(core.SolveOptions())


def test_exact_batch_default_budget(gctx):
    """All instances in one launch at the default budget."""
    by_shape = {}
    for c in CASES:
        by_shape.setdefault((len(c["n"]), len(c["lambda"])), []).append(c)
    for cs in by_shape.values():
        gctx.set_solve_options(core.SolveOptions())
        x, obj, *_ = gctx.solve_batch(np.asarray([c["n"] for c in cs]), np.asarray([c["e"] for c in cs]),
                                      np.asarray([c["lambda"] for c in cs]))
        for i, c in enumerate(cs):
            ref = c["budgets"][1] if c["nodes"] <= 8_000_000 else None
            if ref is not None:
                assert int(obj[i]) == ref["objective"] and x[i].tolist() == ref["x"]


@pytest.mark.parametrize("which", [0, 1, 2])
def test_exact_budget_boundary_wide_values(gctx, which):
    for c in WIDE:
        b = c["budgets"][which]
        gctx.set_solve_options(core.SolveOptions(c["demand_limit"], 20, b["budget"]))
        x, obj, *_ = gctx.solve_batch(np.asarray([c["n"]]), np.asarray([c["e"]]), np.asarray([c["lambda"]]))
        assert int(obj[0]) == b["objective"] and x[0].tolist() == b["x"], (c["nodes"], b["budget"])
    gctx.set_solve_options(core.SolveOptions())
