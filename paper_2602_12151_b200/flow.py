"""oserve::flow::solve_assignment (flowassign.cpp:481-503) on the GPU path:
LCM normalisation (K0b) + greedy/exchange (K1) or branch-and-bound (K4),
batched over many raw tables in one launch."""
from __future__ import annotations

from typing import List, Optional, Sequence

import numpy as np

from . import core
from ._native import GpuContext

_ctx: Optional[GpuContext] = None


def _gpu(opts: Optional[core.SolveOptions]) -> GpuContext:
    global _ctx
    if _ctx is None:
        _ctx = GpuContext(core.cluster(1, 1), core.ModelSpec("none", 1, 1, 1, 1, 1))
    _ctx.set_solve_options(opts or core.SolveOptions())
    return _ctx


def solve_assignment(table: core.CapacityTable, lam: Sequence[int],
                     opts: Optional[core.SolveOptions] = None) -> core.LowerLevel:
    if len(lam) != table.types():
        raise ValueError("solve_assignment: lambda size mismatch")
    return solve_assignment_batch([table.n], [table.e], [list(lam)], opts)[0]


def solve_assignment_batch(n: Sequence, e: Sequence, lam: Sequence,
                           opts: Optional[core.SolveOptions] = None) -> List[core.LowerLevel]:
    """Many independent instances of equal shape [count][R][J]."""
    x, obj, M, unit, used = _gpu(opts).solve_batch(np.asarray(n), np.asarray(e), np.asarray(lam))
    return [core.LowerLevel(core.AssignmentMatrix(x[i].tolist(), int(obj[i])), M[i].tolist(), unit[i].tolist(),
                            used[i].tolist()) for i in range(len(obj))]
