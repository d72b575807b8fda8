"""B200-native OServe scheduling round (arxiv 2602.12151).

enumerate -> cost -> assign -> argmin -> switching cost, as sm_100a kernels
behind the C-ABI in include/oserve_gpu.h.  Python modules mirror the
reference's C++ namespaces: core (L0 types), cost, flow, search, switchplan,
orchestrate (the per-window loop of config 4).
"""
from . import core  # noqa: F401

__all__ = ["core", "cost", "flow", "search", "switchplan", "orchestrate", "workloads"]
