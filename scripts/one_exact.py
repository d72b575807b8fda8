import sys; sys.path.insert(0,'.')
from paper_2602_12151_b200 import workloads
from paper_2602_12151_b200._native import GpuContext
w = workloads.load('cfg1_bnb')
g = GpuContext(w.cluster, w.model, w.params); g.set_workload(w.types, w.lam, w.span_s)
g.exhaustive()
