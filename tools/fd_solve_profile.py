"""One FD config-1 PGMRES solve (n=256, 4th-kind (4,0) half V-cycle) after warm-up
solves, between cudaProfilerStart/Stop, for ncu launch lists."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2210_03179_b200 import chebmg as cm  # noqa: E402

h = cm.build_hierarchy(cm.Domain(1.0, 1.0, 256), 2)
prob = cm.build_problem(h.domain, 1234)
M = cm.vcycle_preconditioner(h, cm.CycleConfig(cm.ChebyshevConfig(cm.Family.fourth, 1, h.lambda_tilde), 4, 0))
for _ in range(3):
    cm.pgmres(h.A, M, prob.b, None, cm.SolveOptions())
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.profiler.start()
e0.record()
_, rep = cm.pgmres(h.A, M, prob.b, None, cm.SolveOptions())
e1.record()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("iterations", rep.iterations, "solve ms", e0.elapsed_time(e1))
