import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import oracle_bind as ob
from paper_2210_03179_b200 import chebmg as cm, sem
np.set_printoptions(linewidth=220, precision=3)
eps = 0.3
P = sem.PMGHierarchy(sem.SemDesc(7, 3, 3, 3, geometry=1, eps=eps), (7, 3, 1))
o = ob.OraclePmg((7, 3, 1), 3, 3, 3, 1, eps)
b = o.sem(0).rhs()
for kp, kq in [(2, 2), (4, 0)]:
    cyc = cm.CycleConfig(cm.ChebyshevConfig(cm.Family.fourth, 1, P.lambda_tilde[0]), kp, kq)
    z = P.A.to_canonical(P.preconditioner_apply(cyc, P.A.from_canonical(b)))
    zo = o.v_cycle(2, kp, kq, b)
    print(kp, kq, "vcycle rel", np.max(np.abs(z - zo)) / np.max(np.abs(zo)))
    # linearity check of the GPU V-cycle (coarse CG is nonlinear at rounding level)
    z2 = P.A.to_canonical(P.preconditioner_apply(cyc, P.A.from_canonical(2 * b)))
    print("  linearity", np.max(np.abs(z2 - 2 * z)) / np.max(np.abs(z)))
    oref = o.solve(1, 2, kp, kq, b, tol=1e-8)
    x, rep = cm.pgmres(P.A, P.preconditioner(cyc), P.A.from_canonical(b), None, cm.SolveOptions(tol=1e-8))
    h, hr = np.array(rep.residual_history), np.array(oref.history)
    print("  its", rep.iterations, oref.iterations, "absdiff/r0", np.abs(h - hr) / hr[0])
rc = ob.random_vector(o.n[2], 7)
C1 = P.ops[2]
ec = C1.to_canonical(P.coarse_solve(C1.from_canonical(rc)))
print("coarse rel", np.max(np.abs(ec - o.coarse_solve(rc))) / np.max(np.abs(ec)))
