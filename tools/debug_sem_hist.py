import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import oracle_bind as ob
from paper_2210_03179_b200 import chebmg as cm, sem
np.set_printoptions(linewidth=200, precision=3)
for geo, eps, kp, kq in [(0, 1.0, 4, 0), (1, 0.05, 8, 0), (1, 0.3, 4, 0)]:
    ex = ey = ez = 3 if geo else 4
    if geo == 0: ey = ez = 3
    P = sem.PMGHierarchy(sem.SemDesc(7, ex, ey, ez, geometry=geo, eps=eps), (7, 3, 1))
    o = ob.OraclePmg((7, 3, 1), ex, ey, ez, geo, eps)
    print("lambda gpu", P.lambda_tilde, "orc", o.lambda_tilde, "rel", [(a-b)/b for a, b in zip(P.lambda_tilde[:2], o.lambda_tilde[:2])])
    b = o.sem(0).rhs()
    rc = ob.random_vector(o.n[2], 7)
    C1 = P.ops[2]
    ec = C1.to_canonical(P.coarse_solve(C1.from_canonical(rc))); eo = o.coarse_solve(rc)
    print("coarse rel err", np.max(np.abs(ec-eo))/np.max(np.abs(eo)))
    oref = o.solve(1, 2, kp, kq, b, tol=1e-8)
    for lam in (P.lambda_tilde[0], o.lambda_tilde[0]):
        cyc = cm.CycleConfig(cm.ChebyshevConfig(cm.Family.fourth, 1, lam), kp, kq)
        x, rep = cm.pgmres(P.A, P.preconditioner(cyc), P.A.from_canonical(b), None, cm.SolveOptions(tol=1e-8))
        h, hr = np.array(rep.residual_history), np.array(oref.history)
        print(geo, eps, "its", rep.iterations, oref.iterations, "relentry", np.abs(h-hr)/hr, "rel_r0 max", np.max(np.abs(h-hr))/hr[0])
