"""Full-size SEM parity against committed fixtures from the reference-template CPU
path (oracle/make_golden_sem.py -> tests/golden/sem_*.json; RefPmg in
oracle/ref_driver.cpp: the reference's pgmres, v_cycle, chebyshev_smooth,
estimate_lambda_max and BandedCholesky over the restated SEM operator, single
threaded, run once in the build container):

  sem_E64_box_4th_8_0  north_star target: N=7, E=64^3 (89.3M unknowns), 4th-kind
                       Chebyshev-Jacobi half V-cycle (8,0), p-MG(7,3,1), PGMRES(30)
  sem_kershaw03_E32    configs[3]: Kershaw eps=0.3, E=32^3, (8,0) vs (4,4)
  sem_ras_E32/asm_E32  configs[2]: E=32^3 Chebyshev-RAS/-ASM, (2,0) vs (1,1)

Criteria (fp64): iterations and fine_matvecs exact; lambda_tilde of every
smoothed level within 1e-11; residual histories entrywise within 1e-12 ||r_0||
(the per-entry relative error is printed; see tests/test_sem_gpu.py for why
1e-10 per entry is below the reference's own reproducibility floor); solution
samples (4096 entries) and ||x|| within 1e-10 relative.  The right-hand side is
rebuilt here with the restatement and must hash to the fixture's sha256.
"""
import glob
import hashlib
import json
import os

import numpy as np
import pytest

import oracle_bind as ob

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
FIXTURES = sorted(glob.glob(os.path.join(HERE, "golden", "sem_*.json")))
FAM = {"first": 0, "first_opt_lambda": 1, "fourth": 2, "fourth_opt": 3}
SM = {"jacobi": 0, "asm": 1, "ras": 2}


def _load(path):
    with open(path) as fh:
        return json.load(fh)


@pytest.fixture(scope="module", params=FIXTURES, ids=[os.path.basename(p)[4:-5] for p in FIXTURES])
def case(request):
    from paper_2210_03179_b200 import sem

    g = _load(request.param)
    Ex, Ey, Ez = g["E"]
    s = ob.OracleSem(7, Ex, Ey, Ez, g["geometry"], g["eps"])
    b = s.rhs()
    del s
    assert hashlib.sha256(b.tobytes()).hexdigest() == g["b_sha256"]
    P = sem.PMGHierarchy(sem.SemDesc(7, Ex, Ey, Ez, geometry=g["geometry"], eps=g["eps"]), tuple(g["orders"]),
                         smoother=SM[g["smoother"]], eigen_iterations=g["eigen_iterations"],
                         eigen_seed=g["eigen_seed"])
    yield g, P, b
    del P


def test_lambda_tilde(case):
    """30 power iterations (smoothers.hpp:61-79) whose norms and Rayleigh quotient use
    the reference's sequential dots on the CPU and a fixed tree on the GPU: 1e-11
    relative (observed 1e-14 .. 1.2e-12, the largest on the Kershaw mesh)."""
    g, P, _ = case
    lt = ob.unhex(g["lambda_tilde"])
    for l in range(len(g["orders"]) - 1):
        d = abs(P.lambda_tilde[l] - lt[l]) / lt[l]
        print(f"\n[{g['case']}] lambda_tilde[{l}] rel diff {d:.3e}")
        assert d <= 1e-11, (l, P.lambda_tilde[l], lt[l])


def test_solves_match_reference_fixture(case):
    from paper_2210_03179_b200 import chebmg as cm

    g, P, b = case
    n = b.size
    idx = np.unique(np.linspace(0, n - 1, 4096).astype(np.int64))
    bd = P.A.from_canonical(b)
    for sv in g["solves"]:
        fam, kpre, kpost = FAM[sv["family"]], sv["k_pre"], sv["k_post"]
        cyc = cm.CycleConfig(cm.ChebyshevConfig(cm.Family(fam), 1, P.lambda_tilde[0]), kpre, kpost)
        x, rep = cm.pgmres(P.A, P.preconditioner(cyc), bd, None,
                           cm.SolveOptions(tol=g["tol"], maxit=g["maxit"], restart=g["restart"]))
        what = f"{g['case']} {sv['family']} ({kpre},{kpost})"
        assert (rep.iterations, rep.fine_matvecs, rep.converged) == (sv["iterations"], sv["fine_matvecs"],
                                                                      sv["converged"]), what
        h, hr = np.array(rep.residual_history), ob.unhex(sv["history"])
        assert h.size == hr.size
        d = np.abs(h - hr)
        print(f"\n[{what}] {rep.iterations} its, {rep.fine_matvecs} mv; history max|h-h_ref|/h0 = "
              f"{np.max(d) / hr[0]:.3e}, max per-entry rel = {np.max(d / hr):.3e}")
        assert np.max(d) <= 1e-12 * hr[0], what
        xc = P.A.to_canonical(x)
        xs, xr = xc[idx], ob.unhex(sv["x_samples"])
        xn, xrn = np.linalg.norm(xc), float.fromhex(sv["x_norm"])
        es = float(np.max(np.abs(xs - xr)) / np.max(np.abs(xr)))
        print(f"[{what}] x samples max rel = {es:.3e}, |x| rel = {abs(xn - xrn) / xrn:.3e}")
        assert es <= 1e-10 and abs(xn - xrn) <= 1e-10 * xrn, what
        del x
