"""The runtime A/B knobs select alternative kernels; every
non-default variant must pass the same parity checks as the default.  Each
knob is read once per process, so each variant runs the relevant parity tests
in a child pytest with the variable set."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

VARIANTS = [
    ("CMG_K1_GREG", "0", "tests/test_sem_gpu.py", "apply_diag_rhs or sweeps_all_families or pmg_solves"),
    ("CMG_K1_PREFETCH", "0", "tests/test_sem_gpu.py", "sweeps_all_families"),
    ("CMG_K1_GREG3", "1", "tests/test_sem_gpu.py", "sweeps_all_families or v_cycle or pmg_solves"),
    ("CMG_PEER_HALO", "0", "tests/test_multigpu.py", "bitwise"),
    # the small test meshes sit below the default peer threshold: force the peer path
    ("CMG_PEER_MIN", "0", "tests/test_multigpu.py", "bitwise"),
    ("CMG_PEER_KWAIT", "0", "tests/test_multigpu.py", "bitwise"),
    ("CMG_SHELL_LEX", "1", "tests/test_sem_gpu.py", "apply_diag_rhs or sweeps_all_families or v_cycle"),
    ("CMG_CGS_FUSE", "0", "tests/test_sem_gpu.py", "pmg_solves"),
    ("CMG_DOTS_UNROLL", "1", "tests/test_sem_gpu.py", "pmg_solves or determinism"),
    ("CMG_CGS_UNROLL", "1", "tests/test_sem_gpu.py", "pmg_solves or determinism"),
    ("CMG_CGS_FUSE", "0", "tests/test_fd_gpu.py", "golden_solves"),
    ("CMG_FD_GRAPHS", "0", "tests/test_fd_gpu.py", "golden_solves or preconditioner_cost"),
    ("CMG_SEM_GRAPHS", "0", "tests/test_sem_gpu.py", "pmg_solves or schwarz_pmg or kershaw or graph_replayed"),
    # the PGMRES least-squares working copy in global memory (the path for restart > ~169)
    ("CMG_LSQ_SMEM_MAX", "0", "tests/test_fd_gpu.py", "any_restart"),
    ("CMG_SCHWARZ_MMA", "1", "tests/test_sem_gpu.py", "schwarz"),
    ("CMG_SCHWARZ_SMALL", "0", "tests/test_sem_gpu.py", "schwarz"),
    ("CMG_SCHWARZ_IL", "1", "tests/test_sem_gpu.py", "schwarz"),
    ("CMG_SCHWARZ_FUSE", "0", "tests/test_sem_gpu.py", "schwarz"),
    ("CMG_COARSE_INV", "0", "tests/test_sem_gpu.py", "kershaw or transfers_and_coarse"),
    ("CMG_TRANSFER_KERNEL", "0", "tests/test_sem_gpu.py", "transfers_and_coarse or v_cycle or pmg_solves"),
    ("CMG_TRANSFER_KERNEL", "1", "tests/test_sem_gpu.py", "transfers_and_coarse or v_cycle or pmg_solves"),
    ("CMG_COARSE_DENSE_MAX", "0", "tests/test_sem_gpu.py", "kershaw or transfers_and_coarse"),
]


@pytest.mark.parametrize("var,val,path,sel", VARIANTS, ids=[f"{v}={x}:{os.path.basename(p)}" for v, x, p, _ in VARIANTS])
def test_variant_parity(var, val, path, sel):
    if "multigpu" in path:
        import torch

        if torch.cuda.device_count() < 2:
            pytest.skip("the multi-GPU parity tests need >= 2 GPUs (they would all skip in the child)")
    env = dict(os.environ, **{var: val})
    r = subprocess.run([sys.executable, "-m", "pytest", path, "-m", "gpu", "-q", "-x", "-k", sel, "-p", "no:cacheprovider"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
