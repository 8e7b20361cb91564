"""Multi-GPU element partition (BASELINE configs[4] shape): the same p-MG(7,3,1)
PGMRES solve at 1, 2 (4, 8) GPUs must give BITWISE identical residual
histories and solutions -- the gather-scatter sums and the inner products are
reduced in a fixed global order -- and the 1-GPU run matches
the oracle (tests/test_sem_gpu.py).  Needs >= 2 GPUs (gpurun --gpus 2)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ngpus():
    try:
        import torch

        return torch.cuda.device_count()
    except Exception:
        return 0


def _worlds():
    return [w for w in (2, 4, 8) if _ngpus() >= w]


def _run(world, out, extra=()):
    script = os.path.join(ROOT, "tools", "mgpu_check.py")
    if world == 1:
        cmd = [sys.executable, script, "--out", out, *extra]
    else:
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
               "--master-addr", "127.0.0.1", "--master-port", str(29500 + world), script, "--out", out, *extra]
    subprocess.run(cmd, check=True, timeout=600, cwd=ROOT)
    with open(out) as fh:
        return json.load(fh)


@pytest.mark.skipif(_ngpus() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("geometry", [0, 1])
def test_partition_bitwise_identical(tmp_path, geometry):
    extra = ("--geometry", str(geometry))
    r1 = _run(1, str(tmp_path / "r1.json"), extra)
    import numpy as np

    x1 = np.load(str(tmp_path / "r1.json") + ".x.npy")
    for w in _worlds():
        rw = _run(w, str(tmp_path / f"r{w}.json"), extra)
        for k in ("iterations", "fine_matvecs", "history", "lambda"):
            assert rw[k] == r1[k], (w, k)
        xw = np.load(str(tmp_path / f"r{w}.json") + ".x.npy")
        diff = np.nonzero(xw != x1)[0]
        print(f"W={w}: {diff.size} entries differ, max |dx| = {np.max(np.abs(xw - x1)) if diff.size else 0}")
        assert diff.size == 0, (w, diff[:10], xw[diff[:10]], x1[diff[:10]])


@pytest.mark.skipif(_ngpus() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("smoother,geometry", [(1, 0), (2, 0), (2, 1)], ids=["asm-box", "ras-box", "ras-kershaw"])
def test_schwarz_partition_bitwise_identical(tmp_path, smoother, geometry):
    """Chebyshev-ASM/RAS p-MG(7,3,1) on the z-slab partition: the extended
    boxes of the first/last owned layer read the neighbouring slabs' node
    planes (and ASM sums their boxes), so the solve is BITWISE the 1-GPU one
    (which tests/test_sem_gpu.py checks against the oracle)."""
    import numpy as np

    extra = ("--smoother", str(smoother), "--geometry", str(geometry), "--kpre", "2")
    r1 = _run(1, str(tmp_path / "s1.json"), extra)
    x1 = np.load(str(tmp_path / "s1.json") + ".x.npy")
    for w in _worlds():
        rw = _run(w, str(tmp_path / f"s{w}.json"), extra)
        for k in ("iterations", "fine_matvecs", "history", "lambda"):
            assert rw[k] == r1[k], (w, k)
        xw = np.load(str(tmp_path / f"s{w}.json") + ".x.npy")
        assert np.array_equal(xw, x1), (w, np.max(np.abs(xw - x1)))


@pytest.mark.skipif(_ngpus() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("smoother,family,kpre,kpost", [(0, 2, 4, 0), (2, 2, 2, 0), (1, 2, 2, 0), (2, 0, 2, 2),
                                                        (1, 0, 2, 2)],
                         ids=["jacobi", "ras", "asm", "ras-1st-2-2", "asm-1st-2-2"])
def test_one_layer_per_rank_bitwise_identical(tmp_path, smoother, family, kpre, kpost):
    """Ez = world: every rank holds ONE element layer (Ezl = 1), so the first and
    the last owned layer coincide -- the face halo, the bottom-face contribution
    return, the Schwarz ghost planes from both neighbours and the ASM box sums
    all touch the same layer.  Bitwise the 1-GPU solve of the same mesh; the
    1st-kind (2,2) Schwarz cases run the fused x += d update at order 2."""
    import numpy as np

    for w in _worlds():
        extra = ("--ez", str(w), "--smoother", str(smoother), "--family", str(family), "--kpre", str(kpre),
                 "--kpost", str(kpost))
        r1 = _run(1, str(tmp_path / f"o1_{w}.json"), extra)
        rw = _run(w, str(tmp_path / f"o{w}.json"), extra)
        for k in ("iterations", "fine_matvecs", "history", "lambda"):
            assert rw[k] == r1[k], (w, k)
        x1 = np.load(str(tmp_path / f"o1_{w}.json") + ".x.npy")
        xw = np.load(str(tmp_path / f"o{w}.json") + ".x.npy")
        assert np.array_equal(xw, x1), (w, np.max(np.abs(xw - x1)))


@pytest.mark.skipif(_ngpus() < 2, reason="needs >= 2 GPUs")
def test_sweep_across_ranks_matches_single_gpu(tmp_path):
    """harness.hpp:297-337 sweep dealt over 2 ranks (tools/sweep.py): the merged
    CSV (timing column off) is byte-identical to the 1-GPU sweep."""
    cfg = tmp_path / "sweep.cfg"
    cfg.write_text("sweep.Lx = 1, 8, 64\nsweep.factor = 2, 4\nsweep.k = 1..2\n"
                   "sweep.family = first, fourth_opt\nsweep.cycle = full, one_sided\ncase.n = 32\n")
    script = os.path.join(ROOT, "tools", "sweep.py")
    out1, out2 = tmp_path / "w1", tmp_path / "w2"
    subprocess.run([sys.executable, script, "--config", str(cfg), "--out", str(out1), "--no-timing"],
                   check=True, timeout=600, cwd=ROOT)
    subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                    "--master-addr", "127.0.0.1", "--master-port", "29611", script, "--config", str(cfg),
                    "--out", str(out2), "--no-timing"], check=True, timeout=600, cwd=ROOT)
    a = (out1 / "sweep.csv").read_text()
    b = (out2 / "sweep.csv").read_text()
    assert a == b and a.count("\n") == 1 + 3 * 2 * 2 * 2 * 2


@pytest.mark.skipif(_ngpus() < 2, reason="needs >= 2 GPUs")
def test_full_size_partition_identity(tmp_path):
    """BASELINE configs[4] at full size (N=7, E=64^3, 89.3M unknowns), the bench's
    (8,0) 4th-kind p-MG PGMRES solve: residual history, iteration count and a
    sha256 of the whole canonical solution are identical at 1, 2 (and 4) GPUs."""
    extra = ("--E", "64", "--ez", "64", "--kpre", "8", "--hash-only")
    r1 = _run(1, str(tmp_path / "f1.json"), extra)
    assert r1["iterations"] == 9
    for w in _worlds():
        rw = _run(w, str(tmp_path / f"f{w}.json"), extra)
        for k in ("iterations", "fine_matvecs", "history", "lambda", "x_sha256"):
            assert rw[k] == r1[k], (w, k)
