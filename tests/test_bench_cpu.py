"""bench.py's measurement bookkeeping (CPU): the workload config is identical for
the GPU arm at every GPU count and for the reference arm, the reference arm's
replica count respects host memory, and the algorithmic sweep bytes follow the
per-pass model of DESIGN.md §7."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def test_config_identical_across_arms_and_gpu_counts():
    n = (7 * 64 - 1) ** 3
    c1 = bench.config_of(64, 8, n, 1)
    for w in (2, 4, 8):
        assert bench.config_of(64, 8, n, w) == c1
    assert c1["unknowns"] == 89314623 and c1["E"] == 64 ** 3


def test_replica_memory_model():
    # one E=64^3 reference sweep context: ~17 GB (levels + 7 vectors)
    assert 16e9 < bench.replica_bytes(64) < 18e9
    assert bench.reference_replicas(64) >= 1


def test_sweep_bytes_model():
    n = (7 * 64 - 1) ** 3
    assert abs(bench.sweep_bytes(64, 8, n) - 93.696e9) < 1e7  # 93.70 GB per sweep
    # one middle step alone is the SURVEY §8(d) 48 N_L + 64 N_G = 12.16 GB
    assert abs((bench.sweep_bytes(64, 3, n) - bench.sweep_bytes(64, 2, n)) - 12.158e9) < 1e7
