"""paper_2210_03179_b200 -- B200-native Chebyshev-smoothed V-cycle preconditioner path.

Host-side mirror of the reference chebmg interface (``chebmg``: 2D FD path,
``sem``: spectral-element p-multigrid path) over the C-ABI library
``lib/libchebmg_b200.so`` (hand-written sm_100a CUDA, see include/chebmg_b200.h).
"""
__all__ = ["chebmg", "sem"]
