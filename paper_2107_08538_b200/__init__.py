"""paper_2107_08538_b200 — B200-native GPU-sharing runtime (arXiv 2107.08538).

Subpackages:
  gpushare   drop-in for the reference's probe/placement API (libgs, sm_100a)
  csrc       CUDA sources: decision engine, workload kernels, executor
"""

__version__ = "0.1.0"
