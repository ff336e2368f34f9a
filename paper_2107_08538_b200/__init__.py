"""paper_2107_08538_b200 — B200-native GPU-sharing runtime (arXiv 2107.08538).

Subpackages:
  gpushare   drop-in for the reference's probe/placement API (libgs, sm_100a)
  csrc       CUDA sources: decision engine, workload kernels, executor
"""

import os as _os

# The persistent decision kernel (probe ring) never ends while jobs run.  CUDA
# multiplexes streams onto CUDA_DEVICE_MAX_CONNECTIONS hardware queues (8 by
# default); a job stream that aliases the ring's queue would queue behind the
# resident kernel.  32 queues keep the ring stream and the executor's worker
# streams distinct.  Must be set before the CUDA context exists.
_os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

__version__ = "0.1.0"
