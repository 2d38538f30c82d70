"""B200-native (sm_100a) drop-in for the data-parallel fork-join code Hercules
generates for the Juno benchmarks (arXiv 2503.10855).

Public surface:
  execute / oracle_execute            -- the reference's execution interface
  matmul, edge_detection, cava, srad, euler, bfs, backprop
  RuntimeError_, DynConstError, OracleLimitError
Kernels live in libjunob200.so (include/junob200.h); build with
``python -m paper_2503_10855_b200.build``.
"""

from .api import (DynConstError, OracleLimitError, RuntimeError_, UnsupportedError, backprop, bfs,
                  cava, edge_detection, edge_detection_stages, euler, euler_flux, euler_step_factor,
                  execute, matmul, oracle_execute, srad)

__all__ = [
    "execute", "oracle_execute", "matmul", "edge_detection", "edge_detection_stages", "cava", "srad",
    "euler", "euler_flux", "euler_step_factor", "bfs", "backprop", "RuntimeError_", "DynConstError",
    "OracleLimitError", "UnsupportedError",
]
