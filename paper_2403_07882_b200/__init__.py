"""B200-native block-coupled linear-solve path (arXiv 2403.07882 hot path).

The product is libbcs.so (hand-written sm_100a kernels behind the C ABI in
include/bcs.h); this package is the host-side mirror of the reference's
solver API plus the synthetic workload generator.
"""
from .bcs import (AmgConfig, Backend, BlockLduMatrix, BlockVector, Context, KrylovMethod, PrecondKind,
                  SolvePipeline, SolveReport, SolverConfig, backend_solve, topology_signature)

__all__ = ["AmgConfig", "Backend", "BlockLduMatrix", "BlockVector", "Context", "KrylovMethod", "PrecondKind",
           "SolvePipeline", "SolveReport", "SolverConfig", "backend_solve", "topology_signature"]
