"""One GMRES+AMG solve on an n^3 5x5 system (profiling target)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_07882_b200 import bcs, gen  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
s = gen.hex_euler(n, scramble_seed=int(sys.argv[3]) if len(sys.argv) > 3 else -1)
mode = bcs.Mode.PERF if len(sys.argv) > 2 and sys.argv[2] == "perf" else bcs.Mode.PARITY
cfg = bcs.SolverConfig(preconditioner=bcs.PrecondKind.AMG, relTol=1e-8, maxIters=1000,
                       amg=bcs.AmgConfig(maxLevels=30, minCoarseRows=8), mode=mode)
ctx = bcs.Context(0)
ctx.set_topology(s.A)
ctx.upload_ldu(s.A)
x = s.x0.values.copy()
r = ctx.solve(s.b.values, x, cfg)
print("iters", r.iterations, "setup", r.timings["amgSetup"], "krylov", r.timings["krylov"])
