"""One profiled solve (BCS_PROFILE=1 per-phase breakdown on stderr)."""
import os
import sys
import time

os.environ.setdefault("BCS_PROFILE", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_07882_b200 import bcs, gen  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
seed = int(sys.argv[2]) if len(sys.argv) > 2 else -1
s = gen.hex_euler(n, scramble_seed=seed)
cfg = bcs.SolverConfig(preconditioner=bcs.PrecondKind.AMG, relTol=1e-8, maxIters=1000,
                       amg=bcs.AmgConfig(maxLevels=30, minCoarseRows=8))
ctx = bcs.Context(0)
ctx.set_topology(s.A)
ctx.upload_ldu(s.A)
for i in range(2):
    x = s.x0.values.copy()
    t = time.perf_counter()
    r = ctx.solve(s.b.values, x, cfg)
    print(f"solve {i}: {time.perf_counter()-t:.3f}s iters={r.iterations} levels={r.amgLevels} "
          f"setup={r.timings['amgSetup']:.3f} krylov={r.timings['krylov']:.3f} coarse_rows={r.coarseRows}", file=sys.stderr, flush=True)
