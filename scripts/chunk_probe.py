"""Chain-scheduled fine-level sweeps: the same solve with BCS_CHAIN as set in
the environment; prints iterations, the solution digest (the schedule must not
change a bit) and the median solve time of a few repeats."""
import hashlib
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_07882_b200 import bcs, gen  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
mode = {"parity": bcs.Mode.PARITY, "exact": bcs.Mode.EXACT}[sys.argv[2] if len(sys.argv) > 2 else "parity"]
s = gen.hex_euler(n)
cfg = bcs.SolverConfig(preconditioner=bcs.PrecondKind.AMG, relTol=1e-8, maxIters=1000,
                       amg=bcs.AmgConfig(maxLevels=30, minCoarseRows=8), mode=mode)
ctx = bcs.Context(0)
ctx.set_topology(s.A)
ctx.upload_ldu(s.A)
ts, dig = [], None
for k in range(4):
    x = s.x0.values.copy()
    t0 = time.perf_counter()
    r = ctx.solve(s.b.values, x, cfg)
    ts.append(time.perf_counter() - t0)
    d = hashlib.sha1(x.tobytes()).hexdigest()[:16]
    assert dig is None or d == dig
    dig = d
ts.sort()
print(f"BCS_CHAIN={os.environ.get('BCS_CHAIN', '1')} mode={sys.argv[2] if len(sys.argv) > 2 else 'parity'}"
      f" iters={r.iterations} digest={dig} solve_ms={1e3 * ts[1]:.1f} amgSetup={r.timings['amgSetup']:.4f}"
      f" krylov={r.timings['krylov']:.4f}")
