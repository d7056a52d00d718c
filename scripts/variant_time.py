"""Timing of one library build (experiments): 1-D chain hop and the 128^3
GMRES+AMG solve (setup / Krylov / sweep time; min over repeats)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2403_07882_b200 import bcs, gen

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
hop = bench.chain_hop_ns(bcs, L=20000, reps=3)
s = gen.hex_euler(n)
cfg = bench.solver_config("gmres")
ctx = bcs.Context(0)
ctx.set_topology(s.A)
ctx.upload_ldu(s.A)
best = None
for i in range(4):
    if i == 1:
        ctx.set_kernel_timing(True)
    x = s.x0.values.copy()
    t = time.perf_counter()
    r = ctx.solve(s.b.values, x, cfg)
    dt = time.perf_counter() - t
    if i >= 1:
        cur = (dt, r.timings["amgSetup"], r.timings["krylov"], r.sweepMs, r.iterations)
        best = cur if best is None or cur[0] < best[0] else best
print(f"hop {hop:.1f} ns | solve {best[0]*1e3:.1f} ms setup {best[1]*1e3:.1f} krylov {best[2]*1e3:.1f} "
      f"sweeps {best[3]:.1f} ms its {best[4]}", flush=True)
