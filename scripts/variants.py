"""Solve times of other workloads: coupled 4x4 (pressure-based) and BiCGStab."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_07882_b200 import bcs, gen

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
for name, mk, method in [("euler5 gmres", lambda: gen.hex_euler(n), bcs.KrylovMethod.GMRES),
                         ("euler5 bicgstab", lambda: gen.hex_euler(n), bcs.KrylovMethod.PBiCGStab),
                         ("coupled4 gmres", lambda: gen.hex_coupled(n), bcs.KrylovMethod.GMRES)]:
    s = mk()
    cfg = bcs.SolverConfig(method=method, preconditioner=bcs.PrecondKind.AMG, relTol=1e-8, maxIters=1000,
                           amg=bcs.AmgConfig(maxLevels=30, minCoarseRows=8))
    ctx = bcs.Context(0)
    ctx.set_topology(s.A)
    ctx.upload_ldu(s.A)
    for i in range(3):
        x = s.x0.values.copy()
        t = time.perf_counter()
        r = ctx.solve(s.b.values, x, cfg)
        dt = time.perf_counter() - t
    print(f"{name} {n}^3: {dt:.3f}s iters={r.iterations} conv={r.converged} levels={r.amgLevels} "
          f"setup={r.timings['amgSetup']:.3f} krylov={r.timings['krylov']:.3f}", flush=True)
    ctx.close()
