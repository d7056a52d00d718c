"""Rows, blocks per row, dependency depth and mean width of every AMG level
of the 128^3 bench system (the lower-dependency count sets the sweeps'
number of poll passes: 6 dependencies per pass for 5x5 blocks)."""
import ctypes, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_07882_b200 import bcs, gen

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
s = gen.hex_euler(n)
ctx = bcs.Context(0)
ctx.set_topology(s.A)
ctx.upload_ldu(s.A)
ctx.precond_setup(bcs.SolverConfig(preconditioner=bcs.PrecondKind.AMG, amg=bcs.AmgConfig(maxLevels=30, minCoarseRows=8)))
for l in range(ctx.amg_depth()):
    ro, ci, _, _ = ctx.amg_level(l, 5) if l < 8 else (None, None, None, None)
    rows, nnz, _ = ctx.amg_level_shape(l, want_agg=False)
    line = f"L{l}: rows {rows} blocks/row {nnz / rows:.2f}"
    if ro is not None:
        r = np.repeat(np.arange(rows), np.diff(ro))
        low = np.bincount(r[ci < r], minlength=rows)
        line += f" lower deps mean {low.mean():.2f} max {low.max()} >6: {np.mean(low > 6) * 100:.1f}% >12: {np.mean(low > 12) * 100:.1f}%"
    if l + 1 < ctx.amg_depth():
        d = ctx.schedule_depth(l)
        line += f" depth {d} width {rows / max(d, 1):.0f}"
    print(line, flush=True)
