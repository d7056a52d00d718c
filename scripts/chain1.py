"""Single 1-D chain DILU apply (hop-latency profiling target)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_07882_b200 import bcs
L = int(sys.argv[1]) if len(sys.argv) > 1 else 4000
owner = np.arange(L - 1, dtype=np.int32); neigh = owner + 1
rng = np.random.default_rng(1)
dg = rng.uniform(-0.1, 0.1, (L, 5, 5))
for i in range(5): dg[:, i, i] += 4.0
A = bcs.BlockLduMatrix(L, owner, neigh, 5, dg.reshape(-1), rng.uniform(-.1, .1, (L - 1) * 25), rng.uniform(-.1, .1, (L - 1) * 25))
ctx = bcs.Context(0); ctx.set_topology(A); ctx.upload_ldu(A)
ctx.precond_setup(bcs.SolverConfig(preconditioner=bcs.PrecondKind.DILU))
z = ctx.precond_apply(rng.uniform(-1, 1, L * 5))
print("ok", float(np.abs(z).max()))
