"""Dependency-hop latency of the sync-free sweeps: DILU application on K
independent 1-D chains of L rows (DAG depth L), time per hop = t/(2L)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_07882_b200 import bcs  # noqa: E402

n = 5
ctx = bcs.Context(0)
for K, L in [(1, 20000), (16, 20000), (256, 4000), (2048, 1000), (8192, 256)]:
    rows = K * L
    # chains interleaved: row r = c + K*s (chain c, step s); faces (r, r+K)
    s_idx = np.arange(L - 1)
    owner = (np.arange(K)[:, None] + K * s_idx[None, :]).reshape(-1).astype(np.int32)
    neigh = owner + K
    order = np.argsort(owner, kind="stable")
    owner, neigh = owner[order], neigh[order]
    rng = np.random.default_rng(1)
    nf = owner.size
    up = rng.uniform(-0.1, 0.1, nf * 25)
    lo = rng.uniform(-0.1, 0.1, nf * 25)
    dg = rng.uniform(-0.1, 0.1, (rows, 5, 5))
    for i in range(5):
        dg[:, i, i] += 4.0
    A = bcs.BlockLduMatrix(rows, owner, neigh, n, dg.reshape(-1), up, lo)
    ctx.set_topology(A)
    ctx.upload_ldu(A)
    ctx.precond_setup(bcs.SolverConfig(preconditioner=bcs.PrecondKind.DILU))
    r = rng.uniform(-1, 1, rows * n)
    z = ctx.precond_apply(r)
    reps = 5
    t0 = time.perf_counter()
    for _ in range(reps):
        z = ctx.precond_apply(r)
    dt = (time.perf_counter() - t0) / reps
    print(f"K={K:5d} L={L:6d} rows={rows:8d} depth={ctx.schedule_depth(0):6d}  apply {dt*1e3:8.3f} ms  "
          f"per hop {dt/(2*L)*1e6:6.3f} us", flush=True)
