"""Per-row timing of the sweep on K interleaved chains (wide levels)."""
import ctypes, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_07882_b200 import bcs, _native
ctx = bcs.Context(0)
for K, L in [(1, 4000), (2048, 200), (8192, 64)]:
    rows = K * L
    s_idx = np.arange(L - 1)
    owner = (np.arange(K)[:, None] + K * s_idx[None, :]).reshape(-1).astype(np.int32)
    neigh = owner + K
    order = np.argsort(owner, kind="stable"); owner, neigh = owner[order], neigh[order]
    rng = np.random.default_rng(1)
    nf = owner.size
    dg = rng.uniform(-0.1, 0.1, (rows, 5, 5))
    for i in range(5): dg[:, i, i] += 4.0
    A = bcs.BlockLduMatrix(rows, owner, neigh, 5, dg.reshape(-1), rng.uniform(-.1, .1, nf * 25), rng.uniform(-.1, .1, nf * 25))
    ctx.set_topology(A); ctx.upload_ldu(A)
    ctx.precond_setup(bcs.SolverConfig(preconditioner=bcs.PrecondKind.DILU))
    r = rng.uniform(-1, 1, rows * 5)
    ctx.precond_apply(r)
    buf = torch.zeros(10 * rows, dtype=torch.int64, device="cuda")
    res = ctypes.c_ulonglong()
    _native.lib().bcs_selftest(20, 1, buf.data_ptr(), ctypes.byref(res))
    ctx.precond_apply(r)
    _native.lib().bcs_selftest(20, 0, 0, ctypes.byref(res))
    tr = buf.cpu().numpy().reshape(rows, 10).astype(np.float64)
    ready, stored, cy0, cy1, start = tr[:, 0], tr[:, 1], tr[:, 2], tr[:, 3], tr[:, 4]
    t0 = start.min()
    span = stored.max() - t0
    print(f"K={K} L={L}: bwd sweep span {span/1e3:.1f} us; start->ready median {np.median(ready-start):.0f} ns "
          f"p90 {np.percentile(ready-start,90):.0f}; ready->stored median {np.median(stored-ready):.0f} ns; "
          f"compute cyc {np.median(cy1-cy0):.0f}", flush=True)
    # per level completion times (level = ticket // K)
    lev_done = stored.reshape(L, K).max(axis=1) - t0
    lev_start = start.reshape(L, K).min(axis=1) - t0
    print("   level done (us) first 6:", np.round(lev_done[:6] / 1e3, 2), " last:", round(lev_done[-1] / 1e3, 2))
    print("   level start (us) first 6:", np.round(lev_start[:6] / 1e3, 2))
