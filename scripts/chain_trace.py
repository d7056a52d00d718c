"""Split the sweep hop on a 1-D chain into compute vs signalling (trace)."""
import ctypes, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_07882_b200 import bcs, _native
L = 4000
owner = np.arange(L - 1, dtype=np.int32); neigh = owner + 1
rng = np.random.default_rng(1)
dg = rng.uniform(-0.1, 0.1, (L, 5, 5))
for i in range(5): dg[:, i, i] += 4.0
A = bcs.BlockLduMatrix(L, owner, neigh, 5, dg.reshape(-1), rng.uniform(-.1, .1, (L - 1) * 25), rng.uniform(-.1, .1, (L - 1) * 25))
ctx = bcs.Context(0); ctx.set_topology(A); ctx.upload_ldu(A)
ctx.precond_setup(bcs.SolverConfig(preconditioner=bcs.PrecondKind.DILU))
r = rng.uniform(-1, 1, L * 5)
ctx.precond_apply(r)
buf = torch.zeros(10 * L, dtype=torch.int64, device="cuda")
res = ctypes.c_ulonglong()
_native.lib().bcs_selftest(20, 1, buf.data_ptr(), ctypes.byref(res))
ctx.precond_apply(r)   # fwd then bwd: trace holds the bwd sweep (last writer)
_native.lib().bcs_selftest(20, 0, 0, ctypes.byref(res))
tr = buf.cpu().numpy().reshape(L, 10).astype(np.float64)
gt0, gt1, cy0, cy1, gts = tr[:, 0], tr[:, 1], tr[:, 2], tr[:, 3], tr[:, 4]
comp = cy1 - cy0
sig = gt0[1:] - gt1[:-1]
print("rows", L)
print("compute cycles (ready->stored): median %.0f p90 %.0f" % (np.median(comp), np.percentile(comp, 90)))
print("compute ns (globaltimer):       median %.0f" % np.median(gt1 - gt0))
print("stored(t-1) -> ready(t) ns:      median %.0f p10 %.0f p90 %.0f" % (np.median(sig), np.percentile(sig, 10), np.percentile(sig, 90)))
print("hop ns (ready->ready):           median %.0f" % np.median(np.diff(gt0)))
