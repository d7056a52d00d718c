"""Per-row timeline of the fine-level forward sweep at 128^3 (traced build of
the one-row-per-warp wide variant, BCS_WIDE_DUAL=0): stage wait, dependency
wait, fold+solve, and the per-dependency-level completion times."""
import ctypes, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_07882_b200 import bcs, gen, _native

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
s = gen.hex_euler(n)
rows = n ** 3
ctx = bcs.Context(0)
ctx.set_topology(s.A)
ctx.upload_ldu(s.A)
ctx.precond_setup(bcs.SolverConfig(preconditioner=bcs.PrecondKind.AMG, amg=bcs.AmgConfig(maxLevels=30, minCoarseRows=8)))
r = np.random.default_rng(1).uniform(-1, 1, rows * 5)
ctx.precond_apply(r)
buf = torch.zeros(10 * rows, dtype=torch.int64, device="cuda")
res = ctypes.c_ulonglong()
lib = _native.lib()
lib.bcs_selftest(20, 2 * rows + 1, buf.data_ptr(), ctypes.byref(res))
ctx.precond_apply(r)
lib.bcs_selftest(20, 0, 0, ctypes.byref(res))
tr = buf.cpu().numpy().reshape(rows, 10).astype(np.int64)
gt0, gt1, gts = tr[:, 0].astype(np.float64), tr[:, 1].astype(np.float64), tr[:, 4].astype(np.float64)
stage_wait = (tr[:, 8] >> 32).astype(np.float64)
spins = (tr[:, 7] & 0xFFFFFFFF).astype(np.float64)
first_poll = (tr[:, 7] >> 32).astype(np.float64)
t0 = gts.min()
print("rows", rows, "sweep span us %.1f" % ((gt1.max() - t0) / 1e3))
print("stage wait cycles: median %.0f p90 %.0f" % (np.median(stage_wait), np.percentile(stage_wait, 90)))
print("spins: mean %.1f median %.0f p90 %.0f" % (spins.mean(), np.median(spins), np.percentile(spins, 90)))
print("first poll cycles: median %.0f" % np.median(first_poll))
print("start->fold done ns: median %.0f p90 %.0f" % (np.median(gt0 - gts), np.percentile(gt0 - gts, 90)))
print("fold done->stored ns: median %.0f p90 %.0f" % (np.median(gt1 - gt0), np.percentile(gt1 - gt0, 90)))
# dependency levels of the natural hex: level d = x + y + z, tickets in level order
cnt = np.bincount((np.add.outer(np.add.outer(np.arange(n), np.arange(n)), np.arange(n))).ravel())
edges = np.concatenate([[0], np.cumsum(cnt)])
done = np.array([gt1[edges[d]:edges[d + 1]].max() for d in range(len(cnt))]) - t0
start = np.array([gts[edges[d]:edges[d + 1]].min() for d in range(len(cnt))]) - t0
per = np.diff(done)
print("levels", len(cnt), "per-level completion ns: median %.0f mean %.0f (levels 100-280: %.0f)" % (
    np.median(per), per.mean(), per[100:280].mean()))
mid = slice(edges[190], edges[191])
print("level 190: rows %d, start spread ns %.0f, done spread ns %.0f" % (
    cnt[190], gts[mid].max() - gts[mid].min(), gt1[mid].max() - gt1[mid].min()))
print("level 190 row: start - prev level done ns: median %.0f" % np.median(gts[mid] - t0 - done[189]))
print("level 190 row: stored - prev level done ns: median %.0f p90 %.0f max %.0f" % (
    np.median(gt1[mid] - t0 - done[189]), np.percentile(gt1[mid] - t0 - done[189], 90), (gt1[mid] - t0 - done[189]).max()))
