"""Per-level timing of one smoother sweep on a real AMG level (diagnostics).

python scripts/level_trace.py N LEVEL : builds the hex_euler N^3 case, sets up
AMG, traces the forward sweep of level LEVEL during one V-cycle and prints the
per-dependency-level span, the spread of row start/ready/stored times."""
import ctypes, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_07882_b200 import bcs, gen, _native

n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
lev = int(sys.argv[2]) if len(sys.argv) > 2 else 1
s = gen.hex_euler(n)
cfg = bcs.SolverConfig(preconditioner=bcs.PrecondKind.AMG, relTol=1e-8, maxIters=1000,
                       amg=bcs.AmgConfig(maxLevels=30, minCoarseRows=8))
ctx = bcs.Context(0)
ctx.set_topology(s.A); ctx.upload_ldu(s.A)
ctx.precond_setup(cfg)
N = s.A.n
ro, ci, _, _ = ctx.amg_level(lev, N)
rows = ro.size - 1
# dependency level of every row for the forward sweep (lower neighbours j < i)
depth = np.zeros(rows, np.int64)
for i in range(rows):
    js = ci[ro[i]:ro[i + 1]]
    js = js[js < i]
    if js.size: depth[i] = depth[js].max() + 1
order = np.lexsort((np.arange(rows), depth))
nlev = depth.max() + 1
r = np.random.default_rng(0).uniform(-1, 1, s.A.n_cells * N)
ctx.precond_apply(r)
buf = torch.zeros(10 * rows, dtype=torch.int64, device="cuda")
res = ctypes.c_ulonglong()
_native.lib().bcs_selftest(20, 2 * rows + 1, buf.data_ptr(), ctypes.byref(res))
ctx.precond_apply(r)
_native.lib().bcs_selftest(20, 0, 0, ctypes.byref(res))
tr = buf.cpu().numpy().reshape(rows, 10).astype(np.float64)
ready, stored, cy0, cy1, start = tr[:, 0], tr[:, 1], tr[:, 2], tr[:, 3], tr[:, 4]
t0 = start.min()
dl = depth[order]  # ticket -> dependency level
width = np.bincount(dl)
print(f"level {lev}: rows {rows} depth {nlev} sweep span {(stored.max()-t0)/1e3:.1f} us "
      f"({(stored.max()-t0)/nlev:.0f} ns per dependency level)")
print(f"  width median {np.median(width):.0f} max {width.max()}")
print(f"  start->ready median {np.median(ready-start):.0f} p90 {np.percentile(ready-start,90):.0f} ns; "
      f"ready->stored median {np.median(stored-ready):.0f} p99 {np.percentile(stored-ready,99):.0f} ns; compute cyc {np.median(cy1-cy0):.0f}")
done = np.array([stored[dl == d].max() for d in range(nlev)]) - t0
first = np.array([ready[dl == d].min() for d in range(nlev)]) - t0
lastready = np.array([ready[dl == d].max() for d in range(nlev)]) - t0
st0 = np.array([start[dl == d].min() for d in range(nlev)]) - t0
st1 = np.array([start[dl == d].max() for d in range(nlev)]) - t0
step = np.diff(done)
print(f"  per-level done step median {np.median(step):.0f} ns p90 {np.percentile(step,90):.0f}")
print(f"  (done[d-1] -> last ready[d]) median {np.median(lastready[1:]-done[:-1]):.0f} ns;"
      f" (done[d-1] -> last start[d]) median {np.median(st1[1:]-done[:-1]):.0f} ns")
print(f"  spread of ready within a level median {np.median(lastready-first):.0f} ns")
# which rows are last in their level: their deps' finishing time vs their ready time
lag = []
inv = np.empty(rows, np.int64); inv[order] = np.arange(rows)
for d in range(1, min(nlev, 400)):
    tk = np.where(dl == d)[0]
    t_last = tk[np.argmax(ready[tk])]
    i = order[t_last]
    js = ci[ro[i]:ro[i + 1]]; js = js[js < i]
    dep_done = stored[inv[js]].max()
    lag.append((ready[t_last] - dep_done, start[t_last] - dep_done, js.size))
lag = np.array(lag)
print(f"  last row of a level: ready - max(dep stored) median {np.median(lag[:,0]):.0f} ns, "
      f"start - max(dep stored) median {np.median(lag[:,1]):.0f} ns, deps median {np.median(lag[:,2]):.0f}")
cys = tr[:, 5]
w6 = buf.cpu().numpy().reshape(rows, 10)[:, 6]
issue = (w6 & 0xFFFFFFFF).astype(np.float64); fac = (w6 >> 32).astype(np.float64)
w7 = buf.cpu().numpy().reshape(rows, 10)[:, 7]
spins = (w7 & 0xFFFFFFFF).astype(np.float64); poll1 = (w7 >> 32).astype(np.float64)
print(f"  cycles: start->issued median {np.median(issue):.0f} p90 {np.percentile(issue,90):.0f}; "
      f"start->factors {np.median(fac):.0f}; start->ready {np.median(cy0-cys):.0f} p90 {np.percentile(cy0-cys,90):.0f}")
print(f"  poll spins: share with 0 {np.mean(spins==0):.2f}, median {np.median(spins):.0f}, p90 {np.percentile(spins,90):.0f}")
z = spins == 0
print(f"  rows with no spin: start->ready cycles median {np.median((cy0-cys)[z]):.0f}  (pure overhead: issue+factors+one poll pass per 6 deps)")
print(f"  no-spin rows: start->first poll returned median {np.median(poll1[z]):.0f} (factors at {np.median(fac[z]):.0f}); "
      f"first poll -> ready {np.median((cy0-cys)[z]-poll1[z]):.0f} cycles")
w9 = buf.cpu().numpy().reshape(rows, 10)[:, 9]
plain = (w9 & 0xFFFFFFFF).astype(np.float64); ry = (w9 >> 32).astype(np.float64)
w8 = buf.cpu().numpy().reshape(rows, 10)[:, 8]
probe = (w8 & 0xFFFFFFFF).astype(np.float64); swait = (w8 >> 32).astype(np.float64)
print(f"  stage wait cycles: median {np.median(swait):.0f} p90 {np.percentile(swait,90):.0f} mean {swait.mean():.0f}")
print(f"  probe RTT (settled rin line): strong median {np.median(probe):.0f} p90 {np.percentile(probe,90):.0f}; "
      f"ld.cg median {np.median(plain):.0f} p90 {np.percentile(plain,90):.0f} cycles")
print(f"  first dependency poll RTT (no-spin rows): median {np.median(ry[z]):.0f} p90 {np.percentile(ry[z],90):.0f}; all rows median {np.median(ry):.0f}")
