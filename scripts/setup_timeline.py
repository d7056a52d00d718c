"""GPU timeline of one AMG setup at 128^3 (torch.profiler / CUPTI records):
kernel time vs the wall span, and the largest idle gaps (host syncs,
allocation, host-side work between launches) with the kernels around them.
(The first gap, ~1.4 ms after the first kernel, is the profiler's own CUPTI
buffer request on the first launch it records.)"""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_07882_b200 import bcs, gen

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
s = gen.hex_euler(n)
cfg = bcs.SolverConfig(preconditioner=bcs.PrecondKind.AMG, relTol=1e-8, maxIters=1000,
                       amg=bcs.AmgConfig(maxLevels=30, minCoarseRows=8))
ctx = bcs.Context(0)
ctx.set_stream(torch.cuda.current_stream().cuda_stream)
ctx.set_topology(s.A)
ctx.upload_ldu(s.A)
for _ in range(2):
    ctx.precond_setup(cfg)
torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    ctx.precond_setup(cfg)
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
iv = sorted((e.time_range.start, e.time_range.end, e.name.split("(")[0].replace("void ", "")[:40]) for e in ev)
span = iv[-1][1] - iv[0][0]
busy = sum(e - s0 for s0, e, _ in iv)
print(f"setup: {len(iv)} GPU records, span {span / 1e3:.2f} ms, kernel/copy time {busy / 1e3:.2f} ms, "
      f"idle {100 * (span - busy) / span:.1f}%")
gaps = []
for a, b in zip(iv, iv[1:]):
    g = b[0] - a[1]
    if g > 0:
        gaps.append((g, a[2], b[2]))
gaps.sort(reverse=True)
print(f"gaps > 20 us: {sum(1 for g in gaps if g[0] > 20)}, total {sum(g[0] for g in gaps if g[0] > 20) / 1e3:.2f} ms")
for g, a, b in gaps[:25]:
    print(f"  {g:8.1f} us  after {a:40s} before {b}")
from collections import Counter
c = Counter()
for s0, e, nm in iv:
    c[nm] += e - s0
for nm, t in c.most_common(15):
    print(f"  {t / 1e3:7.2f} ms  {nm}")
# context of the largest gap
k = max(range(len(iv) - 1), key=lambda i: iv[i + 1][0] - iv[i][1])
t0 = iv[0][0]
for s0, e, nm in iv[max(0, k - 4):k + 5]:
    print(f"    {(s0 - t0) / 1e3:9.3f} ms  {(e - s0):8.1f} us  {nm}")
