"""GPU busy vs idle within one 128^3 solve (torch.profiler / CUPTI kernel records)."""
import os, sys, time, json
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
    x = s.x0.values.copy()
    ctx.solve(s.b.values, x, cfg)
torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    x = s.x0.values.copy()
    t0 = time.perf_counter()
    r = ctx.solve(s.b.values, x, cfg)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
iv = sorted((e.time_range.start, e.time_range.end, e.name) for e in ev)
busy = 0.0
cur_s, cur_e = None, None
for s0, e0, _ in iv:
    if cur_e is None or s0 > cur_e:
        if cur_e is not None:
            busy += cur_e - cur_s
        cur_s, cur_e = s0, e0
    else:
        cur_e = max(cur_e, e0)
if cur_e is not None:
    busy += cur_e - cur_s
span = (iv[-1][1] - iv[0][0]) if iv else 0
print(f"wall {wall*1e3:.1f} ms; GPU span {span/1e3:.1f} ms; busy {busy/1e3:.1f} ms ({100*busy/max(span,1):.1f}%); "
      f"{len(iv)} GPU records")
# largest gaps
gaps = []
for (a0, a1, an), (b0, b1, bn) in zip(iv, iv[1:]):
    if b0 > a1:
        gaps.append((b0 - a1, an[:40], bn[:40]))
gaps.sort(reverse=True)
tot_gap = sum(g[0] for g in gaps)
print(f"idle between records: {tot_gap/1e3:.1f} ms in {len(gaps)} gaps; >20us: {sum(g[0] for g in gaps if g[0]>20)/1e3:.1f} ms")
for g in gaps[:12]:
    print(f"  {g[0]:8.1f} us after {g[1]} before {g[2]}")
from collections import Counter
small = Counter()
for g in gaps:
    b = int(min(g[0], 99) // 5) * 5
    small[b] += g[0]
print("gap histogram (us bucket: total us):", sorted(small.items())[:12])
tot = Counter()
cnt = Counter()
for s0, e0, nm in iv:
    k = nm.split("(")[0][:60]
    tot[k] += e0 - s0
    cnt[k] += 1
print("kernel time by name (ms, count):")
for k, v in tot.most_common(18):
    print(f"  {v/1e3:8.2f}  x{cnt[k]:5d}  {k}")
