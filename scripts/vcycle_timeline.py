"""Real (non-ncu) kernel durations and inter-kernel gaps of one V-cycle in a
128^3 solve (torch.profiler / CUPTI records): which levels and which gaps
the step is made of."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_07882_b200 import bcs, gen

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
method = sys.argv[2] if len(sys.argv) > 2 else "gmres"
mode = {"parity": bcs.Mode.PARITY, "perf": bcs.Mode.PERF, "jacobi": bcs.Mode.PERF_JACOBI}[sys.argv[3] if len(sys.argv) > 3 else "parity"]
s = gen.hex_euler(n)
cfg = bcs.SolverConfig(method=bcs.KrylovMethod.FGMRES if method == "fgmres" else bcs.KrylovMethod.GMRES,
                       preconditioner=bcs.PrecondKind.AMG, relTol=1e-8, maxIters=1000,
                       amg=bcs.AmgConfig(maxLevels=30, minCoarseRows=8), mode=mode)
ctx = bcs.Context(0)
ctx.set_stream(torch.cuda.current_stream().cuda_stream)
ctx.set_topology(s.A)
ctx.upload_ldu(s.A)
for _ in range(2):
    ctx.solve(s.b.values, s.x0.values.copy(), cfg)
torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    r = ctx.solve(s.b.values, s.x0.values.copy(), cfg)
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
iv = sorted((e.time_range.start, e.time_range.end, e.name.split("(")[0].replace("void ", "")) for e in ev)
# the V-cycles: from a k_sweep2 fwd launch following a k_scale_by/k_spmv to the next
starts = [i for i, (_, _, nm) in enumerate(iv) if "k_scale_by" in nm]
for l in range(ctx.amg_depth() - 1):
    import ctypes
    rr, nz = ctypes.c_int(), ctypes.c_int()
    ctx._lib.bcs_amg_level_sizes(ctx.h, l, ctypes.byref(rr), ctypes.byref(nz))
    rows_l, nnz_l = rr.value, nz.value
    d = ctx.schedule_depth(l)
    print(f"level {l}: rows {rows_l} nnz {nnz_l} depth {d} width {rows_l / max(d, 1):.1f}")
print(f"solve: {r.iterations} its, {len(iv)} GPU records, span {(iv[-1][1]-iv[0][0])/1e3:.1f} ms")
if len(starts) >= 3:
    a, b = starts[1], starts[2]
    tot_k = sum(e - s0 for s0, e, _ in iv[a:b])
    tot_g = sum(max(0.0, iv[k + 1][0] - iv[k][1]) for k in range(a, b - 1))
    print(f"one Arnoldi step: {(iv[b][0]-iv[a][0])/1e3:.2f} ms, kernels {tot_k/1e3:.2f} ms, gaps {tot_g/1e3:.2f} ms, {b-a} launches")
    for k in range(a, b):
        s0, e0, nm = iv[k]
        gap = iv[k + 1][0] - e0 if k + 1 < len(iv) else 0
        print(f"  {e0 - s0:9.1f} us  gap {gap:6.1f}  {nm[:60]}")
