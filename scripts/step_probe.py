"""Per-step breakdown of the bench step (upload + solve) with host timers and syncs."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2403_07882_b200 import bcs, gen

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
s = gen.hex_euler(n)
A = s.A
cfg = bcs.SolverConfig(preconditioner=bcs.PrecondKind.AMG, relTol=1e-8, maxIters=1000,
                       amg=bcs.AmgConfig(maxLevels=30, minCoarseRows=8))
dev = torch.device("cuda", 0)
ctx = bcs.Context(0)
st = torch.cuda.current_stream(dev)
ctx.set_stream(st.cuda_stream)
d = [torch.from_numpy(a).to(dev) for a in (A.diag, A.upper, A.lower, s.b.values, s.x0.values)]
dx = torch.empty_like(d[4])
ctx.set_topology(A)
for it in range(6):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ctx.upload_ldu_device(d[0].data_ptr(), d[1].data_ptr(), d[2].data_ptr())
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    dx.copy_(d[4])
    r = ctx.solve_device(d[3].data_ptr(), dx.data_ptr(), cfg)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    free, tot = torch.cuda.mem_get_info(dev)
    print(f"step {it}: upload {1e3*(t1-t0):.1f} ms solve {1e3*(t2-t1):.1f} ms (amgSetup {1e3*r.timings['amgSetup']:.1f} "
          f"krylov {1e3*r.timings['krylov']:.1f}) used {(tot-free)/1e9:.2f} GB", flush=True)
ctx.close()
