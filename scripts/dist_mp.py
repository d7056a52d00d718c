"""Mode R with one process per GPU (NCCL): run with
    python -m torch.distributed.run --nproc-per-node G --master-addr 127.0.0.1 scripts/dist_mp.py [N] [RANKS]
Every rank solves its engine of the N^3 5x5 Euler system decomposed into RANKS
(>= G) RCB ranks consolidated onto G engines; rank 0 then repeats the solve
with all G engines on its own GPU (bcs_dist_solve) and checks that the
solutions are bit-identical, and prints both timings."""
import os
import sys
import time

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_07882_b200 import bcs, gen  # noqa: E402

rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
ranks = int(sys.argv[2]) if len(sys.argv) > 2 else world
torch.cuda.set_device(local)
dist.init_process_group("gloo")  # only to broadcast the NCCL id
uid = [bcs.comm_unique_id() if rank == 0 else None]
dist.broadcast_object_list(uid, src=0)
ctx = bcs.Context(local)
ctx.comm_init(rank, world, uid[0])
s = gen.hex_euler(n)
cfg = bcs.SolverConfig(preconditioner=bcs.PrecondKind.AMG, relTol=1e-8, maxIters=1000,
                       amg=bcs.AmgConfig(maxLevels=30, minCoarseRows=8))
for it in range(3):
    dist.barrier()
    t = time.perf_counter()
    x, r = ctx.dist_solve_mp(s.A, s.b, s.x0, s.centroids, ranks, cfg)
    dt = time.perf_counter() - t
if rank == 0:
    t = time.perf_counter()
    xr, rr = ctx.dist_solve(s.A, s.b, s.x0, s.centroids, ranks, world, cfg)
    dr = time.perf_counter() - t
    same = x.values.tobytes() == xr.values.tobytes()
    print(f"{world} processes, {n}^3, {ranks} ranks: iterations {r.iterations} (one device: {rr.iterations}), "
          f"{dt:.3f} s per solve (one device, {world} engines: {dr:.3f} s), bit-identical: {same}", flush=True)
dist.destroy_process_group()
