"""Host->device LDU upload (bcs_upload_ldu: H2D + replaceValues permutation) at
128^3 5x5 (2.92 GB of values) from pageable numpy arrays (what a std::vector
caller passes) vs page-locked arrays.  Mean of 5 after 2 warm-ups."""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2403_07882_b200 import _native as N, bcs, gen  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
    s = gen.hex_euler(n)
    A = s.A
    ctx = bcs.Context(0)
    ctx.set_topology(A)

    def timed(M):
        ts = []
        for it in range(7):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            ctx.upload_ldu(M)
            torch.cuda.synchronize()
            if it >= 2:
                ts.append(time.perf_counter() - t0)
        return float(np.mean(ts))

    def pin(a):
        p = N.pinned_empty(a.size, a.dtype.type)
        p[:] = a
        return p

    nbytes = A.diag.nbytes + A.upper.nbytes + A.lower.nbytes
    t_pageable = timed(A)
    P = bcs.BlockLduMatrix(A.n_cells, A.owner, A.neighbour, A.n, pin(A.diag), pin(A.upper), pin(A.lower))
    t_pinned = timed(P)
    ctx.close()
    out = {"bytes": nbytes, "pageable_ms": 1e3 * t_pageable, "pinned_ms": 1e3 * t_pinned,
           "pageable_GBps": nbytes / t_pageable / 1e9, "pinned_GBps": nbytes / t_pinned / 1e9}
    # the whole drop-in call (SolvePipeline::solve, GMRES+AMG to 1e-8) from pageable vs pinned inputs
    cfg = bcs.SolverConfig(preconditioner=bcs.PrecondKind.AMG, relTol=1e-8, maxIters=1000,
                           amg=bcs.AmgConfig(maxLevels=30, minCoarseRows=8))
    pb = bcs.BlockVector(A.n_cells, A.n, pin(s.b.values))
    px = bcs.BlockVector(A.n_cells, A.n, pin(s.x0.values))
    pipe = bcs.SolvePipeline(0)
    for name, (M, b, x0) in {"e2e_pageable_s": (A, s.b, s.x0), "e2e_pinned_s": (P, pb, px)}.items():
        ts = []
        for it in range(5):
            t0 = time.perf_counter()
            pipe.solve(M, b, x0, bcs.Backend.EngineCsr, cfg)
            if it >= 2:
                ts.append(time.perf_counter() - t0)
        out[name] = float(np.mean(ts))
    print(json.dumps(out))


if __name__ == "__main__":
    main()
