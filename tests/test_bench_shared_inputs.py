"""bench.py's multi-process Mode R keeps ONE copy of the weak-scaling system
per node (bench.shared_inputs): rank 0 generates it into file-backed shared
mappings, the other ranks map the same pages.  Checked with gloo, world 2,
on CPU: both ranks see exactly the system a direct generation gives, and the
mappings are removed afterwards."""
import argparse
import os
import sys

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _worker(rank, world, port, system, q):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    from paper_2403_07882_b200 import gen
    args = argparse.Namespace(system=system, poly=1 if system == "coupled" else -1, aspect=1.0, scramble=-1)
    dims = (12, 10, 8)
    sh = bench.shared_inputs(args, dims, rank, world)
    ok = sh is not None
    if ok:
        s = sh.system
        ref = (gen.hex_coupled(*dims, poly_seed=1) if system == "coupled" else gen.hex_euler(*dims))
        for a, b in ((s.A.owner, ref.A.owner), (s.A.neighbour, ref.A.neighbour), (s.A.diag, ref.A.diag),
                     (s.A.upper, ref.A.upper), (s.A.lower, ref.A.lower), (s.b.values, ref.b.values),
                     (s.x0.values, ref.x0.values), (s.centroids, ref.centroids)):
            ok = ok and np.array_equal(np.asarray(a), np.asarray(b))
        path = sh.path
        dist.barrier()
        sh.remove(rank)
        dist.barrier()
        ok = ok and not os.path.exists(path)
    q.put((rank, ok))
    dist.destroy_process_group()


@pytest.mark.parametrize("system", ["euler", "coupled"])
def test_shared_inputs_world2(system):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + (os.getpid() % 1000)
    ps = [ctx.Process(target=_worker, args=(r, 2, port, system, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=300) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    assert res == {0: True, 1: True}
