"""Mode-R partition layer (host C++ in libbcs, no device): decompose /
buildPartitioned / consolidate against the reference (partition.cpp:21-248)
and the oracle; plus a world-size-2 gloo check that every rank's send plan
matches its peers' halo columns."""
import os

import numpy as np
import pytest

from oracle_lib import ref_mesh_2d, ref_mesh_tube, ref_partition
from paper_2403_07882_b200 import bcs, gen


def gather_src(A, src):
    nn = A.n * A.n
    allv = np.concatenate([A.diag.reshape(-1, nn), A.upper.reshape(-1, nn), A.lower.reshape(-1, nn)])
    return allv[src].reshape(-1)


CASES = [("hex", lambda: gen.hex_euler(6, 5, 4)), ("hex_scr", lambda: gen.hex_euler(5, 5, 5, scramble_seed=4)),
         ("coupled", lambda: gen.hex_coupled(4, 6, 3))]


@pytest.mark.parametrize("name,maker", CASES)
@pytest.mark.parametrize("ranks,engines", [(1, 0), (2, 0), (3, 0), (4, 0), (8, 0), (2, 1), (4, 2), (4, 4), (3, 2),
                                           (8, 3)])
def test_partition_matches_reference(ref, name, maker, ranks, engines):
    s = maker()
    A = s.A
    P = bcs.Partition(A.n_cells, A.owner, A.neighbour, s.centroids, ranks, engines)
    refparts = ref_partition(ref, A, s.centroids, ranks, engines)
    assert P.count() == len(refparts) == (engines if engines else ranks)
    for i, rp in enumerate(refparts):
        p = P.part(i)
        for k in ("row_start", "row_end"):
            assert p[k] == rp[k]
        for k in ("ro", "ci", "halo_row", "halo_col", "halo_peer", "send_peer", "send_row"):
            assert np.array_equal(p[k], rp[k]), k
        assert gather_src(A, p["src"]).tobytes() == rp["vals"].tobytes()
        assert gather_src(A, p["halo_src"]).tobytes() == rp["halo_vals"].tobytes()


@pytest.mark.parametrize("ranks", [1, 2, 3, 4, 5, 8])
def test_decomposition_matches_oracle(oracle, ranks):
    s = gen.hex_euler(7, 6, 5, scramble_seed=2)
    P = bcs.Partition(s.A.n_cells, s.A.owner, s.A.neighbour, s.centroids, ranks)
    a = P.decomposition()
    b = oracle.decompose(s.centroids, ranks)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)


def test_known_answer_decompositions(ref):
    # test_partition.cpp:48-73: 3x3 mesh on 3 ranks -> rows [0,3,6,9]; tube 100 on 4 -> 25 each
    nc, o, ne, cen = ref_mesh_2d(ref, 3, 3)
    P = bcs.Partition(nc, o, ne, cen, 3)
    assert P.decomposition()[1].tolist() == [0, 3, 6, 9]
    nc, o, ne, cen = ref_mesh_tube(ref, 100)
    P = bcs.Partition(nc, o, ne, cen, 4)
    assert P.decomposition()[1].tolist() == [0, 25, 50, 75, 100]


def test_single_rank_has_no_halo():
    s = gen.hex_euler(4)
    p = bcs.Partition(s.A.n_cells, s.A.owner, s.A.neighbour, s.centroids, 1).part(0)
    assert p["halo_row"].size == 0 and p["send_row"].size == 0


def test_bad_rank_count_is_invalid_argument():
    s = gen.hex_euler(2)
    with pytest.raises(ValueError, match="1 <= nRanks <= nCells"):
        bcs.Partition(s.A.n_cells, s.A.owner, s.A.neighbour, s.centroids, 9)


def _gloo_worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        s = gen.hex_euler(6, 6, 6, scramble_seed=9)
        P = bcs.Partition(s.A.n_cells, s.A.owner, s.A.neighbour, s.centroids, world)
        mine = P.part(rank)
        # what I send to each peer (global rows) and which global columns I need from each peer
        sends = {int(pp): sorted(set((mine["row_start"] + mine["send_row"][mine["send_peer"] == pp]).tolist()))
                 for pp in set(mine["send_peer"].tolist())}
        needs = {int(pp): sorted(set(mine["halo_col"][mine["halo_peer"] == pp].tolist()))
                 for pp in set(mine["halo_peer"].tolist())}
        allsends = [None] * world
        allneeds = [None] * world
        dist.all_gather_object(allsends, sends)
        dist.all_gather_object(allneeds, needs)
        ok = all(allsends[src].get(dst, []) == allneeds[dst].get(src, []) for src in range(world) for dst in range(world)
                 if src != dst)
        q.put((rank, ok, sum(len(v) for v in needs.values())))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_send_plans_match_halos():
    import multiprocessing as mp
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok, _ in res), res
    assert all(n > 0 for _, _, n in res)


def _gloo_exchange_worker(rank, world, port, ranks, q):
    """One process per engine: pack the rows of the exchange plan from this
    engine's slice of a known global vector, exchange them with point-to-point
    gloo messages in the order the NCCL path uses (peers ascending), and check
    every halo entry reads its column's value from the receive buffer."""
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        s = gen.hex_euler(7, 6, 5, scramble_seed=3)
        n = 5
        P = bcs.Partition(s.A.n_cells, s.A.owner, s.A.neighbour, s.centroids, ranks, world)  # engines = processes
        mine = P.part(rank)
        x = P.exchange(rank)
        g = np.arange(s.A.n_cells * n, dtype=np.float64).reshape(-1, n) * 1.5 + 0.25  # global (renumbered) vector
        local = g[mine["row_start"]:mine["row_end"]]
        send = local[x["send_row"]]
        recv = np.zeros((x["recv_global_row"].size, n))
        reqs, so, ro = [], 0, 0
        for peer in range(world):
            c = int(x["send_count"][peer])
            if c:
                reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(send[so:so + c])), peer))
            so += c
        bufs = []
        for peer in range(world):
            c = int(x["recv_count"][peer])
            if c:
                t = torch.zeros((c, n), dtype=torch.float64)
                reqs.append(dist.irecv(t, peer))
                bufs.append((ro, t))
            ro += c
        for r in reqs:
            r.wait()
        for o, t in bufs:
            recv[o:o + t.shape[0]] = t.numpy()
        ok = np.array_equal(recv, g[x["recv_global_row"]])
        ok = ok and np.array_equal(recv[x["halo_recv_idx"]], g[mine["halo_col"]])
        ok = ok and int(x["send_count"].sum()) == x["send_row"].size and int(x["send_count"][rank]) == 0
        q.put((rank, bool(ok), int(mine["halo_col"].size)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("ranks", [2, 5])
def test_gloo_world2_exchange_plan(ranks):
    """The multi-process Mode R halo exchange (bcs_partition_exchange_*, used by
    bcs_dist_solve_mp over NCCL) delivers exactly the halo columns, world size 2."""
    import multiprocessing as mp
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gloo_exchange_worker, args=(r, 2, port, ranks, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok, _ in res), res
    assert all(n > 0 for _, _, n in res)


def _gloo_upload_worker(rank, world, port, ranks, q):
    """One process per engine: the per-rank upload (bcs_partition_gather_values,
    what bcs_dist_solve_mp ships to its GPU) equals the reference's consolidated
    partition of that engine (local BSR values and halo blocks, bit for bit), and
    the engines' uploads together hold every LDU block exactly once as a local
    slot or once per coupling as a halo entry."""
    import torch
    import torch.distributed as dist
    from oracle_lib import Reference, ref_partition
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        s = gen.hex_euler(7, 6, 5, scramble_seed=3)
        A = s.A
        P = bcs.Partition(A.n_cells, A.owner, A.neighbour, s.centroids, ranks, world)
        loc, halo = P.gather_values(rank, A)
        refp = ref_partition(Reference(), A, s.centroids, ranks, world)[rank]
        ok = loc.tobytes() == refp["vals"].tobytes() and halo.tobytes() == refp["halo_vals"].tobytes()
        # every LDU block is uploaded exactly once: a local slot or a halo entry of one engine
        d = P.part(rank)
        mine = np.concatenate([d["src"], d["halo_src"]]).astype(np.int64)
        counts = torch.zeros(A.n_cells + 2 * A.nFaces(), dtype=torch.int64)
        counts.index_add_(0, torch.from_numpy(mine), torch.ones(mine.size, dtype=torch.int64))
        dist.all_reduce(counts)
        ok = ok and bool((counts == 1).all())
        q.put((rank, bool(ok), int(loc.size + halo.size)))
    finally:
        dist.destroy_process_group()


@pytest.mark.skipif(not os.path.exists(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                                    "oracle", "_ref", "libbcs_ref.so")), reason="oracle/_ref not built")
@pytest.mark.parametrize("ranks", [2, 4])
def test_gloo_world2_per_rank_upload(ranks):
    import multiprocessing as mp
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gloo_upload_worker, args=(r, 2, port, ranks, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok, _ in res), res
    s = gen.hex_euler(7, 6, 5, scramble_seed=3)
    # each engine uploads about half of the system, not all of it
    assert all(n < 0.75 * (s.A.diag.size + s.A.upper.size + s.A.lower.size) for _, _, n in res)
