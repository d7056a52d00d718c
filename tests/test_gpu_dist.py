"""Mode R on the device (bcs_dist_solve) against the reference's own
distributedSolve (partition.cpp:370-479, compiled in oracle/_ref): the same
ranks/engines give the same iteration counts (+-1) and solutions, and the
iteration growth with the engine count that SURVEY §8(e) documents."""
import numpy as np
import pytest

from oracle_lib import make_cfg, ref_distributed_solve
from paper_2403_07882_b200 import bcs, gen

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    c = bcs.Context(0)
    yield c
    c.close()


@pytest.mark.parametrize("maker", [lambda: gen.hex_euler(10), lambda: gen.hex_coupled(8),
                                   lambda: gen.hex_euler(9, scramble_seed=3)])
@pytest.mark.parametrize("ranks,engines", [(1, 1), (2, 1), (2, 2), (4, 2), (4, 4), (3, 2), (8, 3), (8, 8)])
@pytest.mark.parametrize("method,pc", [(0, 3), (1, 3), (0, 2)])
def test_dist_solve_matches_reference(ctx, ref, maker, ranks, engines, method, pc):
    s = maker()
    cfg_t = make_cfg(method=method, precond=pc, max_iters=400)
    cfg = bcs.SolverConfig(method=bcs.KrylovMethod(method), preconditioner=bcs.PrecondKind(pc), relTol=1e-8,
                           maxIters=400, amg=bcs.AmgConfig(maxLevels=30, minCoarseRows=8))
    rc, xr, rr = ref_distributed_solve(ref, s.A, s.b.values, s.x0.values, s.centroids, ranks, engines, cfg_t)
    assert rc == 0, ref.err()
    x, r = ctx.dist_solve(s.A, s.b, s.x0, s.centroids, ranks, engines, cfg)
    assert r.converged == bool(rr.converged)
    assert abs(r.iterations - rr.iterations) <= 1, (r.iterations, rr.iterations)
    np.testing.assert_allclose(r.initialResidual, rr.initial_residual, rtol=1e-12)
    if rr.converged:
        np.testing.assert_allclose(x.values, xr, rtol=0, atol=1e-6 * np.abs(xr).max())
        for k in ("convert", "setup", "solve", "retrieve"):
            assert k in r.timings


def test_dist_single_engine_equals_serial(ctx):
    """ranks = engines = 1 is the serial solve (identity renumbering)."""
    s = gen.hex_euler(12)
    cfg = bcs.SolverConfig(preconditioner=bcs.PrecondKind.AMG, relTol=1e-8, maxIters=400,
                           amg=bcs.AmgConfig(maxLevels=30, minCoarseRows=8))
    x1, r1 = ctx.dist_solve(s.A, s.b, s.x0, s.centroids, 1, 1, cfg)
    ctx.set_topology(s.A)
    ctx.upload_ldu(s.A)
    x2 = s.x0.values.copy()
    r2 = ctx.solve(s.b.values, x2, cfg)
    assert r1.iterations == r2.iterations
    assert x1.values.tobytes() == x2.tobytes()


def test_dist_iterations_grow_with_engines(ctx):
    """Block-Jacobi across engines: GMRES+AMG iterations grow with the engine
    count (7/15/18/22 at 32^3)."""
    s = gen.hex_euler(16)
    cfg = bcs.SolverConfig(preconditioner=bcs.PrecondKind.AMG, relTol=1e-8, maxIters=400,
                           amg=bcs.AmgConfig(maxLevels=30, minCoarseRows=8))
    its = [ctx.dist_solve(s.A, s.b, s.x0, s.centroids, g, g, cfg)[1].iterations for g in (1, 2, 4, 8)]
    assert its[0] < its[1] <= its[2] + 1 and its[1] <= its[3] + 1


def test_dist_mp_single_process_equals_one_device(ctx):
    """The multi-process Mode R path (NCCL communicator of one process): the
    same arithmetic as the one-device Mode R with one engine, bit for bit."""
    uid = bcs.comm_unique_id()
    ctx.comm_init(0, 1, uid)
    for ranks in (1, 3):
        s = gen.hex_euler(9, scramble_seed=5)
        cfg = bcs.SolverConfig(preconditioner=bcs.PrecondKind.AMG, relTol=1e-9, maxIters=500,
                               amg=bcs.AmgConfig(maxLevels=30, minCoarseRows=8))
        x1, r1 = ctx.dist_solve(s.A, s.b, s.x0, s.centroids, ranks, 1, cfg)
        x2, r2 = ctx.dist_solve_mp(s.A, s.b, s.x0, s.centroids, ranks, cfg)
        assert r1.iterations == r2.iterations and r2.converged
        assert x1.values.tobytes() == x2.values.tobytes()


def test_dist_mp_requires_comm_init():
    c = bcs.Context(0)
    try:
        s = gen.hex_euler(4)
        cfg = bcs.SolverConfig(preconditioner=bcs.PrecondKind.AMG)
        with pytest.raises(ValueError, match="bcs_comm_init"):
            c.dist_solve_mp(s.A, s.b, s.x0, s.centroids, 2, cfg)
    finally:
        c.close()


@pytest.mark.parametrize("ranks,engines", [(2, 2), (4, 2), (8, 8)])
def test_dist_fgmres_matches_reference_gmres(ctx, ref, ranks, engines):
    """FGMRES in Mode R runs the reference's Arnoldi process: the iteration
    count of the reference's distributedSolve with GMRES, the same solution."""
    s = gen.hex_euler(10)
    cfg_t = make_cfg(method=0, precond=3, max_iters=400)
    cfg = bcs.SolverConfig(method=bcs.KrylovMethod.FGMRES, preconditioner=bcs.PrecondKind.AMG, relTol=1e-8,
                           maxIters=400, amg=bcs.AmgConfig(maxLevels=30, minCoarseRows=8))
    rc, xr, rr = ref_distributed_solve(ref, s.A, s.b.values, s.x0.values, s.centroids, ranks, engines, cfg_t)
    assert rc == 0, ref.err()
    x, r = ctx.dist_solve(s.A, s.b, s.x0, s.centroids, ranks, engines, cfg)
    assert r.converged and rr.converged and r.iterations == rr.iterations
    np.testing.assert_allclose(x.values, xr, rtol=0, atol=1e-6 * np.abs(xr).max())


@pytest.mark.parametrize("maker", [lambda: gen.hex_euler(10), lambda: gen.hex_coupled(8, scramble_seed=3)])
@pytest.mark.parametrize("ranks,engines", [(2, 2), (4, 2), (3, 2), (8, 3)])
@pytest.mark.parametrize("method", [0, 1])
def test_dist_exact_mode_bit_identical_to_reference(ctx, ref, maker, ranks, engines, method):
    """EXACT mode in Mode R: per-engine sequential dot partials folded by the
    reference's pairwise engine tree (partition.cpp:433-450) -- the reference's
    distributedSolve bit for bit: iterations, final residual and solution."""
    s = maker()
    cfg_t = make_cfg(method=method, precond=3, max_iters=400)
    cfg = bcs.SolverConfig(method=bcs.KrylovMethod(method), preconditioner=bcs.PrecondKind.AMG, relTol=1e-8,
                           maxIters=400, amg=bcs.AmgConfig(maxLevels=30, minCoarseRows=8), mode=bcs.Mode.EXACT)
    rc, xr, rr = ref_distributed_solve(ref, s.A, s.b.values, s.x0.values, s.centroids, ranks, engines, cfg_t)
    assert rc == 0, ref.err()
    x, r = ctx.dist_solve(s.A, s.b, s.x0, s.centroids, ranks, engines, cfg)
    assert r.iterations == rr.iterations and r.converged == bool(rr.converged)
    assert r.finalResidual == rr.final_residual
    assert x.values.tobytes() == xr.tobytes()


def test_dist_mp_exact_mode_equals_one_device(ctx):
    """EXACT mode through the NCCL path (one process) equals the one-device engines bit for bit."""
    uid = bcs.comm_unique_id()
    ctx.comm_init(0, 1, uid)
    s = gen.hex_euler(9, scramble_seed=5)
    cfg = bcs.SolverConfig(preconditioner=bcs.PrecondKind.AMG, relTol=1e-9, maxIters=500,
                           amg=bcs.AmgConfig(maxLevels=30, minCoarseRows=8), mode=bcs.Mode.EXACT)
    x1, r1 = ctx.dist_solve(s.A, s.b, s.x0, s.centroids, 3, 1, cfg)
    x2, r2 = ctx.dist_solve_mp(s.A, s.b, s.x0, s.centroids, 3, cfg)
    assert r1.iterations == r2.iterations and r2.converged
    assert x1.values.tobytes() == x2.values.tobytes()


def test_serial_system_survives_a_dist_solve():
    """A Mode R call on another system (other block size and cell count) borrows
    the context's sizes for its Krylov run and restores them: the serial matrix
    uploaded before solves bit-identically afterwards."""
    c = bcs.Context(0)
    try:
        s = gen.hex_euler(6)
        cfg = bcs.SolverConfig(preconditioner=bcs.PrecondKind.AMG, relTol=1e-8, maxIters=400,
                               amg=bcs.AmgConfig(maxLevels=30, minCoarseRows=8))
        c.set_topology(s.A)
        c.upload_ldu(s.A)
        x1 = s.x0.values.copy()
        r1 = c.solve(s.b.values, x1, cfg)
        t = gen.hex_coupled(8)
        xd, rd = c.dist_solve(t.A, t.b, t.x0, t.centroids, 4, 2, cfg)
        assert rd.converged
        x2 = s.x0.values.copy()
        r2 = c.solve(s.b.values, x2, cfg)
        assert r2.iterations == r1.iterations and x2.tobytes() == x1.tobytes()
        assert c.residual(s.b.values, x2) == pytest.approx(r2.finalResidual, rel=1e-9)
    finally:
        c.close()


@pytest.mark.parametrize("mode", [bcs.Mode.PERF, bcs.Mode.PERF_JACOBI])
def test_dist_perf_modes_converge(ctx, mode):
    """The performance smoothers inside Mode R engines: every engine's hierarchy
    is coloured (or Jacobi-smoothed) on its own; the solve reaches the tolerance."""
    s = gen.hex_euler(12)
    cfg = bcs.SolverConfig(preconditioner=bcs.PrecondKind.AMG, relTol=1e-8, maxIters=400,
                           amg=bcs.AmgConfig(maxLevels=30, minCoarseRows=8), mode=mode)
    x, r = ctx.dist_solve(s.A, s.b, s.x0, s.centroids, 4, 2, cfg)
    assert r.converged
    ctx.set_topology(s.A)
    ctx.upload_ldu(s.A)
    assert ctx.residual(s.b.values, x.values) <= 1e-8 * r.initialResidual * 1.01


@pytest.mark.parametrize("maker,ranks,engines", [(lambda: gen.hex_euler(10), 4, 2),
                                                 (lambda: gen.hex_coupled(9, scramble_seed=2, poly_seed=1), 5, 3),
                                                 (lambda: gen.hex_euler(8, 7, 9, aspect=20.0), 3, 3)])
@pytest.mark.parametrize("mode", [bcs.Mode.EXACT, bcs.Mode.PARITY])
def test_dist_solve_parts_matches_dist_solve(ctx, maker, ranks, engines, mode):
    """bcs_dist_solve_parts (distributedSolve on caller-built rank partitions,
    here the host partition layer's buildPartitioned output with its values
    gathered per rank) equals bcs_dist_solve on the same system bit for bit."""
    s = maker()
    A, n = s.A, s.A.n
    cfg = bcs.SolverConfig(preconditioner=bcs.PrecondKind.AMG, relTol=1e-8, maxIters=300,
                           amg=bcs.AmgConfig(maxLevels=30, minCoarseRows=8), mode=mode)
    x_ref, r_ref = ctx.dist_solve(A, s.b, s.x0, s.centroids, ranks, engines, cfg)
    P = bcs.Partition(A.n_cells, A.owner, A.neighbour, s.centroids, ranks)
    _, rro, o2n = P.decomposition()
    parts = []
    for r in range(ranks):
        d = P.part(r)
        loc, halo = P.gather_values(r, A)
        parts.append(dict(row_start=d["row_start"], row_end=d["row_end"], ro=d["ro"], ci=d["ci"], values=loc,
                          halo_row=d["halo_row"], halo_col=d["halo_col"], halo_peer=d["halo_peer"], halo_values=halo))
    # makeConsolidationPlan (partition.cpp:184-199): contiguous rank groups
    r2e = [(r * engines) // ranks for r in range(ranks)]
    ero, acc = [], {}
    for r in range(ranks):
        ero.append(acc.get(r2e[r], 0))
        acc[r2e[r]] = acc.get(r2e[r], 0) + (rro[r + 1] - rro[r])
    # scatterVector: new numbering
    bnew = np.empty_like(s.b.values).reshape(-1, n)
    xnew = np.empty_like(s.x0.values).reshape(-1, n)
    bnew[o2n] = s.b.values.reshape(-1, n)
    xnew[o2n] = s.x0.values.reshape(-1, n)
    x, r = ctx.dist_solve_parts(parts, bnew.reshape(-1), xnew.reshape(-1), n, engines, r2e, ero, cfg)
    assert r.iterations == r_ref.iterations
    assert x.reshape(-1, n)[o2n].tobytes() == np.asarray(x_ref.values).tobytes()


def test_dist_solve_parts_rejects_bad_plans(ctx):
    """The reference's errors on bad consolidation plans (partition.cpp:184-199)
    and rank lists, as invalid_argument -> ValueError, without touching the device state."""
    s = gen.hex_euler(6)
    A, n = s.A, s.A.n
    P = bcs.Partition(A.n_cells, A.owner, A.neighbour, s.centroids, 2)
    parts = []
    for r in range(2):
        d = P.part(r)
        loc, halo = P.gather_values(r, A)
        parts.append(dict(row_start=d["row_start"], row_end=d["row_end"], ro=d["ro"], ci=d["ci"], values=loc,
                          halo_row=d["halo_row"], halo_col=d["halo_col"], halo_peer=d["halo_peer"], halo_values=halo))
    cfg = bcs.SolverConfig(preconditioner=bcs.PrecondKind.AMG, relTol=1e-8, amg=bcs.AmgConfig(maxLevels=30, minCoarseRows=8))
    b = np.ones(A.n_cells * n)
    with pytest.raises(ValueError, match="makeConsolidationPlan"):
        ctx.dist_solve_parts(parts, b, b * 0, n, 3, [0, 1], [0, 0], cfg)
    with pytest.raises(ValueError, match="rank mapped to no engine"):
        ctx.dist_solve_parts(parts, b, b * 0, n, 1, [0, 1], [0, 0], cfg)
    with pytest.raises(ValueError, match="block size"):
        ctx.dist_solve_parts(parts, b, b * 0, 7, 1, [0, 0], [0, 0], cfg)
    # the context still solves afterwards
    x, r = ctx.dist_solve_parts(parts, b, b * 0, n, 1, [0, 0], [0, parts[0]["row_end"] - parts[0]["row_start"]], cfg)
    assert r.converged
