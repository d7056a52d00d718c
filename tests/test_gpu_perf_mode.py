"""Performance mode (bcs Mode.PERF): multicolour block DILU smoothing.

The smoother of every coloured level is, by construction, the reference's
natural-order DILU (preconditioner.cpp:101-156) of the level matrix
symmetrically permuted by colour.  So its application is checked BIT-EXACTLY
against the CPU oracle's DILU on the permuted system (the permutation read back
through bcs_level_coloring), the colouring is checked to be a proper colouring
of every coloured level's pattern, and AMG-preconditioned solves are checked to
converge to the requested tolerance, with their iteration counts next to the
parity mode's (reported, not claimed equal).
"""
import numpy as np
import pytest

from oracle_lib import make_cfg
from paper_2403_07882_b200 import bcs, gen
from test_gpu_parity import random_system

pytestmark = pytest.mark.gpu

AMG = bcs.AmgConfig(maxLevels=30, minCoarseRows=8)


@pytest.fixture(scope="module")
def ctx():
    c = bcs.Context(0)
    yield c
    c.close()


def permuted_ldu(A, perm):
    """The LDU system with cells renumbered new = inv[old] (perm[new] = old):
    faces keep their order, owner < neighbour is restored by swapping the
    upper and lower blocks of a face whose ends change order."""
    nc, n, nn = A.n_cells, A.n, A.n * A.n
    inv = np.empty(nc, np.int64)
    inv[perm] = np.arange(nc)
    o, ne = inv[A.owner], inv[A.neighbour]
    flip = o > ne
    up = A.upper.reshape(-1, nn).copy()
    lo = A.lower.reshape(-1, nn).copy()
    up[flip], lo[flip] = A.lower.reshape(-1, nn)[flip], A.upper.reshape(-1, nn)[flip]
    owner = np.where(flip, ne, o).astype(np.int32)
    neigh = np.where(flip, o, ne).astype(np.int32)
    diag = A.diag.reshape(nc, nn)[perm].reshape(-1)
    return bcs.BlockLduMatrix(nc, owner, neigh, n, np.ascontiguousarray(diag), up.reshape(-1), lo.reshape(-1))


SYSTEMS = {
    "euler8": lambda: gen.hex_euler(8).A,
    # >= 16384 rows per colour: one streaming launch per colour (k_mc_colour)
    "euler56": lambda: gen.hex_euler(56).A,
    "coupled56p": lambda: gen.hex_coupled(56, poly_seed=2).A,
    "euler7s": lambda: gen.hex_euler(7, scramble_seed=3).A,
    "coupled7p": lambda: gen.hex_coupled(7, poly_seed=2).A,
    "rand4": lambda: random_system(9, 7, 6, 4, 5)[0],
    "rand3": lambda: random_system(6, 5, 7, 3, 8)[0],
}


@pytest.mark.parametrize("name", list(SYSTEMS))
def test_perf_dilu_is_the_natural_dilu_of_the_colour_permuted_matrix(ctx, oracle, name):
    A = SYSTEMS[name]()
    ctx.set_topology(A)
    ctx.upload_ldu(A)
    ctx.precond_setup(bcs.SolverConfig(preconditioner=bcs.PrecondKind.DILU, mode=bcs.Mode.PERF))
    ncol, perm, off = ctx.level_coloring(0)
    assert 2 <= ncol <= 64
    if name.endswith("56") or name.endswith("56p"):
        assert A.n_cells >= 16384 * ncol  # one launch per colour (engine mcLaunchMin_)
    r = np.random.default_rng(7).uniform(-1, 1, A.n_cells * A.n)
    z = ctx.precond_apply(r)
    P = permuted_ldu(A, perm)
    rp = r.reshape(-1, A.n)[perm].reshape(-1)
    zp = oracle.precond_apply(P, make_cfg(precond=2), rp)
    zo = np.empty_like(zp).reshape(-1, A.n)
    zo[perm] = zp.reshape(-1, A.n)
    assert z.tobytes() == zo.reshape(-1).tobytes()


def _check_coloring(ro, ci, perm, off):
    color = np.empty(perm.size, np.int64)
    for c in range(off.size - 1):
        color[perm[off[c]:off[c + 1]]] = c
    rows = np.repeat(np.arange(ro.size - 1), np.diff(ro))
    off_diag = rows != ci
    assert not np.any(color[rows[off_diag]] == color[ci[off_diag]]), "coupled rows share a colour"
    # rows of one colour are in index order (deterministic placement)
    for c in range(off.size - 1):
        seg = perm[off[c]:off[c + 1]]
        assert np.all(np.diff(seg) > 0)


@pytest.mark.parametrize("maker", [lambda: gen.hex_euler(24), lambda: gen.hex_coupled(16, poly_seed=1),
                                   lambda: gen.hex_euler(16, 16, 12, aspect=100.0, scramble_seed=4)])
@pytest.mark.parametrize("method", [bcs.KrylovMethod.GMRES, bcs.KrylovMethod.PBiCGStab])
def test_perf_amg_solve(ctx, maker, method):
    s = maker()
    A = s.A
    ctx.set_topology(A)
    ctx.upload_ldu(A)
    base = dict(method=method, preconditioner=bcs.PrecondKind.AMG, relTol=1e-8, maxIters=1000, amg=AMG)
    xp = s.x0.values.copy()
    rp = ctx.solve(s.b.values, xp, bcs.SolverConfig(mode=bcs.Mode.PERF, **base))
    assert rp.converged
    # the true residual meets the tolerance (the smoother is a different operator)
    assert ctx.residual(s.b.values, xp) <= 1e-8 * rp.initialResidual * 1.0000001
    coloured = 0
    for lvl in range(ctx.amg_depth() - 1):
        ncol, perm, off = ctx.level_coloring(lvl)
        if ncol == 0:
            continue
        coloured += 1
        ro, ci, _, _ = ctx.amg_level(lvl, A.n)
        _check_coloring(ro, ci, perm, off)
    assert coloured >= 1
    x = s.x0.values.copy()
    r = ctx.solve(s.b.values, x, bcs.SolverConfig(**base))
    assert r.converged
    # reported, not claimed equal: the colour-ordered smoother costs some iterations
    assert rp.iterations <= 3 * r.iterations + 2, (rp.iterations, r.iterations)
    np.testing.assert_allclose(xp, x, rtol=0, atol=1e-6 * np.abs(x).max())


@pytest.mark.parametrize("maker", [lambda: gen.hex_euler(24), lambda: gen.hex_coupled(16, poly_seed=1),
                                   lambda: gen.hex_euler(16, 16, 12, aspect=100.0, scramble_seed=4)])
def test_perf_block_jacobi_amg_solve(ctx, maker):
    """Mode.PERF_JACOBI: block-Jacobi smoothing (0.8 D^-1 per block row) on the
    levels above the one-CTA tail: converges to the requested tolerance (true
    residual), iterations reported next to the parity mode's."""
    s = maker()
    A = s.A
    ctx.set_topology(A)
    ctx.upload_ldu(A)
    base = dict(preconditioner=bcs.PrecondKind.AMG, relTol=1e-8, maxIters=1000, amg=AMG)
    xj = s.x0.values.copy()
    rj = ctx.solve(s.b.values, xj, bcs.SolverConfig(mode=bcs.Mode.PERF_JACOBI, **base))
    assert rj.converged
    assert ctx.residual(s.b.values, xj) <= 1e-8 * rj.initialResidual * 1.0000001
    r = ctx.solve(s.b.values, s.x0.values.copy(), bcs.SolverConfig(**base))
    assert rj.iterations <= 6 * r.iterations + 5, (rj.iterations, r.iterations)


def _bsr_matvec(ro, ci, v, n, x):
    blocks = v.reshape(-1, n, n)
    xb = x.reshape(-1, n)
    rows = np.repeat(np.arange(ro.size - 1), np.diff(ro))
    y = np.zeros_like(xb)
    np.add.at(y, rows, np.einsum("kab,kb->ka", blocks, xb[ci]))
    return y.reshape(-1)


@pytest.mark.parametrize("maker", [lambda: gen.hex_euler(12), lambda: gen.hex_coupled(12, poly_seed=2)])
def test_block_jacobi_vcycle_against_numpy(ctx, maker):
    """Two-level V-cycle of Mode.PERF_JACOBI against a numpy restatement:
    z = w D^-1 r, res = r - A z, z += P A_c^-1 R res, z += w D^-1 (r - A z)
    (w = 0.8; D the diagonal blocks; R/P the aggregate sum/injection)."""
    s = maker()
    A = s.A
    n = A.n
    ctx.set_topology(A)
    ctx.upload_ldu(A)
    ctx.precond_setup(bcs.SolverConfig(preconditioner=bcs.PrecondKind.AMG, mode=bcs.Mode.PERF_JACOBI,
                                       amg=bcs.AmgConfig(maxLevels=2, minCoarseRows=8)))
    assert ctx.amg_depth() == 2
    ro, ci, v, agg = ctx.amg_level(0, n)
    cro, cci, cv, _ = ctx.amg_level(1, n)
    assert ro.size - 1 > 512  # above the one-CTA tail: smoothed by block Jacobi
    r = np.random.default_rng(5).uniform(-1, 1, A.n_cells * n)
    z = ctx.precond_apply(r)

    rows = np.repeat(np.arange(ro.size - 1), np.diff(ro))
    D = v.reshape(-1, n, n)[ci == rows]  # one diagonal block per row, in row order
    def smooth(x):
        return 0.8 * np.linalg.solve(D, x.reshape(-1, n, 1)).reshape(-1)
    zn = smooth(r)
    res = r - _bsr_matvec(ro, ci, v, n, zn)
    nc = cro.size - 1
    rc = np.zeros((nc, n))
    np.add.at(rc, agg, res.reshape(-1, n))
    Ac = np.zeros((nc * n, nc * n))
    crows = np.repeat(np.arange(nc), np.diff(cro))
    for k, (i, j) in enumerate(zip(crows, cci)):
        Ac[i * n:(i + 1) * n, j * n:(j + 1) * n] = cv.reshape(-1, n, n)[k]
    ec = np.linalg.solve(Ac, rc.reshape(-1)).reshape(-1, n)
    zn = zn + ec[agg].reshape(-1)
    zn = zn + smooth(r - _bsr_matvec(ro, ci, v, n, zn))
    np.testing.assert_allclose(z, zn, rtol=0, atol=1e-10 * np.abs(zn).max())
