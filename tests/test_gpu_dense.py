"""Large coarsest levels (scrambled inputs): the blocked
dense LU and solve (csrc/k_dense.cu) against the oracle's denseFactor /
denseSolve restatement through whole V-cycle applications, bit for bit."""
import os

import numpy as np
import pytest

from oracle_lib import make_cfg
from paper_2403_07882_b200 import bcs, gen

pytestmark = pytest.mark.gpu


def _apply(ctx, s, cfg_t, r):
    ctx.set_topology(s.A)
    ctx.upload_ldu(s.A)
    ctx.precond_setup(bcs.SolverConfig(preconditioner=bcs.PrecondKind.AMG,
                                       amg=bcs.AmgConfig(maxLevels=cfg_t[6], minCoarseRows=cfg_t[7])))
    return ctx.precond_apply(r)


@pytest.mark.parametrize("threshold", ["1", "64", "65"])
def test_blocked_dense_forced_small(oracle, threshold, monkeypatch):
    """Scrambled 32^3: the blocked path forced on a small coarsest level
    (threshold 1 / 64 / 65 covers one- and two-panel factorisations)."""
    monkeypatch.setenv("BCS_DENSE_BLOCKED_MIN", threshold)
    ctx = bcs.Context(0)
    try:
        s = gen.hex_euler(32, scramble_seed=7)
        cfg = make_cfg(precond=3, max_levels=30, min_coarse=8)
        r = np.random.default_rng(5).uniform(-1, 1, s.A.n_cells * s.A.n)
        z = _apply(ctx, s, cfg, r)
        zo = oracle.precond_apply(s.A, cfg, r)
        assert z.tobytes() == zo.tobytes()
    finally:
        ctx.close()


def test_blocked_dense_scrambled64(oracle):
    """Scrambled 64^3 hits the 30-level cap with m = 665: the blocked path by default."""
    ctx = bcs.Context(0)
    try:
        s = gen.hex_euler(64, scramble_seed=7)
        cfg = make_cfg(precond=3, max_levels=30, min_coarse=8)
        r = np.random.default_rng(6).uniform(-1, 1, s.A.n_cells * s.A.n)
        z = _apply(ctx, s, cfg, r)
        assert ctx.amg_depth() == 30
        rows, _ = ctx.amg_level(29, s.A.n)[0].size - 1, None
        assert rows * s.A.n >= 256, "expected a coarsest level large enough for the blocked path"
        zo = oracle.precond_apply(s.A, cfg, r)
        assert z.tobytes() == zo.tobytes()
    finally:
        ctx.close()


def test_sweep_variants_bit_exact(oracle):
    """Natural 64^3 (fine level ~1.4 K rows per dependency level: the medium
    sweep variant) and scrambled 48^3 (shallow fine level, thousands of rows per
    level: the wide cp.async variant), V-cycle applications bit for bit."""
    ctx = bcs.Context(0)
    try:
        for s in (gen.hex_euler(64), gen.hex_euler(48, scramble_seed=11)):
            cfg = make_cfg(precond=3, max_levels=30, min_coarse=8)
            r = np.random.default_rng(8).uniform(-1, 1, s.A.n_cells * s.A.n)
            z = _apply(ctx, s, cfg, r)
            width = s.A.n_cells / max(1, ctx.schedule_depth(0))
            assert width > 1184, f"{s.name}: fine-level width {width:.0f} too narrow for the variants under test"
            zo = oracle.precond_apply(s.A, cfg, r)
            assert z.tobytes() == zo.tobytes(), s.name
    finally:
        ctx.close()


@pytest.mark.parametrize("env", [{"BCS_AGG_MODE": "1"}, {"BCS_DILU_MODE": "1"}, {"BCS_TAIL_ROWS": "0"},
                                 {"BCS_TAIL_ROWS": "100000"}])
def test_alternative_schedules_bit_exact(oracle, env, monkeypatch):
    """The alternative schedules (cooperative-round aggregation, Kahn-level DILU
    setup, no one-CTA tail, everything in the tail) give the same bits."""
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    ctx = bcs.Context(0)
    try:
        s = gen.hex_euler(12, scramble_seed=2)
        cfg = make_cfg(precond=3, max_levels=30, min_coarse=8)
        r = np.random.default_rng(9).uniform(-1, 1, s.A.n_cells * s.A.n)
        z = _apply(ctx, s, cfg, r)
        zo = oracle.precond_apply(s.A, cfg, r)
        assert z.tobytes() == zo.tobytes()
    finally:
        ctx.close()


def test_tiled_dense_solve_tolerance_level(oracle, monkeypatch):
    """Large coarsest levels (m >= 2048 by default; forced here from 64): the
    backward substitution runs by tiles (tolerance-level): the
    V-cycle application agrees with the reference-order one to rounding."""
    monkeypatch.setenv("BCS_DENSE_TILED_MIN", "64")
    monkeypatch.setenv("BCS_DENSE_BLOCKED_MIN", "64")
    ctx = bcs.Context(0)
    try:
        s = gen.hex_euler(32, scramble_seed=7)
        cfg = make_cfg(precond=3, max_levels=30, min_coarse=8)
        r = np.random.default_rng(5).uniform(-1, 1, s.A.n_cells * s.A.n)
        z = _apply(ctx, s, cfg, r)
        m = (ctx.amg_level(ctx.amg_depth() - 1, s.A.n)[0].size - 1) * s.A.n
        assert m >= 64
        zo = oracle.precond_apply(s.A, cfg, r)
        np.testing.assert_allclose(z, zo, rtol=0, atol=1e-10 * np.abs(zo).max())
        # EXACT mode keeps the reference order (bit-identical solve)
        rexact = ctx.solve(s.b.values, xe := s.x0.values.copy(),
                           bcs.SolverConfig(preconditioner=bcs.PrecondKind.AMG, relTol=1e-8, maxIters=200,
                                            amg=bcs.AmgConfig(maxLevels=30, minCoarseRows=8), mode=bcs.Mode.EXACT))
        rc, xo, rep, ho = oracle.solve(s.A, s.b.values, s.x0.values, cfg)
        assert rexact.iterations == rep.iterations and xe.tobytes() == xo.tobytes()
        # default mode: tiled, iterations within +-1
        rd = ctx.solve(s.b.values, s.x0.values.copy(),
                       bcs.SolverConfig(preconditioner=bcs.PrecondKind.AMG, relTol=1e-8, maxIters=200,
                                        amg=bcs.AmgConfig(maxLevels=30, minCoarseRows=8)))
        assert rd.converged and abs(rd.iterations - rep.iterations) <= 1
    finally:
        ctx.close()
