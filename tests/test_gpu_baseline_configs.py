"""Parity at the BASELINE.json configurations against the LIVE reference
(oracle/_ref: the unmodified reference compiled from its sources).

* C1 (configs[0]): 32^3 4x4 pressure-based coupled system, GMRES+AMG and
  BiCGStab+AMG to 1e-8 (the reference takes ~3 s per solve).
* C2 (configs[1], the bench headline): 128^3 5x5 density-based system,
  GMRES+AMG to 1e-8 (the reference takes ~70-130 s; marked slow).

Each checks the AMG depth, every level's row/block counts and every level's
aggregates (integer, bit-exact) and then:
  * EXACT mode (the reference's sequential dot order + its libm hypot): the
    residual history (from the reference's own KrylovOps::dot stream, SURVEY
    §8(c)) and the solution are BIT-IDENTICAL to the reference's;
  * default PARITY mode (tree dots): iterations within +-1, converged, the
    solution to the reference's own tolerance, and the maximum relative
    history deviation recorded (parity_log).
"""
import dataclasses

import numpy as np
import pytest

from oracle_lib import make_cfg
from paper_2403_07882_b200 import bcs, gen
from test_gpu_parity import check_history, history_rel_dev

pytestmark = pytest.mark.gpu

AMG = bcs.AmgConfig(maxLevels=30, minCoarseRows=8)


def _against_reference(ref, parity_log, s, method, what):
    cfg_t = make_cfg(method=method, precond=3, max_iters=1000)
    # calls=0: the reference's solveCsr with the recording dot only (engine.cpp:31-45)
    rc, xr, rr, hr = ref.solve(s.A, s.b.values, s.x0.values, cfg_t, calls=0)
    assert rc == 0, ref.err()
    shape = ref.amg_shape(s.A, 30, 8)
    ctx = bcs.Context(0)
    cfg = bcs.SolverConfig(method=bcs.KrylovMethod(method), preconditioner=bcs.PrecondKind.AMG, relTol=1e-8,
                           maxIters=1000, amg=AMG)
    try:
        ctx.set_topology(s.A)
        ctx.upload_ldu(s.A)
        xe = s.x0.values.copy()
        re = ctx.solve(s.b.values, xe, dataclasses.replace(cfg, mode=bcs.Mode.EXACT))
        he = ctx.residual_history()
        x = s.x0.values.copy()
        r = ctx.solve(s.b.values, x, cfg)
        h = ctx.residual_history()
        # hierarchy: depth, per-level sizes and aggregates (bit-exact integers)
        assert ctx.amg_depth() == len(shape)
        assert r.amgLevels == len(shape)
        for lvl, (rows, nnz, agg) in enumerate(shape):
            grows, gnnz, gagg = ctx.amg_level_shape(lvl, want_agg=agg is not None)
            assert (grows, gnnz) == (rows, nnz), f"level {lvl}"
            if agg is not None:
                assert np.array_equal(gagg, agg), f"level {lvl} aggregates"
        assert r.coarseRows == shape[-1][0]
    finally:
        ctx.close()
    # exact mode: bit-identical to the live reference
    assert re.iterations == rr.iterations and re.converged and rr.converged
    assert he.tobytes() == hr.tobytes(), (he, hr)
    assert xe.tobytes() == xr.tobytes()
    check_history(he, hr, what + " [exact]")
    # default mode
    assert r.converged
    assert abs(r.iterations - rr.iterations) <= 1, (r.iterations, rr.iterations)
    np.testing.assert_allclose(r.initialResidual, rr.initial_residual, rtol=1e-12)
    parity_log(what, dict(max_rel_dev=history_rel_dev(h, hr), n=min(len(h), len(hr)), iters=r.iterations,
                          ref_iters=rr.iterations, levels=len(shape), coarse_rows=shape[-1][0],
                          final_rel=float(r.finalResidual / r.initialResidual), exact_bit_identical=True))
    np.testing.assert_allclose(x, xr, rtol=0, atol=1e-8 * np.abs(xr).max())
    return r, rr


@pytest.mark.parametrize("method", [0, 1])
def test_c1_coupled_32_against_reference(ref, parity_log, method):
    s = gen.hex_coupled(32)
    _against_reference(ref, parity_log, s, method, f"C1 32^3 4x4 coupled method={method}")


@pytest.mark.slow
def test_c2_euler_128_gmres_amg_against_reference(ref, parity_log):
    s = gen.hex_euler(128)
    r, rr = _against_reference(ref, parity_log, s, 0, "C2 128^3 5x5 euler GMRES+AMG")
    assert r.iterations == rr.iterations == 7
