"""State isolation across the C ABI: long random sequences of operations on
ONE context (topology changes, value uploads, solves in every method /
preconditioner / mode, the pipeline in both backends, the one-device Mode R,
preconditioner-only setups and applications, residual and SpMV queries) must
give, operation by operation, bit for bit what the same operation gives on a
fresh context.  A state leak between phases (a buffer borrowed from a
recycled arena, a stale schedule, a preconditioner built for another matrix)
shows up as a mismatch or a fault.  Seeded; small systems so each sequence
runs in seconds."""
import dataclasses

import numpy as np
import pytest

from paper_2403_07882_b200 import bcs, gen
from test_gpu_parity import random_system

pytestmark = pytest.mark.gpu

AMG = bcs.AmgConfig(maxLevels=30, minCoarseRows=8)

def _rand(nx, ny, nz, n, seed):
    """a random diagonally dominant n x n block system (n = 1..3) as a
    gen.System-like record"""
    A, b = random_system(nx, ny, nz, n, seed)
    base = gen.hex_euler(nx, ny, nz)
    return gen.System(A=A, b=bcs.BlockVector(A.n_cells, n, values=b), x0=bcs.BlockVector(A.n_cells, n),
                      centroids=base.centroids, name=f"rand{n}_{nx}x{ny}x{nz}")


SYSTEMS = [
    lambda: gen.hex_euler(9),
    lambda: gen.hex_euler(8, 7, 6, scramble_seed=3),
    lambda: gen.hex_coupled(8, poly_seed=2),
    lambda: gen.hex_coupled(7, scramble_seed=1),
    lambda: _rand(9, 8, 7, 1, 11),
    lambda: _rand(7, 7, 6, 2, 12),
    lambda: _rand(6, 7, 5, 3, 13),
]


def _configs():
    out = []
    for method in (bcs.KrylovMethod.GMRES, bcs.KrylovMethod.PBiCGStab, bcs.KrylovMethod.FGMRES):
        for pc in (bcs.PrecondKind.AMG, bcs.PrecondKind.DILU, bcs.PrecondKind.LUSGS, bcs.PrecondKind.none):
            for mode in (bcs.Mode.PARITY, bcs.Mode.EXACT, bcs.Mode.PERF, bcs.Mode.PERF_JACOBI):
                if mode in (bcs.Mode.PERF, bcs.Mode.PERF_JACOBI) and pc != bcs.PrecondKind.AMG:
                    continue
                out.append(bcs.SolverConfig(method=method, preconditioner=pc, relTol=1e-8, maxIters=300,
                                            amg=AMG, mode=mode))
    return out


CONFIGS = _configs()


def _op(ctx, kind, s, cfg, rng_vec):
    """Run one operation; returns bytes to compare (results + iteration counts)."""
    A = s.A
    if kind == "solve":
        ctx.set_topology(A)
        ctx.upload_ldu(A)
        x = s.x0.values.copy()
        r = ctx.solve(s.b.values, x, cfg)
        return x.tobytes() + ctx.residual_history().tobytes() + bytes([r.iterations % 256])
    if kind == "pipe_engine":
        x, r = ctx.pipeline_solve(A, s.b, s.x0, bcs.Backend.EngineCsr, cfg)
        return np.asarray(x.values).tobytes() + bytes([r.iterations % 256])
    if kind == "pipe_host":
        c = dataclasses.replace(cfg, preconditioner=bcs.PrecondKind.LUSGS,
                                mode=bcs.Mode.EXACT if cfg.mode == bcs.Mode.EXACT else bcs.Mode.PARITY)
        x, r = ctx.pipeline_solve(A, s.b, s.x0, bcs.Backend.HostLdu, c)
        return np.asarray(x.values).tobytes() + bytes([r.iterations % 256])
    if kind == "precond":
        ctx.set_topology(A)
        ctx.upload_ldu(A)
        ctx.precond_setup(cfg if cfg.preconditioner != bcs.PrecondKind.none else
                          dataclasses.replace(cfg, preconditioner=bcs.PrecondKind.DILU))
        return ctx.precond_apply(rng_vec).tobytes()
    if kind == "spmv":
        ctx.set_topology(A)
        ctx.upload_ldu(A)
        return ctx.spmv(rng_vec).tobytes() + np.float64(ctx.residual(s.b.values, rng_vec)).tobytes()
    if kind == "dist":
        c = dataclasses.replace(cfg, mode=bcs.Mode.EXACT if cfg.mode == bcs.Mode.EXACT else bcs.Mode.PARITY,
                                preconditioner=bcs.PrecondKind.AMG if cfg.preconditioner == bcs.PrecondKind.none
                                else cfg.preconditioner)
        x, r = ctx.dist_solve(A, s.b, s.x0, s.centroids, 3, 2, c)
        return np.asarray(x.values).tobytes() + bytes([r.iterations % 256])
    raise AssertionError(kind)


KINDS = ["solve", "solve", "pipe_engine", "pipe_host", "precond", "spmv", "dist"]


@pytest.mark.parametrize("seed", list(range(1, 9)))
def test_random_operation_sequences_match_fresh_contexts(seed):
    rng = np.random.default_rng(seed)
    systems = [m() for m in SYSTEMS]
    ctx = bcs.Context(0)
    try:
        for step in range(32):
            s = systems[rng.integers(len(systems))]
            kind = KINDS[rng.integers(len(KINDS))]
            cfg = CONFIGS[rng.integers(len(CONFIGS))]
            vec = np.random.default_rng(100 * seed + step).uniform(-1, 1, s.A.n_cells * s.A.n)
            got = _op(ctx, kind, s, cfg, vec)
            fresh = bcs.Context(0)
            try:
                want = _op(fresh, kind, s, cfg, vec)
            finally:
                fresh.close()
            assert got == want, (seed, step, kind, s.name, cfg)
    finally:
        ctx.close()
