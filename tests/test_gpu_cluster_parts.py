"""Cluster sweep variant spread over several clusters (opt-in, BCS_CL_PARTS):
each cluster takes one contiguous row range of a level in level order, hands
dependencies inside its range over through distributed shared memory and the
others through global memory.  It only reorders work, so every solve must be
bit-identical to the default schedule's; run in subprocesses because the switch
is read once per process."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROBE = r"""
import hashlib, json, sys
sys.path.insert(0, %r)
from paper_2403_07882_b200 import bcs, gen
out = {}
for name, s in [("euler40", gen.hex_euler(40)), ("coupled32", gen.hex_coupled(32, poly_seed=1)),
                ("euler40s", gen.hex_euler(40, scramble_seed=5))]:
    for method in (bcs.KrylovMethod.GMRES, bcs.KrylovMethod.PBiCGStab):
        ctx = bcs.Context(0)
        ctx.set_topology(s.A)
        ctx.upload_ldu(s.A)
        x = s.x0.values.copy()
        r = ctx.solve(s.b.values, x, bcs.SolverConfig(method=method, preconditioner=bcs.PrecondKind.AMG, relTol=1e-8,
                                                      maxIters=500, amg=bcs.AmgConfig(maxLevels=30, minCoarseRows=8)))
        ctx.close()
        out[f"{name}/{int(method)}"] = [r.iterations, hashlib.sha1(x.tobytes()).hexdigest()]
print(json.dumps(out))
""" % ROOT


def _run(env_extra):
    env = dict(os.environ, **env_extra)
    p = subprocess.run([sys.executable, "-c", PROBE], env=env, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    return json.loads(p.stdout.strip().splitlines()[-1])


def test_multi_cluster_levels_are_bit_identical():
    base = _run({"BCS_CL_PARTS": "1"})
    # narrow cluster widths so that several levels spread over 2..9 clusters
    multi = _run({"BCS_CL_PARTS": "9", "BCS_CL_WIDTH": "12"})
    assert multi == base
