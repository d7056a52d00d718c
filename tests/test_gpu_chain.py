"""Chain schedule (opt-in, BCS_CHAIN=1): the sweeps of natural-order levels
taken chain by chain (k_sweep_chain, warp-major tickets).  The schedule only
reorders work, so every solve must be bit-identical to the level-order
schedule's; run in subprocesses because the switch is read once per process."""
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
for name, s in [("euler24", gen.hex_euler(24)), ("coupled16", gen.hex_coupled(16, poly_seed=1)),
                ("euler20x12x9", gen.hex_euler(20, 12, 9, aspect=30.0))]:
    for mode in (bcs.Mode.PARITY, bcs.Mode.EXACT):
        for pc in (bcs.PrecondKind.AMG, bcs.PrecondKind.DILU):
            ctx = bcs.Context(0)
            ctx.set_topology(s.A)
            ctx.upload_ldu(s.A)
            x = s.x0.values.copy()
            r = ctx.solve(s.b.values, x, bcs.SolverConfig(preconditioner=pc, relTol=1e-8, maxIters=500, mode=mode,
                                                          amg=bcs.AmgConfig(maxLevels=30, minCoarseRows=8)))
            ctx.close()
            out[f"{name}/{int(mode)}/{int(pc)}"] = [r.iterations, hashlib.sha1(x.tobytes()).hexdigest()]
print(json.dumps(out))
""" % ROOT


def _run(env_extra):
    env = dict(os.environ, **env_extra)
    p = subprocess.run([sys.executable, "-c", PROBE], env=env, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    return json.loads(p.stdout.strip().splitlines()[-1]), p.stderr


def test_chain_schedule_is_bit_identical_to_level_order():
    base, _ = _run({"BCS_CHAIN": "0"})
    chain, err = _run({"BCS_CHAIN": "1", "BCS_CHAIN_MIN_WIDTH": "1", "BCS_CHAIN_VERBOSE": "1"})
    assert "chain schedule" in err  # the chain kernel actually ran
    assert chain == base
