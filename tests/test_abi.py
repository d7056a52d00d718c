"""C ABI checks that need no GPU: the library loads, exports every symbol
declared in include/bcs.h, and its host-only entry points behave."""
import os
import re

import numpy as np
import pytest

from paper_2403_07882_b200 import _native, bcs, gen

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "bcs.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(bcs_[a-z_]+)\s*\(", src)))


def test_library_exports_all_declared_symbols():
    lib = _native.lib()
    syms = declared_symbols()
    assert len(syms) >= 25
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_native.SIGNATURES), set(syms) ^ set(_native.SIGNATURES)


def test_version_and_default_config():
    lib = _native.lib()
    assert b"sm_100a" in lib.bcs_version()
    c = _native.SolverConfigC()
    lib.bcs_default_config(c)
    # SolverConfig / AmgConfig defaults (krylov.hpp:18-37)
    assert (c.method, c.precond, c.rel_tol, c.abs_tol, c.max_iters, c.gmres_restart) == (0, 1, 1e-6, 1e-300, 500, 30)
    assert (c.amg_max_levels, c.amg_min_coarse_rows, c.amg_pre_sweeps, c.amg_post_sweeps) == (10, 8, 1, 1)
    d = bcs.SolverConfig()
    assert (d.relTol, d.maxIters, d.gmresRestart, d.amg.maxLevels) == (1e-6, 500, 30, 10)


@pytest.mark.parametrize("seed", [-1, 4])
def test_topology_signature_exact(oracle, seed):
    s = gen.hex_euler(6, 5, 4, scramble_seed=seed)
    assert bcs.topology_signature(s.A) == oracle.signature(s.A)


def test_topology_signature_live(ref):
    s = gen.hex_euler(7, 3, 5, scramble_seed=2)
    assert bcs.topology_signature(s.A) == ref.signature(s.A)


def test_create_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(RuntimeError):
        bcs.Context(0)


def test_struct_layouts_match_header():
    # bcs_solver_config: 6 ints + 2 doubles + ... ; bcs_report field count
    assert [f for f, _ in _native.SolverConfigC._fields_][:6] == [
        "method", "precond", "rel_tol", "abs_tol", "max_iters", "gmres_restart"]
    hdr = open(os.path.join(ROOT, "include", "bcs.h")).read()
    body = hdr[hdr.index("typedef struct {\n    int iterations;"):hdr.index("} bcs_report;")]
    body = re.sub(r"/\*.*?\*/", "", body, flags=re.S)
    names = re.findall(r"\b([a-z_]+)\s*[;,]", body)
    assert [f for f, _ in _native.ReportC._fields_] == names


def test_ldu_dump_round_trip_and_corruption(tmp_path):
    """Binary LDU dump (bcs_ldu_save/load, host only): exact round trip of a
    generator system, optional vectors, and the error paths."""
    from paper_2403_07882_b200 import bcs, gen
    s = gen.hex_coupled(5, 4, 3, poly_seed=2)
    p = tmp_path / "sys.bcsldu"
    bcs.save_ldu(p, s.A, s.b, s.x0)
    A, b, x0 = bcs.load_ldu(p)
    for x, y in ((A.owner, s.A.owner), (A.neighbour, s.A.neighbour), (A.diag, s.A.diag), (A.upper, s.A.upper),
                 (A.lower, s.A.lower), (b.values, s.b.values), (x0.values, s.x0.values)):
        assert x.tobytes() == y.tobytes()
    assert A.n == 4 and A.n_cells == s.A.n_cells
    q = tmp_path / "nob.bcsldu"
    bcs.save_ldu(q, s.A)
    A2, b2, x02 = bcs.load_ldu(q)
    assert b2 is None and x02 is None and A2.upper.tobytes() == s.A.upper.tobytes()
    raw = bytearray(p.read_bytes())
    raw[100] ^= 0x40  # payload bit flip
    (tmp_path / "bad.bcsldu").write_bytes(bytes(raw))
    with pytest.raises(RuntimeError, match="checksum"):
        bcs.load_ldu(tmp_path / "bad.bcsldu")
    (tmp_path / "short.bcsldu").write_bytes(p.read_bytes()[:1000])
    with pytest.raises(RuntimeError, match="truncated"):
        bcs.load_ldu(tmp_path / "short.bcsldu")
    (tmp_path / "junk.bcsldu").write_bytes(b"\0" * 128)
    with pytest.raises(RuntimeError, match="not a BCSLDU01"):
        bcs.load_ldu(tmp_path / "junk.bcsldu")
