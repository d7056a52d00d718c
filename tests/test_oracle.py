"""The CPU oracle pinned: the C restatement (oracle/bcs_oracle.c) against the
golden vectors produced by the reference itself (tests/golden, made by
oracle/make_golden.py) and, where oracle/_ref is built, against the live
reference on fresh inputs.  Everything here is bit-exact."""
import hashlib
import json
import os

import numpy as np
import pytest

from oracle_lib import make_cfg
from paper_2403_07882_b200 import bcs, gen

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
INDEX = json.load(open(os.path.join(GOLD, "index.json")))
HEX = [k for k in INDEX if k != "known_answers"]
SOLVES = [(0, 3), (1, 3), (0, 2), (1, 2), (0, 1), (0, 0)]


def sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def hex_from_index(name):
    p = INDEX[name]
    f = gen.hex_euler if p["kind"] == "euler" else gen.hex_coupled
    return f(p["nx"], p["ny"], p["nz"], aspect=p["aspect"], scramble_seed=p["seed"])


@pytest.fixture(scope="module")
def ka():
    return np.load(os.path.join(GOLD, "known_answers.npz"))


def test_known_answer_ldu_matvec(oracle, ka):
    A = bcs.BlockLduMatrix(2, [0], [1], 1, [2.0, 3.0], [1.0], [4.0])
    y = oracle.matvec(A, np.ones(2))
    assert y.tolist() == [3.0, 7.0] == ka["ldu2_y"].tolist()
    assert oracle.ldu_matvec(A, np.ones(2)).tolist() == [3.0, 7.0]


def test_known_answer_plans(oracle, ka):
    A4 = bcs.BlockLduMatrix(2, [0], [1], 4)
    ro, ci, _, _ = oracle.csr(A4)
    assert ro.tolist() == [0, 2, 4] == ka["plan2_ro"].tolist()
    assert ci.tolist() == [0, 1, 0, 1] == ka["plan2_ci"].tolist()
    # 3x3 mesh: 9 + 2*12 = 33 blocks, centre row has 5 entries
    ro9 = ka["mesh3x3_ro"]
    assert ro9[-1] == 33 and ro9[5] - ro9[4] == 5


def test_known_answer_spd2(oracle, ka):
    A = bcs.BlockLduMatrix(2, [0], [1], 1, [4.0, 3.0], [1.0], [1.0])
    rc, x, rep, h = oracle.solve(A, np.array([1.0, 2.0]), np.zeros(2), make_cfg(precond=0, rel_tol=1e-10))
    assert rc == 0 and rep.converged and rep.iterations <= 2
    np.testing.assert_allclose(x, [1 / 11, 7 / 11], atol=1e-12)
    assert x.tobytes() == ka["spd2_x"].tobytes()


def test_known_answer_aggregation(oracle, ka):
    assert ka["chain4_agg"].tolist() == [0, 0, 1, 1]
    A = bcs.BlockLduMatrix(4, [0, 1, 2], [1, 2, 3], 1, np.full(4, 2.0), np.full(3, -1.0), np.full(3, -1.0))
    lv = oracle.amg_levels(A, 10, 1)
    assert lv[0][3].tolist() == [0, 0, 1, 1]
    assert len(set(ka["tube16_agg"].tolist())) == 8


def test_known_answer_galerkin(oracle, ka):
    g = np.load(os.path.join(GOLD, "galerkin6x6_n3.npz"))
    A = bcs.BlockLduMatrix(36, g["owner"], g["neigh"], 3, g["diag"], g["upper"], g["lower"])
    lv = oracle.amg_levels(A, 2, 1)
    assert np.array_equal(lv[0][3], ka["galerkin6x6_agg"])
    assert np.array_equal(lv[1][0], ka["galerkin6x6_c_ro"])
    assert np.array_equal(lv[1][1], ka["galerkin6x6_c_ci"])
    assert lv[1][2].tobytes() == ka["galerkin6x6_c_v"].tobytes()
    # block sums preserved (test_krylov.cpp:194-210)
    assert abs(lv[1][2].sum() - lv[0][2].sum()) <= 1e-12 * abs(lv[0][2]).sum()


def test_known_answer_decomposition(oracle, ka):
    assert ka["decomp9_rro"].tolist() == [0, 3, 6, 9]
    assert ka["decomp_tube100_rro"].tolist() == [0, 25, 50, 75, 100]


@pytest.mark.parametrize("name", HEX)
def test_restatement_matches_reference_goldens(oracle, name):
    g = np.load(os.path.join(GOLD, name + ".npz"))
    s = hex_from_index(name)
    A = s.A
    assert sha(A.owner, A.neighbour, A.diag, A.upper, A.lower, s.b.values, s.x0.values) == str(g["ldu_sha"])
    assert oracle.signature(A) == int(g["signature"])
    ro, ci, src, v = oracle.csr(A)
    assert np.array_equal(ro, g["plan_ro"]) and np.array_equal(ci, g["plan_ci"])
    assert sha(v) == str(g["plan_v_sha"])
    lv = oracle.amg_levels(A, 30, 8)
    assert len(lv) == int(g["amg_depth"][0])
    for i, (lro, lci, lvv, agg) in enumerate(lv):
        assert np.array_equal(lro, g[f"amg{i}_ro"]) and np.array_equal(lci, g[f"amg{i}_ci"])
        assert sha(lvv) == str(g[f"amg{i}_v_sha"])
        if agg is not None:
            assert np.array_equal(agg, g[f"amg{i}_agg"])
    for method, pc in SOLVES:
        tag = f"m{method}p{pc}"
        rc, x, rep, h = oracle.solve(A, s.b.values, s.x0.values, make_cfg(method=method, precond=pc, max_iters=300))
        assert rc == int(g[f"{tag}_rc"][0])
        assert rep.iterations == int(g[f"{tag}_iters"][0])
        assert h.tobytes() == g[f"{tag}_hist"].tobytes()
        assert x.tobytes() == g[f"{tag}_x"].tobytes()


def _random_2d(ref, nx, ny, n, seed):
    from oracle_lib import ref_mesh_2d, ref_randomize
    nc, o, ne, cen = ref_mesh_2d(ref, nx, ny)
    d, u, lo = ref_randomize(ref, nc, o, ne, n, seed)
    return bcs.BlockLduMatrix(nc, o, ne, n, d, u, lo)


@pytest.mark.parametrize("n", [1, 3, 4, 5])
@pytest.mark.parametrize("pc", [0, 1, 2, 3])
@pytest.mark.parametrize("method", [0, 1])
def test_restatement_matches_live_reference(oracle, ref, n, pc, method):
    from oracle_lib import ref_random_vector
    A = _random_2d(ref, 9, 7, n, 100 + n)
    b = ref_random_vector(ref, A.n_cells, n, 5)
    x0 = np.zeros_like(b)
    cfg = make_cfg(method=method, precond=pc, rel_tol=1e-10, max_iters=200, max_levels=30, min_coarse=4)
    rc1, x1, r1, h1 = ref.solve(A, b, x0, cfg)
    rc2, x2, r2, h2 = oracle.solve(A, b, x0, cfg)
    assert rc1 == rc2 and r1.iterations == r2.iterations
    assert x1.tobytes() == x2.tobytes()
    assert h1.tobytes() == h2.tobytes()
    z1 = ref.precond_apply(A, cfg, b)
    z2 = oracle.precond_apply(A, cfg, b)
    assert z1.tobytes() == z2.tobytes()


def test_restatement_plan_signature_live(oracle, ref):
    s = gen.hex_euler(5, 6, 7, scramble_seed=9)
    assert oracle.signature(s.A) == ref.signature(s.A)
    ro, ci, _, v = oracle.csr(s.A)
    rro, rci, rv = ref.csr(s.A)
    assert np.array_equal(ro, rro) and np.array_equal(ci, rci) and v.tobytes() == rv.tobytes()


@pytest.mark.parametrize("ranks", [1, 2, 3, 4, 8])
def test_restatement_decompose_live(oracle, ref, ranks):
    s = gen.hex_euler(6, 5, 4, scramble_seed=3)
    a = oracle.decompose(s.centroids, ranks)
    b = ref.decompose(s.centroids, ranks)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)


def _glibc_hypot(x, y):
    """The reference libm's hypot (glibc >= 2.35 sysdeps/ieee754/dbl-64/e_hypot.c,
    non-FMA kernel), restated in Python double arithmetic -- the algorithm the
    device Givens rotation runs (k_krylov.cu glibc_hypot)."""
    import math
    if not math.isfinite(x) or not math.isfinite(y):
        return math.inf if (math.isinf(x) or math.isinf(y)) else x + y
    x, y = abs(x), abs(y)
    ax, ay = max(x, y), min(x, y)

    def kernel(ax, ay):
        h = math.sqrt(ax * ax + ay * ay)
        if h <= 2.0 * ay:
            delta = h - ay
            t1 = ax * (2.0 * delta - ax)
            t2 = (delta - 2.0 * (ax - ay)) * delta
        else:
            delta = h - ax
            t1 = 2.0 * delta * (ax - 2.0 * ay)
            t2 = (4.0 * delta - ay) * ay + delta * delta
        return h - (t1 + t2) / (2.0 * h)

    scale, large, tiny, eps = 2.0 ** -600, 2.0 ** 511, 2.0 ** -459, 2.0 ** -54
    if ax > large:
        return ax + ay if ay <= ax * eps else kernel(ax * scale, ay * scale) / scale
    if ay < tiny:
        return ax + ay if ax >= ay / eps else kernel(ax / scale, ay / scale) * scale
    return ax + ay if ay <= ax * eps else kernel(ax, ay)


def test_glibc_hypot_restatement_matches_libm():
    """The restated hypot equals this host's libm bit for bit (the reference
    links the same libm); the device copy is pinned on the GPU
    (test_device_hypot_is_the_reference_libm_hypot)."""
    import ctypes
    import random
    libm = ctypes.CDLL("libm.so.6")
    libm.hypot.restype = ctypes.c_double
    libm.hypot.argtypes = [ctypes.c_double, ctypes.c_double]
    rnd = random.Random(11)
    for _ in range(50000):
        e1 = rnd.randint(-1070, 1020)
        e2 = max(-1070, min(1020, e1 + rnd.randint(-70, 70))) if rnd.random() < 0.7 else rnd.randint(-1070, 1020)
        x = rnd.uniform(-1, 1) * 2.0 ** e1
        y = 0.0 if rnd.random() < 0.03 else rnd.uniform(-1, 1) * 2.0 ** e2
        assert _glibc_hypot(x, y) == libm.hypot(x, y), (x.hex(), y.hex())
