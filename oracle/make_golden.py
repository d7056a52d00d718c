"""TEST INFRASTRUCTURE ONLY — writes tests/golden/*.npz from the reference.

Run in the container where /root/reference is mounted (after
``make -C oracle``).  Every number comes from the unmodified reference
compiled into oracle/_ref/libbcs_ref.so:

  * known-answer cases of the reference's own spec/tests (SPEC.md:139, 202-204,
    221, 247; test_krylov.cpp:181-260; test_partition.cpp:48-73);
  * synthetic hex systems from the reference producers
    (assembleJacobian / assembleCoupled): a SHA-256 of the LDU arrays (pins the
    generator), the BSR plan, every AMG level (aggregates + value hash), and
    full SolvePipeline solves (iterations, residuals, history, x).

    python oracle/make_golden.py
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from oracle_lib import (Reference, make_cfg, ref_mesh_2d, ref_mesh_tube, ref_random_vector,  # noqa: E402
                        ref_randomize)
from paper_2403_07882_b200.bcs import BlockLduMatrix  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")


def sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def hex_system(R, kind, nx, ny, nz, aspect, seed):
    if kind == "euler":
        o, ne, d, u, lo, b, cen = R.gen_euler(nx, ny, nz, aspect, seed)
        x0 = np.zeros_like(b)
        n = 5
    else:
        o, ne, d, u, lo, b, x0, cen = R.gen_coupled(nx, ny, nz, aspect, seed)
        n = 4
    return BlockLduMatrix(nx * ny * nz, o, ne, n, d, u, lo), b, x0, cen


SOLVES = [(0, 3), (1, 3), (0, 2), (1, 2), (0, 1), (0, 0)]


def main():
    R = Reference()
    os.makedirs(OUT, exist_ok=True)
    index = {}

    # ---- known answers -------------------------------------------------
    ka = {}
    # 2-cell LDU matvec [[2,1],[4,3]]·[1,1] = [3,7]
    A = BlockLduMatrix(2, [0], [1], 1, [2.0, 3.0], [1.0], [4.0])
    ycsr, yldu = R.matvec(A, np.ones(2))
    ka["ldu2_y"] = ycsr
    # 2-cell n=4 plan
    A4 = BlockLduMatrix(2, [0], [1], 4, np.arange(32.0), np.arange(16.0), -np.arange(16.0))
    ro, ci, v = R.csr(A4)
    ka["plan2_ro"], ka["plan2_ci"] = ro, ci
    # 3x3 mesh: nnz 33, centre row 5 entries
    nc, o, ne, cen = ref_mesh_2d(R, 3, 3)
    A9 = BlockLduMatrix(nc, o, ne, 1, np.ones(nc), np.ones(o.size), np.ones(o.size))
    ro, ci, v = R.csr(A9)
    ka["mesh3x3_ro"], ka["mesh3x3_ci"] = ro, ci
    # SPD 2x2 [[4,1],[1,3]] b=[1,2] -> x=[1/11, 7/11]
    S = BlockLduMatrix(2, [0], [1], 1, [4.0, 3.0], [1.0], [1.0])
    rc, x, rep, h = R.solve(S, np.array([1.0, 2.0]), np.zeros(2), make_cfg(precond=0, rel_tol=1e-10))
    ka["spd2_x"], ka["spd2_iters"] = x, np.array([rep.iterations])
    # 4-row chain -> {0,1},{2,3}
    nc, o, ne, cen = ref_mesh_tube(R, 4)
    C4 = BlockLduMatrix(nc, o, ne, 1, np.full(nc, 2.0), np.full(o.size, -1.0), np.full(o.size, -1.0))
    lv = R.amg_levels(C4, 10, 1)
    ka["chain4_agg"] = lv[0][3]
    # test_krylov.cpp:181-192 — tube 16, randomize(rng 2), n=1 -> 8 aggregates
    nc, o, ne, cen = ref_mesh_tube(R, 16)
    d, u, lo = ref_randomize(R, nc, o, ne, 1, 2)
    T = BlockLduMatrix(nc, o, ne, 1, d, u, lo)
    lv = R.amg_levels(T, 2, 1)
    ka["tube16_agg"] = lv[0][3]
    # test_krylov.cpp:194-210 — 6x6, n=3, randomize(rng 29): Galerkin coarse matrix
    nc, o, ne, cen = ref_mesh_2d(R, 6, 6)
    d, u, lo = ref_randomize(R, nc, o, ne, 3, 29)
    G = BlockLduMatrix(nc, o, ne, 3, d, u, lo)
    np.savez_compressed(os.path.join(OUT, "galerkin6x6_n3.npz"), owner=o, neigh=ne, diag=d, upper=u, lower=lo)
    lv = R.amg_levels(G, 2, 1)
    ka["galerkin6x6_agg"] = lv[0][3]
    ka["galerkin6x6_c_ro"], ka["galerkin6x6_c_ci"], ka["galerkin6x6_c_v"] = lv[1][0], lv[1][1], lv[1][2]
    # test_krylov.cpp:212-237 — 12x12 Poisson, AmgConfig{} hierarchy + one V-cycle
    nc, o, ne, cen = ref_mesh_2d(R, 12, 12)
    P = BlockLduMatrix(nc, o, ne, 1, np.full(nc, 4.0), np.full(o.size, -1.0), np.full(o.size, -1.0))
    lv = R.amg_levels(P, 10, 8)
    ka["poisson12_rows"] = np.array([lvl[0].size - 1 for lvl in lv])
    r = ref_random_vector(R, nc, 1, 4)
    ka["poisson12_r"] = r
    ka["poisson12_z"] = R.precond_apply(P, make_cfg(precond=3, max_levels=10, min_coarse=8), r)
    # test_krylov.cpp:239-260 — 20x20 Poisson (+1e-3), GMRES relTol 1e-10, AMG vs plain
    nc, o, ne, cen = ref_mesh_2d(R, 20, 20)
    P20 = BlockLduMatrix(nc, o, ne, 1, np.full(nc, 4.0 + 1e-3), np.full(o.size, -1.0), np.full(o.size, -1.0))
    b20 = ref_random_vector(R, nc, 1, 8)
    ka["poisson20_b"] = b20
    for pc in (3, 0):
        rc, x, rep, h = R.solve(P20, b20, np.zeros(nc), make_cfg(precond=pc, rel_tol=1e-10, max_iters=500,
                                                                 max_levels=10))
        ka[f"poisson20_iters_pc{pc}"] = np.array([rep.iterations])
        ka[f"poisson20_x_pc{pc}"] = x
        ka[f"poisson20_hist_pc{pc}"] = h
    # test_partition.cpp:48-73 — decompositions
    nc, o, ne, cen = ref_mesh_2d(R, 3, 3)
    c2r, rro, o2n = R.decompose(cen, 3)
    ka["decomp9_rro"], ka["decomp9_c2r"] = rro, c2r
    nc, o, ne, cen = ref_mesh_tube(R, 100)
    c2r, rro, o2n = R.decompose(cen, 4)
    ka["decomp_tube100_rro"] = rro
    np.savez_compressed(os.path.join(OUT, "known_answers.npz"), **ka)
    index["known_answers"] = sorted(ka)

    # ---- synthetic hex systems -----------------------------------------
    cases = [("euler", 5, 4, 3, 1.0, -1), ("euler", 6, 6, 6, 1.0, 7), ("euler", 4, 5, 6, 100.0, -1),
             ("coupled", 5, 5, 5, 1.0, -1), ("coupled", 6, 5, 4, 1.0, 11)]
    for kind, nx, ny, nz, asp, seed in cases:
        name = f"{kind}_{nx}x{ny}x{nz}_ar{asp:g}_s{seed}"
        A, b, x0, cen = hex_system(R, kind, nx, ny, nz, asp, seed)
        g = {"ldu_sha": np.array(sha(A.owner, A.neighbour, A.diag, A.upper, A.lower, b, x0)),
             "signature": np.array(R.signature(A), dtype=np.uint64)}
        ro, ci, v = R.csr(A)
        g["plan_ro"], g["plan_ci"], g["plan_v_sha"] = ro, ci, np.array(sha(v))
        lv = R.amg_levels(A, 30, 8)
        g["amg_depth"] = np.array([len(lv)])
        for i, (lro, lci, lv_, agg) in enumerate(lv):
            g[f"amg{i}_ro"], g[f"amg{i}_ci"], g[f"amg{i}_v_sha"] = lro, lci, np.array(sha(lv_))
            if agg is not None:
                g[f"amg{i}_agg"] = agg
        for method, pc in SOLVES:
            cfg = make_cfg(method=method, precond=pc, max_iters=300)
            rc, x, rep, h = R.solve(A, b, x0, cfg)
            tag = f"m{method}p{pc}"
            g[f"{tag}_rc"] = np.array([rc])
            g[f"{tag}_iters"] = np.array([rep.iterations])
            g[f"{tag}_conv"] = np.array([rep.converged])
            g[f"{tag}_res"] = np.array([rep.initial_residual, rep.final_residual])
            g[f"{tag}_hist"] = h
            g[f"{tag}_x"] = x
        np.savez_compressed(os.path.join(OUT, name + ".npz"), **g)
        index[name] = {"kind": kind, "nx": nx, "ny": ny, "nz": nz, "aspect": asp, "seed": seed}
    with open(os.path.join(OUT, "index.json"), "w") as f:
        json.dump(index, f, indent=1, sort_keys=True)
    print("wrote", len(index), "golden sets to", OUT)


if __name__ == "__main__":
    main()
