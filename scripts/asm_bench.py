"""Device Euler assembly cost at 128^3: first-order Roe with
farfield patches vs the second-order variants (MUSCL + Barth-Jespersen, Roe /
HLLC / Rusanov, mixed patch kinds).  Wall time of one bcs_assemble_euler[_ex]
call from pinned host buffers (state + geometry H2D, rhs D2H included), mean
of 10 after 3 warm-ups.  Usage: python scripts/asm_bench.py [n]"""
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2403_07882_b200 import _native as N, bcs, gen  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
    s = gen.hex_euler(n)
    area, bcell, barea, q, q_inf = gen.hex_euler_inputs(n)
    geo = gen.hex_coupled_inputs(n)
    kinds = gen.hex_patch_kinds(n, n, n, (0, 1, 2, 3, 4, 5))
    ctx = bcs.Context(0)

    def pin(a):
        p = N.pinned_empty(a.size, a.dtype.type)
        p[:] = a
        return p

    p_area, p_barea, p_q = pin(area), pin(barea), pin(q)
    p_fx, p_cen = pin(geo["face_fx"]), pin(geo["cell_centroid"])
    rhs = N.pinned_empty(q.size)
    variants = {
        "roe_first_farfield": dict(),
        "roe_first_mixed_patches": dict(bface_kind=kinds),
        "roe_muscl_bj": dict(bface_kind=kinds, muscl="BarthJespersen"),
        "hllc_muscl_bj": dict(bface_kind=kinds, muscl="BarthJespersen", flux="hllc"),
        "rusanov_muscl_bj": dict(bface_kind=kinds, muscl="BarthJespersen", flux="rusanov"),
    }
    out = {"cells": s.A.n_cells, "faces": int(s.A.owner.size), "ms": {}}
    for name, kw in variants.items():
        extra = dict(face_fx=p_fx, cell_centroid=p_cen) if "muscl" in kw else {}
        times = []
        for it in range(13):
            t0 = time.perf_counter()
            ctx.assemble_euler(s.A.owner, s.A.neighbour, p_area, bcell, p_barea, p_q, q_inf, 50.0, out=rhs, **kw,
                               **extra)
            if it >= 3:
                times.append(time.perf_counter() - t0)
        out["ms"][name] = round(1e3 * float(np.mean(times)), 3)
    ctx.close()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
