"""Test-side access to the CPU checkers (TEST INFRASTRUCTURE ONLY).

* ``Restatement`` — oracle/_build/libbcs_oracle.so, the C restatement of the
  reference hot path (oracle/bcs_oracle.c).  Always available (built by
  __graft_entry__.build()).
* ``Reference``   — oracle/_ref/libbcs_ref.so, the reference itself compiled
  from /root/reference by oracle/Makefile.  Present wherever build() ran with
  the reference mounted; the .so travels to the GPU box with the snapshot.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_SO = os.path.join(ROOT, "oracle", "_build", "libbcs_oracle.so")
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libbcs_ref.so")

c_int, c_double, c_void_p = ctypes.c_int, ctypes.c_double, ctypes.c_void_p


def ptr(a):
    return None if a is None else a.ctypes.data_as(c_void_p)


class OrCfg(ctypes.Structure):
    _fields_ = [("method", c_int), ("precond", c_int), ("rel_tol", c_double), ("abs_tol", c_double),
                ("max_iters", c_int), ("gmres_restart", c_int), ("amg_max_levels", c_int),
                ("amg_min_coarse_rows", c_int), ("amg_pre_sweeps", c_int), ("amg_post_sweeps", c_int)]


class OrReport(ctypes.Structure):
    _fields_ = [("iterations", c_int), ("converged", c_int), ("breakdown", c_int), ("amg_levels", c_int),
                ("initial_residual", c_double), ("final_residual", c_double)]


class RefReport(ctypes.Structure):
    _fields_ = [("iterations", c_int), ("converged", c_int), ("breakdown", c_int), ("setupBranch", c_int),
                ("initial_residual", c_double), ("final_residual", c_double)] + \
               [(k, c_double) for k in ("tConvert", "tSetup", "tReplace", "tSolve", "tRetrieve")]


def cfg_tuple(cfg):
    """(method, precond, relTol, absTol, maxIters, restart, maxLevels, minCoarse, pre, post)"""
    return tuple(cfg)


def make_cfg(method=0, precond=3, rel_tol=1e-8, abs_tol=1e-300, max_iters=1000, restart=30, max_levels=30,
             min_coarse=8, pre=1, post=1):
    return (method, precond, rel_tol, abs_tol, max_iters, restart, max_levels, min_coarse, pre, post)


def _sys_args(A):
    return (A.n_cells, A.nFaces(), A.n, ptr(A.owner), ptr(A.neighbour), ptr(A.diag), ptr(A.upper), ptr(A.lower))


class Restatement:
    def __init__(self):
        if not os.path.exists(ORACLE_SO):
            raise FileNotFoundError(f"{ORACLE_SO} missing: run __graft_entry__.build()")
        self.L = ctypes.CDLL(ORACLE_SO)
        self.L.or_signature.restype = ctypes.c_ulonglong
        self.L.or_amg_build.restype = c_void_p
        self.L.or_amg_depth.argtypes = [c_void_p]
        self.L.or_amg_level_sizes.argtypes = [c_void_p, c_int] + [ctypes.POINTER(c_int)] * 3
        self.L.or_amg_level_get.argtypes = [c_void_p, c_int] + [c_void_p] * 4
        self.L.or_amg_free.argtypes = [c_void_p]
        self.L.or_last_error.restype = ctypes.c_char_p

    def err(self):
        return self.L.or_last_error().decode()

    def csr(self, A):
        nnz = A.n_cells + 2 * A.nFaces()
        ro = np.zeros(A.n_cells + 1, np.int32)
        ci = np.zeros(nnz, np.int32)
        src = np.zeros(nnz, np.int32)
        self.L.or_csr_plan(A.n_cells, A.nFaces(), ptr(A.owner), ptr(A.neighbour), ptr(ro), ptr(ci), ptr(src))
        v = np.zeros(nnz * A.n * A.n)
        self.L.or_csr_values(A.n_cells, A.nFaces(), A.n, ptr(src), ptr(A.diag), ptr(A.upper), ptr(A.lower), ptr(v))
        return ro, ci, src, v

    def signature(self, A):
        return int(self.L.or_signature(A.n_cells, A.nFaces(), ptr(A.owner), ptr(A.neighbour)))

    def matvec(self, A, x):
        ro, ci, _, v = self.csr(A)
        y = np.zeros_like(x)
        self.L.or_csr_matvec(A.n_cells, A.n, ptr(ro), ptr(ci), ptr(v), ptr(x), ptr(y))
        return y

    def ldu_matvec(self, A, x):
        y = np.zeros_like(x)
        self.L.or_ldu_matvec(*_sys_args(A), ptr(x), ptr(y))
        return y

    def aggregate(self, ro, ci, v, n):
        rows = ro.size - 1
        agg = np.zeros(rows, np.int32)
        nc = self.L.or_aggregate(rows, n, ptr(ro), ptr(ci), ptr(v), ptr(agg))
        return agg, nc

    def precond_apply(self, A, cfg, r):
        c = OrCfg(*cfg)
        z = np.zeros_like(r)
        rc = self.L.or_precond_apply(*_sys_args(A), ctypes.byref(c), ptr(r), ptr(z))
        if rc:
            raise RuntimeError(self.err())
        return z

    def solve(self, A, b, x0, cfg, hist_cap=100000, dot_mode=0):
        self.L.or_set_dot_mode(int(dot_mode))
        try:
            return self._solve(A, b, x0, cfg, hist_cap)
        finally:
            self.L.or_set_dot_mode(0)

    def _solve(self, A, b, x0, cfg, hist_cap):
        c = OrCfg(*cfg)
        x = np.zeros_like(b)
        rep = OrReport()
        h = np.zeros(hist_cap)
        hn = c_int()
        rc = self.L.or_solve(*_sys_args(A), ptr(b), ptr(x0), ctypes.byref(c), ptr(x), ctypes.byref(rep), ptr(h),
                             hist_cap, ctypes.byref(hn))
        return rc, x, rep, h[: min(hn.value, hist_cap)]

    def amg_levels(self, A, max_levels=30, min_coarse=8):
        h = self.L.or_amg_build(*_sys_args(A), max_levels, min_coarse)
        if not h:
            raise RuntimeError(self.err())
        out = []
        try:
            for lvl in range(self.L.or_amg_depth(h)):
                rows, nnz, alen = c_int(), c_int(), c_int()
                self.L.or_amg_level_sizes(h, lvl, ctypes.byref(rows), ctypes.byref(nnz), ctypes.byref(alen))
                ro = np.zeros(rows.value + 1, np.int32)
                ci = np.zeros(nnz.value, np.int32)
                v = np.zeros(nnz.value * A.n * A.n)
                agg = np.full(rows.value, -1, np.int32)
                self.L.or_amg_level_get(h, lvl, ptr(ro), ptr(ci), ptr(v), ptr(agg) if alen.value else None)
                out.append((ro, ci, v, agg if alen.value else None))
        finally:
            self.L.or_amg_free(h)
        return out

    def decompose(self, centroids, n_ranks):
        nc = centroids.shape[0]
        c2r = np.zeros(nc, np.int32)
        rro = np.zeros(n_ranks + 1, np.int32)
        o2n = np.zeros(nc, np.int32)
        cen = np.ascontiguousarray(centroids, np.float64)
        rc = self.L.or_decompose(nc, ptr(cen), n_ranks, ptr(c2r), ptr(rro), ptr(o2n))
        if rc:
            raise ValueError(self.err())
        return c2r, rro, o2n


def reference_available():
    return os.path.exists(REF_SO)


class Reference:
    """The unmodified reference (oracle/_ref) through oracle/ref_driver.cpp."""

    def __init__(self):
        if not os.path.exists(REF_SO):
            raise FileNotFoundError(REF_SO)
        L = self.L = ctypes.CDLL(REF_SO)
        L.ref_last_error.restype = ctypes.c_char_p
        L.ref_signature.restype = ctypes.c_ulonglong
        L.ref_gen_euler.argtypes = [c_int] * 3 + [c_double, ctypes.c_longlong] + [c_void_p] * 7
        L.ref_gen_coupled.argtypes = [c_int] * 3 + [c_double, ctypes.c_longlong] + [c_void_p] * 8
        L.ref_gen_euler_poly.argtypes = [c_int] * 3 + [c_double, ctypes.c_longlong, ctypes.c_longlong] + [c_void_p] * 7
        L.ref_gen_euler_kinds.argtypes = ([c_int] * 3 + [c_double, ctypes.c_longlong, ctypes.c_longlong, c_void_p, c_int,
                                           c_int] + [c_void_p] * 7)
        L.ref_gen_coupled_poly.argtypes = [c_int] * 3 + [c_double, ctypes.c_longlong, ctypes.c_longlong] + [c_void_p] * 8
        L.ref_gen_coupled_bcs.argtypes = ([c_int] * 3 + [c_double, ctypes.c_longlong, ctypes.c_longlong]
                                          + [c_void_p] * 3 + [c_int] + [c_void_p] * 9)
        L.ref_amg_build.restype = c_void_p
        L.ref_amg_depth.argtypes = [c_void_p]
        L.ref_amg_level_sizes.argtypes = [c_void_p, c_int] + [ctypes.POINTER(c_int)] * 3
        L.ref_amg_level_get.argtypes = [c_void_p, c_int] + [c_void_p] * 4
        L.ref_amg_free.argtypes = [c_void_p]
        L.ref_pipe_new.restype = c_void_p
        L.ref_pipe_new.argtypes = [c_int, c_int, c_int] + [c_void_p] * 7
        L.ref_pipe_solve.argtypes = [c_void_p, c_int, c_void_p, c_void_p, c_void_p, c_void_p]
        L.ref_pipe_free.argtypes = [c_void_p]
        L.ref_partition.restype = c_void_p
        L.ref_part_count.argtypes = [c_void_p]
        L.ref_part_sizes.argtypes = [c_void_p, c_int] + [ctypes.POINTER(c_int)] * 5
        L.ref_part_get.argtypes = [c_void_p, c_int] + [c_void_p] * 9
        L.ref_part_free.argtypes = [c_void_p]

    def err(self):
        return self.L.ref_last_error().decode()

    @staticmethod
    def _faces(nx, ny, nz, poly):
        nf = (nx - 1) * ny * nz + nx * (ny - 1) * nz + nx * ny * (nz - 1)
        if poly >= 0:  # the augmented count (sizing only; contents are compared)
            from paper_2403_07882_b200 import gen
            nf = gen.hex_sizes(nx, ny, nz, poly)[1]
        return nx * ny * nz, nf

    def gen_euler(self, nx, ny, nz, aspect=1.0, seed=-1, poly=-1):
        nc, nf = self._faces(nx, ny, nz, poly)
        a = [np.zeros(nf, np.int32), np.zeros(nf, np.int32), np.zeros(nc * 25), np.zeros(nf * 25),
             np.zeros(nf * 25), np.zeros(nc * 5), np.zeros(nc * 3)]
        rc = self.L.ref_gen_euler_poly(nx, ny, nz, aspect, seed, poly, *[ptr(x) for x in a])
        assert rc == 0, self.err()
        return a

    def gen_euler_kinds(self, nx, ny, nz, kinds, aspect=1.0, seed=-1, poly=-1, recon=0, flux=0):
        """gen_euler with EulerCase::patchOverride: kinds = 6 PatchKind values
        for the xmin xmax ymin ymax zmin zmax patches (euler.cpp:345-348);
        recon 0 first order, 1 MUSCL (no limiter), 2 MUSCL + Barth-Jespersen;
        flux 0 Roe, 1 HLLC, 2 Rusanov."""
        nc, nf = self._faces(nx, ny, nz, poly)
        k = np.ascontiguousarray(kinds, np.int32)
        assert k.size == 6
        a = [np.zeros(nf, np.int32), np.zeros(nf, np.int32), np.zeros(nc * 25), np.zeros(nf * 25),
             np.zeros(nf * 25), np.zeros(nc * 5), np.zeros(nc * 3)]
        rc = self.L.ref_gen_euler_kinds(nx, ny, nz, aspect, seed, poly, ptr(k), recon, flux, *[ptr(x) for x in a])
        assert rc == 0, self.err()
        return a

    def gen_coupled_bcs(self, nx, ny, nz, kinds, u, p, aspect=1.0, seed=-1, poly=-1, pin=0):
        """gen_coupled with one IncompressibleBc per hex patch (kinds: Kind
        order wall, movingWall, inlet, outlet; u: 6x3; p: 6).  Returns owner,
        neighbour, diag, upper, lower, rhs, state, centroids, phi."""
        nc, nf = self._faces(nx, ny, nz, poly)
        k = np.ascontiguousarray(kinds, np.int32)
        uu = np.ascontiguousarray(u, np.float64).reshape(-1)
        pp = np.ascontiguousarray(p, np.float64)
        a = [np.zeros(nf, np.int32), np.zeros(nf, np.int32), np.zeros(nc * 16), np.zeros(nf * 16),
             np.zeros(nf * 16), np.zeros(nc * 4), np.zeros(nc * 4), np.zeros(nc * 3), np.zeros(nf)]
        rc = self.L.ref_gen_coupled_bcs(nx, ny, nz, aspect, seed, poly, ptr(k), ptr(uu), ptr(pp), pin,
                                        *[ptr(x) for x in a])
        assert rc == 0, self.err()
        return a

    def gen_coupled(self, nx, ny, nz, aspect=1.0, seed=-1, poly=-1):
        nc, nf = self._faces(nx, ny, nz, poly)
        a = [np.zeros(nf, np.int32), np.zeros(nf, np.int32), np.zeros(nc * 16), np.zeros(nf * 16),
             np.zeros(nf * 16), np.zeros(nc * 4), np.zeros(nc * 4), np.zeros(nc * 3)]
        rc = self.L.ref_gen_coupled_poly(nx, ny, nz, aspect, seed, poly, *[ptr(x) for x in a])
        assert rc == 0, self.err()
        return a

    def signature(self, A):
        return int(self.L.ref_signature(A.n_cells, A.nFaces(), ptr(A.owner), ptr(A.neighbour)))

    def csr(self, A):
        nnz = A.n_cells + 2 * A.nFaces()
        ro = np.zeros(A.n_cells + 1, np.int32)
        ci = np.zeros(nnz, np.int32)
        v = np.zeros(nnz * A.n * A.n)
        rc = self.L.ref_csr(*_sys_args(A), ptr(ro), ptr(ci), ptr(v))
        assert rc == 0, self.err()
        return ro, ci, v

    def matvec(self, A, x):
        y = np.zeros_like(x)
        y2 = np.zeros_like(x)
        rc = self.L.ref_matvec(*_sys_args(A), ptr(x), ptr(y), ptr(y2))
        assert rc == 0, self.err()
        return y, y2

    def precond_apply(self, A, cfg, r):
        c = OrCfg(*cfg)
        z = np.zeros_like(r)
        rc = self.L.ref_precond_apply(*_sys_args(A), ctypes.byref(c), ptr(r), ptr(z))
        if rc:
            raise RuntimeError(self.err())
        return z

    def solve(self, A, b, x0, cfg, backend=1, calls=1, hist=True, hist_cap=100000):
        c = OrCfg(*cfg)
        x = np.zeros_like(b)
        rep = RefReport()
        h = np.zeros(hist_cap) if hist else None
        hn = c_int()
        rc = self.L.ref_solve(*_sys_args(A), ptr(b), ptr(x0), backend, ctypes.byref(c), calls, ptr(x),
                              ctypes.byref(rep), ptr(h), hist_cap, ctypes.byref(hn) if hist else None)
        return rc, x, rep, (h[: min(hn.value, hist_cap)] if hist else None)

    def amg_shape(self, A, max_levels=30, min_coarse=8):
        """[(rows, nnz, aggregate or None)] per level of the reference's AmgHierarchy (amg.cpp:73-105),
        without copying level values (cheap enough at 128^3)."""
        h = self.L.ref_amg_build(*_sys_args(A), max_levels, min_coarse)
        if not h:
            raise RuntimeError(self.err())
        out = []
        try:
            for lvl in range(self.L.ref_amg_depth(h)):
                rows, nnz, alen = c_int(), c_int(), c_int()
                self.L.ref_amg_level_sizes(h, lvl, ctypes.byref(rows), ctypes.byref(nnz), ctypes.byref(alen))
                agg = np.full(rows.value, -1, np.int32) if alen.value else None
                if agg is not None:
                    self.L.ref_amg_level_get(h, lvl, None, None, None, ptr(agg))
                out.append((rows.value, nnz.value, agg))
        finally:
            self.L.ref_amg_free(h)
        return out

    def pipeline(self, A, b, x0):
        return RefPipeline(self, A, b, x0)

    def amg_levels(self, A, max_levels=30, min_coarse=8):
        h = self.L.ref_amg_build(*_sys_args(A), max_levels, min_coarse)
        if not h:
            raise RuntimeError(self.err())
        out = []
        try:
            for lvl in range(self.L.ref_amg_depth(h)):
                rows, nnz, alen = c_int(), c_int(), c_int()
                self.L.ref_amg_level_sizes(h, lvl, ctypes.byref(rows), ctypes.byref(nnz), ctypes.byref(alen))
                ro = np.zeros(rows.value + 1, np.int32)
                ci = np.zeros(nnz.value, np.int32)
                v = np.zeros(nnz.value * A.n * A.n)
                agg = np.full(rows.value, -1, np.int32)
                self.L.ref_amg_level_get(h, lvl, ptr(ro), ptr(ci), ptr(v), ptr(agg) if alen.value else None)
                out.append((ro, ci, v, agg if alen.value else None))
        finally:
            self.L.ref_amg_free(h)
        return out

    def decompose(self, centroids, n_ranks):
        nc = centroids.shape[0]
        c2r = np.zeros(nc, np.int32)
        rro = np.zeros(n_ranks + 1, np.int32)
        o2n = np.zeros(nc, np.int32)
        cen = np.ascontiguousarray(centroids, np.float64)
        rc = self.L.ref_decompose(nc, ptr(cen), n_ranks, ptr(c2r), ptr(rro), ptr(o2n))
        if rc:
            raise ValueError(self.err())
        return c2r, rro, o2n


class RefPipeline:
    """One persistent reference SolvePipeline (engine.hpp:28-38) over a fixed
    system: the first solve takes the setup branch, later ones the replace
    branch (engine.cpp:85-98).  solve() returns (wall seconds, report, x)."""

    def __init__(self, R, A, b, x0):
        self.R = R
        self._keep = (A, b, x0)
        self.h = R.L.ref_pipe_new(*_sys_args(A), ptr(b), ptr(x0))
        if not self.h:
            raise RuntimeError(R.err())
        self.size = b.size

    def solve(self, cfg, backend=1, want_x=False):
        c = OrCfg(*cfg)
        rep = RefReport()
        wall = c_double()
        x = np.zeros(self.size) if want_x else None
        rc = self.R.L.ref_pipe_solve(self.h, backend, ctypes.byref(c), ptr(x), ctypes.byref(rep), ctypes.byref(wall))
        if rc:
            raise RuntimeError(self.R.err())
        return wall.value, rep, x

    def close(self):
        if self.h:
            self.R.L.ref_pipe_free(self.h)
            self.h = None

    def __del__(self):
        self.close()


# --- reference test-suite fixtures (tests/support/test_helpers.hpp via ref_driver)
def _ref_mesh(L, fn, *args):
    nc, nf = c_int(), c_int()
    rc = fn(*args, ctypes.byref(nc), ctypes.byref(nf), None, None, None)
    assert rc == 0
    owner = np.zeros(nf.value, np.int32)
    neigh = np.zeros(nf.value, np.int32)
    cen = np.zeros(nc.value * 3)
    rc = fn(*args, ctypes.byref(nc), ctypes.byref(nf), ptr(owner), ptr(neigh), ptr(cen))
    assert rc == 0
    return nc.value, owner, neigh, cen.reshape(-1, 3)


def ref_mesh_2d(R, nx, ny, lx=1.0, ly=1.0):
    R.L.ref_mesh_2d.argtypes = [c_int, c_int, c_double, c_double] + [c_void_p] * 5
    return _ref_mesh(R.L, R.L.ref_mesh_2d, nx, ny, lx, ly)


def ref_mesh_tube(R, n, length=1.0):
    R.L.ref_mesh_tube.argtypes = [c_int, c_double] + [c_void_p] * 5
    return _ref_mesh(R.L, R.L.ref_mesh_tube, n, length)


def ref_randomize(R, nc, owner, neigh, n, seed, boost=4.0):
    R.L.ref_randomize.argtypes = [c_int, c_int, c_int, c_void_p, c_void_p, ctypes.c_uint, c_double] + [c_void_p] * 3
    nf, nn = owner.size, n * n
    d, u, lo = np.zeros(nc * nn), np.zeros(nf * nn), np.zeros(nf * nn)
    rc = R.L.ref_randomize(nc, nf, n, ptr(owner), ptr(neigh), seed, boost, ptr(d), ptr(u), ptr(lo))
    assert rc == 0
    return d, u, lo


def ref_random_vector(R, nc, n, seed):
    R.L.ref_random_vector.argtypes = [c_int, c_int, ctypes.c_uint, c_void_p]
    out = np.zeros(nc * n)
    R.L.ref_random_vector(nc, n, seed, ptr(out))
    return out


def ref_partition(R, A, centroids, n_ranks, n_engines):
    """The reference's buildPartitioned (+consolidate when n_engines > 0) as a list of dicts."""
    L = R.L
    cen = np.ascontiguousarray(centroids, np.float64).reshape(-1)
    h = L.ref_partition(A.n_cells, A.nFaces(), A.n, ptr(A.owner), ptr(A.neighbour), ptr(cen), ptr(A.diag),
                        ptr(A.upper), ptr(A.lower), n_ranks, n_engines)
    assert h, R.err()
    out = []
    try:
        for p in range(L.ref_part_count(h)):
            rs, re, nnz, nh, ns = (c_int() for _ in range(5))
            L.ref_part_sizes(h, p, *(ctypes.byref(x) for x in (rs, re, nnz, nh, ns)))
            nb = A.n * A.n
            d = {"row_start": rs.value, "row_end": re.value, "ro": np.zeros(re.value - rs.value + 1, np.int32),
                 "ci": np.zeros(nnz.value, np.int32), "vals": np.zeros(nnz.value * nb),
                 "halo_row": np.zeros(nh.value, np.int32), "halo_col": np.zeros(nh.value, np.int32),
                 "halo_peer": np.zeros(nh.value, np.int32), "halo_vals": np.zeros(nh.value * nb),
                 "send_peer": np.zeros(ns.value, np.int32), "send_row": np.zeros(ns.value, np.int32)}
            L.ref_part_get(h, p, *(ptr(d[k]) for k in ("ro", "ci", "vals", "halo_row", "halo_col", "halo_peer",
                                                        "halo_vals", "send_peer", "send_row")))
            out.append(d)
    finally:
        L.ref_part_free(h)
    return out


def ref_distributed_solve(R, A, b, x0, centroids, n_ranks, n_engines, cfg):
    L = R.L
    L.ref_distributed_solve.argtypes = [c_int, c_int, c_int] + [c_void_p] * 8 + [c_int, c_int, c_void_p, c_void_p,
                                                                                  c_void_p]
    cen = np.ascontiguousarray(centroids, np.float64).reshape(-1)
    c = OrCfg(*cfg)
    x = np.zeros_like(b)
    rep = RefReport()
    rc = L.ref_distributed_solve(A.n_cells, A.nFaces(), A.n, ptr(A.owner), ptr(A.neighbour), ptr(cen), ptr(A.diag),
                                 ptr(A.upper), ptr(A.lower), ptr(b), ptr(x0), n_ranks, n_engines, ctypes.byref(c),
                                 ptr(x), ctypes.byref(rep))
    return rc, x, rep
