"""Synthetic workloads of SURVEY §8(d) via libbcs_gen.so (csrc/gen/bcs_gen.cpp).

``hex_euler``   — 5x5 density-based Jacobian (restates euler.cpp:390-455)
``hex_coupled`` — 4x4 pressure-based coupled p-U system (incompressible.cpp:143-264)

``poly_seed >= 0`` adds the polyhedral augmentation of SURVEY §8(d) (C5): a
seeded 30% of the cells get an extra face to their edge-diagonal neighbour
(i+1, j+1, k), so rows have mixed 6/7/8... couplings.

Both are bit-identical to the reference producers (tests/test_generator.py).
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .bcs import BlockLduMatrix, BlockVector


@dataclass
class System:
    A: BlockLduMatrix
    b: BlockVector
    x0: BlockVector
    centroids: np.ndarray  # (n_cells, 3)
    name: str


def hex_sizes(nx: int, ny: int, nz: int, poly_seed: int = -1):
    nc, nf = ctypes.c_int(), ctypes.c_int()
    N.gen().bcsgen_hex_sizes_poly(nx, ny, nz, int(poly_seed), ctypes.byref(nc), ctypes.byref(nf))
    return nc.value, nf.value


def _alloc(nx, ny, nz, n, pinned_alloc=None, poly_seed=-1):
    nc, nf = hex_sizes(nx, ny, nz, poly_seed)
    mk = pinned_alloc or (lambda size, dt: np.zeros(size, dt))
    owner = mk(nf, np.int32)
    neigh = mk(nf, np.int32)
    diag = mk(nc * n * n, np.float64)
    upper = mk(nf * n * n, np.float64)
    lower = mk(nf * n * n, np.float64)
    rhs = mk(nc * n, np.float64)
    cen = mk(nc * 3, np.float64) if pinned_alloc else np.zeros(nc * 3)
    return nc, nf, owner, neigh, diag, upper, lower, rhs, cen


def _tag(scramble_seed, poly_seed):
    return ("scrambled" if scramble_seed >= 0 else "natural") + (f" poly{poly_seed}" if poly_seed >= 0 else "")


def hex_euler(nx: int, ny: int = None, nz: int = None, aspect: float = 1.0, scramble_seed: int = -1,
              alloc=None, poly_seed: int = -1, fill: bool = True) -> System:
    """fill=False: the arrays `alloc` returns already hold this system (e.g.
    mappings of a copy another process generated); nothing is written."""
    ny = nx if ny is None else ny
    nz = nx if nz is None else nz
    nc, nf, owner, neigh, diag, upper, lower, rhs, cen = _alloc(nx, ny, nz, 5, alloc, poly_seed)
    if fill:
        rc = N.gen().bcsgen_hex_euler_poly(nx, ny, nz, float(aspect), int(scramble_seed), int(poly_seed),
                                           N.ptr(owner), N.ptr(neigh), N.ptr(diag), N.ptr(upper), N.ptr(lower),
                                           N.ptr(rhs), N.ptr(cen))
        if rc:
            raise ValueError("bcsgen_hex_euler: bad arguments")
    A = BlockLduMatrix(nc, owner, neigh, 5, diag, upper, lower)
    x0 = (alloc or (lambda size, dt: np.zeros(size, dt)))(nc * 5, np.float64)
    if fill:
        x0[:] = 0.0
    return System(A, BlockVector(nc, 5, rhs), BlockVector(nc, 5, x0), cen.reshape(nc, 3),
                  f"euler5 {nx}x{ny}x{nz} {_tag(scramble_seed, poly_seed)} AR{aspect:g}")


def hex_coupled(nx: int, ny: int = None, nz: int = None, aspect: float = 1.0, scramble_seed: int = -1,
                alloc=None, poly_seed: int = -1, fill: bool = True) -> System:
    """fill=False: as hex_euler."""
    ny = nx if ny is None else ny
    nz = nx if nz is None else nz
    nc, nf, owner, neigh, diag, upper, lower, rhs, cen = _alloc(nx, ny, nz, 4, alloc, poly_seed)
    x0 = (alloc or (lambda size, dt: np.zeros(size, dt)))(nc * 4, np.float64)
    if fill:
        rc = N.gen().bcsgen_hex_coupled_poly(nx, ny, nz, float(aspect), int(scramble_seed), int(poly_seed),
                                             N.ptr(owner), N.ptr(neigh), N.ptr(diag), N.ptr(upper), N.ptr(lower),
                                             N.ptr(rhs), N.ptr(x0), N.ptr(cen))
        if rc:
            raise ValueError("bcsgen_hex_coupled: bad arguments")
    A = BlockLduMatrix(nc, owner, neigh, 4, diag, upper, lower)
    return System(A, BlockVector(nc, 4, rhs), BlockVector(nc, 4, x0), cen.reshape(nc, 3),
                  f"coupled4 {nx}x{ny}x{nz} {_tag(scramble_seed, poly_seed)} AR{aspect:g}")


def hex_euler_inputs(nx: int, ny: int = None, nz: int = None, aspect: float = 1.0, scramble_seed: int = -1,
                     poly_seed: int = -1):
    """Inputs of the 5x5 assembly on the hex mesh of ``hex_euler`` (same
    arguments): face area vectors, boundary faces (cell, area) in patch order,
    the seeded primitive state q and the freestream -- for the device assembly."""
    ny = nx if ny is None else ny
    nz = nx if nz is None else nz
    nc, nf = hex_sizes(nx, ny, nz, poly_seed)
    nb = ctypes.c_int()
    N.gen().bcsgen_hex_boundary_count(nx, ny, nz, ctypes.byref(nb))
    area = np.zeros(3 * nf)
    bcell = np.zeros(nb.value, np.int32)
    barea = np.zeros(3 * nb.value)
    q = np.zeros(5 * nc)
    rc = N.gen().bcsgen_hex_euler_inputs(nx, ny, nz, float(aspect), int(scramble_seed), int(poly_seed), N.ptr(area),
                                         N.ptr(bcell), N.ptr(barea), N.ptr(q))
    if rc:
        raise ValueError("bcsgen_hex_euler_inputs: bad arguments")
    q_inf = np.array([1.0, 0.5, 0.1, 0.0, 1.0 / 1.4])
    return area, bcell, barea, q, q_inf


PATCH_KINDS = {"wall": 0, "inlet": 1, "outlet": 2, "farfield": 3, "slip": 4, "symmetry": 5}


def hex_patch_kinds(nx: int, ny: int = None, nz: int = None, kinds=(3, 3, 3, 3, 3, 3)) -> np.ndarray:
    """Per-boundary-face PatchKind (the reference's enum order, PATCH_KINDS)
    for the hex mesh's six patches xmin xmax ymin ymax zmin zmax, in the patch
    order of ``hex_euler_inputs``' boundary faces."""
    ny = nx if ny is None else ny
    nz = nx if nz is None else nz
    k = [PATCH_KINDS[x] if isinstance(x, str) else int(x) for x in kinds]
    if len(k) != 6:
        raise ValueError("hex_patch_kinds: six patch kinds (xmin xmax ymin ymax zmin zmax)")
    sizes = [ny * nz, ny * nz, nx * nz, nx * nz, nx * ny, nx * ny]
    return np.concatenate([np.full(n, v, np.int32) for n, v in zip(sizes, k)])


def hex_patch_values(nx: int, ny: int = None, nz: int = None, values=None, width: int = 1) -> np.ndarray:
    """Per-boundary-face copy of one value (width doubles) per hex patch, in
    the patch order of the boundary faces (see hex_patch_kinds)."""
    ny = nx if ny is None else ny
    nz = nx if nz is None else nz
    v = np.asarray(values, np.float64).reshape(6, width)
    sizes = [ny * nz, ny * nz, nx * nz, nx * nz, nx * ny, nx * ny]
    return np.concatenate([np.tile(v[i], n) for i, n in enumerate(sizes)])


def hex_coupled_inputs(nx: int, ny: int = None, nz: int = None, aspect: float = 1.0, scramble_seed: int = -1,
                       poly_seed: int = -1) -> dict:
    """Inputs of assembleCoupled on the mesh of ``hex_coupled`` (same
    arguments): geometry, wall / moving-lid boundary faces, the seeded state and
    the Rhie-Chow face fluxes -- for the device assembly."""
    ny = nx if ny is None else ny
    nz = nx if nz is None else nz
    nc, nf = hex_sizes(nx, ny, nz, poly_seed)
    nb = ctypes.c_int()
    N.gen().bcsgen_hex_boundary_count(nx, ny, nz, ctypes.byref(nb))
    nb = nb.value
    d = dict(face_area=np.zeros(3 * nf), face_fx=np.zeros(nf), cell_vol=np.zeros(nc), cell_centroid=np.zeros(3 * nc),
             bface_cell=np.zeros(nb, np.int32), bface_area=np.zeros(3 * nb), bface_kind=np.zeros(nb, np.int32),
             bface_u=np.zeros(3 * nb), state=np.zeros(4 * nc), phi=np.zeros(nf))
    rc = N.gen().bcsgen_hex_coupled_inputs(nx, ny, nz, float(aspect), int(scramble_seed), int(poly_seed),
                                           *[N.ptr(d[k]) for k in ("face_area", "face_fx", "cell_vol", "cell_centroid",
                                                                   "bface_cell", "bface_area", "bface_kind", "bface_u",
                                                                   "state", "phi")])
    if rc:
        raise ValueError("bcsgen_hex_coupled_inputs: bad arguments")
    return d
