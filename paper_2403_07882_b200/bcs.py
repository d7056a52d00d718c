"""Host-side mirror of the reference solver API over the C ABI.

Reference interface (blockfv, proj/core/include/blockfv):
  * ``SolverConfig`` / ``AmgConfig`` / ``SolveReport``   krylov.hpp:18-50
  * ``KrylovMethod`` / ``PrecondKind``                  krylov.hpp:15-16
  * ``Backend``, ``SolvePipeline.solve``, ``backend_solve`` engine.hpp:17-43
  * ``BlockLduMatrix`` / ``BlockVector`` (layout only)   block_matrix.hpp:20-87

Errors keep the reference's semantics: ``std::invalid_argument`` surfaces as
``ValueError`` and ``std::runtime_error`` as ``RuntimeError`` with the
reference's message text.  Everything numerical runs on the B200 through
libbcs.so; there is no CPU path.
"""
from __future__ import annotations

import ctypes
import enum
from dataclasses import dataclass, field
from typing import Dict, Optional, Tuple

import numpy as np

from . import _native as N


class KrylovMethod(enum.IntEnum):
    GMRES = 0
    PBiCGStab = 1
    FGMRES = 2  # flexible GMRES (x += Z y); same Arnoldi scalars as GMRES


class PrecondKind(enum.IntEnum):
    none = 0
    LUSGS = 1
    DILU = 2
    AMG = 3


class Backend(enum.IntEnum):
    HostLdu = 0
    EngineCsr = 1


@dataclass
class AmgConfig:
    maxLevels: int = 10
    minCoarseRows: int = 8
    preSweeps: int = 1
    postSweeps: int = 1
    aggregationSize: int = 2


class Mode(enum.IntEnum):
    """bcs_solver_config.mode (include/bcs.h): PARITY (default: reference order
    except the global dot association), PERF (multicolour smoothers), EXACT
    (the reference's sequential dot order too: bit-identical histories)."""
    PARITY = 0
    PERF = 1
    EXACT = 2
    PERF_JACOBI = 3


@dataclass
class SolverConfig:
    method: KrylovMethod = KrylovMethod.GMRES
    preconditioner: PrecondKind = PrecondKind.LUSGS
    relTol: float = 1e-6
    absTol: float = 1e-300
    maxIters: int = 500
    gmresRestart: int = 30
    amg: AmgConfig = field(default_factory=AmgConfig)
    mode: Mode = Mode.PARITY

    def to_c(self) -> N.SolverConfigC:
        return N.SolverConfigC(
            int(self.method), int(self.preconditioner), float(self.relTol), float(self.absTol),
            int(self.maxIters), int(self.gmresRestart), int(self.amg.maxLevels), int(self.amg.minCoarseRows),
            int(self.amg.preSweeps), int(self.amg.postSweeps), int(self.mode),
        )


@dataclass
class SolveReport:
    iterations: int = 0
    initialResidual: float = 0.0
    finalResidual: float = 0.0
    converged: bool = False
    breakdown: bool = False
    timings: Dict[str, float] = field(default_factory=dict)
    amgLevels: int = 0
    coarseRows: int = 0
    spmvLaunches: int = 0
    spmvMs: float = 0.0
    kernelLaunches: int = 0
    sweepLaunches: int = 0
    sweepMs: float = 0.0
    sweepBytes: float = 0.0

    @staticmethod
    def from_c(r: N.ReportC, backend: Optional[Backend] = None) -> "SolveReport":
        t = {"convert": r.t_convert, "solve": r.t_solve, "retrieve": r.t_retrieve,
             "amgSetup": r.t_amg_setup, "krylov": r.t_krylov}
        if backend is None or backend == Backend.EngineCsr:
            t["setup"] = r.t_setup
            t["replace"] = r.t_replace
        else:
            t["setup"] = 0.0
        return SolveReport(r.iterations, r.initial_residual, r.final_residual, bool(r.converged),
                           bool(r.breakdown), t, r.amg_levels, r.coarse_rows, r.spmv_launches, r.spmv_ms,
                           r.kernel_launches, r.sweep_launches, r.sweep_ms, r.sweep_bytes)

    def csvRow(self) -> str:  # krylov.cpp:24-34
        g = self.timings.get
        return ",".join(f"{v:.12g}" for v in (self.iterations, self.initialResidual, self.finalResidual,
                                              g("convert", 0.0), g("setup", 0.0), g("solve", 0.0),
                                              g("retrieve", 0.0)))

    @staticmethod
    def csvHeader() -> str:
        return "iter,initRes,finalRes,tConvert,tSetup,tSolve,tRetrieve"


class BlockVector:
    """AoS block vector: n_cells * block_size doubles (block_matrix.hpp:20-30)."""

    def __init__(self, n_cells: int = 0, block_size: int = 0, values: Optional[np.ndarray] = None):
        self.blockSize = int(block_size)
        if values is None:
            values = np.zeros(int(n_cells) * int(block_size))
        self.values = np.ascontiguousarray(values, dtype=np.float64).reshape(-1)

    def nCells(self) -> int:
        return self.values.size // self.blockSize if self.blockSize else 0


class BlockLduMatrix:
    """Face-addressed block LDU operator (block_matrix.hpp:40-87), layout only.

    owner/neighbour: int32 per internal face with owner < neighbour;
    diag (n_cells, n, n), upper/lower (n_faces, n, n), row-major blocks.
    """

    def __init__(self, n_cells: int, owner, neighbour, block_size: int, diag=None, upper=None, lower=None):
        self.n_cells = int(n_cells)
        self.owner = np.ascontiguousarray(owner, dtype=np.int32)
        self.neighbour = np.ascontiguousarray(neighbour, dtype=np.int32)
        self.n = int(block_size)
        nn = self.n * self.n
        nf = self.owner.size
        self.diag = np.zeros(self.n_cells * nn) if diag is None else np.ascontiguousarray(diag, np.float64).reshape(-1)
        self.upper = np.zeros(nf * nn) if upper is None else np.ascontiguousarray(upper, np.float64).reshape(-1)
        self.lower = np.zeros(nf * nn) if lower is None else np.ascontiguousarray(lower, np.float64).reshape(-1)

    def blockSize(self) -> int:
        return self.n

    def nCells(self) -> int:
        return self.n_cells

    def nFaces(self) -> int:
        return int(self.owner.size)


def _raise(status: int, msg: str):
    if status == N.BCS_INVALID_ARGUMENT:
        raise ValueError(msg)
    if status == N.BCS_OUT_OF_MEMORY:
        raise MemoryError(msg)
    raise RuntimeError(msg)


class Context:
    """One bcs_ctx (one B200)."""

    def __init__(self, device: int = 0):
        self._lib = N.lib()
        h = ctypes.c_void_p()
        st = self._lib.bcs_create(ctypes.byref(h), int(device))
        if st != N.BCS_OK:
            _raise(st, self._lib.bcs_last_error(None).decode())
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            self._lib.bcs_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _ck(self, st: int):
        if st != N.BCS_OK:
            _raise(st, self._lib.bcs_last_error(self.h).decode())

    # --- staged interface
    def set_stream(self, stream_ptr: int):
        self._ck(self._lib.bcs_set_stream(self.h, ctypes.c_void_p(stream_ptr)))

    def set_kernel_timing(self, on: bool):
        self._ck(self._lib.bcs_set_kernel_timing(self.h, 1 if on else 0))

    def set_topology(self, A: BlockLduMatrix):
        self._ck(self._lib.bcs_set_topology(self.h, A.n_cells, A.nFaces(), A.n, N.ptr(A.owner), N.ptr(A.neighbour)))

    def upload_ldu(self, A: BlockLduMatrix):
        self._ck(self._lib.bcs_upload_ldu(self.h, N.ptr(A.diag), N.ptr(A.upper), N.ptr(A.lower)))

    def upload_ldu_device(self, d_diag: int, d_upper: int, d_lower: int):
        self._ck(self._lib.bcs_upload_ldu_device(self.h, c_ptr(d_diag), c_ptr(d_upper), c_ptr(d_lower)))

    def assemble_euler(self, owner, neighbour, face_area, bface_cell, bface_area, q, q_inf, cfl: float,
                       out: Optional[np.ndarray] = None, bface_kind=None, muscl: Optional[str] = None,
                       face_fx=None, cell_centroid=None, flux: str = "roe") -> np.ndarray:
        """Device assembleJacobian + computeResidual (Roe): the matrix goes into
        this context; returns the right-hand side.  ``bface_kind``: the
        reference's PatchKind per boundary face (0 wall, 1 inlet, 2 outlet,
        3 farfield, 4 slip, 5 symmetry); None = all farfield.  ``muscl``: None
        (first order), "none" or "BarthJespersen" (ReconstructionConfig::limiter;
        needs ``face_fx`` and ``cell_centroid``).  ``flux``: "roe", "hllc" or
        "rusanov" (fluxSchemeFromString names) for the residual."""
        owner = np.ascontiguousarray(owner, np.int32)
        neighbour = np.ascontiguousarray(neighbour, np.int32)
        face_area = np.ascontiguousarray(face_area, np.float64)
        bface_cell = np.ascontiguousarray(bface_cell, np.int32)
        bface_area = np.ascontiguousarray(bface_area, np.float64)
        q = np.ascontiguousarray(q, np.float64)
        q_inf = np.ascontiguousarray(q_inf, np.float64)
        nc = q.size // 5
        rhs = np.zeros(nc * 5) if out is None else out
        if muscl is not None or flux != "roe":
            recon = {None: 0, "none": 1, "BarthJespersen": 2}.get(muscl, -1)
            if recon < 0:
                raise ValueError(f"assemble_euler: unknown limiter {muscl!r}")
            scheme = {"roe": 0, "hllc": 1, "rusanov": 2}.get(flux)
            if scheme is None:
                raise ValueError(f"unknown flux scheme: {flux}")
            if recon and (face_fx is None or cell_centroid is None):
                raise ValueError("assemble_euler: MUSCL needs face_fx and cell_centroid")
            fx = None if face_fx is None else np.ascontiguousarray(face_fx, np.float64)
            cen = None if cell_centroid is None else np.ascontiguousarray(cell_centroid, np.float64)
            bk = None if bface_kind is None else np.ascontiguousarray(bface_kind, np.int32)
            if bk is not None and bk.size != bface_cell.size:
                raise ValueError("assemble_euler: bface_kind needs one entry per boundary face")
            self._ck(self._lib.bcs_assemble_euler_ex(self.h, nc, owner.size, N.ptr(owner), N.ptr(neighbour),
                                                     N.ptr(face_area), N.ptr(fx), N.ptr(cen), bface_cell.size,
                                                     N.ptr(bface_cell), N.ptr(bface_area), N.ptr(bk), N.ptr(q),
                                                     N.ptr(q_inf), recon, scheme, float(cfl), N.ptr(rhs)))
        elif bface_kind is None:
            self._ck(self._lib.bcs_assemble_euler(self.h, nc, owner.size, N.ptr(owner), N.ptr(neighbour),
                                                  N.ptr(face_area), bface_cell.size, N.ptr(bface_cell),
                                                  N.ptr(bface_area), N.ptr(q), N.ptr(q_inf), float(cfl), N.ptr(rhs)))
        else:
            bface_kind = np.ascontiguousarray(bface_kind, np.int32)
            if bface_kind.size != bface_cell.size:
                raise ValueError("assemble_euler: bface_kind needs one entry per boundary face")
            self._ck(self._lib.bcs_assemble_euler_patches(self.h, nc, owner.size, N.ptr(owner), N.ptr(neighbour),
                                                          N.ptr(face_area), bface_cell.size, N.ptr(bface_cell),
                                                          N.ptr(bface_area), N.ptr(bface_kind), N.ptr(q), N.ptr(q_inf),
                                                          float(cfl), N.ptr(rhs)))
        return rhs

    def assemble_coupled(self, owner, neighbour, face_area, face_fx, cell_vol, cell_centroid, bface_cell, bface_area,
                         bface_kind, bface_u, state, phi, nu: float, pin_cell: int = 0, pin_value: float = 0.0,
                         out: Optional[np.ndarray] = None, bface_p=None) -> np.ndarray:
        """Device assembleCoupled + pinPressure: the matrix goes into this
        context; returns the right-hand side.  ``bface_kind``: the
        IncompressibleBc kind per boundary face (0 wall, 1 moving wall, 2 inlet,
        3 outlet); ``bface_u`` the wall / inlet velocity, ``bface_p`` the outlet
        pressure (needed when there is an outlet)."""
        i32 = lambda a: np.ascontiguousarray(a, np.int32)  # noqa: E731
        f64 = lambda a: np.ascontiguousarray(a, np.float64)  # noqa: E731
        owner, neighbour, bface_cell, bface_kind = i32(owner), i32(neighbour), i32(bface_cell), i32(bface_kind)
        face_area, face_fx, cell_vol, cell_centroid = f64(face_area), f64(face_fx), f64(cell_vol), f64(cell_centroid)
        bface_area, bface_u, state, phi = f64(bface_area), f64(bface_u), f64(state), f64(phi)
        nc = cell_vol.size
        rhs = np.zeros(nc * 4) if out is None else out
        bp = None if bface_p is None else f64(bface_p)
        self._ck(self._lib.bcs_assemble_coupled_ex(
            self.h, nc, owner.size, N.ptr(owner), N.ptr(neighbour), N.ptr(face_area), N.ptr(face_fx), N.ptr(cell_vol),
            N.ptr(cell_centroid), bface_cell.size, N.ptr(bface_cell), N.ptr(bface_area), N.ptr(bface_kind),
            N.ptr(bface_u), N.ptr(bp), N.ptr(state), N.ptr(phi), float(nu), int(pin_cell), float(pin_value),
            N.ptr(rhs)))
        return rhs

    def solve(self, b: np.ndarray, x: np.ndarray, cfg: SolverConfig) -> SolveReport:
        rep = N.ReportC()
        c = cfg.to_c()
        self._ck(self._lib.bcs_solve(self.h, N.ptr(b), N.ptr(x), ctypes.byref(c), ctypes.byref(rep)))
        return SolveReport.from_c(rep)

    def solve_device(self, d_b: int, d_x: int, cfg: SolverConfig) -> SolveReport:
        rep = N.ReportC()
        c = cfg.to_c()
        self._ck(self._lib.bcs_solve_device(self.h, c_ptr(d_b), c_ptr(d_x), ctypes.byref(c), ctypes.byref(rep)))
        return SolveReport.from_c(rep)

    def residual(self, b: np.ndarray, x: np.ndarray) -> float:
        v = ctypes.c_double()
        self._ck(self._lib.bcs_residual(self.h, N.ptr(b), N.ptr(x), ctypes.byref(v)))
        return v.value

    def residual_history(self) -> np.ndarray:
        n = ctypes.c_int()
        self._ck(self._lib.bcs_residual_history(self.h, None, 0, ctypes.byref(n)))
        out = np.zeros(n.value)
        self._ck(self._lib.bcs_residual_history(self.h, N.ptr(out), n.value, ctypes.byref(n)))
        return out

    def spmv(self, x: np.ndarray) -> np.ndarray:
        y = np.zeros_like(x)
        self._ck(self._lib.bcs_spmv(self.h, N.ptr(x), N.ptr(y)))
        return y

    def spmv_device(self, d_x: int, d_y: int):
        self._ck(self._lib.bcs_spmv_device(self.h, c_ptr(d_x), c_ptr(d_y)))

    def csr(self, n_cells: int, nnz: int, n: int):
        ro = np.zeros(n_cells + 1, np.int32)
        ci = np.zeros(nnz, np.int32)
        v = np.zeros(nnz * n * n)
        self._ck(self._lib.bcs_csr_get(self.h, N.ptr(ro), N.ptr(ci), N.ptr(v)))
        return ro, ci, v

    def precond_setup(self, cfg: SolverConfig):
        c = cfg.to_c()
        self._ck(self._lib.bcs_precond_setup(self.h, ctypes.byref(c)))

    def precond_apply(self, r: np.ndarray) -> np.ndarray:
        z = np.zeros_like(r)
        self._ck(self._lib.bcs_precond_apply(self.h, N.ptr(r), N.ptr(z)))
        return z

    def amg_depth(self) -> int:
        d = ctypes.c_int()
        self._ck(self._lib.bcs_amg_depth(self.h, ctypes.byref(d)))
        return d.value

    def amg_level(self, level: int, n: int):
        rows, nnz = ctypes.c_int(), ctypes.c_int()
        self._ck(self._lib.bcs_amg_level_sizes(self.h, level, ctypes.byref(rows), ctypes.byref(nnz)))
        ro = np.zeros(rows.value + 1, np.int32)
        ci = np.zeros(nnz.value, np.int32)
        v = np.zeros(nnz.value * n * n)
        agg = np.full(rows.value, -1, np.int32)
        self._ck(self._lib.bcs_amg_level_get(self.h, level, N.ptr(ro), N.ptr(ci), N.ptr(v), N.ptr(agg)))
        return ro, ci, v, agg

    def amg_level_shape(self, level: int, want_agg: bool = True):
        """(rows, nnz, aggregate or None) of one level without copying its values."""
        rows, nnz = ctypes.c_int(), ctypes.c_int()
        self._ck(self._lib.bcs_amg_level_sizes(self.h, level, ctypes.byref(rows), ctypes.byref(nnz)))
        agg = None
        if want_agg:
            agg = np.full(rows.value, -1, np.int32)
            self._ck(self._lib.bcs_amg_level_get(self.h, level, None, None, None, N.ptr(agg)))
        return rows.value, nnz.value, agg

    def amg_level_rows(self, level: int) -> int:
        rows, nnz = ctypes.c_int(), ctypes.c_int()
        self._ck(self._lib.bcs_amg_level_sizes(self.h, level, ctypes.byref(rows), ctypes.byref(nnz)))
        return rows.value

    def memory_report(self) -> dict:
        """Device bytes held by this context per category (bcs_memory_report)."""
        import json
        need = ctypes.c_size_t()
        self._ck(self._lib.bcs_memory_report(self.h, None, 0, ctypes.byref(need)))
        buf = ctypes.create_string_buffer(need.value + 16)
        self._ck(self._lib.bcs_memory_report(self.h, buf, need.value + 16, ctypes.byref(need)))
        return json.loads(buf.value.decode())

    def level_coloring(self, level: int):
        """(n_colors, perm, color_offsets) of a level's performance-mode smoother
        (n_colors 0: natural order; perm[new] = row; colour c = perm[off[c]:off[c+1]])."""
        nc = ctypes.c_int()
        self._ck(self._lib.bcs_level_coloring(self.h, level, ctypes.byref(nc), None, None))
        if nc.value == 0:
            return 0, None, None
        perm = np.zeros(self.amg_level_rows(level), np.int32)
        off = np.zeros(nc.value + 1, np.int32)
        self._ck(self._lib.bcs_level_coloring(self.h, level, ctypes.byref(nc), N.ptr(perm), N.ptr(off)))
        return nc.value, perm, off

    def schedule_depth(self, level: int) -> int:
        d = ctypes.c_int()
        self._ck(self._lib.bcs_level_schedule_depth(self.h, level, ctypes.byref(d)))
        return d.value

    def pipeline_solve(self, A: BlockLduMatrix, b: BlockVector, x0: BlockVector, backend: Backend,
                       cfg: SolverConfig) -> Tuple[BlockVector, SolveReport]:
        # the result lives in cached page-locked memory: full-rate D2H, no page faults
        x = BlockVector(A.n_cells, A.n, values=N.pinned_empty(A.n_cells * A.n))
        rep = N.ReportC()
        c = cfg.to_c()
        st = self._lib.bcs_pipeline_solve(
            self.h, A.n_cells, A.nFaces(), A.n, N.ptr(A.owner), N.ptr(A.neighbour), N.ptr(A.diag),
            N.ptr(A.upper), N.ptr(A.lower), N.ptr(b.values), b.values.size, N.ptr(x0.values), x0.values.size,
            N.ptr(x.values), int(backend), ctypes.byref(c), ctypes.byref(rep))
        self._ck(st)
        return x, SolveReport.from_c(rep, backend)


    def dist_solve(self, A: BlockLduMatrix, b: BlockVector, x0: BlockVector, centroids: np.ndarray, n_ranks: int,
                   n_engines: int, cfg: SolverConfig) -> Tuple[BlockVector, SolveReport]:
        """Mode R: the reference's distributedSolve (partition.cpp:370-479) on this device."""
        x = BlockVector(A.n_cells, A.n)
        cen = np.ascontiguousarray(centroids, dtype=np.float64).reshape(-1)
        rep = N.ReportC()
        c = cfg.to_c()
        self._ck(self._lib.bcs_dist_solve(self.h, A.n_cells, A.nFaces(), A.n, N.ptr(A.owner), N.ptr(A.neighbour),
                                          N.ptr(cen), N.ptr(A.diag), N.ptr(A.upper), N.ptr(A.lower),
                                          N.ptr(b.values), N.ptr(x0.values), N.ptr(x.values), int(n_ranks),
                                          int(n_engines), ctypes.byref(c), ctypes.byref(rep)))
        r = SolveReport.from_c(rep)
        r.timings = {"convert": rep.t_convert, "setup": rep.t_setup, "solve": rep.t_solve, "retrieve": rep.t_retrieve}
        return x, r

    def dist_solve_parts(self, parts, b: np.ndarray, x0: np.ndarray, n: int, n_engines: int,
                         rank_to_engine, engine_row_offset, cfg: SolverConfig) -> Tuple[np.ndarray, SolveReport]:
        """distributedSolve on caller-built rank partitions (bcs_dist_solve_parts).
        parts: one dict per rank with row_start, row_end, ro, ci, values (nnz*n*n),
        halo_row, halo_col, halo_peer, halo_values; b, x0 and the result are global
        vectors in the new (rank-major) numbering."""
        R = len(parts)
        keep = []  # keep every array alive for the call

        def arr(a, dt):
            a = np.ascontiguousarray(a, dt)
            keep.append(a)
            return a

        def ptrs(key, dt):
            ps = (ctypes.c_void_p * R)(*[arr(p[key], dt).ctypes.data for p in parts])
            keep.append(ps)
            return ctypes.cast(ps, ctypes.c_void_p)
        rro = arr([parts[0]["row_start"]] + [p["row_end"] for p in parts], np.int32)
        hcnt = arr([len(p["halo_col"]) for p in parts], np.int32)
        bb, xx = arr(b, np.float64), arr(x0, np.float64)
        x = np.zeros_like(bb)
        r2e, ero = arr(rank_to_engine, np.int32), arr(engine_row_offset, np.int32)
        c = cfg.to_c()
        rep = N.ReportC()
        st = self._lib.bcs_dist_solve_parts(
            self.h, R, int(n), N.ptr(rro), ptrs("ro", np.int32), ptrs("ci", np.int32), ptrs("values", np.float64),
            N.ptr(hcnt), ptrs("halo_row", np.int32), ptrs("halo_col", np.int32), ptrs("halo_peer", np.int32),
            ptrs("halo_values", np.float64), int(n_engines), N.ptr(r2e), N.ptr(ero), N.ptr(bb), N.ptr(xx),
            N.ptr(x), ctypes.byref(c), ctypes.byref(rep))
        self._ck(st)
        return x, SolveReport.from_c(rep)

    def comm_init(self, rank: int, size: int, uid: bytes):
        """Collective: this context joins an NCCL communicator of `size` processes (one per GPU)."""
        buf = (ctypes.c_ubyte * 128).from_buffer_copy(uid)
        self._ck(self._lib.bcs_comm_init(self.h, int(rank), int(size), buf))

    def dist_solve_mp(self, A: BlockLduMatrix, b: BlockVector, x0: BlockVector, centroids: np.ndarray, n_ranks: int,
                      cfg: SolverConfig) -> Tuple[BlockVector, SolveReport]:
        """Collective Mode R over processes: this process solves engine `rank` (comm_init), exchanging halos and
        dot partials with NCCL; returns the whole solution (original cell order) on every rank."""
        x = BlockVector(A.n_cells, A.n)
        cen = np.ascontiguousarray(centroids, dtype=np.float64).reshape(-1)
        rep = N.ReportC()
        c = cfg.to_c()
        self._ck(self._lib.bcs_dist_solve_mp(self.h, A.n_cells, A.nFaces(), A.n, N.ptr(A.owner), N.ptr(A.neighbour),
                                             N.ptr(cen), N.ptr(A.diag), N.ptr(A.upper), N.ptr(A.lower),
                                             N.ptr(b.values), N.ptr(x0.values), N.ptr(x.values), int(n_ranks),
                                             ctypes.byref(c), ctypes.byref(rep)))
        r = SolveReport.from_c(rep)
        r.timings = {"convert": rep.t_convert, "setup": rep.t_setup, "solve": rep.t_solve, "retrieve": rep.t_retrieve}
        return x, r


class Partition:
    """Host partition layer (decompose + buildPartitioned [+ consolidate]); no device needed."""

    def __init__(self, n_cells, owner, neighbour, centroids, n_ranks, n_engines=0):
        self._lib = N.lib()
        self.n_cells = int(n_cells)
        self.n_ranks = int(n_ranks)
        o = np.ascontiguousarray(owner, np.int32)
        nb = np.ascontiguousarray(neighbour, np.int32)
        cen = np.ascontiguousarray(centroids, np.float64).reshape(-1)
        h = ctypes.c_void_p()
        st = self._lib.bcs_partition_create(ctypes.byref(h), self.n_cells, o.size, N.ptr(o), N.ptr(nb), N.ptr(cen),
                                            self.n_ranks, int(n_engines))
        if st != N.BCS_OK:
            _raise(st, self._lib.bcs_last_error(None).decode())
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            self._lib.bcs_partition_destroy(self.h)
            self.h = None

    def count(self) -> int:
        return int(self._lib.bcs_partition_count(self.h))

    def decomposition(self):
        c2r = np.zeros(self.n_cells, np.int32)
        rro = np.zeros(self.n_ranks + 1, np.int32)
        o2n = np.zeros(self.n_cells, np.int32)
        self._lib.bcs_partition_decomposition(self.h, N.ptr(c2r), N.ptr(rro), N.ptr(o2n))
        return c2r, rro, o2n

    def part(self, i: int) -> dict:
        rs, re, nnz, nh, ns = (ctypes.c_int() for _ in range(5))
        st = self._lib.bcs_partition_sizes(self.h, i, ctypes.byref(rs), ctypes.byref(re), ctypes.byref(nnz),
                                           ctypes.byref(nh), ctypes.byref(ns))
        if st != N.BCS_OK:
            _raise(st, self._lib.bcs_last_error(None).decode())
        d = {"row_start": rs.value, "row_end": re.value,
             "ro": np.zeros(re.value - rs.value + 1, np.int32), "ci": np.zeros(nnz.value, np.int32),
             "src": np.zeros(nnz.value, np.int32), "halo_row": np.zeros(nh.value, np.int32),
             "halo_col": np.zeros(nh.value, np.int32), "halo_peer": np.zeros(nh.value, np.int32),
             "halo_src": np.zeros(nh.value, np.int32), "send_peer": np.zeros(ns.value, np.int32),
             "send_row": np.zeros(ns.value, np.int32)}
        self._lib.bcs_partition_get(self.h, i, *(N.ptr(d[k]) for k in ("ro", "ci", "src", "halo_row", "halo_col",
                                                                        "halo_peer", "halo_src", "send_peer",
                                                                        "send_row")))
        return d

    def gather_values(self, i: int, A: "BlockLduMatrix"):
        """The per-rank upload of engine i (bcs_partition_gather_values): its local
        slots' and halo entries' LDU blocks, gathered on the host in slot order."""
        d = self.part(i)
        nn = A.n * A.n
        loc = np.zeros(d["ci"].size * nn)
        halo = np.zeros(d["halo_col"].size * nn)
        st = self._lib.bcs_partition_gather_values(self.h, i, A.n_cells, A.nFaces(), A.n, N.ptr(A.diag),
                                                   N.ptr(A.upper), N.ptr(A.lower), N.ptr(loc), N.ptr(halo))
        if st != N.BCS_OK:
            _raise(st, self._lib.bcs_last_error(None).decode())
        return loc, halo

    def exchange(self, i: int) -> dict:
        """Per-process halo exchange plan of engine i (see bcs_partition_exchange_get)."""
        ns, nr = ctypes.c_int(), ctypes.c_int()
        st = self._lib.bcs_partition_exchange_sizes(self.h, i, ctypes.byref(ns), ctypes.byref(nr))
        if st != N.BCS_OK:
            _raise(st, self._lib.bcs_last_error(None).decode())
        G = self.count()
        nh = self.part(i)["halo_col"].size
        d = {"send_row": np.zeros(ns.value, np.int32), "send_count": np.zeros(G, np.int32),
             "recv_global_row": np.zeros(nr.value, np.int32), "recv_count": np.zeros(G, np.int32),
             "halo_recv_idx": np.zeros(nh, np.int32)}
        st = self._lib.bcs_partition_exchange_get(self.h, i, *(N.ptr(d[k]) for k in (
            "send_row", "send_count", "recv_global_row", "recv_count", "halo_recv_idx")))
        if st != N.BCS_OK:
            _raise(st, self._lib.bcs_last_error(None).decode())
        return d


def comm_unique_id() -> bytes:
    """128-byte NCCL unique id for bcs_comm_init (create on one rank, broadcast)."""
    buf = (ctypes.c_ubyte * 128)()
    st = N.lib().bcs_comm_unique_id(buf)
    if st != N.BCS_OK:
        _raise(st, N.lib().bcs_last_error(None).decode())
    return bytes(buf)


def c_ptr(p) -> ctypes.c_void_p:
    return ctypes.c_void_p(int(p))


def topology_signature(A: BlockLduMatrix) -> int:
    return int(N.lib().bcs_topology_signature(A.n_cells, A.nFaces(), N.ptr(A.owner), N.ptr(A.neighbour)))


_default_ctx: Optional[Context] = None


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(0)
    return _default_ctx


class SolvePipeline:
    """Stateful pipeline (engine.hpp:28-38): setup on first call / topology
    change, value replace otherwise.  Each pipeline owns one device context."""

    def __init__(self, device: int = 0):
        self.ctx = Context(device)

    def solve(self, A: BlockLduMatrix, b: BlockVector, x0: BlockVector, backend: Backend,
              cfg: SolverConfig) -> Tuple[BlockVector, SolveReport]:
        if b.blockSize != A.n or x0.blockSize != A.n or b.nCells() != A.n_cells or x0.nCells() != A.n_cells:
            raise ValueError("SolvePipeline::solve: dimension mismatch")
        return self.ctx.pipeline_solve(A, b, x0, backend, cfg)


def backend_solve(A: BlockLduMatrix, b: BlockVector, x0: BlockVector, backend: Backend,
                  cfg: SolverConfig) -> Tuple[BlockVector, SolveReport]:
    """One-shot fresh pipeline (engine.cpp:122-127)."""
    p = SolvePipeline()
    try:
        return p.solve(A, b, x0, backend, cfg)
    finally:
        p.ctx.close()


def _ck_global(st: int):
    if st != 0:
        _raise(st, N.lib().bcs_last_error(None).decode())


def save_ldu(path: str, A: BlockLduMatrix, b: Optional[BlockVector] = None, x0: Optional[BlockVector] = None):
    """Binary LDU dump (bcs_ldu_save): topology, blocks and optionally b / x0."""
    n = A.n
    _ck_global(N.lib().bcs_ldu_save(
        str(path).encode(), A.n_cells, A.nFaces(), n, N.ptr(A.owner), N.ptr(A.neighbour), N.ptr(A.diag),
        N.ptr(A.upper), N.ptr(A.lower), N.ptr(b.values) if b is not None else None,
        N.ptr(x0.values) if x0 is not None else None))


def load_ldu(path: str) -> Tuple[BlockLduMatrix, Optional[BlockVector], Optional[BlockVector]]:
    """Read a bcs_ldu_save file; raises RuntimeError on a bad magic, truncation or checksum mismatch."""
    nc, nf, n, hb, hx = (ctypes.c_int() for _ in range(5))
    L = N.lib()
    _ck_global(L.bcs_ldu_load_sizes(str(path).encode(), ctypes.byref(nc), ctypes.byref(nf), ctypes.byref(n),
                                    ctypes.byref(hb), ctypes.byref(hx)))
    nc, nf, n = nc.value, nf.value, n.value
    owner, neigh = np.zeros(nf, np.int32), np.zeros(nf, np.int32)
    diag, upper, lower = np.zeros(nc * n * n), np.zeros(nf * n * n), np.zeros(nf * n * n)
    b = np.zeros(nc * n) if hb.value else None
    x0 = np.zeros(nc * n) if hx.value else None
    _ck_global(L.bcs_ldu_load(str(path).encode(), N.ptr(owner), N.ptr(neigh), N.ptr(diag), N.ptr(upper), N.ptr(lower),
                              N.ptr(b) if b is not None else None, N.ptr(x0) if x0 is not None else None))
    A = BlockLduMatrix(nc, owner, neigh, n, diag, upper, lower)
    return A, (BlockVector(nc, n, b) if b is not None else None), (BlockVector(nc, n, x0) if x0 is not None else None)
