"""ctypes binding of the C ABI in include/bcs.h (libbcs.so, sm_100a).

The library is built in-tree by ``__graft_entry__.build()`` /
``make -C paper_2403_07882_b200/csrc``.  There is deliberately no fallback:
if the extension is missing, importing the solver raises.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_DIR = os.path.join(_HERE, "lib")
LIB_PATH = os.path.join(LIB_DIR, "libbcs.so")
GEN_PATH = os.path.join(LIB_DIR, "libbcs_gen.so")

c_int = ctypes.c_int
c_double = ctypes.c_double
c_size_t = ctypes.c_size_t
c_void_p = ctypes.c_void_p
c_uint64 = ctypes.c_uint64
P = ctypes.POINTER

BCS_OK = 0
BCS_INVALID_ARGUMENT = 1
BCS_RUNTIME_ERROR = 2
BCS_CUDA_ERROR = 3
BCS_NCCL_ERROR = 4
BCS_OUT_OF_MEMORY = 5


class SolverConfigC(ctypes.Structure):
    """bcs_solver_config (include/bcs.h) == SolverConfig + AmgConfig (krylov.hpp:18-37)."""

    _fields_ = [
        ("method", c_int),
        ("precond", c_int),
        ("rel_tol", c_double),
        ("abs_tol", c_double),
        ("max_iters", c_int),
        ("gmres_restart", c_int),
        ("amg_max_levels", c_int),
        ("amg_min_coarse_rows", c_int),
        ("amg_pre_sweeps", c_int),
        ("amg_post_sweeps", c_int),
        ("mode", c_int),
    ]


class ReportC(ctypes.Structure):
    """bcs_report == SolveReport (krylov.hpp:39-50) + stage timings."""

    _fields_ = [
        ("iterations", c_int),
        ("converged", c_int),
        ("breakdown", c_int),
        ("setup_branch", c_int),
        ("initial_residual", c_double),
        ("final_residual", c_double),
        ("t_convert", c_double),
        ("t_setup", c_double),
        ("t_replace", c_double),
        ("t_solve", c_double),
        ("t_retrieve", c_double),
        ("t_amg_setup", c_double),
        ("t_krylov", c_double),
        ("amg_levels", c_int),
        ("coarse_rows", c_int),
        ("spmv_launches", c_int),
        ("spmv_ms", c_double),
        ("kernel_launches", c_int),
        ("sweep_launches", c_int),
        ("sweep_ms", c_double),
        ("sweep_bytes", c_double),
    ]


# name -> (restype, argtypes); every symbol declared in include/bcs.h
SIGNATURES = {
    "bcs_default_config": (None, [P(SolverConfigC)]),
    "bcs_version": (ctypes.c_char_p, []),
    "bcs_create": (c_int, [P(c_void_p), c_int]),
    "bcs_destroy": (c_int, [c_void_p]),
    "bcs_last_error": (ctypes.c_char_p, [c_void_p]),
    "bcs_set_stream": (c_int, [c_void_p, c_void_p]),
    "bcs_set_kernel_timing": (c_int, [c_void_p, c_int]),
    "bcs_host_alloc": (c_int, [c_size_t, P(c_void_p)]),
    "bcs_host_free": (None, [c_void_p]),
    "bcs_ldu_save": (c_int, [ctypes.c_char_p, c_int, c_int, c_int] + [c_void_p] * 7),
    "bcs_ldu_load_sizes": (c_int, [ctypes.c_char_p] + [P(c_int)] * 5),
    "bcs_ldu_load": (c_int, [ctypes.c_char_p] + [c_void_p] * 7),
    "bcs_topology_signature": (c_uint64, [c_int, c_int, c_void_p, c_void_p]),
    "bcs_pipeline_solve": (
        c_int,
        [c_void_p, c_int, c_int, c_int, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_size_t,
         c_void_p, c_size_t, c_void_p, c_int, P(SolverConfigC), P(ReportC)],
    ),
    "bcs_set_topology": (c_int, [c_void_p, c_int, c_int, c_int, c_void_p, c_void_p]),
    "bcs_upload_ldu": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p]),
    "bcs_upload_ldu_device": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p]),
    "bcs_assemble_euler": (c_int, [c_void_p, c_int, c_int, c_void_p, c_void_p, c_void_p, c_int, c_void_p, c_void_p,
                                   c_void_p, c_void_p, c_double, c_void_p]),
    "bcs_assemble_euler_patches": (c_int, [c_void_p, c_int, c_int, c_void_p, c_void_p, c_void_p, c_int, c_void_p,
                                           c_void_p, c_void_p, c_void_p, c_void_p, c_double, c_void_p]),
    "bcs_assemble_euler_ex": (c_int, [c_void_p, c_int, c_int] + [c_void_p] * 5 + [c_int] + [c_void_p] * 5
                              + [c_int, c_int, c_double, c_void_p]),
    "bcs_assemble_coupled": (c_int, [c_void_p, c_int, c_int] + [c_void_p] * 6 + [c_int] + [c_void_p] * 6
                             + [c_double, c_int, c_double, c_void_p]),
    "bcs_assemble_coupled_ex": (c_int, [c_void_p, c_int, c_int] + [c_void_p] * 6 + [c_int] + [c_void_p] * 7
                                + [c_double, c_int, c_double, c_void_p]),
    "bcs_solve": (c_int, [c_void_p, c_void_p, c_void_p, P(SolverConfigC), P(ReportC)]),
    "bcs_solve_device": (c_int, [c_void_p, c_void_p, c_void_p, P(SolverConfigC), P(ReportC)]),
    "bcs_residual": (c_int, [c_void_p, c_void_p, c_void_p, P(c_double)]),
    "bcs_residual_history": (c_int, [c_void_p, c_void_p, c_int, P(c_int)]),
    "bcs_spmv": (c_int, [c_void_p, c_void_p, c_void_p]),
    "bcs_spmv_device": (c_int, [c_void_p, c_void_p, c_void_p]),
    "bcs_csr_get": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p]),
    "bcs_precond_setup": (c_int, [c_void_p, P(SolverConfigC)]),
    "bcs_precond_apply": (c_int, [c_void_p, c_void_p, c_void_p]),
    "bcs_amg_depth": (c_int, [c_void_p, P(c_int)]),
    "bcs_amg_level_sizes": (c_int, [c_void_p, c_int, P(c_int), P(c_int)]),
    "bcs_amg_level_get": (c_int, [c_void_p, c_int, c_void_p, c_void_p, c_void_p, c_void_p]),
    "bcs_level_schedule_depth": (c_int, [c_void_p, c_int, P(c_int)]),
    "bcs_memory_report": (c_int, [c_void_p, ctypes.c_char_p, ctypes.c_size_t, P(ctypes.c_size_t)]),
    "bcs_selftest_hypot": (c_int, [c_void_p, c_void_p, c_void_p, c_int]),
    "bcs_level_coloring": (c_int, [c_void_p, c_int, P(c_int), c_void_p, c_void_p]),
    "bcs_partition_gather_values": (c_int, [c_void_p, c_int, c_int, c_int, c_int, c_void_p, c_void_p, c_void_p,
                                            c_void_p, c_void_p]),
    "bcs_dist_solve": (c_int, [c_void_p, c_int, c_int, c_int] + [c_void_p] * 9 + [c_int, c_int, P(SolverConfigC), P(ReportC)]),
    "bcs_dist_solve_parts": (c_int, [c_void_p, c_int, c_int] + [c_void_p] * 9 + [c_int] + [c_void_p] * 5 +
                             [P(SolverConfigC), P(ReportC)]),
    "bcs_partition_create": (c_int, [P(c_void_p), c_int, c_int, c_void_p, c_void_p, c_void_p, c_int, c_int]),
    "bcs_partition_destroy": (None, [c_void_p]),
    "bcs_partition_count": (c_int, [c_void_p]),
    "bcs_partition_decomposition": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p]),
    "bcs_partition_sizes": (c_int, [c_void_p, c_int, P(c_int), P(c_int), P(c_int), P(c_int), P(c_int)]),
    "bcs_partition_get": (c_int, [c_void_p, c_int] + [c_void_p] * 9),
    "bcs_partition_exchange_sizes": (c_int, [c_void_p, c_int, P(c_int), P(c_int)]),
    "bcs_partition_exchange_get": (c_int, [c_void_p, c_int] + [c_void_p] * 5),
    "bcs_comm_unique_id": (c_int, [c_void_p]),
    "bcs_comm_init": (c_int, [c_void_p, c_int, c_int, c_void_p]),
    "bcs_dist_solve_mp": (c_int, [c_void_p, c_int, c_int, c_int] + [c_void_p] * 9 + [c_int, P(SolverConfigC), P(ReportC)]),
    "bcs_selftest": (c_int, [c_int, ctypes.c_ulonglong, ctypes.c_ulonglong, P(ctypes.c_ulonglong)]),
}

GEN_SIGNATURES = {
    "bcsgen_hex_sizes": (None, [c_int, c_int, c_int, P(c_int), P(c_int)]),
    "bcsgen_hex_euler": (c_int, [c_int, c_int, c_int, c_double, ctypes.c_longlong] + [c_void_p] * 7),
    "bcsgen_hex_coupled": (c_int, [c_int, c_int, c_int, c_double, ctypes.c_longlong] + [c_void_p] * 8),
    "bcsgen_hex_boundary_count": (None, [c_int, c_int, c_int, P(c_int)]),
    "bcsgen_hex_euler_inputs": (c_int, [c_int, c_int, c_int, c_double, ctypes.c_longlong, ctypes.c_longlong]
                                + [c_void_p] * 4),
    "bcsgen_hex_coupled_inputs": (c_int, [c_int, c_int, c_int, c_double, ctypes.c_longlong, ctypes.c_longlong]
                                  + [c_void_p] * 10),
    "bcsgen_hex_sizes_poly": (None, [c_int, c_int, c_int, ctypes.c_longlong, P(c_int), P(c_int)]),
    "bcsgen_hex_euler_poly": (c_int, [c_int, c_int, c_int, c_double, ctypes.c_longlong, ctypes.c_longlong]
                              + [c_void_p] * 7),
    "bcsgen_hex_coupled_poly": (c_int, [c_int, c_int, c_int, c_double, ctypes.c_longlong, ctypes.c_longlong]
                                + [c_void_p] * 8),
}

_lib = None
_gen = None


def pinned_empty(count: int, dtype=np.float64) -> np.ndarray:
    """Uninitialised array in page-locked host memory from the library's
    pinned-buffer cache (bcs_host_alloc); the block returns to the cache when
    the array is garbage-collected."""
    import weakref
    dt = np.dtype(dtype)
    nbytes = max(1, int(count) * dt.itemsize)
    p = c_void_p()
    L = lib()
    if L.bcs_host_alloc(nbytes, ctypes.byref(p)) != 0 or not p.value:
        raise MemoryError(f"bcs_host_alloc({nbytes}) failed")
    raw = (ctypes.c_ubyte * nbytes).from_address(p.value)
    weakref.finalize(raw, L.bcs_host_free, p.value)
    return np.frombuffer(raw, dtype=dt, count=int(count))


def _bind(lib, sigs):
    for name, (res, args) in sigs.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


def lib():
    """The loaded libbcs.so; raises if it has not been built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build the CUDA extension first "
                "(python -c 'import __graft_entry__ as g; g.build()')"
            )
        _lib = _bind(ctypes.CDLL(LIB_PATH), SIGNATURES)
    return _lib


def gen():
    global _gen
    if _gen is None:
        if not os.path.exists(GEN_PATH):
            raise ImportError(f"{GEN_PATH} is missing: build first")
        _gen = _bind(ctypes.CDLL(GEN_PATH), GEN_SIGNATURES)
    return _gen


def ptr(a):
    """Raw pointer of a contiguous numpy array (or None)."""
    if a is None:
        return None
    return a.ctypes.data_as(c_void_p)
