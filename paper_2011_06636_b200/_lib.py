"""ctypes binding of libsrj.so (the C ABI in include/srj.h).

The library is the only compute path: importing the package works without it
(host-side scheme construction, problem metadata), but every device call goes
through `lib()`, which raises if the shared object is missing or was built
against a different ABI.  There is no CPU fallback.
"""

from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_double, c_int32, c_int64, c_uint64, c_void_p

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libsrj.so")
ABI_VERSION = 2

SRJ_OK, SRJ_DIVERGED, SRJ_BAD_ARGUMENT, SRJ_CUDA_ERROR = 0, 1, 2, 3
SRJ_STENCIL_1D3, SRJ_STENCIL_2D5, SRJ_STENCIL_3D7, SRJ_STENCIL_2D5_VAR, SRJ_CSR = 1, 2, 3, 4, 5
SRJ_STENCIL_3D7_VAR, SRJ_STENCIL_1D3_VAR = 6, 7
CYCLE_RAN, CYCLE_CONVERGED, CYCLE_DIVERGED = 0, 1, 2

# Every symbol include/srj.h declares (checked by tests/test_abi.py).
EXPORTED_SYMBOLS = (
    "srj_abi_version", "srj_last_error", "srj_op_create", "srj_op_destroy",
    "srj_op_layout", "srj_op_diag", "srj_op_set_sweeps_per_pass", "srj_op_describe",
    "srj_residual_sq",
    "srj_run_cycle", "srj_sweep", "srj_matvec", "srj_fill_uniform_rhs",
    "srj_op_planes", "srj_sweep_planes", "srj_run_cycle_diffinf", "srj_batch_cycles_1d",
    "srj_op_set_temporal_kernel", "srj_tb_pass", "srj_op_solve_supported", "srj_solve",
    "srj_op_set_reserved_sms", "srj_skew_plan",
    "srj_nccl_available", "srj_nccl_last_error", "srj_nccl_unique_id", "srj_nccl_comm_init",
    "srj_nccl_comm_destroy", "srj_slab_exchange", "srj_allgather_sums", "srj_slab_cycle_forward",
    "srj_slab_exchange_plan",
)
SOLVE_PAUSED, SOLVE_CONVERGED, SOLVE_DIVERGED, SOLVE_BUDGET = 0, 1, 2, 3
SOLVE_HEURISTIC, SOLVE_INCREASING, SOLVE_FIXED = 0, 1, 2
TB_TILE = 0


class BatchJob(ctypes.Structure):
    _fields_ = [("n", c_int32), ("M", c_int32), ("omega_off", c_int64),
                ("x_in_off", c_int64), ("x_out_off", c_int64), ("b_off", c_int64)]


class OpDesc(ctypes.Structure):
    _fields_ = [
        ("family", c_int32), ("device", c_int32),
        ("nx", c_int64), ("ny", c_int64), ("nz", c_int64),
        ("dx2", c_double),
        ("face_x", c_void_p), ("face_y", c_void_p),
        ("nnz", c_int64), ("row_ptr", c_void_p), ("col_idx", c_void_p),
        ("values", c_void_p), ("inv_diag", c_void_p),
        ("face_z", c_void_p),
    ]


class CycleOut(ctypes.Structure):
    _fields_ = [
        ("executed", c_int32), ("status", c_int32), ("result_in_alt", c_int32),
        ("launches", c_int32), ("res_before", c_double), ("res_after", c_double),
    ]


class SolveArgs(ctypes.Structure):
    _fields_ = [
        ("omegas_all", c_void_p), ("level_off", c_void_p),
        ("n_levels", c_int32), ("mode", c_int32), ("level0", c_int32), ("max_cycles", c_int32),
        ("t_hi", c_double), ("t_lo", c_double), ("res0", c_double), ("prev_ratio0", c_double),
        ("budget", c_int64), ("hist_cap", c_int64),
    ]


class SolveRec(ctypes.Structure):
    _fields_ = [("level", c_int32), ("M", c_int32), ("executed", c_int32), ("status", c_int32),
                ("res_before", c_double), ("res_after", c_double)]


class SolveOut(ctypes.Structure):
    _fields_ = [("cycles", c_int32), ("stop", c_int32), ("result_in_alt", c_int32),
                ("next_level", c_int32), ("res_next", c_double), ("prev_ratio", c_double),
                ("sweeps", c_int64)]


class OpInfo(ctypes.Structure):
    _fields_ = [(name, c_int32) for name in (
        "num_sms", "cycle_blocks", "cycle_threads", "sweeps_per_pass", "tb_supported",
        "tb_blocks", "tb_occupancy", "tb_tiles", "cycle_kernel")]

    KERNELS = {0: "srj::k_cycle (generic row walker)",
               1: "srj::k_tb2d_cycle (TMA temporal blocking)",
               2: "srj::k_cycle2d (TMA tile streaming)",
               3: "srj::k_cycle3d (TMA plane ring)",
               5: "srj::k_tb3d_cycle (TMA z-wavefront temporal blocking)",
               6: "srj::k_tbvar_cycle (TMA var-coef temporal blocking)",
               7: "srj::k_small_cycle_1d (single-CTA shared-memory cycle)",
               8: "srj::k_reg_cycle_1d (single-CTA register-resident cycle)",
               9: "srj::k_cycle3dv (TMA plane ring, variable coefficient)",
               10: "srj::k_tb3v_cycle (TMA z-wavefront temporal blocking, variable coefficient)",
               11: "srj::k_tbs_cycle (TMA temporal blocking, skewed tiles)"}

    def as_dict(self):
        return {name: int(getattr(self, name)) for name, _ in self._fields_}


class SrjLibraryError(RuntimeError):
    pass


_lib = None


def _declare(L):
    L.srj_abi_version.restype = c_int32
    L.srj_last_error.restype = ctypes.c_char_p
    L.srj_op_create.argtypes = [POINTER(OpDesc), POINTER(c_void_p)]
    L.srj_op_destroy.argtypes = [c_void_p]
    L.srj_op_layout.argtypes = [c_void_p, POINTER(c_int64), POINTER(c_int64)]
    L.srj_op_diag.argtypes = [c_void_p, POINTER(c_double), POINTER(c_double)]
    L.srj_op_set_sweeps_per_pass.argtypes = [c_void_p, c_int32]
    L.srj_op_describe.argtypes = [c_void_p, POINTER(OpInfo)]
    L.srj_residual_sq.argtypes = [c_void_p, c_void_p, c_void_p, POINTER(c_double), c_void_p]
    L.srj_run_cycle.argtypes = [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_int32,
                                c_double, c_double, c_double, c_int64, c_void_p,
                                POINTER(CycleOut), c_void_p]
    L.srj_sweep.argtypes = [c_void_p, c_void_p, c_void_p, c_void_p, c_double, c_void_p]
    L.srj_matvec.argtypes = [c_void_p, c_void_p, c_void_p, c_void_p]
    L.srj_fill_uniform_rhs.argtypes = [c_void_p, c_int64, c_uint64, c_int64, c_int32, c_void_p]
    L.srj_op_planes.argtypes = [c_void_p]
    L.srj_op_set_temporal_kernel.argtypes = [c_void_p, c_int32]
    L.srj_batch_cycles_1d.argtypes = [c_void_p, c_int32, c_int32, c_void_p, c_void_p, c_void_p,
                                      c_void_p, c_int32, c_void_p]
    L.srj_run_cycle_diffinf.argtypes = [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                        c_int32, c_double, c_double, c_int64, c_void_p,
                                        POINTER(CycleOut), c_void_p]
    L.srj_sweep_planes.argtypes = [c_void_p, c_void_p, c_void_p, c_void_p, c_double, c_int64,
                                   c_int64, c_void_p, c_int32, c_void_p]
    L.srj_tb_pass.argtypes = [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_int32,
                              c_int64, c_int64, c_void_p, c_void_p]
    L.srj_op_solve_supported.argtypes = [c_void_p]
    L.srj_op_set_reserved_sms.argtypes = [c_void_p, c_int32]
    L.srj_solve.argtypes = [c_void_p, c_void_p, c_void_p, c_void_p, POINTER(SolveArgs), c_double,
                            c_double, c_void_p, c_void_p, POINTER(SolveOut), c_void_p]
    L.srj_nccl_last_error.restype = ctypes.c_char_p
    L.srj_nccl_unique_id.argtypes = [c_void_p]
    L.srj_nccl_comm_init.argtypes = [c_int32, c_void_p, c_int32, c_int32, POINTER(c_void_p)]
    L.srj_nccl_comm_destroy.argtypes = [c_void_p]
    L.srj_slab_exchange.argtypes = [c_void_p, c_void_p, c_int32, c_int32, c_void_p, c_int64,
                                    c_int64, c_int64, c_int32, c_void_p]
    L.srj_slab_exchange_plan.argtypes = [c_int64, c_int32, c_int32, c_int64, c_int64, c_int64,
                                         c_int32, POINTER(c_int64)]
    L.srj_allgather_sums.argtypes = [c_void_p, c_int32, c_void_p, c_void_p, c_int64, c_void_p]
    L.srj_slab_cycle_forward.argtypes = [c_void_p, c_void_p, c_int32, c_int32, c_void_p,
                                         c_void_p, c_void_p, c_void_p, c_void_p, c_int32,
                                         c_int32, c_int64, c_int64, c_int64, c_void_p, c_void_p,
                                         POINTER(c_int32), c_void_p]
    for name in EXPORTED_SYMBOLS:
        if name not in ("srj_abi_version", "srj_last_error", "srj_nccl_last_error"):
            getattr(L, name).restype = c_int32
    L.srj_op_planes.restype = c_int64


def skew_plan(nx: int, ny: int, num_ctas: int = 148):
    """Work plan of the skewed-tile 2D kernel (srj_skew_plan; host only, no GPU
    needed): dict with tiles_per_cta, ctas_used, tile_rows, tile_cols, sweeps
    and `tiles`, one list of (ox, oy, lo, hi) per CTA."""
    L = load()
    T, used, rows, cols, sw = (c_int32() for _ in range(5))
    byref = ctypes.byref
    check(L.srj_skew_plan(c_int64(nx), c_int64(ny), c_int32(num_ctas), byref(T), byref(used),
                          byref(rows), byref(cols), byref(sw), None, c_int64(0)), "srj_skew_plan")
    n = 4 * num_ctas * T.value
    table = (c_int32 * n)()
    check(L.srj_skew_plan(c_int64(nx), c_int64(ny), c_int32(num_ctas), byref(T), byref(used),
                          byref(rows), byref(cols), byref(sw), table, c_int64(n)), "srj_skew_plan")
    tiles = []
    for c in range(num_ctas):
        mine = []
        for i in range(T.value):
            ox, oy, lo, hi = table[4 * (c * T.value + i):4 * (c * T.value + i) + 4]
            if hi <= lo:
                break
            mine.append((ox, oy, lo, hi))
        tiles.append(mine)
    return {"tiles_per_cta": T.value, "ctas_used": used.value, "tile_rows": rows.value,
            "tile_cols": cols.value, "sweeps": sw.value, "tiles": tiles}


STRESS_LIB_PATH = os.path.join(_HERE, "libsrj_stress.so")


def load(path: str | None = None):
    """Load and type the shared library (no CUDA call is made).  SRJ_LIBRARY
    selects another build of the same ABI (tests: the race/bounds stress
    build libsrj_stress.so, csrc/srj_stress.cuh)."""
    global _lib
    if _lib is not None:
        return _lib
    if path is None:
        path = os.environ.get("SRJ_LIBRARY") or LIB_PATH
    if not os.path.exists(path):
        raise SrjLibraryError(
            f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
            " (there is no CPU fallback)")
    L = ctypes.CDLL(path)
    _declare(L)
    if L.srj_abi_version() != ABI_VERSION:
        raise SrjLibraryError(f"libsrj ABI {L.srj_abi_version()} != expected {ABI_VERSION}")
    _lib = L
    return L


def lib():
    return load()


def check(rc: int, what: str) -> None:
    if rc != SRJ_OK:
        msg = lib().srj_last_error().decode(errors="replace")
        raise SrjLibraryError(f"{what} failed (status {rc}): {msg}")


def check_nccl(rc: int, what: str) -> None:
    if rc != SRJ_OK:
        msg = lib().srj_nccl_last_error().decode(errors="replace")
        raise SrjLibraryError(f"{what} failed (status {rc}): {msg}")
