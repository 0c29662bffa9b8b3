"""Device-resident operators: the drop-in for `sparse.SparseMatrix` on the
solve path.

The reference's `run_cycle` touches only `A.inv_diag` and `A.scipy_csr().dot`
(reference solver.py:192-193,209,225,233); `ProblemInstance` checks `A.n`
(problems.py:37-39).  Every operator here exposes that surface (`n`, `diag`,
`inv_diag`, `scipy_csr()` for interop) and runs its sweeps in libsrj:

* `StencilOperator` -- structured Dirichlet stencils; the sm_100a kernels
  recompute the constant-coefficient stencil, or read two face-coefficient
  streams, in the exact CSR column order; no matrix is stored.
* `sparse.SparseMatrix` -- any canonical CSR matrix (unstructured problems,
  Neumann grids, random tridiagonals), swept by the generic CSR kernel.

Device vectors are `Field`s: n interior fp64 values with `halo` ghost elements
before and after (one grid plane for stencils, zero for CSR).  Every C-ABI
pointer addresses the first interior element.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np

from . import _lib

FAMILIES = {
    "1d3": _lib.SRJ_STENCIL_1D3,
    "2d5": _lib.SRJ_STENCIL_2D5,
    "3d7": _lib.SRJ_STENCIL_3D7,
    "2d5var": _lib.SRJ_STENCIL_2D5_VAR,
    "3d7var": _lib.SRJ_STENCIL_3D7_VAR,
    "1d3var": _lib.SRJ_STENCIL_1D3_VAR,
}


def _torch():
    import torch
    return torch


def _stream_handle(device):
    torch = _torch()
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


class Field:
    """n interior fp64 values in a buffer with `halo` ghosts per side."""

    def __init__(self, n: int, halo: int, device, buf=None):
        torch = _torch()
        self.n = int(n)
        self.halo = int(halo)
        self.device = torch.device(device)
        if buf is None:
            buf = torch.zeros(self.n + 2 * self.halo, dtype=torch.float64, device=self.device)
        self.buf = buf

    @property
    def interior(self):
        return self.buf[self.halo:self.halo + self.n]

    @property
    def ptr(self) -> int:
        return self.buf.data_ptr() + 8 * self.halo

    def copy_(self, values) -> "Field":
        torch = _torch()
        if isinstance(values, Field):
            values = values.interior
        if isinstance(values, np.ndarray):
            values = torch.from_numpy(np.ascontiguousarray(values, dtype=np.float64))
        self.interior.copy_(values.reshape(-1), non_blocking=False)
        return self

    def clone(self) -> "Field":
        return Field(self.n, self.halo, self.device, self.buf.clone())


class DeviceOperator:
    """Device plumbing shared by every operator: handle, Fields, sweeps,
    residuals and the per-cycle C-ABI calls.  Subclasses set `n`, `halo`,
    `_device` and implement `_fill_desc`."""

    n: int
    halo: int

    def _init_device(self, device) -> None:
        self._device = device
        self._handle = None
        self._keep = ()  # device arrays the native handle points into

    @property
    def device(self):
        torch = _torch()
        if self._device is None:
            self._device = torch.device("cuda", torch.cuda.current_device())
        return torch.device(self._device)

    @property
    def handle(self):
        if self._handle is None:
            self._handle = self._create()
        return self._handle

    def _fill_desc(self, desc, dev) -> None:
        raise NotImplementedError

    def _create(self):
        torch = _torch()
        L = _lib.lib()
        if not torch.cuda.is_available():
            raise _lib.SrjLibraryError("the SRJ device path needs a CUDA device (no CPU fallback)")
        dev = self.device
        desc = _lib.OpDesc()
        desc.device = dev.index if dev.index is not None else torch.cuda.current_device()
        self._fill_desc(desc, dev)
        h = ctypes.c_void_p()
        _lib.check(L.srj_op_create(ctypes.byref(desc), ctypes.byref(h)), "srj_op_create")
        return h

    def set_sweeps_per_pass(self, s: int) -> None:
        _lib.check(_lib.lib().srj_op_set_sweeps_per_pass(self.handle, int(s)),
                   "srj_op_set_sweeps_per_pass")

    def set_temporal_kernel(self, kind: str) -> None:
        """'tile' (TMA overlapped tiles): the temporally blocked 2D kernel that
        serves sweeps_per_pass > 1 (the round-1 'warp_stream' experiment was
        removed; any other kind raises ValueError)."""
        if kind != "tile":
            raise ValueError(f"unknown temporal kernel {kind!r} (only 'tile')")
        code = _lib.TB_TILE
        _lib.check(_lib.lib().srj_op_set_temporal_kernel(self.handle, code),
                   "srj_op_set_temporal_kernel")

    def describe(self) -> dict:
        """Launch configuration libsrj chose for this operator."""
        info = _lib.OpInfo()
        _lib.check(_lib.lib().srj_op_describe(self.handle, ctypes.byref(info)), "srj_op_describe")
        return info.as_dict()

    def new_field(self) -> Field:
        return Field(self.n, self.halo, self.device)

    def field(self, values) -> Field:
        """A fresh zero-ghost device Field holding `values` (numpy or torch)."""
        if isinstance(values, Field):
            return values.clone()
        n = values.shape[0] if values.ndim == 1 else int(np.prod(values.shape))
        if n != self.n:
            raise ValueError(f"dimension mismatch: operator {self.n}, vector {n}")
        return self.new_field().copy_(values)

    def residual_sq(self, x: Field, b: Field) -> float:
        out = ctypes.c_double()
        _lib.check(_lib.lib().srj_residual_sq(self.handle, x.ptr, b.ptr, ctypes.byref(out),
                                              _stream_handle(self.device)), "srj_residual_sq")
        return out.value

    def sweep(self, x: Field, b: Field, omega: float, out: Field | None = None) -> Field:
        out = out if out is not None else self.new_field()
        _lib.check(_lib.lib().srj_sweep(self.handle, x.ptr, out.ptr, b.ptr, float(omega),
                                        _stream_handle(self.device)), "srj_sweep")
        return out

    def sweep_planes(self, x: Field, x_out: Field | None, b: Field, omega: float, z_begin: int,
                     z_end: int, partial_ptr: int, slot: int = 0) -> None:
        """Sweep (or residual, x_out None) of slab planes [z_begin, z_end);
        the planes' sum of r^2 lands at device address `partial_ptr`."""
        _lib.check(_lib.lib().srj_sweep_planes(
            self.handle, x.ptr, x_out.ptr if x_out is not None else None, b.ptr, float(omega),
            int(z_begin), int(z_end), ctypes.c_void_p(partial_ptr), int(slot),
            _stream_handle(self.device)), "srj_sweep_planes")

    def tb_pass(self, x: Field, x_alt: Field, b: Field, omegas_ptr: int, h: int, row_lo: int,
                row_hi: int, sums_ptr: int) -> None:
        """One temporally blocked pass (h <= 6 sweeps in 2D, <= 2 in 3D) storing
        only the owned rows (3D: planes) [row_lo, row_hi) into x_alt; owned sums
        of r^2 per sweep at `sums_ptr` (device).  Rows outside are a slab's deep
        ghost rows (srj_tb_pass)."""
        _lib.check(_lib.lib().srj_tb_pass(
            self.handle, x.ptr, x_alt.ptr, b.ptr, ctypes.c_void_p(omegas_ptr), int(h),
            int(row_lo), int(row_hi), ctypes.c_void_p(sums_ptr), _stream_handle(self.device)),
            "srj_tb_pass")

    def matvec(self, x: Field):
        torch = _torch()
        y = torch.empty(self.n, dtype=torch.float64, device=self.device)
        _lib.check(_lib.lib().srj_matvec(self.handle, x.ptr, y.data_ptr(),
                                         _stream_handle(self.device)), "srj_matvec")
        return y

    def run_cycle(self, x: Field, x_alt: Field, b: Field, omegas_dev, M: int, tol: float,
                  baseline: float, res_before: float, budget: int, history: np.ndarray | None):
        out = _lib.CycleOut()
        hist_ptr = history.ctypes.data if history is not None else None
        _lib.check(_lib.lib().srj_run_cycle(
            self.handle, x.ptr, x_alt.ptr, b.ptr, omegas_dev.data_ptr(), int(M), float(tol),
            float(baseline), float(res_before), int(budget), hist_ptr, ctypes.byref(out),
            _stream_handle(self.device)), "srj_run_cycle")
        return out

    def set_reserved_sms(self, k: int) -> None:
        """Leave k SMs free in the temporally blocked kernels (srj_op_set_reserved_sms)."""
        _lib.check(_lib.lib().srj_op_set_reserved_sms(self.handle, int(k)), "srj_op_set_reserved_sms")

    def solve_supported(self) -> bool:
        """True when whole solves can run on the device (srj_solve)."""
        return bool(_lib.lib().srj_op_solve_supported(self.handle))

    def solve_device(self, x: Field, x_alt: Field, b: Field, omegas_all, level_off,
                     mode: int, level0: int, t_hi: float, t_lo: float, res0: float,
                     prev_ratio: float, budget: int, tol: float, baseline: float,
                     max_cycles: int, hist_cap: int, history: np.ndarray | None):
        """Device-resident solve from x (srj_solve): returns (SolveOut, records)."""
        args = _lib.SolveArgs(omegas_all.data_ptr(), level_off.data_ptr(), int(level_off.numel() - 1),
                              int(mode), int(level0), int(max_cycles), float(t_hi), float(t_lo),
                              float(res0), float(prev_ratio), int(budget), int(hist_cap))
        recs = (_lib.SolveRec * int(max_cycles))()
        out = _lib.SolveOut()
        hist_ptr = history.ctypes.data if history is not None else None
        _lib.check(_lib.lib().srj_solve(
            self.handle, x.ptr, x_alt.ptr, b.ptr, ctypes.byref(args), float(tol), float(baseline),
            ctypes.cast(recs, ctypes.c_void_p), hist_ptr, ctypes.byref(out),
            _stream_handle(self.device)), "srj_solve")
        return out, recs[:out.cycles]

    def run_cycle_diffinf(self, x: Field, x_alt: Field, b: Field, omegas_dev, M: int,
                          tol: float, res_before: float | None, budget: int,
                          history: np.ndarray | None):
        out = _lib.CycleOut()
        hist_ptr = history.ctypes.data if history is not None else None
        rb = float("nan") if res_before is None else float(res_before)
        _lib.check(_lib.lib().srj_run_cycle_diffinf(
            self.handle, x.ptr, x_alt.ptr, b.ptr, omegas_dev.data_ptr(), int(M), float(tol),
            rb, int(budget), hist_ptr, ctypes.byref(out), _stream_handle(self.device)),
            "srj_run_cycle_diffinf")
        return out

    def __del__(self):
        h = getattr(self, "_handle", None)
        if h is not None and _lib._lib is not None:
            try:
                _lib._lib.srj_op_destroy(h)
            except Exception:
                pass


@dataclass(frozen=True)
class Grid:
    family: str
    nx: int
    ny: int = 1
    nz: int = 1

    @property
    def n(self) -> int:
        return self.nx * self.ny * self.nz

    @property
    def halo(self) -> int:
        return {"1d3": 1, "1d3var": 1, "2d5": self.nx, "2d5var": self.nx,
                "3d7": self.nx * self.ny, "3d7var": self.nx * self.ny}[self.family]


VAR_FAMILIES = ("1d3var", "2d5var", "3d7var")
DIMS = {"1d3": 1, "1d3var": 1, "2d5": 2, "2d5var": 2, "3d7": 3, "3d7var": 3}


def face_shapes(family: str, dims) -> tuple:
    """Expected face-array shapes of a variable-coefficient family (numpy
    index order, slowest axis first): face_x couples x-neighbours (one more
    face than points along x), face_y y-neighbours, face_z z-neighbours."""
    if family == "1d3var":
        (nx,) = dims
        return ((nx + 1,),)
    if family == "2d5var":
        nx, ny = dims
        return ((ny, nx + 1), (ny + 1, nx))
    nx, ny, nz = dims
    return ((nz, ny, nx + 1), (nz, ny + 1, nx), (nz + 1, ny, nx))


class StencilOperator(DeviceOperator):
    """Symmetric Dirichlet stencil operator on a structured grid.

    Constant coefficient ("1d3", "2d5", "3d7"): off-diagonals -dx2 and diagonal
    2d*dx2 with dx2 = (N+1)^2, as `poisson_1d` / `poisson_3d` assemble them
    (reference problems.py:50-69,148-177).  Variable coefficient ("1d3var",
    "2d5var", "3d7var"): `face_x` / `face_y` / `face_z` hold the dx2-scaled
    face coefficients (shapes: `face_shapes`); off-diagonals are -face and the
    diagonal is the sum of the point's faces in the order west, east, south,
    north, bottom, top (2D: ((c_w + c_e) + c_s) + c_n).  Face arrays are
    captured when the native handle is created.
    """

    def __init__(self, family: str, shape, dx2: float | None = None,
                 face_x=None, face_y=None, device=None, face_z=None):
        if family not in FAMILIES:
            raise ValueError(f"unknown stencil family {family!r}")
        dims = tuple(int(v) for v in (shape if isinstance(shape, (tuple, list)) else (shape,)))
        want = DIMS[family]
        if len(dims) != want or min(dims) < 1:
            raise ValueError(f"{family} needs {want} positive extents, got {shape!r}")
        self.family = family
        self.shape = dims
        self.grid = Grid(family, *dims)
        self.n = self.grid.n
        self.halo = self.grid.halo
        self._init_device(device)
        self.face_x = self.face_y = self.face_z = None
        if family in VAR_FAMILIES:
            faces = (face_x, face_y, face_z)[:want]
            if any(f is None for f in faces):
                names = ("face_x", "face_y", "face_z")[:want]
                raise ValueError(f"variable-coefficient operator needs {', '.join(names)}")
            faces = [np.asarray(f, dtype=np.float64) if isinstance(f, np.ndarray) else f
                     for f in faces]
            shapes = face_shapes(family, dims)
            for f, shp in zip(faces, shapes):
                if tuple(f.shape) != shp:
                    raise ValueError(f"face arrays must have shapes {shapes}")
            self.face_x = faces[0]
            if want >= 2:
                self.face_y = faces[1]
            if want == 3:
                self.face_z = faces[2]
            self.dx2 = None
        else:
            if dx2 is None:
                dx2 = (dims[0] + 1.0) ** 2
            if not dx2 > 0.0:
                raise ValueError("dx2 must be positive")
            self.dx2 = float(dx2)
        self._diag = None

    @property
    def is_var(self) -> bool:
        return self.family in VAR_FAMILIES

    # ------------------------------------------------------------ SparseMatrix surface
    @property
    def diag_value(self) -> float:
        d = {"1d3": 2.0, "2d5": 4.0, "3d7": 6.0}[self.family]
        return d * self.dx2

    @property
    def diag(self) -> np.ndarray:
        if self._diag is None:
            if self.family == "2d5var":
                fx = _as_numpy(self.face_x)
                fy = _as_numpy(self.face_y)
                self._diag = (((fx[:, :-1] + fx[:, 1:]) + fy[:-1, :]) + fy[1:, :]).reshape(-1)
            elif self.family == "3d7var":
                fx = _as_numpy(self.face_x)
                fy = _as_numpy(self.face_y)
                fz = _as_numpy(self.face_z)
                self._diag = (((((fx[:, :, :-1] + fx[:, :, 1:]) + fy[:, :-1, :]) + fy[:, 1:, :])
                               + fz[:-1]) + fz[1:]).reshape(-1)
            elif self.family == "1d3var":
                fx = _as_numpy(self.face_x)
                self._diag = fx[:-1] + fx[1:]
            else:
                self._diag = np.full(self.n, self.diag_value)
        return self._diag

    @property
    def inv_diag(self) -> np.ndarray:
        return 1.0 / self.diag

    def scipy_csr(self):
        """Host CSR with the reference's canonical layout (interop and tests)."""
        import scipy.sparse
        rows, cols, vals = self.coo()
        m = scipy.sparse.csr_matrix((vals, (rows, cols)), shape=(self.n, self.n))
        m.sum_duplicates()
        m.sort_indices()
        return m

    def coo(self):
        g = self.grid
        ids = np.arange(self.n).reshape(g.nz, g.ny, g.nx)
        diag = self.diag
        rows, cols, vals = [ids.reshape(-1)], [ids.reshape(-1)], [diag]
        if self.is_var:
            # inner faces of each axis (numpy axis 2 = x, 1 = y, 0 = z)
            faces = {2: self.face_x, 1: self.face_y, 0: self.face_z}
            for axis in (2, 1, 0):
                if ids.shape[axis] < 2 or faces[axis] is None:
                    continue
                f = _as_numpy(faces[axis]).reshape(
                    tuple(ids.shape[a] + (1 if a == axis else 0) for a in range(3)))
                inner = np.take(f, np.arange(1, ids.shape[axis]), axis=axis).reshape(-1)
                lo = np.take(ids, np.arange(ids.shape[axis] - 1), axis=axis).reshape(-1)
                hi = np.take(ids, np.arange(1, ids.shape[axis]), axis=axis).reshape(-1)
                rows += [lo, hi]; cols += [hi, lo]; vals += [-inner] * 2
        else:
            off = -1.0 * self.dx2
            for axis in (2, 1, 0):
                if ids.shape[axis] < 2:
                    continue
                lo = np.take(ids, np.arange(ids.shape[axis] - 1), axis=axis).reshape(-1)
                hi = np.take(ids, np.arange(1, ids.shape[axis]), axis=axis).reshape(-1)
                rows += [lo, hi]; cols += [hi, lo]; vals += [np.full(lo.size, off)] * 2
        return np.concatenate(rows), np.concatenate(cols), np.concatenate(vals)

    @property
    def planes(self) -> int:
        """Planes along the slab axis (z in 3D, rows in 2D, 1 in 1D)."""
        return 1 if DIMS[self.family] == 1 else self.shape[-1]

    # ------------------------------------------------------------ device side
    def _fill_desc(self, desc, dev) -> None:
        g = self.grid
        desc.family = FAMILIES[self.family]
        desc.nx, desc.ny, desc.nz = g.nx, g.ny, g.nz
        desc.dx2 = self.dx2 if self.dx2 is not None else 0.0
        if self.is_var:
            keep = []
            for name in ("face_x", "face_y", "face_z"):
                f = getattr(self, name)
                if f is not None:
                    t = _to_device(f, dev).contiguous()
                    keep.append(t)
                    setattr(desc, name, t.data_ptr())
            self._keep = tuple(keep)


def _as_numpy(a) -> np.ndarray:
    if isinstance(a, np.ndarray):
        return a
    return a.detach().cpu().numpy()


def _to_device(a, device):
    torch = _torch()
    if isinstance(a, np.ndarray):
        return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(device)
    return a.to(device=device, dtype=torch.float64)


def fill_uniform_rhs(field_or_tensor, seed: int, start: int = 0) -> None:
    """f_i = 2 u_i - 1 with u the SplitMix64(seed) stream, generated on device."""
    torch = _torch()
    if isinstance(field_or_tensor, Field):
        ptr, n, dev = field_or_tensor.ptr, field_or_tensor.n, field_or_tensor.device
    else:
        t = field_or_tensor
        if not (t.is_cuda and t.dtype == torch.float64 and t.is_contiguous()):
            raise ValueError("need a contiguous float64 CUDA tensor")
        ptr, n, dev = t.data_ptr(), t.numel(), t.device
    _lib.check(_lib.lib().srj_fill_uniform_rhs(
        ctypes.c_void_p(ptr), int(n), int(seed) & ((1 << 64) - 1), int(start),
        dev.index if dev.index is not None else torch.cuda.current_device(),
        _stream_handle(dev)), "srj_fill_uniform_rhs")


def relative_residual(op: DeviceOperator, x: Field, b: Field, x0: Field) -> float:
    r0 = math.sqrt(op.residual_sq(x0, b))
    if r0 == 0.0:
        raise ValueError("initial residual is zero; relative residual undefined")
    return math.sqrt(op.residual_sq(x, b)) / r0
