"""General CSR operator on the device and the standalone
sweep / norm helpers (§8 a6).

`SparseMatrix` keeps the reference constructor's contract (reference
sparse.py:20-75): the matrix is converted to float CSR, duplicate entries are
summed and column indices sorted (canonical CSR -- the order csr_matvec sums
in), it must be square, symmetric to 1e-12 relative and have a nonzero
diagonal; `inv_diag = 1.0 / diag`.  The device copy is the same CSR (int64 row
pointers, int32 columns) plus inv_diag, swept by libsrj's generic kernel with
the reference's exact summation order, so iterates stay bit-identical.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .operators import DeviceOperator, Field, _torch

SYMMETRY_RTOL = 1e-12


class SparseMatrix(DeviceOperator):
    def __init__(self, csr, device=None):
        import scipy.sparse
        m = scipy.sparse.csr_matrix(csr).astype(np.float64)
        m.sum_duplicates()
        m.sort_indices()
        rows, cols = m.shape
        if rows != cols:
            raise ValueError(f"matrix must be square, got {rows}x{cols}")
        scale = max(1.0, float(abs(m).max()) if m.nnz else 0.0)
        asym = abs(m - m.T)
        if asym.nnz and asym.max() > SYMMETRY_RTOL * scale:
            raise ValueError("matrix is not symmetric")
        d = m.diagonal()
        if not np.all(d != 0.0):
            raise ValueError("every row needs a structurally present nonzero diagonal")
        self._csr = m
        self.n = rows
        self.halo = 0
        self.diag = d
        self.inv_diag = 1.0 / d
        self._init_device(device)

    # ------------------------------------------------------------ reference surface
    @property
    def row_ptr(self) -> np.ndarray:
        return self._csr.indptr

    @property
    def col_idx(self) -> np.ndarray:
        return self._csr.indices

    @property
    def vals(self) -> np.ndarray:
        return self._csr.data

    @property
    def nnz(self) -> int:
        return self._csr.nnz

    @classmethod
    def from_coo(cls, n: int, rows, cols, vals, device=None) -> "SparseMatrix":
        import scipy.sparse
        return cls(scipy.sparse.coo_matrix((vals, (rows, cols)), shape=(n, n)).tocsr(),
                   device=device)

    @classmethod
    def from_dense(cls, dense, device=None) -> "SparseMatrix":
        import scipy.sparse
        return cls(scipy.sparse.csr_matrix(np.asarray(dense, dtype=np.float64)), device=device)

    def to_dense(self) -> np.ndarray:
        return self._csr.toarray()

    def scipy_csr(self):
        return self._csr

    @property
    def planes(self) -> int:
        return 1

    # ------------------------------------------------------------ device side
    def _fill_desc(self, desc, dev) -> None:
        torch = _torch()
        rp = torch.from_numpy(np.ascontiguousarray(self._csr.indptr, dtype=np.int64)).to(dev)
        ci = torch.from_numpy(np.ascontiguousarray(self._csr.indices, dtype=np.int32)).to(dev)
        cv = torch.from_numpy(np.ascontiguousarray(self._csr.data, dtype=np.float64)).to(dev)
        inv = torch.from_numpy(np.ascontiguousarray(self.inv_diag, dtype=np.float64)).to(dev)
        self._keep = (rp, ci, cv, inv)
        desc.family = _lib.SRJ_CSR
        desc.nx, desc.ny, desc.nz = self.n, 1, 1
        desc.nnz = self._csr.nnz
        desc.row_ptr, desc.col_idx = rp.data_ptr(), ci.data_ptr()
        desc.values, desc.inv_diag = cv.data_ptr(), inv.data_ptr()


# ---------------------------------------------------------------------------
# Standalone helpers (reference sparse.py:78-111), device computed
# ---------------------------------------------------------------------------

def _kind(v):
    return "numpy" if isinstance(v, np.ndarray) else "torch"


def _back(template, t):
    return t.cpu().numpy() if _kind(template) == "numpy" else t


def _check_len(A, *vs, what):
    for v in vs:
        if tuple(v.shape) != (A.n,):
            raise ValueError(f"dimension mismatch in {what}")


def matvec(A: DeviceOperator, x):
    """A x (reference sparse.py:78-81)."""
    if tuple(x.shape) != (A.n,):
        raise ValueError(f"dimension mismatch: matrix {A.n}, vector {tuple(x.shape)}")
    return _back(x, A.matvec(A.field(x)))


def weighted_jacobi_sweep(A: DeviceOperator, x, b, omega: float):
    """x + omega * D^{-1} (b - A x) (reference sparse.py:84-93)."""
    _check_len(A, x, b, what="weighted_jacobi_sweep")
    out = A.sweep(A.field(x), A.field(b), omega)
    return _back(x, out.interior)


def residual_l2(A: DeviceOperator, x, b) -> float:
    _check_len(A, x, b, what="residual_l2")
    return float(np.sqrt(A.residual_sq(A.field(x), A.field(b))))


def relative_residual_l2(A: DeviceOperator, x, b, x0) -> float:
    r0 = residual_l2(A, x0, b)
    if r0 == 0.0:
        raise ValueError("initial residual is zero; relative residual undefined")
    return residual_l2(A, x, b) / r0


def diff_inf(x_new, x_old) -> float:
    """max |x_new - x_old| (reference sparse.py:108-111)."""
    if tuple(x_new.shape) != tuple(x_old.shape):
        raise ValueError("dimension mismatch in diff_inf")
    if _kind(x_new) == "numpy":
        return float(np.max(np.abs(x_new - x_old))) if x_new.size else 0.0
    return float((x_new - x_old).abs().max()) if x_new.numel() else 0.0


__all__ = ["SparseMatrix", "matvec", "weighted_jacobi_sweep", "residual_l2",
           "relative_residual_l2", "diff_inf", "Field"]
