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
    def wrap(cls, csr, inv_diag, device=None) -> "SparseMatrix":
        """Device copy of a foreign operator's CSR exactly as stored (no
        canonicalisation, no symmetry check) with its own `inv_diag`: the
        reference's run_cycle only reads `A.inv_diag` and sums
        `A.scipy_csr().dot(x)` in stored column order (reference
        solver.py:192-193,233), so both are taken as they are."""
        import scipy.sparse
        m = csr if scipy.sparse.isspmatrix_csr(csr) or isinstance(csr, scipy.sparse.csr_array) \
            else scipy.sparse.csr_matrix(csr)
        if m.dtype != np.float64:
            m = m.astype(np.float64)
        rows, cols = m.shape
        if rows != cols:
            raise ValueError(f"matrix must be square, got {rows}x{cols}")
        inv = np.ascontiguousarray(np.asarray(inv_diag, dtype=np.float64).reshape(-1))
        if inv.shape != (rows,):
            raise ValueError("inv_diag length does not match matrix dimension")
        self = cls.__new__(cls)
        self._csr = m
        self.n = rows
        self.halo = 0
        self.diag = 1.0 / inv
        self.inv_diag = inv
        self._init_device(device)
        return self

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
# Duck-typed operators (reference boundary: solver.py:192-193, problems.py:37-39)
# ---------------------------------------------------------------------------

_WRAPPED: dict = {}


def _structured_from_csr(csr, inv: np.ndarray, device):
    """The StencilOperator equal to `csr` entry for entry, or None.

    Matches the reference's own Dirichlet generators (poisson_1d / poisson_3d,
    problems.py:50-69,148-177, and the 2D 5-point analogue): canonical CSR on
    an m^d grid with the d-dimensional nearest-neighbour pattern, every
    off-diagonal equal to one value -dx2 < 0, every diagonal equal to
    2d*dx2 and inv_diag equal to 1/diag bit for bit.  Then the structured
    kernels compute exactly what csr_matvec computes (same ascending column
    order, same products)."""
    from .operators import StencilOperator
    n = csr.shape[0]
    if n < 2 or not csr.has_canonical_format:
        return None
    for d, fam in ((1, "1d3"), (2, "2d5"), (3, "3d7")):
        m = int(round(n ** (1.0 / d)))
        if m < 2 or m ** d != n:
            continue
        if csr.nnz != (2 * d + 1) * n - 2 * d * m ** (d - 1):
            continue
        op = StencilOperator(fam, (m,) * d, dx2=1.0, device=device)
        pat = op.scipy_csr()
        if not (np.array_equal(pat.indptr, csr.indptr) and np.array_equal(pat.indices, csr.indices)):
            continue
        data = csr.data
        is_diag = pat.data > 0.0
        off = data[~is_diag]
        v = off[0]
        if not (v < 0.0 and np.all(off == v)):
            return None
        dx2 = -v
        if not (np.all(data[is_diag] == 2.0 * d * dx2) and np.all(inv == 1.0 / (2.0 * d * dx2))):
            return None
        return StencilOperator(fam, (m,) * d, dx2=dx2, device=device)
    return None


def device_operator(A, device=None) -> DeviceOperator:
    """The device operator that runs a reference-style duck-typed operator.

    Anything exposing `.n` (or a square `scipy_csr()`), `.inv_diag` and
    `.scipy_csr()` -- e.g. the reference's own `srj.sparse.SparseMatrix` -- is
    accepted, as the reference's run_cycle / solve accept it.  A CSR that is
    exactly a 1D/2D/3D Dirichlet stencil goes to the structured kernels;
    anything else to the general CSR kernel with the operator's own inv_diag.
    The wrapped operator is cached per object for the object's lifetime (a
    weak-keyed table, else an attribute on the object)."""
    if isinstance(A, DeviceOperator):
        return A
    if not (hasattr(A, "scipy_csr") and hasattr(A, "inv_diag")):
        raise TypeError("the SRJ device path needs an operator exposing inv_diag and "
                        f"scipy_csr() (reference solver.py:192-193); got {type(A).__name__}")
    key = id(A)
    hit = _WRAPPED.get(key)
    if hit is not None and hit[0]() is A:
        return hit[1]
    hit = getattr(A, "_srj_device_operator", None)
    if isinstance(hit, DeviceOperator):
        return hit
    import scipy.sparse
    csr = A.scipy_csr()
    if not (scipy.sparse.isspmatrix_csr(csr) or isinstance(csr, scipy.sparse.csr_array)):
        csr = scipy.sparse.csr_matrix(csr)
    inv = np.asarray(A.inv_diag, dtype=np.float64).reshape(-1)
    op = _structured_from_csr(csr, inv, device)
    if op is None:
        op = SparseMatrix.wrap(csr, inv, device=device)
    import weakref
    try:
        ref = weakref.ref(A)
        weakref.finalize(A, _WRAPPED.pop, key, None)
        _WRAPPED[key] = (ref, op)
    except TypeError:  # not weak-referenceable: keep it on the object if possible
        try:
            setattr(A, "_srj_device_operator", op)
        except (AttributeError, TypeError):
            pass
    return op


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
    A = device_operator(A)
    if tuple(x.shape) != (A.n,):
        raise ValueError(f"dimension mismatch: matrix {A.n}, vector {tuple(x.shape)}")
    return _back(x, A.matvec(A.field(x)))


def weighted_jacobi_sweep(A: DeviceOperator, x, b, omega: float):
    """x + omega * D^{-1} (b - A x) (reference sparse.py:84-93)."""
    A = device_operator(A)
    _check_len(A, x, b, what="weighted_jacobi_sweep")
    out = A.sweep(A.field(x), A.field(b), omega)
    return _back(x, out.interior)


def residual_l2(A: DeviceOperator, x, b) -> float:
    A = device_operator(A)
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


__all__ = ["SparseMatrix", "device_operator", "matvec", "weighted_jacobi_sweep", "residual_l2",
           "relative_residual_l2", "diff_inf", "Field"]
