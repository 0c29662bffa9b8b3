"""Problem instances for the device solve path.

`ProblemInstance` mirrors the reference container (reference problems.py:26-47):
operator, right-hand side, initial guess, the stopping norm the experiment
uses and optional CJM bounds.  The operator is a device `StencilOperator`;
b and x0 may be numpy arrays (copied to HBM by `solve`) or CUDA tensors.

Generators:
  poisson_1d(N)              reference problems.py:50-69 (b = 1, x0 = 0, absolute L2)
  poisson_3d(n)              reference problems.py:148-177 (b = 1, x0 = 0, relative L2)
  poisson_2d(n)              2D Dirichlet 5-point analogue (no reference generator,
                             SPEC.md:372; diag 4*dx2, off -dx2 as SURVEY §8d)
  diffusion_2d_varcoef(n, seed)  BASELINE config 4 (definition in DESIGN.md §2)
  baseline_config(name, ...) the BASELINE.json configs with f ~ U[-1, 1) from SplitMix64
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .operators import StencilOperator
from .rng import derive_seed, uniform_rhs, uniforms_counter

ABSOLUTE_L2 = "absolute_l2"
RELATIVE_L2 = "relative_l2"
SOLUTION_DIFF_INF = "solution_diff_inf"


@dataclass
class ProblemInstance:
    A: StencilOperator
    b: object
    x0: object
    stopping_norm: str
    cjm_bounds: tuple[float, float] | None = None
    label: str = ""

    def __post_init__(self):
        n = self.A.n
        if _length(self.b) != n or _length(self.x0) != n:
            raise ValueError("vector length does not match matrix dimension")
        if self.cjm_bounds is not None:
            lo, hi = self.cjm_bounds
            if not (-1.0 <= lo < hi < 1.0):
                raise ValueError("cjm_bounds must lie inside [-1, 1)")

    @property
    def n(self) -> int:
        return self.A.n


def _length(v) -> int:
    shape = tuple(v.shape)
    if len(shape) != 1:
        return -1
    return int(shape[0])


def poisson_1d(N: int, device=None) -> ProblemInstance:
    if N < 1:
        raise ValueError("N must be positive")
    A = StencilOperator("1d3", (N,), dx2=(N + 1.0) ** 2, device=device)
    mu = float(np.cos(np.pi / (N + 1)))
    return ProblemInstance(A=A, b=np.ones(N), x0=np.zeros(N), stopping_norm=ABSOLUTE_L2,
                           cjm_bounds=(-mu, mu), label=f"poisson1d:{N}")


def poisson_2d(n: int, device=None) -> ProblemInstance:
    if n < 2:
        raise ValueError("n must be at least 2")
    A = StencilOperator("2d5", (n, n), dx2=(n + 1.0) ** 2, device=device)
    mu = float(np.cos(np.pi / (n + 1)))
    return ProblemInstance(A=A, b=np.ones(n * n), x0=np.zeros(n * n), stopping_norm=RELATIVE_L2,
                           cjm_bounds=(-mu, mu), label=f"poisson2d:{n}")


def poisson_3d(n: int, device=None) -> ProblemInstance:
    if n < 2:
        raise ValueError("n must be at least 2")
    A = StencilOperator("3d7", (n, n, n), dx2=(n + 1.0) ** 2, device=device)
    mu = float(np.cos(np.pi / (n + 1)))
    N = n ** 3
    return ProblemInstance(A=A, b=np.ones(N), x0=np.zeros(N), stopping_norm=RELATIVE_L2,
                           cjm_bounds=(-mu, mu), label=f"poisson3d:{n}")


# ---------------------------------------------------------------------------
# General-CSR problems: device SparseMatrix operators
# ---------------------------------------------------------------------------

def random_tridiagonal(N: int, seed: int, device=None) -> ProblemInstance:
    """Random symmetric weakly diagonally dominant tridiagonal system
    (reference problems.py:72-98): off-diagonals then diagonals drawn from one
    SplitMix64 stream, non-dominant diagonals raised to the neighbour sum, the
    end diagonals set to twice their single neighbour."""
    from .sparse import SparseMatrix
    if N < 2:
        raise ValueError("N must be at least 2")
    u = uniforms_counter(seed, 2 * N - 1)
    off, diag = u[:N - 1], u[N - 1:]
    nsum = np.zeros(N)
    nsum[:-1] += off
    nsum[1:] += off
    diag = np.where(diag >= nsum, diag, nsum)
    diag[0] = 2.0 * off[0]
    diag[-1] = 2.0 * off[-1]
    i = np.arange(N)
    rows = np.concatenate([i, i[:-1], i[1:]])
    cols = np.concatenate([i, i[1:], i[:-1]])
    A = SparseMatrix.from_coo(N, rows, cols, np.concatenate([diag, off, off]), device=device)
    return ProblemInstance(A=A, b=np.ones(N), x0=np.zeros(N), stopping_norm=ABSOLUTE_L2,
                           cjm_bounds=None, label=f"tridiag:{N}:seed{seed}")


def laplace_2d_neumann(n: int, seed: int, device=None) -> ProblemInstance:
    """2D Laplace with homogeneous Neumann faces, A x = 0 (reference
    problems.py:101-145): ghost nodes reflect onto the inward neighbour and
    boundary rows are scaled by 1/2 per boundary direction (symmetric, same
    Jacobi iteration); x0 uniform in [0, 1) from SplitMix64(seed); judged on
    the solution-difference infinity norm."""
    from .sparse import SparseMatrix
    if n < 2:
        raise ValueError("n must be at least 2")
    dx = 1.0 / (n + 1)
    dx2 = 1.0 / dx ** 2
    jj, ii = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    ii, jj = ii.ravel(), jj.ravel()
    wt = np.where((ii == 0) | (ii == n - 1), 0.5, 1.0) * np.where((jj == 0) | (jj == n - 1),
                                                                  0.5, 1.0)
    k = ii + n * jj
    rows, cols, vals = [k], [k], [4.0 * wt * dx2]
    for di, dj in ((1, 0), (-1, 0), (0, 1), (0, -1)):
        ni, nj = ii + di, jj + dj
        inside = (ni >= 0) & (ni < n) & (nj >= 0) & (nj < n)
        ci = np.where(inside, ni, ii - di)   # ghost reflects to the inward neighbour
        cj = np.where(inside, nj, jj - dj)
        rows.append(k)
        cols.append(ci + n * cj)
        vals.append(-wt * dx2)
    A = SparseMatrix.from_coo(n * n, np.concatenate(rows), np.concatenate(cols),
                              np.concatenate(vals), device=device)
    mu = (np.cos(np.pi * dx) + 1.0) / 2.0
    return ProblemInstance(A=A, b=np.zeros(n * n), x0=uniforms_counter(seed, n * n),
                           stopping_norm=SOLUTION_DIFF_INF, cjm_bounds=(-mu, mu),
                           label=f"laplace2d:{n}:seed{seed}")


# ---------------------------------------------------------------------------
# Config 4: variable-coefficient diffusion -div(k grad u) = f on n x n
# ---------------------------------------------------------------------------

BOX = 9          # box filter width
PAD = BOX // 2   # extra ring of xi so the filter never needs boundary handling
FIELD_WORD = 0x6B  # derive_seed word for the Gaussian field stream


def gaussian_field(n: int, seed: int) -> np.ndarray:
    """g on the (n+2)^2 node grid (interior plus Dirichlet boundary nodes).

    xi: i.i.d. N(0,1) on an (n+2+2*PAD)^2 grid (x fastest) by Box-Muller from
    SplitMix64(derive_seed(seed, FIELD_WORD)) uniforms taken in pairs
    (u1, u2) -> sqrt(-2 ln(1-u1)) * (cos 2 pi u2, sin 2 pi u2).
    g = (9x9 box sum of xi) / 9, summed x-direction first, left to right, then
    y-direction bottom to top; the 1/9 restores unit variance (sigma = 1).
    """
    m = n + 2 + 2 * PAD
    cnt = m * m
    u = uniforms_counter(derive_seed(seed, FIELD_WORD), 2 * ((cnt + 1) // 2))
    u1, u2 = u[0::2], u[1::2]
    rad = np.sqrt(-2.0 * np.log1p(-u1))
    ang = 2.0 * np.pi * u2
    xi = np.empty(2 * u1.size)
    xi[0::2] = rad * np.cos(ang)
    xi[1::2] = rad * np.sin(ang)
    xi = xi[:cnt].reshape(m, m)
    sx = xi[:, 0:m - 2 * PAD].copy()
    for d in range(1, BOX):
        sx = sx + xi[:, d:d + m - 2 * PAD]
    s = sx[0:m - 2 * PAD, :].copy()
    for d in range(1, BOX):
        s = s + sx[d:d + m - 2 * PAD, :]
    return s / 9.0


def _normals(seed: int, cnt: int) -> np.ndarray:
    """cnt i.i.d. N(0,1) by Box-Muller from SplitMix64(derive_seed(seed,
    FIELD_WORD)) uniforms taken in pairs (as gaussian_field)."""
    u = uniforms_counter(derive_seed(seed, FIELD_WORD), 2 * ((cnt + 1) // 2))
    u1, u2 = u[0::2], u[1::2]
    rad = np.sqrt(-2.0 * np.log1p(-u1))
    ang = 2.0 * np.pi * u2
    xi = np.empty(2 * u1.size)
    xi[0::2] = rad * np.cos(ang)
    xi[1::2] = rad * np.sin(ang)
    return xi[:cnt]


BOX3 = 5          # 3D box filter width (5 x 5 x 5)
PAD3 = BOX3 // 2


def gaussian_field_3d(n: int, seed: int) -> np.ndarray:
    """g on the (n+2)^3 node grid (z slowest, x fastest) for the 3D
    variable-coefficient problem: xi i.i.d. N(0,1) (`_normals`, x fastest) on
    an (n+2+2*PAD3)^3 grid, g = (5x5x5 box sum of xi) / sqrt(125), summed
    along x first, then y, then z, each left to right (unit variance)."""
    m = n + 2 + 2 * PAD3
    o = m - 2 * PAD3
    xi = _normals(seed, m * m * m).reshape(m, m, m)
    sx = xi[:, :, 0:o].copy()
    for d in range(1, BOX3):
        sx += xi[:, :, d:d + o]
    del xi
    sy = sx[:, 0:o, :].copy()
    for d in range(1, BOX3):
        sy += sx[:, d:d + o, :]
    del sx
    s = sy[0:o].copy()
    for d in range(1, BOX3):
        s += sy[d:d + o]
    del sy
    s /= np.sqrt(125.0)
    return s


def gaussian_field_1d(n: int, seed: int) -> np.ndarray:
    """g on the n+2 nodes of the 1D variable-coefficient problem: xi
    (`_normals`) on n+2+2*PAD nodes, g = (9-point box sum, left to right) / 3."""
    m = n + 2 + 2 * PAD
    xi = _normals(seed, m)
    s = xi[0:m - 2 * PAD].copy()
    for d in range(1, BOX):
        s = s + xi[d:d + m - 2 * PAD]
    return s / 3.0


def _hm(a, b, dx2):
    return (2.0 * a * b) / (a + b) * dx2


def harmonic_faces_3d(k: np.ndarray, dx2: float):
    """dx2-scaled harmonic-mean faces from the (n+2)^3 node coefficients
    (index [z, y, x], boundary nodes included): face_x[z, j, i] couples x-nodes
    i-1 and i of interior row (j, z) (i = 0 and i = nx are boundary faces);
    face_y[z, j, i] couples rows j-1 and j; face_z[z, j, i] planes z-1 and z."""
    c = k[1:-1, 1:-1, :]
    face_x = _hm(c[:, :, :-1], c[:, :, 1:], dx2)
    c = k[1:-1, :, 1:-1]
    face_y = _hm(c[:, :-1, :], c[:, 1:, :], dx2)
    c = k[:, 1:-1, 1:-1]
    face_z = _hm(c[:-1], c[1:], dx2)
    return (np.ascontiguousarray(face_x), np.ascontiguousarray(face_y),
            np.ascontiguousarray(face_z))


def harmonic_faces_1d(k: np.ndarray, dx2: float) -> np.ndarray:
    """face_x[i] couples nodes i-1 and i of the n+2 node coefficients."""
    return np.ascontiguousarray(_hm(k[:-1], k[1:], dx2))


def harmonic_faces(k: np.ndarray, dx2: float) -> tuple[np.ndarray, np.ndarray]:
    """dx2-scaled harmonic-mean faces from the (n+2)^2 node coefficients.

    face_x[j, i] couples nodes (i-1, j) and (i, j) of the interior numbering
    (i = 0 and i = n are the boundary faces); face_y[j, i] couples rows j-1, j.
    """
    def hm(a, b):
        return (2.0 * a * b) / (a + b) * dx2
    inner = k[1:-1, :]                 # interior rows, all columns
    face_x = hm(inner[:, :-1], inner[:, 1:])
    cols = k[:, 1:-1]                  # interior columns, all rows
    face_y = hm(cols[:-1, :], cols[1:, :])
    return np.ascontiguousarray(face_x), np.ascontiguousarray(face_y)


def diffusion_2d_varcoef(n: int, seed: int = 0, device=None) -> ProblemInstance:
    if n < 2:
        raise ValueError("n must be at least 2")
    dx2 = (n + 1.0) ** 2
    k = np.exp(gaussian_field(n, seed))
    fx, fy = harmonic_faces(k, dx2)
    A = StencilOperator("2d5var", (n, n), face_x=fx, face_y=fy, device=device)
    N = n * n
    return ProblemInstance(A=A, b=uniform_rhs(seed, N), x0=np.zeros(N),
                           stopping_norm=RELATIVE_L2, label=f"varcoef2d:{n}:seed{seed}")


def diffusion_3d_varcoef(n: int, seed: int = 0, device=None) -> ProblemInstance:
    """-div(k grad u) = f on n^3 interior points, 7-point stencil with
    harmonic-mean faces, k = exp(g) (`gaussian_field_3d`), Dirichlet, f and
    x0 as the BASELINE recipe (north_star: 3D variable-coefficient stencil)."""
    if n < 2:
        raise ValueError("n must be at least 2")
    dx2 = (n + 1.0) ** 2
    fx, fy, fz = harmonic_faces_3d(np.exp(gaussian_field_3d(n, seed)), dx2)
    A = StencilOperator("3d7var", (n, n, n), face_x=fx, face_y=fy, face_z=fz, device=device)
    N = n ** 3
    return ProblemInstance(A=A, b=uniform_rhs(seed, N), x0=np.zeros(N),
                           stopping_norm=RELATIVE_L2, label=f"varcoef3d:{n}:seed{seed}")


def diffusion_1d_varcoef(n: int, seed: int = 0, device=None) -> ProblemInstance:
    """-(k u')' = f on n interior points, 3-point stencil with harmonic-mean
    faces, k = exp(g) (`gaussian_field_1d`), Dirichlet (north_star: 1D
    variable-coefficient stencil)."""
    if n < 2:
        raise ValueError("n must be at least 2")
    dx2 = (n + 1.0) ** 2
    fx = harmonic_faces_1d(np.exp(gaussian_field_1d(n, seed)), dx2)
    A = StencilOperator("1d3var", (n,), face_x=fx, device=device)
    return ProblemInstance(A=A, b=uniform_rhs(seed, n), x0=np.zeros(n),
                           stopping_norm=RELATIVE_L2, label=f"varcoef1d:{n}:seed{seed}")


# ---------------------------------------------------------------------------
# BASELINE.json configs
# ---------------------------------------------------------------------------

CONFIGS = {
    # name: (family, extent, description)
    "c1": ("1d3", 1024, "1D Poisson N=1024"),
    "c2": ("2d5", 2048, "2D Poisson 2048^2"),
    "c3": ("3d7", 512, "3D Poisson 512^3"),
    "c4": ("2d5var", 4096, "2D variable-coefficient diffusion 4096^2"),
    "c5": ("3d7", 1024, "3D Poisson 1024^3"),
    # north_star's variable-coefficient stencils in 3D and 1D (not BASELINE
    # configs: same recipe as C3 / C1 with k = exp(g) faces)
    "c3v": ("3d7var", 512, "3D variable-coefficient diffusion 512^3"),
    "c1v": ("1d3var", 1024, "1D variable-coefficient diffusion N=1024"),
}


def baseline_problem(family: str, n: int, seed: int = 0, device=None,
                     rhs_on_device: bool = False) -> ProblemInstance:
    """A BASELINE recipe: f_i = 2 u_i - 1 (SplitMix64(seed), x fastest), x0 = 0,
    relative L2 stopping norm."""
    if family == "2d5var":
        return diffusion_2d_varcoef(n, seed, device=device)
    if family == "3d7var":
        return diffusion_3d_varcoef(n, seed, device=device)
    if family == "1d3var":
        return diffusion_1d_varcoef(n, seed, device=device)
    dims = {"1d3": (n,), "2d5": (n, n), "3d7": (n, n, n)}[family]
    A = StencilOperator(family, dims, dx2=(n + 1.0) ** 2, device=device)
    N = A.n
    if rhs_on_device:
        import torch

        from .operators import fill_uniform_rhs
        b = torch.empty(N, dtype=torch.float64, device=A.device)
        fill_uniform_rhs(b, seed)
        x0 = torch.zeros(N, dtype=torch.float64, device=A.device)
    else:
        b = uniform_rhs(seed, N)
        x0 = np.zeros(N)
    return ProblemInstance(A=A, b=b, x0=x0, stopping_norm=RELATIVE_L2,
                           label=f"{family}:{n}:seed{seed}")


def config_problem(name: str, seed: int = 0, device=None, size: int | None = None,
                   rhs_on_device: bool = False) -> ProblemInstance:
    family, extent, _ = CONFIGS[name]
    return baseline_problem(family, size or extent, seed, device=device,
                            rhs_on_device=rhs_on_device)
