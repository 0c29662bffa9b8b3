"""Slab-decomposed SRJ solve: one z-slab (3D) or row-slab (2D) per GPU.

The reference has no parallelism beyond a process pool of independent runs
(reference cli.py:196-198); this module is the multi-GPU form of the same
solve.  Each rank owns `count` consecutive planes of the global
grid in a Field whose ghost planes hold the neighbours' boundary planes (zero
on a Dirichlet face), so every per-point computation -- and therefore every
iterate -- is bit-identical to the single-GPU solve.

Protocol per cycle (M sweeps, identical on every rank):
  0. snapshot x_0 (device copy, 16 B/point once per cycle);
  1. for each sweep k: exchange ghost planes of x_k with the z-/y-neighbours
     (overlapped with the interior planes' sweep), sweep the boundary planes,
     record the slab's sum of (b - A x_k)^2 -- three deterministic device
     partials (interior, low face, high face);
  2. residual of x_M (same exchange);
  3. ONE all-gather of the (M+1) x 3 partials; every rank sums them in rank
     order -- bit-identical global norms everywhere -- and applies the
     reference's per-sweep stopping rule (solver.py:216-222,235-239) to
     res_1 .. res_M;
  4. a stop at sweep k < M restores the snapshot and re-runs k sweeps.
So the data path has one ghost-plane exchange per sweep and one small
collective per cycle; the host reads one gathered vector per cycle.

Exchangers: `TorchExchanger` (one slab per process; torch.distributed P2P --
NCCL over NVLink between GPUs, gloo on CPU for the tests) and
`LocalExchanger` (several slabs in one process, e.g. virtual ranks on one GPU,
exchanging by device copies).  Engines: `DeviceEngine` (libsrj's
srj_sweep_planes) or any object with the same `apply` method (the CPU tests
plug in a numpy engine).
"""

from __future__ import annotations

import ctypes
import math
import time
from dataclasses import dataclass

import numpy as np

from . import _lib
from .operators import Field, StencilOperator, fill_uniform_rhs
from .problems import ABSOLUTE_L2, RELATIVE_L2
from .schemes import MAX_LEVEL, ORDER_GRID_SIZE
from .solver import (CycleStats, Heuristic, Increasing, SolveDivergedError, SolveReport,
                     SolverState, StoppingRule, _l2_norm_parts, _next_scheme,
                     average_convergence_rate, heuristic_next_level)

PARTS = 3  # interior planes, low face, high face


def _torch():
    import torch
    return torch


# ---------------------------------------------------------------------------
# Layout
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class SlabLayout:
    """Global grid split into `world` slabs of whole planes along the slowest
    axis (z in 3D, y in 2D); slab sizes differ by at most one plane."""

    family: str
    shape: tuple
    world: int

    def __post_init__(self):
        if self.family in ("1d3", "1d3var") and self.world != 1:
            raise ValueError("a 1D grid is not sharded (replicas only)")
        if self.world < 1 or self.world > self.planes:
            raise ValueError(f"{self.world} slabs for {self.planes} planes")

    @property
    def planes(self) -> int:
        return 1 if self.family in ("1d3", "1d3var") else int(self.shape[-1])

    @property
    def plane_points(self) -> int:
        return (int(np.prod(self.shape[:-1])) if self.family not in ("1d3", "1d3var")
                else int(self.shape[0]))

    @property
    def n(self) -> int:
        return int(np.prod(self.shape))

    def span(self, rank: int) -> tuple[int, int]:
        base, extra = divmod(self.planes, self.world)
        count = base + (1 if rank < extra else 0)
        start = rank * base + min(rank, extra)
        return start, count

    def local_shape(self, rank: int) -> tuple:
        if self.family in ("1d3", "1d3var"):
            return tuple(self.shape)
        return tuple(self.shape[:-1]) + (self.span(rank)[1],)


class Slab:
    """One rank's planes: operator, right-hand side, iterate, ping-pong partner
    and the cycle-start snapshot (all Fields with ghost planes)."""

    def __init__(self, layout: SlabLayout, rank: int, device, dx2: float | None = None,
                 face_x=None, face_y=None, face_z=None):
        self.layout = layout
        self.rank = rank
        self.start, self.count = layout.span(rank)
        nx = layout.shape[0]
        lo, hi = self.start, self.start + self.count
        if dx2 is None and layout.family not in ("2d5var", "3d7var", "1d3var"):
            dx2 = (nx + 1.0) ** 2
        if layout.family == "2d5var":
            fx = face_x[lo:hi, :]
            fy = face_y[lo:hi + 1, :]
            self.A = StencilOperator("2d5var", layout.local_shape(rank), face_x=fx, face_y=fy,
                                     device=device)
        elif layout.family == "3d7var":
            # z-slab: its planes' x/y faces and the nz+1 z-faces bounding them
            self.A = StencilOperator("3d7var", layout.local_shape(rank), face_x=face_x[lo:hi],
                                     face_y=face_y[lo:hi], face_z=face_z[lo:hi + 1],
                                     device=device)
        elif layout.family == "1d3var":
            self.A = StencilOperator("1d3var", layout.local_shape(rank), face_x=face_x,
                                     device=device)
        else:
            self.A = StencilOperator(layout.family, layout.local_shape(rank), dx2=dx2,
                                     device=device)
        self.device = device
        self.x = self.A.new_field()
        self.x_alt = self.A.new_field()
        self.snap = self.A.new_field()
        self.b = self.A.new_field()

    @property
    def offset(self) -> int:
        """Global flat index of the slab's first interior point."""
        return self.start * self.layout.plane_points

    @property
    def planes(self) -> int:
        return self.count if self.layout.family not in ("1d3", "1d3var") else 1

    def swap(self) -> None:
        self.x, self.x_alt = self.x_alt, self.x


def _plane(field: Field, which: str):
    """Views of a Field: 'lo_ghost', 'first', 'last', 'hi_ghost'."""
    h, n = field.halo, field.n
    buf = field.buf
    return {"lo_ghost": buf[0:h], "first": buf[h:2 * h], "last": buf[n:n + h],
            "hi_ghost": buf[n + h:n + 2 * h]}[which]


# ---------------------------------------------------------------------------
# Exchangers
# ---------------------------------------------------------------------------

class LocalExchanger:
    """All slabs live in this process (virtual ranks): ghost planes are filled
    by device copies; the gather is a stack."""

    def __init__(self, world: int):
        self.world = world

    def start(self, fields):
        for lo, hi in zip(fields[:-1], fields[1:]):
            _plane(hi, "lo_ghost").copy_(_plane(lo, "last"))
            _plane(lo, "hi_ghost").copy_(_plane(hi, "first"))
        return None

    def finish(self, handle) -> None:
        return None

    def exchange(self, fields) -> None:
        self.finish(self.start(fields))

    def allgather(self, tensors):
        torch = _torch()
        dev = tensors[0].device
        return torch.stack([t.to(dev) for t in tensors])


class TorchExchanger:
    """One slab per process; torch.distributed point-to-point for the ghost
    planes (NCCL over NVLink/NVSwitch on GPUs, gloo on CPU) and all_gather for
    the per-cycle partials."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)

    def start(self, fields):
        (f,) = fields
        dist = self.dist
        ops = []
        if self.rank > 0:
            ops.append(dist.P2POp(dist.isend, _plane(f, "first"), self.rank - 1, self.group))
            ops.append(dist.P2POp(dist.irecv, _plane(f, "lo_ghost"), self.rank - 1, self.group))
        if self.rank < self.world - 1:
            ops.append(dist.P2POp(dist.isend, _plane(f, "last"), self.rank + 1, self.group))
            ops.append(dist.P2POp(dist.irecv, _plane(f, "hi_ghost"), self.rank + 1, self.group))
        return dist.batch_isend_irecv(ops) if ops else []

    def finish(self, reqs) -> None:
        for r in reqs:
            r.wait()

    def exchange(self, fields) -> None:
        self.finish(self.start(fields))

    def allgather(self, tensors):
        torch = _torch()
        (t,) = tensors
        out = [torch.empty_like(t) for _ in range(self.world)]
        self.dist.all_gather(out, t, group=self.group)
        return torch.stack(out)


# ---------------------------------------------------------------------------
# Engines
# ---------------------------------------------------------------------------

class DeviceEngine:
    """libsrj slab kernels: srj_sweep_planes (sum of r^2 written on device)."""

    overlap = True

    def apply(self, slab: Slab, xin: Field, xout: Field | None, w: float, z0: int, z1: int,
              out, slot: int) -> None:
        slab.A.sweep_planes(xin, xout, slab.b, w, z0, z1, out.data_ptr(), slot)


# ---------------------------------------------------------------------------
# Solver
# ---------------------------------------------------------------------------

class SlabSolver:
    """`solve` over slabs (drop-in semantics of reference solver.py:289-331)."""

    def __init__(self, slabs: list[Slab], exchanger, engine=None):
        if not slabs:
            raise ValueError("no slabs")
        self.slabs = slabs
        self.ex = exchanger
        self.engine = engine if engine is not None else DeviceEngine()
        self.layout = slabs[0].layout
        self._parts = None
        self.launches = 0  # kernel launches issued by this solver (bench evidence)

    # -- data ---------------------------------------------------------------
    def load(self, b=None, x0=None, seed: int | None = None) -> None:
        """b: global numpy vector (sliced per slab) or None with `seed` for the
        SplitMix64 right-hand side generated in place on each slab's device;
        x0: global numpy vector or None (zero)."""
        for s in self.slabs:
            lo, hi = s.offset, s.offset + s.A.n
            if b is not None:
                s.b.copy_(np.asarray(b)[lo:hi])
            elif seed is not None and s.b.device.type == "cuda":
                fill_uniform_rhs(s.b, seed, start=lo)
            elif seed is not None:
                from .rng import uniforms_counter
                s.b.copy_(2.0 * uniforms_counter(seed, hi - lo, start=lo) - 1.0)
            else:
                raise ValueError("need b or seed")
            s.x.buf.zero_()
            s.x_alt.buf.zero_()
            if x0 is not None:
                s.x.copy_(np.asarray(x0)[lo:hi])

    def gather(self) -> np.ndarray:
        """The global iterate on the host (tests and small problems)."""
        torch = _torch()
        parts = self.ex.allgather([self._padded_interior(s) for s in self.slabs])
        total = []
        for r in range(self.layout.world):
            start, count = self.layout.span(r)
            total.append(parts[r][:count * self.layout.plane_points].cpu().numpy())
        del torch
        return np.concatenate(total)

    def _padded_interior(self, s: Slab):
        torch = _torch()
        base, extra = divmod(self.layout.planes, self.layout.world)
        size = (base + (1 if extra else 0)) * self.layout.plane_points
        out = torch.zeros(size, dtype=torch.float64, device=s.x.buf.device)
        out[:s.A.n].copy_(s.x.interior)
        return out

    # -- kernels over all local slabs ----------------------------------------
    def _parts_buffer(self, K: int):
        torch = _torch()
        return [torch.zeros((K, PARTS), dtype=torch.float64, device=s.x.buf.device)
                for s in self.slabs]

    def _sweep(self, w: float, parts, k: int) -> None:
        eng = self.engine
        P = [s.planes for s in self.slabs]
        # the interior/boundary split only pays when a halo exchange can overlap
        if getattr(eng, "overlap", False) and min(P) >= 3 and self.layout.world > 1:
            handle = self.ex.start([s.x for s in self.slabs])
            for s, p in zip(self.slabs, parts):
                eng.apply(s, s.x, s.x_alt, w, 1, s.planes - 1, p[k, 0], 0)
            self.ex.finish(handle)
            for s, p in zip(self.slabs, parts):
                eng.apply(s, s.x, s.x_alt, w, 0, 1, p[k, 1], 1)
                eng.apply(s, s.x, s.x_alt, w, s.planes - 1, s.planes, p[k, 2], 1)
            self.launches += 3 * len(self.slabs)
        else:
            self.ex.exchange([s.x for s in self.slabs])
            for s, p in zip(self.slabs, parts):
                eng.apply(s, s.x, s.x_alt, w, 0, s.planes, p[k, 0], 0)
            self.launches += len(self.slabs)
        for s in self.slabs:
            s.swap()

    def _residual(self, parts, k: int) -> None:
        self.ex.exchange([s.x for s in self.slabs])
        for s, p in zip(self.slabs, parts):
            self.engine.apply(s, s.x, None, 0.0, 0, s.planes, p[k, 0], 0)
        self.launches += len(self.slabs)

    def _global_sums(self, parts, K: int) -> np.ndarray:
        g = self.ex.allgather(parts).cpu().numpy()  # [world, K, PARTS]
        acc = np.zeros(K)
        for r in range(g.shape[0]):  # fixed rank order: identical bits on every rank
            acc = acc + ((g[r, :K, 0] + g[r, :K, 1]) + g[r, :K, 2])
        return acc

    def residual_norm(self) -> float:
        parts = self._parts_buffer(1)
        self._residual(parts, 0)
        return math.sqrt(self._global_sums(parts, 1)[0])

    # -- cycle / solve ----------------------------------------------------------
    def cycle(self, ordered_omegas, res_before: float, tol: float, baseline: float,
              budget: int):
        """Returns (executed, status, res_after, history[1..executed])."""
        M = len(ordered_omegas)
        if res_before <= tol:
            return 0, "converged", res_before, []
        Meff = min(M, max(budget, 0))
        if Meff == 0:
            return 0, "ran", res_before, []
        for s in self.slabs:
            s.snap.buf.copy_(s.x.buf)
        parts = self._parts_buffer(Meff + 1)
        for k in range(Meff):
            self._sweep(ordered_omegas[k], parts, k)
        self._residual(parts, Meff)
        sums = self._global_sums(parts, Meff + 1)
        res = np.sqrt(sums) / baseline
        stop, status = None, "ran"
        for k in range(1, Meff + 1):
            if not math.isfinite(res[k]):
                stop, status = k, "diverged"
                break
            if res[k] <= tol:
                stop, status = k, "converged"
                break
        executed = Meff if stop is None else stop
        if executed < Meff:
            # roll back: x_executed from the cycle-start snapshot
            for s in self.slabs:
                s.x.buf.copy_(s.snap.buf)
            scratch = self._parts_buffer(max(executed, 1))
            for k in range(executed):
                self._sweep(ordered_omegas[k], scratch, k)
        return executed, status, float(res[executed]), [float(v) for v in res[1:executed + 1]]

    def solve(self, controller, stopping: StoppingRule, order_grid: int = ORDER_GRID_SIZE,
              record_history: bool = True, max_cycles: int | None = None) -> SolveReport:
        """`max_cycles` caps the number of cycles (throughput mode, BASELINE
        config 5: a fixed count of heuristic-selected cycles)."""
        t0 = time.perf_counter()
        _l2_norm_parts(stopping.norm)
        r0 = self.residual_norm()
        baseline = 1.0
        if stopping.norm == RELATIVE_L2:
            baseline = r0
            if baseline == 0.0:
                raise ValueError("initial residual is zero; relative norm undefined")
        res_now = r0 / baseline
        state = SolverState(x=None, level=0)
        history = [(0, res_now)] if record_history else []
        cycles: list[CycleStats] = []
        converged = False
        while True:
            scheme = _next_scheme(controller, state, order_grid)
            ordered = scheme.ordered_omegas()
            budget = stopping.max_iterations - state.total_iterations
            res_before = res_now
            executed, status, res_after, hist = self.cycle(
                ordered, res_before, stopping.tolerance, baseline, budget)
            if status == "diverged":
                raise SolveDivergedError({
                    "cycle": state.cycle_index, "sweep": executed,
                    "omega": ordered[executed - 1], "level": scheme.level, "M": scheme.M})
            if record_history:
                history.extend((state.total_iterations + i + 1, r) for i, r in enumerate(hist))
            res_now = res_after
            if executed > 0 and res_before > 0.0 and res_after > 0.0:
                rate = average_convergence_rate(res_before, res_after, executed)
                ratio = res_after / res_before
            else:
                rate = math.inf if executed > 0 else 0.0
                ratio = state.prev_residual_ratio
            if executed > 0:
                cycles.append(CycleStats(
                    cycle=state.cycle_index,
                    level=scheme.level if scheme.level is not None else -1, M=scheme.M,
                    executed=executed, residual_before=res_before, residual_after=res_after,
                    average_rate=rate))
                state.prev_residual_ratio = ratio
            state.level = scheme.level if scheme.level is not None else state.level
            state.cycle_index += 1
            state.total_iterations += executed
            if res_now <= stopping.tolerance:
                converged = True
                break
            if state.total_iterations >= stopping.max_iterations:
                break
            if max_cycles is not None and state.cycle_index >= max_cycles:
                break
            if isinstance(controller, Heuristic):
                r = state.prev_residual_ratio
                if r is not None and math.isfinite(r):
                    state.level = heuristic_next_level(r, state.level, controller.t_hi,
                                                       controller.t_lo)
            elif isinstance(controller, Increasing):
                state.level = min(state.level + 1, MAX_LEVEL)
        return SolveReport(converged=converged, total_iterations=state.total_iterations,
                           cycles=cycles, wall_time=time.perf_counter() - t0,
                           x=[s.x.interior for s in self.slabs], residual_history=history)


def local_slabs(family: str, shape, world: int, ranks, device, face_x=None, face_y=None,
                dx2: float | None = None, face_z=None) -> list[Slab]:
    layout = SlabLayout(family, tuple(shape), world)
    return [Slab(layout, r, device, dx2=dx2, face_x=face_x, face_y=face_y, face_z=face_z)
            for r in ranks]


# ---------------------------------------------------------------------------
# Temporally blocked row slabs (2D): deep ghost rows, one exchange per pass
# ---------------------------------------------------------------------------

TB_GHOST = 6   # 2D: ghost rows per interior side = sweeps per pass (srj_tb_pass)
TB3_GHOST = 2  # 3D: ghost planes per interior side = sweeps per pass


def tb_ghost(family: str) -> int:
    """Deep-halo width (= most sweeps one srj_tb_pass fuses) of a family."""
    return TB3_GHOST if family == "3d7" else TB_GHOST


class TbSlab:
    """A 2D row slab (3D z slab) extended by `ghost` ghost rows (planes) toward
    each neighbour (none on a Dirichlet face): TB_GHOST = 6 rows in 2D,
    TB3_GHOST = 2 planes in 3D.  Its operator covers the extended rows -- faces,
    b and the iterate of the ghost rows included -- so one srj_tb_pass of up to
    `ghost` sweeps updates the ghost rows as ring points and stores the owned
    rows exactly as the single-GPU solve would.  A "row" is one x-row in 2D and
    one xy plane in 3D (`unit` points)."""

    def __init__(self, layout: SlabLayout, rank: int, device, dx2: float | None = None,
                 face_x=None, face_y=None):
        if layout.family not in ("2d5", "2d5var", "3d7"):
            raise ValueError("temporally blocked slabs are 2D row slabs or 3D z slabs")
        self.layout = layout
        self.rank = rank
        self.start, self.count = layout.span(rank)
        nx = layout.shape[0]
        g = self.ghost = tb_ghost(layout.family)
        self.g_lo = g if rank > 0 else 0
        self.g_hi = g if rank < layout.world - 1 else 0
        rows = self.count + self.g_lo + self.g_hi
        r0 = self.start - self.g_lo  # global row of extended row 0
        if layout.family == "2d5var":
            fx = np.ascontiguousarray(face_x[r0:r0 + rows, :])
            fy = np.ascontiguousarray(face_y[r0:r0 + rows + 1, :])
            self.A = StencilOperator("2d5var", (nx, rows), face_x=fx, face_y=fy, device=device)
        else:
            if dx2 is None:
                dx2 = (nx + 1.0) ** 2
            shape = (nx, rows) if layout.family == "2d5" else (nx, layout.shape[1], rows)
            self.A = StencilOperator(layout.family, shape, dx2=dx2, device=device)
        if not self.A.describe()["tb_supported"]:
            raise ValueError("no temporally blocked kernel for this grid (odd nx?)")
        self.device = device
        self.unit = layout.plane_points  # points per row (2D) / plane (3D)
        self.nx = self.unit
        self.row0 = r0
        self.x = self.A.new_field()
        self.x_alt = self.A.new_field()
        self.pair = (self.x, self.x_alt)  # fixed identities (CUDA-graph keys)
        self.snap = self.A.new_field()
        self.b = self.A.new_field()

    @property
    def offset(self) -> int:
        """Global flat index of the slab's first OWNED point."""
        return self.start * self.unit

    @property
    def owned(self) -> tuple[int, int]:
        return self.g_lo, self.g_lo + self.count

    def rows(self, field: Field, r0: int, r1: int):
        """View of extended rows (planes) [r0, r1) of a Field."""
        h = field.halo
        return field.buf[h + r0 * self.unit:h + r1 * self.unit]

    def interior(self, field: Field):
        lo, hi = self.owned
        return self.rows(field, lo, hi)

    def swap(self) -> None:
        self.x, self.x_alt = self.x_alt, self.x


def exchange_plan(s, rank: int, world: int) -> tuple:
    """srj_slab_exchange_plan of a slab: element offsets (from the first
    interior point) of the planes sent to / received from rank-1 and rank+1 and
    the values per message -- the same plan srj_slab_exchange sends by."""
    plan = (ctypes.c_int64 * 5)()
    lo, hi = s.owned
    _lib.check_nccl(_lib.lib().srj_slab_exchange_plan(
        s.nx, rank, world, lo, hi - lo, s.g_hi, s.ghost, plan), "srj_slab_exchange_plan")
    return tuple(plan)


class LocalTbExchanger(LocalExchanger):
    """Virtual ranks in one process: deep ghost rows by device copies, at the
    offsets of the native exchange plan (srj_slab_exchange_plan)."""

    graph_capturable = True

    def start_rows(self, slabs, fields):
        world = len(slabs)
        plans = [exchange_plan(s, r, world) for r, s in enumerate(slabs)]
        for flo, fhi, plo, phi in zip(fields[:-1], fields[1:], plans[:-1], plans[1:]):
            m = plo[4]
            h = flo.halo
            xl, xh = flo.buf, fhi.buf
            xh[h + phi[1]:h + phi[1] + m].copy_(xl[h + plo[2]:h + plo[2] + m])  # lo's last owned
            xl[h + plo[3]:h + plo[3] + m].copy_(xh[h + phi[0]:h + phi[0] + m])  # hi's first owned
        return None


class NcclTbExchanger:
    """One slab per process; the deep-halo exchange and the per-cycle
    all-gather run natively through libsrj's NCCL entry points
    (srj_slab_exchange, srj_allgather_sums) on a communicator libsrj creates
    (srj_nccl_comm_init; the unique id travels over torch.distributed).  With
    it, TbSlabSolver issues each cycle's forward work as ONE C call
    (srj_slab_cycle_forward) when the exchange is not split for overlap."""

    graph_capturable = False  # NCCL inside graph capture: not exercised here

    def __init__(self, device, group=None):
        import torch
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        L = _lib.lib()
        if not L.srj_nccl_available():
            raise _lib.SrjLibraryError("libnccl.so.2 not available: "
                                       + L.srj_nccl_last_error().decode(errors="replace"))
        uid = (ctypes.c_uint8 * 128)()
        if self.rank == 0:
            _lib.check_nccl(L.srj_nccl_unique_id(uid), "srj_nccl_unique_id")
        obj = [bytes(uid)]
        dist.broadcast_object_list(obj, src=0, group=group)
        uid = (ctypes.c_uint8 * 128).from_buffer_copy(obj[0])
        self.device = torch.device(device)
        comm = ctypes.c_void_p()
        _lib.check_nccl(L.srj_nccl_comm_init(self.world, uid, self.rank, self.device.index or 0,
                                             ctypes.byref(comm)), "srj_nccl_comm_init")
        self.comm = comm

    def close(self) -> None:
        if self.comm:
            _lib.lib().srj_nccl_comm_destroy(self.comm)
            self.comm = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _stream(self):
        import torch
        return ctypes.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)

    def start_rows(self, slabs, fields):
        (s,), (f,) = slabs, fields
        lo, hi = s.owned
        _lib.check_nccl(_lib.lib().srj_slab_exchange(
            s.A.handle, self.comm, self.rank, self.world, f.ptr, lo, hi - lo, s.g_hi, s.ghost,
            self._stream()), "srj_slab_exchange")
        return None

    def finish(self, handle) -> None:
        return None

    def allgather(self, tensors):
        import torch
        (t,) = tensors
        K = t.numel()
        out = torch.empty(self.world * K, dtype=torch.float64, device=t.device)
        _lib.check_nccl(_lib.lib().srj_allgather_sums(self.comm, self.world, t.data_ptr(),
                                                      out.data_ptr(), K, self._stream()),
                        "srj_allgather_sums")
        return out.view(self.world, K)


class TorchTbExchanger(TorchExchanger):
    """One slab per process: deep ghost rows over torch.distributed P2P."""

    # NCCL P2P inside CUDA-graph capture is not exercised here (one GPU per
    # call): opt in with TbSlabSolver(graphs=True)
    graph_capturable = False

    def start_rows(self, slabs, fields):
        (s,), (f,) = slabs, fields
        dist = self.dist
        g = s.ghost
        a, b = s.owned
        ops = []
        if self.rank > 0:
            ops.append(dist.P2POp(dist.isend, s.rows(f, a, a + g), self.rank - 1, self.group))
            ops.append(dist.P2POp(dist.irecv, s.rows(f, 0, g), self.rank - 1, self.group))
        if self.rank < self.world - 1:
            ops.append(dist.P2POp(dist.isend, s.rows(f, b - g, b), self.rank + 1, self.group))
            ops.append(dist.P2POp(dist.irecv, s.rows(f, b, b + g), self.rank + 1, self.group))
        return dist.batch_isend_irecv(ops) if ops else []


class TbSlabSolver(SlabSolver):
    NCCL_SMS = 4  # SMs the pass kernels leave to NCCL when the exchange overlaps
    """`solve` over temporally blocked slabs: per cycle, passes of up to
    `ghost` sweeps, each one deep ghost-row exchange plus one srj_tb_pass;
    the residual of x_M over the owned rows; one all-gather of the per-sweep
    owned sums; the same stop / rollback protocol as SlabSolver.

    overlap (None: on for 2D, off for 3D): a pass of a slab with a neighbour is
    split into an interior launch -- the owned rows at least `ghost` rows away
    from every ghost row, which never read a ghost row -- issued while the
    exchange is in flight, then one launch per boundary band of `ghost` rows
    once it has arrived.  Iterates are identical either way; the per-sweep sums
    are added interior + lower + upper (fixed order)."""

    def __init__(self, slabs: list[TbSlab], exchanger, overlap: bool | None = None,
                 graphs: bool | None = None):
        super().__init__(slabs, exchanger, engine=None)
        # graphs (None: where the exchanger is capturable): the forward part of
        # a cycle -- snapshot, every pass with its exchange, the residual of
        # x_M -- is captured once per (sweeps, scheme, buffer parity) into a
        # CUDA graph and replayed: one graph launch per cycle instead of
        # ~M/ghost rounds of host work (tensor-map encodes, cooperative
        # launches, exchange calls)
        self.graphs = (getattr(exchanger, "graph_capturable", False) if graphs is None
                       else bool(graphs))
        self._graph_cache = {}
        self._graph_seen = set()
        g = slabs[0].ghost
        if any(s.count < g for s in slabs):
            raise ValueError(f"every slab needs at least {g} rows")
        self.ghost = g
        self._omega_cache = {}
        if overlap is None:
            overlap = slabs[0].layout.family != "3d7"
        self.overlap = overlap
        self._band_sums = None
        if overlap and isinstance(exchanger, TorchTbExchanger) and exchanger.world > 1:
            # NCCL's P2P kernels need SMs while the interior launch runs
            for s in slabs:
                s.A.set_reserved_sms(self.NCCL_SMS)

    # -- data ---------------------------------------------------------------
    def load(self, b=None, x0=None, seed: int | None = None) -> None:
        """As SlabSolver.load; b covers the extended rows (ghost rows hold the
        neighbours' b, which never changes)."""
        for s in self.slabs:
            n_ext = s.A.n
            lo = s.row0 * s.unit
            if b is not None:
                s.b.copy_(np.asarray(b)[lo:lo + n_ext])
            elif seed is not None:
                fill_uniform_rhs(s.b, seed, start=lo)
            else:
                raise ValueError("need b or seed")
            s.x.buf.zero_()
            s.x_alt.buf.zero_()
            if x0 is not None:
                s.x.copy_(np.asarray(x0)[lo:lo + n_ext])

    def _padded_interior(self, s: TbSlab):
        torch = _torch()
        base, extra = divmod(self.layout.planes, self.layout.world)
        size = (base + (1 if extra else 0)) * self.layout.plane_points
        out = torch.zeros(size, dtype=torch.float64, device=s.x.buf.device)
        out[:s.count * s.unit].copy_(s.interior(s.x))
        return out

    # -- kernels over all local slabs ----------------------------------------
    def _exchange_rows(self) -> None:
        self.ex.finish(self.ex.start_rows(self.slabs, [s.x for s in self.slabs]))

    def _omegas(self, ordered):
        torch = _torch()
        key = tuple(ordered)
        t = self._omega_cache.get(key)
        if t is None:
            t = torch.tensor(key, dtype=torch.float64, device=self.slabs[0].x.buf.device)
            self._omega_cache[key] = t
        return t

    def _bands(self, s: TbSlab):
        """(interior, [boundary bands]) owned row ranges of a split pass, or
        None when the pass is not split."""
        g = self.ghost
        lo, hi = s.owned
        a = lo + (g if s.g_lo else 0)
        b = hi - (g if s.g_hi else 0)
        if not self.overlap or (a == lo and b == hi) or b <= a:
            return None
        bands = ([(lo, a)] if a > lo else []) + ([(b, hi)] if b < hi else [])
        return (a, b), bands

    def _passes(self, om, sums, k_end: int) -> None:
        """Sweeps 0 .. k_end-1 of the cycle in passes of <= ghost."""
        torch = _torch()
        k = 0
        while k < k_end:
            h = min(self.ghost, k_end - k)
            split = [self._bands(s) for s in self.slabs]
            if not any(split):
                self._exchange_rows()
                for s, sm in zip(self.slabs, sums):
                    lo, hi = s.owned
                    s.A.tb_pass(s.x, s.x_alt, s.b, om.data_ptr() + 8 * k, h, lo, hi,
                                sm.data_ptr() + 8 * k)
                self.launches += len(self.slabs)
            else:
                if self._band_sums is None:
                    self._band_sums = [torch.zeros((3, 8), dtype=torch.float64,
                                                   device=s.x.buf.device) for s in self.slabs]
                handle = self.ex.start_rows(self.slabs, [s.x for s in self.slabs])
                # interior rows: no ghost row is read, so they run under the exchange
                for s, sm, sp, bs in zip(self.slabs, sums, split, self._band_sums):
                    lo, hi = sp[0] if sp else s.owned
                    dst = bs[0].data_ptr() if sp else sm.data_ptr() + 8 * k
                    s.A.tb_pass(s.x, s.x_alt, s.b, om.data_ptr() + 8 * k, h, lo, hi, dst)
                self.ex.finish(handle)
                for s, sm, sp, bs in zip(self.slabs, sums, split, self._band_sums):
                    if not sp:
                        continue
                    bs[1:].zero_()
                    for i, (lo, hi) in enumerate(sp[1]):
                        s.A.tb_pass(s.x, s.x_alt, s.b, om.data_ptr() + 8 * k, h, lo, hi,
                                    bs[1 + i].data_ptr())
                    sm[k:k + h] = (bs[0, :h] + bs[1, :h]) + bs[2, :h]
                self.launches += sum(1 + (len(sp[1]) if sp else 0) for sp in split)
            for s in self.slabs:
                s.swap()
            k += h

    def _residual_into(self, sums, k: int) -> None:
        self._exchange_rows()
        for s, sm in zip(self.slabs, sums):
            lo, hi = s.owned
            s.A.sweep_planes(s.x, None, s.b, 0.0, lo, hi, sm.data_ptr() + 8 * k, 0)
        self.launches += len(self.slabs)

    def _sums_buffer(self, K: int):
        torch = _torch()
        return [torch.zeros(K, dtype=torch.float64, device=s.x.buf.device) for s in self.slabs]

    def _global(self, sums, K: int) -> np.ndarray:
        if getattr(self, "_gathered", None) is not None and self._gathered.shape[1] == K \
                and isinstance(self.ex, NcclTbExchanger):
            g = self._gathered.cpu().numpy()  # gathered inside srj_slab_cycle_forward
            self._gathered = None
        else:
            g = self.ex.allgather(sums).cpu().numpy()  # [world, K]
        acc = np.zeros(K)
        for r in range(g.shape[0]):  # fixed rank order: identical bits on every rank
            acc = acc + g[r, :K]
        return acc

    def residual_norm(self) -> float:
        sums = self._sums_buffer(1)
        self._residual_into(sums, 0)
        return math.sqrt(self._global(sums, 1)[0])

    def cycle(self, ordered_omegas, res_before: float, tol: float, baseline: float,
              budget: int):
        M = len(ordered_omegas)
        if res_before <= tol:
            return 0, "converged", res_before, []
        Meff = min(M, max(budget, 0))
        if Meff == 0:
            return 0, "ran", res_before, []
        om = self._omegas(ordered_omegas)
        sums = self._forward(om, Meff)
        res = np.sqrt(self._global(sums, Meff + 1)) / baseline
        stop, status = None, "ran"
        for k in range(1, Meff + 1):
            if not math.isfinite(res[k]):
                stop, status = k, "diverged"
                break
            if res[k] <= tol:
                stop, status = k, "converged"
                break
        executed = Meff if stop is None else stop
        if executed < Meff:
            # roll back: x_executed from the cycle-start snapshot
            for s in self.slabs:
                s.x.buf.copy_(s.snap.buf)
            self._passes(om, self._sums_buffer(Meff + 1), executed)
        return executed, status, float(res[executed]), [float(v) for v in res[1:executed + 1]]

    def _forward_native(self, om, Meff: int):
        """The whole forward part of the cycle in one libsrj call
        (srj_slab_cycle_forward: snapshot, passes with NCCL deep-halo
        exchanges, residual of x_Meff, NCCL all-gather of the sums)."""
        torch = _torch()
        (s,) = self.slabs
        sums = torch.empty(Meff + 1, dtype=torch.float64, device=s.x.buf.device)
        self._gathered = torch.empty((self.ex.world, Meff + 1), dtype=torch.float64,
                                     device=s.x.buf.device)
        lo, hi = s.owned
        alt = ctypes.c_int32()
        _lib.check_nccl(_lib.lib().srj_slab_cycle_forward(
            s.A.handle, self.ex.comm, self.ex.rank, self.ex.world, s.x.ptr, s.x_alt.ptr,
            s.snap.ptr, s.b.ptr, om.data_ptr(), Meff, self.ghost, lo, hi - lo, s.g_hi,
            sums.data_ptr(), self._gathered.data_ptr(), ctypes.byref(alt),
            self.ex._stream()), "srj_slab_cycle_forward")
        if alt.value:
            s.swap()
        self.launches += -(-Meff // self.ghost) + 1
        return [sums]

    def _forward_eager(self, om, Meff: int, sums) -> None:
        for s in self.slabs:
            s.snap.buf.copy_(s.x.buf)
        for sm in sums:
            sm.zero_()
        self._passes(om, sums, Meff)
        self._residual_into(sums, Meff)

    def _forward(self, om, Meff: int):
        """Snapshot, Meff sweeps in passes, residual of x_Meff; returns the
        per-slab per-sweep sums (device).  Graph mode: the first cycle of a
        key runs eagerly (it also creates every handle and workspace), the
        second captures, later ones replay."""
        if isinstance(self.ex, NcclTbExchanger) and not self.overlap:
            return self._forward_native(om, Meff)
        if not self.graphs:
            sums = self._sums_buffer(Meff + 1)
            self._forward_eager(om, Meff, sums)
            return sums
        torch = _torch()
        parity = tuple(s.x is s.pair[0] for s in self.slabs)
        key = (Meff, om.data_ptr(), parity)
        hit = self._graph_cache.get(key)
        if hit is None and key not in self._graph_seen:
            self._graph_seen.add(key)
            sums = self._sums_buffer(Meff + 1)
            self._forward_eager(om, Meff, sums)
            return sums
        if hit is None:
            sums = self._sums_buffer(Meff + 1)
            launches0 = self.launches
            g = torch.cuda.CUDAGraph()
            dev = self.slabs[0].x.buf.device
            torch.cuda.synchronize(dev)
            with torch.cuda.graph(g):
                self._forward_eager(om, Meff, sums)
            end = tuple(s.x is s.pair[0] for s in self.slabs)
            hit = self._graph_cache[key] = (g, sums, end, self.launches - launches0)
            # capture recorded the work and moved the Python-side buffer roles
            # exactly as an execution would; now run it
            self.launches = launches0
        g, sums, end, nl = hit
        g.replay()
        for s, e in zip(self.slabs, end):
            s.x, s.x_alt = (s.pair[0], s.pair[1]) if e else (s.pair[1], s.pair[0])
        self.launches += nl
        return sums

    def solve(self, *args, **kwargs) -> SolveReport:
        rep = super().solve(*args, **kwargs)
        rep.x = [s.interior(s.x) for s in self.slabs]
        return rep


def local_tb_slabs(family: str, shape, world: int, ranks, device, face_x=None, face_y=None,
                   dx2: float | None = None) -> list[TbSlab]:
    layout = SlabLayout(family, tuple(shape), world)
    return [TbSlab(layout, r, device, dx2=dx2, face_x=face_x, face_y=face_y) for r in ranks]


__all__ = ["SlabLayout", "Slab", "LocalExchanger", "TorchExchanger", "DeviceEngine",
           "SlabSolver", "local_slabs", "PARTS", "ABSOLUTE_L2", "TB_GHOST", "TB3_GHOST",
           "tb_ghost", "TbSlab",
           "LocalTbExchanger", "TorchTbExchanger", "NcclTbExchanger", "TbSlabSolver",
           "local_tb_slabs", "exchange_plan"]
