"""Deep ghost-row exchange of the temporally blocked row slabs, on CPU.

The exchangers only use a slab's owned-row range and row views, so a minimal
stand-in slab over CPU tensors exercises them: in process (LocalTbExchanger,
3 virtual ranks) and over torch.distributed gloo with world_size 2
(TorchTbExchanger).  Each ghost row must receive exactly the neighbour's
boundary rows; owned rows are never touched.
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch

from paper_2011_06636_b200.distributed import TB_GHOST, SlabLayout

NX = 8


class FakeField:
    def __init__(self, rows):
        self.halo = NX  # one zero ghost row at each end, as a Field of the extended grid
        self.buf = torch.zeros((rows + 2) * NX, dtype=torch.float64)


class FakeTbSlab:
    """What the exchangers use of a TbSlab: owned rows and row views."""

    def __init__(self, layout, rank):
        self.layout = layout
        self.start, self.count = layout.span(rank)
        self.ghost = TB_GHOST
        self.g_lo = TB_GHOST if rank > 0 else 0
        self.g_hi = TB_GHOST if rank < layout.world - 1 else 0
        self.nx = NX
        self.x = FakeField(self.count + self.g_lo + self.g_hi)

    @property
    def owned(self):
        return self.g_lo, self.g_lo + self.count

    def rows(self, field, r0, r1):
        h = field.halo
        return field.buf[h + r0 * NX:h + r1 * NX]


def _fill_owned(s):
    lo, hi = s.owned
    for r in range(lo, hi):
        s.rows(s.x, r, r + 1).fill_(float(s.start + r - lo))  # = global row index


def _check(slabs):
    for s in slabs:
        lo, hi = s.owned
        view = s.x.buf[s.x.halo:s.x.halo + (hi + s.g_hi) * NX].view(-1, NX)
        for r in range(view.shape[0]):
            want = float(s.start - s.g_lo + r)  # every extended row holds its global row
            assert torch.all(view[r] == want), (s.start, r)


def test_local_deep_row_exchange():
    from paper_2011_06636_b200.distributed import LocalTbExchanger
    layout = SlabLayout("2d5", (NX, 40), 3)
    slabs = [FakeTbSlab(layout, r) for r in range(3)]
    for s in slabs:
        _fill_owned(s)
    ex = LocalTbExchanger(3)
    ex.finish(ex.start_rows(slabs, [s.x for s in slabs]))
    _check(slabs)


def _free_port():
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def _worker(rank, world, port, result_path):
    import torch.distributed as dist

    from paper_2011_06636_b200.distributed import TorchTbExchanger
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        layout = SlabLayout("2d5var", (NX, 31), world)
        s = FakeTbSlab(layout, rank)
        _fill_owned(s)
        ex = TorchTbExchanger()
        ex.finish(ex.start_rows([s], [s.x]))
        _check([s])
        np.save(result_path + f".{rank}.npy", np.array([1]))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_deep_row_exchange(tmp_path):
    import torch.multiprocessing as mp
    out = str(tmp_path / "ok")
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    for r in range(2):
        assert np.load(out + f".{r}.npy")[0] == 1


def test_layout_rejects_thin_tb_slabs():
    from paper_2011_06636_b200.distributed import TbSlabSolver
    layout = SlabLayout("2d5", (NX, 10), 2)
    slabs = [FakeTbSlab(layout, r) for r in range(2)]
    with pytest.raises(ValueError):
        TbSlabSolver(slabs, None)
