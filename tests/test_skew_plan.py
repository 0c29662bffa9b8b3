"""Host-side work plan of the skewed-tile 2D kernel (srj_skew_plan, CPU only).

The kernel trusts the table: every grid row of every strip must be owned by
exactly one segment, a segment's tiles must start 2 * sweeps rows above it
(sweeps at the grid's top) and follow each other every tile_rows rows until
their slots cover it (plus the skew at the grid's bottom), cuts inside the
grid must fall on multiples of the rows per warp, a
CTA's tiles of one segment must be consecutive (the carry rows go from one
tile to the next), and no CTA may exceed the budget.
"""

from __future__ import annotations

import os

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2011_06636_b200", "libsrj.so")

pytestmark = pytest.mark.skipif(not os.path.exists(LIB), reason="libsrj.so not built")

SHAPES = [(2048, 2048, 148), (4096, 4096, 148), (1024, 1024, 148), (96, 96, 148), (2, 300, 148),
          (400, 1, 148), (52, 96, 148), (130, 250, 148), (1100, 1100, 148), (2048, 2048, 144),
          (8192, 8192, 148), (3000, 700, 132), (64, 5000, 7), (100000, 8, 148)]


@pytest.mark.parametrize("nx,ny,ncta", SHAPES)
def test_plan_covers_every_row_once(nx, ny, ncta):
    from paper_2011_06636_b200 import _lib
    p = _lib.skew_plan(nx, ny, ncta)
    T, RY, TX, S = p["tiles_per_cta"], p["tile_rows"], p["tile_cols"], p["sweeps"]
    strips = -(-nx // TX)
    owned = {sx: [] for sx in range(strips)}
    used = 0
    for tiles in p["tiles"]:
        assert len(tiles) <= T
        used += bool(tiles)
        i = 0
        while i < len(tiles):
            ox, oy, lo, hi = tiles[i]
            assert ox % TX == 0 and 0 <= ox < nx
            assert 0 <= lo < hi <= ny
            lead = 2 * S if lo > 0 else S  # restart inside the grid: 2S rows early; top: S
            assert oy == lo - lead
            if hi < ny:  # cut inside the grid: whole warps (V = S rows) own or not
                assert (hi - lo) % S == 0
                k = -(-(hi - lo + lead) // RY)
            else:        # to the grid's bottom: S more rows of skew
                k = -(-(hi - lo + lead + S) // RY)
            seg = tiles[i:i + k]
            assert len(seg) == k, "a segment's tiles stay on one CTA"
            for j, t in enumerate(seg):
                assert t == (ox, oy + j * RY, lo, hi)
            owned[ox // TX].append((lo, hi))
            i += k
    assert used == p["ctas_used"] <= ncta
    for sx, segs in owned.items():
        segs.sort()
        assert segs[0][0] == 0 and segs[-1][1] == ny, (sx, segs)
        for (a0, a1), (b0, b1) in zip(segs, segs[1:]):
            assert a1 == b0, (sx, segs)


def test_plan_budget_is_tight():
    """No smaller budget packs the grid; 2048^2 (C2) takes 6 tiles of 96 rows on
    147 CTAs, against ten rounds of 72-row square tiles."""
    from paper_2011_06636_b200 import _lib
    p = _lib.skew_plan(2048, 2048, 148)
    assert (p["tiles_per_cta"], p["tile_rows"], p["tile_cols"], p["sweeps"]) == (6, 96, 52, 6)
    assert p["ctas_used"] == 147
    total = sum(len(t) for t in p["tiles"])
    assert total == 880, total
    for nx, ny, ncta in SHAPES:
        q = _lib.skew_plan(nx, ny, ncta)
        T, RY, TX, S = q["tiles_per_cta"], q["tile_rows"], q["tile_cols"], q["sweeps"]
        need = -(-nx // TX) * (ny + 2 * S)  # region rows if every strip were one segment
        assert T * RY * ncta >= need
        # the greedy packing needed more than (T - 1) tiles per CTA: the tiles it places
        # with budget T already exceed what ncta CTAs hold with one tile less
        ntiles = sum(len(t) for t in q["tiles"])
        assert ntiles <= T * ncta
        if T > 1 and q["ctas_used"] == ncta:
            assert ntiles > (T - 1) * (ncta - 1)


def test_plan_rejects_bad_arguments():
    from paper_2011_06636_b200 import _lib
    L = _lib.load()
    assert L.srj_skew_plan(0, 5, 148, None, None, None, None, None, None, 0) == _lib.SRJ_BAD_ARGUMENT
    import ctypes
    small = (ctypes.c_int32 * 4)()
    assert L.srj_skew_plan(2048, 2048, 148, None, None, None, None, None, small, 4) == _lib.SRJ_BAD_ARGUMENT
    assert b"capacity" in L.srj_last_error()
