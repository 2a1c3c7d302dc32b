"""Host logic of the SGS tile kernel (csrc/ops.cu, k_sgs_tile): the halo of its staged window
covers the dependency cone of one symmetric sweep in the colour order 0,1,2,3,P0 | 3,2,1,0
(reading R7).  Entries read from outside the window are garbage; an entry is valid after a step
when everything its update reads is valid.  The tile the kernel writes must be valid."""
import os
import re

import numpy as np

SRC = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                   "paper_2303_10233_b200", "csrc", "ops.cu")


def _const(name):
    m = re.search(r"constexpr int[^;]*\b" + name + r"\s*=\s*(\d+)", open(SRC).read())
    assert m, name
    return int(m.group(1))


def _valid_after_sweep(W):
    V = np.ones((W, W), bool)     # [y, x]
    C = np.ones((W, W), bool)     # cell (e, f) with lower-left vertex (e, f)

    def gv(x, y):
        return 0 <= x < W and 0 <= y < W and V[y, x]

    def gc(e, f):
        return 0 <= e < W and 0 <= f < W and C[f, e]

    def colour(px, py):
        new = V.copy()
        for y in range(py, W, 2):
            for x in range(px, W, 2):
                ok = all(gv(x + dx, y + dy) for dx in (-1, 0, 1) for dy in (-1, 0, 1) if dx or dy)
                ok = ok and all(gc(x + de, y + df) for de in (-1, 0) for df in (-1, 0))
                new[y, x] = ok
        V[:] = new

    for c in ((0, 0), (1, 0), (0, 1), (1, 1)):
        colour(*c)
    C[:] = np.array([[gv(e, f) and gv(e + 1, f) and gv(e, f + 1) and gv(e + 1, f + 1)
                      for e in range(W)] for f in range(W)])
    for c in ((1, 1), (0, 1), (1, 0), (0, 0)):
        colour(*c)
    return V & C


def test_sgs_tile_halo_covers_dependency_cone():
    W, hx, hy, tx, ty = (_const(k) for k in ("SGS_W", "SGS_HX", "SGS_HY", "SGS_TTX", "SGS_TTY"))
    ok = _valid_after_sweep(W)
    assert ok[hy:hy + ty, hx:hx + tx].all()
    # the halos are tight: one entry less on any side leaves an invalid entry in the tile
    assert not ok[hy - 2:hy + ty, hx:hx + tx].all() or hy - 2 < 0
    assert not ok[hy:hy + ty, hx - 2:hx + tx].all()
    assert not ok[hy:hy + ty + 2, hx:hx + tx].all() or hy + ty + 2 > W
    assert not ok[hy:hy + ty, hx:hx + tx + 2].all() or hx + tx + 2 > W
    assert hx % 2 == 0 and hy % 2 == 0 and tx % 2 == 0 and ty % 2 == 0
