"""CPU model of H1's tile-local reach prefilter (csrc/ef_hyst.cu, warp_reach).

The claims the CUDA kernels rely on, checked on random label tiles with scipy's
connected components (no GPU needed):

1. Every weak pixel of the tile is in exactly one of: reached from a seed (final
   at once), an unreached component touching the tile perimeter (handed to the
   union-find), or an unreached interior component (not an edge: it cannot
   reach a strong pixel without leaving the tile).
2. The union-find over the reduced set (unreached perimeter components plus
   the reached perimeter pixels) gives every unreached perimeter component the
   node id the full per-tile CCL gives it (tile * 256 + its smallest perimeter
   slot) -- H4's overflow path re-runs the full CCL and looks those ids up.
3. Reached components are strong, so their perimeter pixels may be exported as
   strong nodes of any grouping.
"""

import numpy as np
import pytest
from scipy import ndimage

EIGHT = np.ones((3, 3), dtype=bool)


def perim_slot(y, x, vh, vw):
    s = None
    if x == vw - 1:
        s = 192 + y
    if x == 0:
        s = 128 + y
    if y == vh - 1:
        s = 64 + x
    if y == 0:
        s = x
    return s


def node_ids(mask, vh, vw):
    """{component label: smallest perimeter slot} of the 8-connected components of mask."""
    lab, n = ndimage.label(mask, structure=EIGHT)
    best = {}
    for y, x in zip(*np.nonzero(mask)):
        p = perim_slot(int(y), int(x), vh, vw)
        if p is not None:
            k = lab[y, x]
            best[k] = min(best.get(k, 1 << 30), p)
    return lab, best


def reach(weak, seeds):
    """x <- weak & dilate8(x) to the fixpoint (tile-local)."""
    x = seeds & weak
    while True:
        nx = weak & ndimage.binary_dilation(x, structure=EIGHT)
        if (nx == x).all():
            return x
        x = nx


@pytest.mark.parametrize("seed", range(12))
def test_reach_prefilter_keeps_full_ccl_node_ids(seed):
    rng = np.random.default_rng(seed)
    vh, vw = (64, 64) if seed % 3 else (int(rng.integers(1, 65)), int(rng.integers(1, 65)))
    density = rng.uniform(0.05, 0.45)
    labels = np.zeros((vh + 2, vw + 2), dtype=np.uint8)  # one ring of neighbour-tile pixels
    r = rng.random(labels.shape)
    labels[r < density] = 1
    labels[r < density * rng.uniform(0.05, 0.5)] = 2
    tile = labels[1:-1, 1:-1]
    weak = tile == 1
    strong_ring = labels == 2
    seeds = weak & ndimage.binary_dilation(strong_ring, structure=EIGHT)[1:-1, 1:-1]

    reached = reach(weak, seeds)
    unreached = weak & ~reached
    perim = np.zeros_like(weak)
    perim[0, :] = perim[-1, :] = perim[:, 0] = perim[:, -1] = True
    ulab, un = ndimage.label(unreached, structure=EIGHT)
    touching = set(np.unique(ulab[unreached & perim])) - {0}
    border_unreached = np.isin(ulab, list(touching)) & unreached

    # claim 1: a partition of the weak pixels
    interior = unreached & ~border_unreached
    assert not (reached & unreached).any()
    assert ((reached | border_unreached | interior) == weak).all()
    # ... and exactly the full CCL's answer inside the tile: a component is
    # reached iff it holds a seed
    flab, fn = ndimage.label(weak, structure=EIGHT)
    seeded = set(np.unique(flab[seeds])) - {0}
    assert (reached == (np.isin(flab, list(seeded)) & weak)).all()

    # claim 2: node ids of the unreached perimeter components agree
    _, full_best = node_ids(weak, vh, vw)
    reduced = border_unreached | (reached & perim)
    rlab, red_best = node_ids(reduced, vh, vw)
    for y, x in zip(*np.nonzero(border_unreached & perim)):
        assert red_best[rlab[y, x]] == full_best[flab[y, x]]

    # claim 3: reduced components never mix reached and unreached pixels
    for k in range(1, rlab.max() + 1):
        comp = rlab == k
        assert not ((comp & reached).any() and (comp & unreached).any())
