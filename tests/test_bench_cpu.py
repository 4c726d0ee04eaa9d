"""CPU checks of bench.py's host logic: the patch-grid block partition used for --gpus N."""
import collections

import pytest

import bench


@pytest.mark.parametrize("grid,world,expect", [((8, 8, 4), 2, (128, 2)), ((8, 8, 4), 4, (64, 4)),
                                               ((8, 8, 4), 8, (32, 8)), ((4, 4), 2, (8, 2)),
                                               ((4, 4, 4), 8, (8, 8))])
def test_block_owner_balanced_contiguous(grid, world, expect):
    own = bench.block_owner(grid, world)
    cnt = collections.Counter(own)
    assert len(cnt) == expect[1] and set(cnt.values()) == {expect[0]}
    # every rank's patches form a box of the patch grid
    import itertools
    for r in range(world):
        idx = [i for i, o in enumerate(own) if o == r]
        coords = []
        for k in idx:
            c, t = [], k
            for g in grid:
                c.append(t % g)
                t //= g
            coords.append(c)
        lo = [min(c[d] for c in coords) for d in range(len(grid))]
        hi = [max(c[d] for c in coords) for d in range(len(grid))]
        vol = 1
        for a, b in zip(lo, hi):
            vol *= b - a + 1
        assert vol == len(idx)


def test_block_owner_falls_back():
    assert bench.block_owner((3, 3), 2) is None
