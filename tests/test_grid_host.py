"""Host-side grid logic: known answers from the reference's test_grid.py / driver.py."""

import numpy as np
import pytest

from paper_1909_01149_b200.grid import CommCounters, Grid, RankLayout, block_partition


def test_linearization_known_answers():
    g = Grid((3, 3, 3))
    assert g.coord_of(5) == (2, 1, 0) and g.rank_of((2, 1, 0)) == 5      # test_grid.py:10-13
    g = Grid((4, 2))
    assert g.coord_of(1) == (1, 0) and g.coord_of(4) == (0, 1)           # test_grid.py:22-25
    with pytest.raises(ValueError):
        Grid((2, 2)).rank_of((2, 0))
    g = Grid((2, 3, 2))
    assert sorted(g.coord_of(r) for r in range(g.total)) == sorted(set(g.coord_of(r) for r in range(g.total)))


def test_slice_groups_known_answers():
    g = Grid((4, 1, 1))                                                  # test_grid.py:34-39
    assert [grp.ranks for grp in g.slice_groups[0]] == [(0,), (1,), (2,), (3,)]
    assert g.slice_groups[1][0].ranks == (0, 1, 2, 3)
    g = Grid((2, 2, 2))
    for n in range(3):
        for c, grp in enumerate(g.slice_groups[n]):
            assert all(g.coord_of(r)[n] == c for r in grp.ranks)


def test_block_partition_known_answers():
    assert block_partition(10, 4).lengths == (3, 3, 2, 2)               # test_grid.py:64-71
    assert block_partition(8, 4).lengths == (2, 2, 2, 2)
    assert block_partition(3, 5).lengths == (1, 1, 1, 0, 0)
    m = block_partition(17, 5)
    assert m.total == 17 and list(m.offsets) == sorted(m.offsets)
    with pytest.raises(ValueError):
        block_partition(-1, 2)
    with pytest.raises(ValueError):
        block_partition(4, 0)


@pytest.mark.parametrize("grid,dims", [((2, 2, 1), (7, 5, 6)), ((1, 2, 4), (5, 3, 4)), ((2, 2, 2, 1), (9, 8, 7, 6))])
def test_rank_layout_covers_everything(grid, dims):
    g = Grid(grid)
    owned = [np.zeros(d, dtype=int) for d in dims]
    cells = np.zeros(dims, dtype=int)
    for r in range(g.total):
        lay = RankLayout(g, r, dims)
        cells[tuple(lay.slice_rows)] += 1
        for n, s in enumerate(lay.owned_rows):
            owned[n][s] += 1
            assert lay.slice_rows[n].start <= s.start and s.stop <= lay.slice_rows[n].stop
    assert (cells == 1).all()
    for n in range(len(dims)):
        # every factor row is owned by exactly one rank (driver.py:239-246)
        assert (owned[n] == 1).all()


def test_counters_merge():
    a, b = CommCounters(), CommCounters()
    a.record("AllReduce", 3, 3)
    b.record("AllReduce", 2, 2)
    b.record("AllGather", 4, 8)
    m = a.merged_with(b)
    assert m.calls == {"AllReduce": 2, "AllGather": 1}
    assert m.total_words() == 3 + 3 + 2 + 2 + 4 + 8


def test_counters_graph_replay_delta():
    """A sweep captured once as a CUDA graph records its collectives once; every later
    replay re-adds exactly that delta, and a failed capture restores the snapshot."""
    c = CommCounters()
    c.record("AllReduce", 4, 4)
    snap = c.snapshot()
    sweep = [("ReduceScatter", 32, 16), ("AllReduce", 2, 2), ("AllGather", 16, 32), ("AllReduce", 4, 4)]
    for name, a, b in sweep:          # the capture records the sweep once
        c.record(name, a, b)
    delta = c.since(snap)
    assert delta["calls"] == {"AllReduce": 2, "ReduceScatter": 1, "AllGather": 1}
    for _ in range(3):                # three more replays
        c.add(delta)
    ref = CommCounters()
    ref.record("AllReduce", 4, 4)
    for _ in range(4):
        for name, a, b in sweep:
            ref.record(name, a, b)
    assert c.snapshot() == ref.snapshot()
    c.restore(snap)
    assert c.snapshot() == snap
