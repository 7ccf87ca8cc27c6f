"""Height export and the mean-height accumulators on the device.

* the row-scan export (heights.cu / lozenge.cu: per-row prefix sums chained
  through one vertical link per row, every other edge checked) and the
  min-plus relaxation it falls back to are both bit-identical to the
  reference's height_function (lattice.py:537-580) and loz_heights
  (lozenge.py:414-447) on the reference-generated goldens, including the
  non-row-convex random domains;
* inconsistent states raise InconsistencyError on both paths;
* DeviceDensity(handle, "height") sums heights exactly: its counts equal the
  sum of the per-state height grids (the mean height function).
"""

import os

import numpy as np
import pytest

import golden_cases as gc
import paper_1804_07250_b200 as ts
from paper_1804_07250_b200.lozenge import LozengeHandle, loz_p_up_grid
from paper_1804_07250_b200.stats import DeviceDensity
from paper_1804_07250_b200.sweeps import DominoHandle

pytestmark = pytest.mark.gpu
G = os.path.join(os.path.dirname(__file__), "golden")


def _dom_heights(d, states, relax, monkeypatch):
    monkeypatch.setenv("TSB_HEIGHTS_RELAX", "1" if relax else "0")
    h = DominoHandle(d, d.n + 1, 1)  # fresh handle: the path is chosen per handle
    h.upload(states[None])
    return h.heights(0, d.reference_vertex)


@pytest.mark.parametrize("relax", [False, True])
def test_domino_heights_golden_both_paths(relax, monkeypatch):
    g = np.load(os.path.join(G, "domino_extremal.npz"))
    n = 0
    for i, d in enumerate(gc.extremal_domains(ts)):
        if f"d{i}_none" in g.files:
            continue
        for k in ("max", "min", "mixed"):
            got = _dom_heights(d, g[f"d{i}_t{k}"] if k != "mixed" else g[f"d{i}_mixed"], relax, monkeypatch)
            assert np.array_equal(got, g[f"d{i}_h{k}"]), (i, k)
            n += 1
    assert n > 30
    c1 = np.load(os.path.join(G, "domino_c1.npz"))
    d = ts.Domain.aztec(64)
    assert np.array_equal(_dom_heights(d, c1["final"], relax, monkeypatch), c1["heights"])
    assert np.array_equal(_dom_heights(d, c1["t_max"], relax, monkeypatch), c1["heights_tmax"])


def test_domino_scan_and_relax_agree_large(monkeypatch):
    """Aztec 700 after a walk, and a rectangle: both paths identical."""
    for d, steps in ((ts.Domain.aztec(700), 300), (ts.Domain.rectangle(130, 90), 200)):
        t_max, _ = ts.extremal_tilings(d)
        st = ts.random_walk(t_max, 99, steps, ts.SweepPlan(d)).states
        a = _dom_heights(d, st, False, monkeypatch)
        b = _dom_heights(d, st, True, monkeypatch)
        assert np.array_equal(a, b)


@pytest.mark.parametrize("relax", [False, True])
def test_domino_heights_inconsistent_raises(relax, monkeypatch):
    """A tiling with one domino removed (its interior edge cleared on both
    endpoints: edge-consistent, so upload accepts it) has no height function."""
    d = ts.Domain.aztec(8)
    t_max, _ = ts.extremal_tilings(d)
    st = t_max.states.copy()
    r, c = np.argwhere((st & 2) != 0)[5]  # a vertical interior edge (r,c)-(r+1,c)
    st[r, c] &= ~np.uint8(2)
    st[r + 1, c] &= ~np.uint8(1)
    with pytest.raises(ts.InconsistencyError):
        _dom_heights(d, st, relax, monkeypatch)


@pytest.mark.parametrize("relax", [False, True])
def test_lozenge_heights_golden_both_paths(relax, monkeypatch):
    g = np.load(os.path.join(G, "lozenge.npz"))
    monkeypatch.setenv("TSB_HEIGHTS_RELAX", "1" if relax else "0")
    for abc in gc.LOZ_EXTREMAL:
        d = ts.TriDomain.hexagon(*abc)
        key = "x" + "_".join(map(str, abc))
        h = LozengeHandle(d, 2)
        h.upload(np.stack([g[key + "_max"], g[key + "_min"]]))
        assert np.array_equal(h.heights(0, d.reference_vertex), g[key + "_hmax"]), abc
        assert np.array_equal(h.heights(1, d.reference_vertex), g[key + "_hmin"]), abc
    for i, abc in enumerate([(8, 8, 8), (3, 4, 5), (5, 2, 6)]):
        d = ts.TriDomain.hexagon(*abc)
        h = LozengeHandle(d, 1)
        h.upload(g[f"l{i}_out"][None])
        assert np.array_equal(h.heights(0, d.reference_vertex), g[f"l{i}_heights"]), abc


def test_lozenge_scan_and_relax_agree_large(monkeypatch):
    d = ts.TriDomain.hexagon(150, 200, 170)
    t_max, t_min = ts.loz_extremal(d)
    h0 = LozengeHandle(d, 2)
    h0.set_p_up(loz_p_up_grid(d, ts.Uniform()))
    h0.upload(np.stack([t_max.edges, t_min.edges]))
    h0.walk(np.array([5, 6], dtype=np.uint64), 500)
    st = h0.download()
    res = []
    for relax in (False, True):
        monkeypatch.setenv("TSB_HEIGHTS_RELAX", "1" if relax else "0")
        h = LozengeHandle(d, 2)
        h.upload(st)
        res.append([h.heights(k, d.reference_vertex) for k in (0, 1)])
    assert all(np.array_equal(a, b) for a, b in zip(*res))


def test_domino_mean_height_accumulator():
    d = ts.Domain.aztec(120)
    plan = ts.SweepPlan(d)
    t_max, t_min = ts.extremal_tilings(d)
    chains = 4
    h = DominoHandle(d, d.n + 1, chains)
    h.set_plan(plan)
    h.upload(np.stack([t_max.states, t_min.states] * 2))
    acc = DeviceDensity(h, "height")
    ref = np.zeros((d.n + 1, d.n + 1), dtype=np.int64)
    seeds = np.arange(11, 11 + chains, dtype=np.uint64)
    for k in range(3):
        h.walk(seeds, 50, step0=50 * k)
        acc.add()
        for s in h.download():
            ref += ts.height_function(ts.Tiling(d, s)).heights
    assert np.array_equal(acc.counts(), ref)
    res = acc.result()
    assert res.samples == 3 * chains
    assert np.array_equal(res.grid, ref / (3 * chains))


def test_lozenge_mean_height_accumulator():
    d = ts.TriDomain.hexagon(30, 40, 25)
    t_max, t_min = ts.loz_extremal(d)
    h = LozengeHandle(d, 2)
    h.set_p_up(loz_p_up_grid(d, ts.VolumeWeights(0.95)))
    h.upload(np.stack([t_max.edges, t_min.edges]))
    acc = DeviceDensity(h, "height")
    ref = np.zeros((d.size[0] + 1, d.size[1] + 1), dtype=np.int64)
    for k in range(4):
        h.walk(np.array([3, 4], dtype=np.uint64), 60, step0=60 * k)
        acc.add()
        for e in h.download():
            ref += ts.loz_heights(ts.LozengeTiling(d, e)).heights
    assert np.array_equal(acc.counts(), ref)
    assert acc.result().samples == 8
