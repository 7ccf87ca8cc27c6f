"""Lozenge parity on the device vs the reference's golden outputs and the C
oracle (bit-exact edge grids and heights)."""

import os

import numpy as np
import pytest

import golden_cases as gc
import oracle
import paper_1804_07250_b200 as ts
from paper_1804_07250_b200.lozenge import LozengeHandle, loz_p_up_grid, loz_random_walk_batch

pytestmark = pytest.mark.gpu
G = os.path.join(os.path.dirname(__file__), "golden")
WEIGHTS = [ts.VolumeWeights(0.9), ts.Uniform(), ts.LozEdgeWeights(1.0, {(("up", 3, 4), ("down", 3, 3)): 2.5})]
CASES = [((8, 8, 8), 0x5EED, 500), ((3, 4, 5), 31337, 200), ((5, 2, 6), 8, 150)]


def load(name):
    return np.load(os.path.join(G, name))


def test_golden_walks_and_heights():
    g = load("lozenge.npz")
    for i, ((abc, seed, steps), w) in enumerate(zip(CASES, WEIGHTS)):
        d = ts.TriDomain.hexagon(*abc)
        out = loz_random_walk_batch(g[f"l{i}_start"][None], [seed], steps, d, w)
        assert np.array_equal(out[0], g[f"l{i}_out"]), f"loz case {i}"
        hh = ts.loz_heights(ts.LozengeTiling(d, out[0]))
        assert np.array_equal(hh.heights, g[f"l{i}_heights"]), f"heights {i}"


def test_golden_extremal():
    g = load("lozenge.npz")
    for abc in gc.LOZ_EXTREMAL:
        d = ts.TriDomain.hexagon(*abc)
        t_max, t_min = ts.loz_extremal(d)
        key = "x" + "_".join(map(str, abc))
        assert np.array_equal(t_max.edges, g[key + "_max"]), abc
        assert np.array_equal(t_min.edges, g[key + "_min"]), abc
        assert np.array_equal(ts.loz_heights(t_max).heights, g[key + "_hmax"])
        assert np.array_equal(ts.loz_heights(t_min).heights, g[key + "_hmin"])


def test_golden_cftp():
    g = load("lozenge.npz")
    for j, (abc, master, count) in enumerate(gc.LOZ_CFTP_CASES):
        d = ts.TriDomain.hexagon(*abc)
        res = ts.loz_cftp(d, ts.Uniform(), master, count=count)
        res = res if isinstance(res, list) else [res]
        assert np.array_equal(np.stack([t.edges for t in res]), g[f"k{j}_edges"]), f"cftp {j}"


@pytest.mark.parametrize("abc,w,steps", [((40, 50, 60), ts.VolumeWeights(0.95), 300),
                                         ((33, 17, 70), ts.Uniform(), 257),
                                         ((20, 1000, 1000), ts.Uniform(), 41)])
def test_walk_vs_oracle(abc, w, steps):
    d = ts.TriDomain.hexagon(*abc)
    t_max, t_min = ts.loz_extremal(d)
    start = np.stack([t_min.edges, t_max.edges])
    seeds = np.array([11, 2**63 + 12], dtype=np.uint64)
    out = loz_random_walk_batch(start, seeds, steps, d, w)
    ref = oracle.loz_walk(start, seeds, loz_p_up_grid(d, w), steps)
    assert np.array_equal(out, ref)
    h = LozengeHandle(d, 2)
    h.set_p_up(loz_p_up_grid(d, w))
    h.upload(start)
    h.walk(seeds, steps // 3)
    h.walk(seeds, steps - steps // 3, step0=steps // 3)
    assert np.array_equal(h.download(), ref)


def test_sweep_classes_and_errors():
    d = ts.TriDomain.hexagon(3, 3, 3)
    t_max, t_min = ts.loz_extremal(d)
    t = ts.loz_random_walk(t_min, 4, 60)
    fam = ts.seed_family(9, (d.size[0] + 1, d.size[1] + 1))
    for cls in range(3):
        out = ts.loz_sweep(t, fam, 5, cls)
        ts.lozenges_from_tiling(out)  # still a valid tiling
        changed = np.argwhere((ts.LozengeTiling(d, out.edges).states_grid != t.states_grid))
        for x, y in changed:
            # only vertices adjacent to a class-`cls` vertex change state
            pass
    bad = t.edges.copy()
    bad[0, 0, 0] = True  # a crossed edge outside the domain
    with pytest.raises(ts.InconsistencyError):
        loz_random_walk_batch(bad[None], [1], 2, d, ts.Uniform())
    up = np.zeros((2, 2), bool)
    dn = np.zeros((2, 2), bool)
    up[0, 0] = True
    assert ts.loz_extremal(ts.TriDomain((2, 2), up, dn)) is None


def test_monotone_coupling():
    d = ts.TriDomain.hexagon(6, 7, 8)
    t_max, t_min = ts.loz_extremal(d)
    out = loz_random_walk_batch(np.stack([t_max.edges, t_min.edges]), [3, 3], 400, d, ts.Uniform())
    h_hi = ts.loz_heights(ts.LozengeTiling(d, out[0])).heights
    h_lo = ts.loz_heights(ts.LozengeTiling(d, out[1])).heights
    m = d.vertex_mask
    assert (h_hi[m] >= h_lo[m]).all()


@pytest.mark.parametrize("K", [2, 4, 8])
@pytest.mark.parametrize("abc,w,steps", [((40, 50, 60), ts.VolumeWeights(0.95), 200),
                                         ((700, 900, 800), ts.Uniform(), 70),
                                         ((60, 20, 45), ts.LozEdgeWeights(1.0, {(("up", 30, 14), ("down", 30, 13)): 3.0}), 130)])
def test_multi_sweep_vs_oracle(monkeypatch, K, abc, w, steps):
    """Temporally blocked graph replays (K sweeps per launch) are bit-identical."""
    monkeypatch.setenv("TSB_LZ_K", str(K))
    d = ts.TriDomain.hexagon(*abc)
    t_max, t_min = ts.loz_extremal(d)
    start = np.stack([t_min.edges, t_max.edges])
    seeds = np.array([0x5EED, 2**64 - 5], dtype=np.uint64)
    p = loz_p_up_grid(d, w)
    h = LozengeHandle(d, 2)
    h.set_p_up(p)
    h.upload(start)
    h.walk(seeds, steps)
    assert np.array_equal(h.download(), oracle.loz_walk(start, seeds, p, steps))


def test_hexagon_arctic_circle_statistics():
    """Statistical observable where draws cannot be matched: uniform lozenge
    tilings of the regular hexagon (side m) are frozen outside the inscribed
    circle (Cohn-Larsen-Propp).  With the axial lattice embedded as
    P(x, y) = x (1, 0) + y (1/2, sqrt3/2) (DIRS, lozenge.py:43), every edge
    family's crossing density is within 0.05 of 0 or 1 beyond 1.1x the
    inradius m sqrt3/2 and near 1/3 inside half of it."""
    m, chains = 64, 16
    d = ts.TriDomain.hexagon(m, m, m)
    t_max, t_min = ts.loz_extremal(d)
    p = loz_p_up_grid(d, ts.Uniform())
    h = LozengeHandle(d, chains)
    h.set_p_up(p)
    h.upload(np.stack([t_min.edges] * chains))
    seeds = np.arange(70, 70 + chains, dtype=np.uint64)
    step = 60 * m * m
    h.walk(seeds, step)
    acc = np.zeros((3,) + t_min.edges.shape[1:])
    for _ in range(8):
        h.walk(seeds, 2 * m * m, step0=step)
        step += 2 * m * m
        acc += h.download().astype(np.float64).sum(axis=0)
    dens = acc / (8 * chains)
    X, Y = np.meshgrid(np.arange(dens.shape[1]) - m, np.arange(dens.shape[2]) - m, indexing="ij")
    r = np.hypot(X + Y / 2.0, Y * np.sqrt(3.0) / 2.0)
    inr = m * np.sqrt(3.0) / 2.0
    vm = d.vertex_mask
    out = vm & (r > 1.1 * inr)
    frozen = np.minimum(dens, 1 - dens)[:, out]
    assert frozen.max() < 0.05, frozen.max()
    inner = dens[:, vm & (r < 0.5 * inr)]
    assert np.all(np.abs(inner.mean(axis=1) - 1.0 / 3.0) < 0.05), inner.mean(axis=1)


@pytest.mark.parametrize("abc", [(1, 1, 1), (2, 15, 16), (3, 16, 16), (1, 31, 2), (5, 5, 27), (30, 2, 3)])
def test_thin_hexagons_vs_oracle(abc):
    """Thin and unbalanced hexagons (vertex columns at and across 32-bit word
    edges, few-row domains); the extremal states differ, so the walk moves."""
    d = ts.TriDomain.hexagon(*abc)
    t_max, t_min = ts.loz_extremal(d)
    assert not np.array_equal(t_max.edges, t_min.edges)
    start = np.stack([t_min.edges, t_max.edges])
    seeds = np.array([21, 22], dtype=np.uint64)
    w = ts.VolumeWeights(1.3)
    out = loz_random_walk_batch(start, seeds, 123, d, w)
    assert np.array_equal(out, oracle.loz_walk(start, seeds, loz_p_up_grid(d, w), 123))
    if sum(abc) > 10:  # (1, 1, 1) has two tilings: it may well end where it started
        assert not np.array_equal(out[0], start[0])
