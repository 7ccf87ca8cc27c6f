"""On-device observables (density maps, mean heights) vs the oracle's
restatement of the reference's stats.py and the reference's own golden
density maps (tests/golden/observables.npz)."""

import os

import numpy as np
import pytest

import oracle
import paper_1804_07250_b200 as ts
from paper_1804_07250_b200.sixvertex import SixVertexHandle
from paper_1804_07250_b200.stats import DeviceDensity
from paper_1804_07250_b200.sweeps import DominoHandle

pytestmark = pytest.mark.gpu
G = os.path.join(os.path.dirname(__file__), "golden")


def test_domino_density_golden():
    g = np.load(os.path.join(G, "observables.npz"))
    d = ts.Domain.aztec(32)
    st = g["dom_states"]
    h = DominoHandle(d, d.n + 1, len(st))
    h.upload(st)
    acc = DeviceDensity(h, "domino-orientation")
    acc.add()
    res = acc.result()
    assert res.samples == len(st)
    # counts are exact; the mean equals the reference's acc / len up to the
    # order of the float sum (the reference adds float grids)
    assert np.allclose(res.grid, g["dom_density"], equal_nan=True, rtol=0, atol=1e-15)
    counts = acc.counts()
    ref = sum(np.nan_to_num(oracle.domino_orientation(s, d.faces)) for s in st)
    assert np.array_equal(counts, ref.astype(np.int64))


@pytest.mark.parametrize("order,chains,rounds", [(64, 8, 5), (300, 3, 4)])
def test_domino_density_accumulates_walks(order, chains, rounds):
    d = ts.Domain.aztec(order)
    plan = ts.SweepPlan(d)
    t_max, _ = ts.extremal_tilings(d)
    h = DominoHandle(d, d.n + 1, chains)
    h.set_p_up(plan.p_up)
    h.upload(np.stack([t_max.states] * chains))
    acc = DeviceDensity(h, "domino-orientation")
    seeds = np.arange(1, chains + 1, dtype=np.uint64)
    ref = np.zeros((d.n, d.n))
    step = 0
    for _ in range(rounds):
        h.walk(seeds, 37, step0=step)
        step += 37
        acc.add()
        for s in h.download():
            ref += np.nan_to_num(oracle.domino_orientation(s, d.faces))
    assert np.array_equal(acc.counts(), ref.astype(np.int64))
    res = acc.result()
    assert np.isnan(res.grid[~d.faces]).all()
    y = ts.aztec_y_intercept_from_density(oracle.domino_orientation(h.download()[0], d.faces))
    assert y == oracle.aztec_y_intercept(oracle.domino_orientation(h.download()[0], d.faces))


def test_sixvertex_density_golden_and_walks():
    g = np.load(os.path.join(G, "observables.npz"))
    hs = g["sv_heights"]
    n = hs.shape[1] - 1
    h = SixVertexHandle(n, len(hs))
    h.upload(hs)
    for name in ("h-edge", "v-edge", "c-vertex"):
        acc = DeviceDensity(h, name)
        acc.add()
        assert np.array_equal(acc.result().grid, g["sv_" + name.replace("-", "_")]), name
    hsum = DeviceDensity(h, "height")
    hsum.add()
    assert np.array_equal(hsum.counts(), hs.astype(np.int64).sum(0))
    # larger walked batch vs the oracle's restatement
    n = 70
    R, C = np.meshgrid(np.arange(n + 1), np.arange(n + 1), indexing="ij")
    lo = np.maximum(-(R + C), R + C - 2 * n).astype(np.int32)
    h = SixVertexHandle(n, 4)
    h.set_weights(ts.SVWeights(1.0, 1.0, 1.3))
    h.upload(np.stack([lo] * 4))
    accs = {k: DeviceDensity(h, k) for k in ("h-edge", "v-edge", "c-vertex", "height")}
    ref = {k: 0 for k in accs}
    seeds = np.array([3, 4, 5, 6], dtype=np.uint64)
    for r in range(3):
        h.walk(seeds, 45, step0=45 * r)
        for a in accs.values():
            a.add()
        for x in h.download():
            he, ve = oracle.sv_edges(x)
            ref["h-edge"] = ref["h-edge"] + he
            ref["v-edge"] = ref["v-edge"] + ve
            ref["c-vertex"] = ref["c-vertex"] + oracle.sv_c_vertex(he, ve)
            ref["height"] = ref["height"] + x.astype(np.int64)
    for k, a in accs.items():
        assert np.array_equal(a.counts(), np.asarray(ref[k]).astype(np.int64)), k


def test_arctic_circle_statistics():
    """Statistical observables where draws cannot be matched (north_star):
    the reference's acceptance C8 (test_acceptance.py:264-296: the four
    corners outside 1.1x the arctic circle are frozen >= 0.95, top/bottom
    horizontal, left/right vertical) at order 128 from 32 long device walks,
    plus the centre density ~ 1/2 and the y-intercept ~ -order/sqrt(2)."""
    order, chains = 128, 32
    d = ts.Domain.aztec(order)
    plan = ts.SweepPlan(d)
    t_max, _ = ts.extremal_tilings(d)
    h = DominoHandle(d, d.n + 1, chains)
    h.set_p_up(plan.p_up)
    h.upload(np.stack([t_max.states] * chains))
    seeds = np.arange(100, 100 + chains, dtype=np.uint64)
    burn = 1 << 18  # 16 n^2 sweeps
    h.walk(seeds, burn)
    acc = DeviceDensity(h, "domino-orientation")
    step, yints = burn, []
    for _ in range(8):
        h.walk(seeds, 4096, step0=step)
        step += 4096
        acc.add()
        for s in h.download()[:4]:
            yints.append(ts.aztec_y_intercept_from_density(oracle.domino_orientation(s, d.faces)))
    grid = acc.result().grid
    n = d.n
    rr, cc = np.meshgrid(np.arange(n) + 0.5 - order, np.arange(n) + 0.5 - order, indexing="ij")
    radius = 1.1 * order / np.sqrt(2.0)
    outside = (rr ** 2 + cc ** 2 > radius ** 2) & d.faces
    regions = {"top": outside & (-rr > np.abs(cc)), "bottom": outside & (rr > np.abs(cc)),
               "left": outside & (-cc >= np.abs(rr)), "right": outside & (cc >= np.abs(rr))}
    frac = {k: float(np.nanmean(grid[v])) for k, v in regions.items()}
    assert frac["top"] >= 0.95 and frac["bottom"] >= 0.95, frac  # horizontal bricks
    assert frac["left"] <= 0.05 and frac["right"] <= 0.05, frac  # vertical bricks
    centre = (rr ** 2 + cc ** 2 < (0.25 * order) ** 2)
    assert abs(float(np.nanmean(grid[centre])) - 0.5) < 0.05
    y = float(np.mean(yints))
    assert abs(y + order / np.sqrt(2.0)) < 0.12 * order / np.sqrt(2.0), y


def test_sixvertex_free_fermion_arctic_circle():
    """Statistical observable where draws cannot be matched: DWBC six-vertex at
    the free-fermion point (a = b = 1, c = sqrt 2, Delta = 0) has the arctic
    circle inscribed in the square; outside 1.1x its radius the four corners
    are frozen (every edge-occupancy density within 0.05 of 0 or 1), inside
    0.5x the edges fluctuate.  Device densities over 16 chains x 8 samples."""
    import math

    n, chains = 96, 16
    R, C = np.meshgrid(np.arange(n + 1), np.arange(n + 1), indexing="ij")
    lo = np.maximum(-(R + C), R + C - 2 * n).astype(np.int32)
    h = SixVertexHandle(n, chains)
    h.set_weights(ts.SVWeights(1.0, 1.0, math.sqrt(2.0)))
    h.upload(np.stack([lo] * chains))
    seeds = np.arange(50, 50 + chains, dtype=np.uint64)
    burn = 40 * n * n
    h.walk(seeds, burn)
    acc = DeviceDensity(h, "h-edge")
    step = burn
    for _ in range(8):
        h.walk(seeds, 2 * n * n, step0=step)
        step += 2 * n * n
        acc.add()
    grid = acc.result().grid  # (n, n+1): h_edges[r, c] between faces (r, c), (r+1, c)
    rr, cc = np.meshgrid(np.arange(n) + 1.0 - (n + 1) / 2, np.arange(n + 1) + 0.5 - (n + 1) / 2, indexing="ij")
    rad = np.hypot(rr, cc)
    frozen = grid[rad > 1.1 * n / 2]
    assert np.minimum(frozen, 1 - frozen).max() < 0.05, np.minimum(frozen, 1 - frozen).max()
    inner = grid[rad < 0.5 * n / 2]
    assert 0.2 < inner.mean() < 0.8 and np.minimum(inner, 1 - inner).mean() > 0.15
