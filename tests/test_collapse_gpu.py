"""Run collapsing (tsb_*_set_collapse) is exact: with it on and off every
model's walks equal the C oracle (which executes every sweep, like the
reference's _kernels.py:35-69, sixvertex.py:445-467, lozenge.py:600-622),
for single chains and batches, across graph replays, remainder launches and
single sweeps, and for walks that start mid-stream (step0 > 0)."""

import numpy as np
import pytest

import oracle
import paper_1804_07250_b200 as ts
from paper_1804_07250_b200.lattice import aztec_extremal_states
from paper_1804_07250_b200.lozenge import LozengeHandle, loz_p_up_grid
from paper_1804_07250_b200.sixvertex import SixVertexHandle
from paper_1804_07250_b200.sweeps import DominoHandle

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("order,chains,steps,step0", [(40, 3, 257, 0), (300, 2, 131, 17), (700, 1, 200, 5),
                                                      (1100, 1, 67, 1000)])
def test_domino_collapse_exact(order, chains, steps, step0):
    d = ts.Domain.aztec(order)
    plan = ts.SweepPlan(d)
    t_max, t_min = aztec_extremal_states(order)
    start = np.stack([t_max, t_min] * chains)[:chains]
    seeds = np.arange(21, 21 + chains, dtype=np.uint64)
    ref = oracle.domino_walk(start, seeds, plan.p_up, steps, step0=step0)
    for on in (True, False):
        h = DominoHandle(d, d.n + 1, chains)
        h.set_collapse(on)
        h.set_plan(plan)
        h.upload(start)
        h.walk(seeds, steps, step0=step0)
        assert np.array_equal(h.download(), ref), on


def test_domino_collapse_split_walks():
    """A walk split into pieces (each piece's last sweep is never skipped)
    equals one walk."""
    order = 200
    d = ts.Domain.aztec(order)
    plan = ts.SweepPlan(d)
    t_max, _ = aztec_extremal_states(order)
    ref = oracle.domino_walk(t_max[None], [9], plan.p_up, 300)
    h = DominoHandle(d, d.n + 1, 1)
    h.set_plan(plan)
    h.upload(t_max[None])
    s = 0
    for n in (1, 2, 3, 64, 65, 100, 65):
        h.walk([9], n, step0=s)
        s += n
    assert s == 300
    assert np.array_equal(h.download(), ref)


@pytest.mark.parametrize("n,chains,steps", [(60, 2, 300), (1100, 1, 133)])
def test_sixvertex_collapse_exact(n, chains, steps):
    hi, lo = ts.sv_extremal(n, ts.dwbc(n))
    start = np.stack([lo.heights, hi.heights] * chains)[:chains].astype(np.int32)
    seeds = np.arange(5, 5 + chains, dtype=np.uint64)
    w = ts.SVWeights(1.0, 1.0, 1.5)
    ref = oracle.sv_walk(start, seeds, w.table(), steps, step0=3)
    for on in (True, False):
        h = SixVertexHandle(n, chains)
        h.set_collapse(on)
        h.set_weights(w)
        h.upload(start)
        h.walk(seeds, steps, step0=3)
        assert np.array_equal(h.download(), ref), on


@pytest.mark.parametrize("abc,chains,steps", [((30, 40, 50), 2, 301), ((300, 200, 250), 1, 290)])
def test_lozenge_collapse_exact(abc, chains, steps):
    d = ts.TriDomain.hexagon(*abc)
    t_max, t_min = ts.loz_extremal(d)
    start = np.stack([t_min.edges, t_max.edges] * chains)[:chains]
    seeds = np.arange(7, 7 + chains, dtype=np.uint64)
    w = ts.VolumeWeights(0.97)
    p = loz_p_up_grid(d, w)
    ref = oracle.loz_walk(start, seeds, p, steps, step0=11)
    for on in (True, False):
        h = LozengeHandle(d, chains)
        h.set_collapse(on)
        h.set_p_up(p)
        h.upload(start)
        h.walk(seeds, steps, step0=11)
        assert np.array_equal(h.download(), ref), on


def test_random_walk_batch_pipelined():
    """random_walk_batch on large lattices alternates the chains between two
    one-chain handles on their own streams (copies of one chain overlap the
    sweeps of the next): equal to the oracle for odd and even batch sizes."""
    order = 1100  # 2201^2 = 4.8 MB of tilestates per chain: the pipelined path
    d = ts.Domain.aztec(order)
    plan = ts.SweepPlan(d)
    t_max, t_min = aztec_extremal_states(order)
    for b in (2, 3):
        start = np.stack([t_max, t_min, t_max][:b])
        seeds = np.arange(40, 40 + b, dtype=np.uint64)
        out = ts.random_walk_batch(start, seeds, 37, plan)
        assert np.array_equal(out, oracle.domino_walk(start, seeds, plan.p_up, 37)), b
        assert out is not start and np.array_equal(start[0], t_max)  # a new array; input untouched
