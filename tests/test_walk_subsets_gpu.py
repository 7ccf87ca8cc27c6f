"""Walks of a chain subset with every remainder shape (graph replays, direct
multi-sweep launches, single sweeps): the walked chains match the oracle and
the other chains of the handle are untouched (buffer parity bookkeeping)."""

import math

import numpy as np
import pytest

import oracle
import paper_1804_07250_b200 as ts
from paper_1804_07250_b200.lozenge import LozengeHandle, loz_p_up_grid
from paper_1804_07250_b200.sixvertex import SixVertexHandle
from paper_1804_07250_b200.sweeps import DominoHandle

pytestmark = pytest.mark.gpu
STEPS = [1, 2, 3, 5, 7, 9, 17, 33, 70]


@pytest.mark.parametrize("steps", STEPS)
def test_domino_subset(steps):
    d = ts.Domain.aztec(40)
    plan = ts.SweepPlan(d)
    t_max, t_min = ts.extremal_tilings(d)
    start = np.stack([t_max.states, t_min.states, t_max.states])
    h = DominoHandle(d, d.n + 1, 3)
    h.set_p_up(plan.p_up)
    h.upload(start)
    h.walk([9], steps, step0=4, chain0=1)
    out = h.download()
    assert np.array_equal(out[0], start[0]) and np.array_equal(out[2], start[2])
    ref = oracle.domino_walk(start[1:2].copy(), [9], plan.p_up, steps, step0=4)
    assert np.array_equal(out[1], ref[0])


@pytest.mark.parametrize("steps", STEPS)
def test_lozenge_subset(steps):
    d = ts.TriDomain.hexagon(9, 12, 7)
    t_max, t_min = ts.loz_extremal(d)
    start = np.stack([t_max.edges, t_min.edges, t_max.edges])
    p = loz_p_up_grid(d, ts.Uniform())
    h = LozengeHandle(d, 3)
    h.set_p_up(p)
    h.upload(start)
    h.walk([5], steps, step0=3, chain0=1)
    out = h.download()
    assert np.array_equal(out[0], start[0]) and np.array_equal(out[2], start[2])
    assert np.array_equal(out[1], oracle.loz_walk(start[1:2].copy(), [5], p, steps, step0=3)[0])


@pytest.mark.parametrize("steps", STEPS)
def test_sixvertex_subset(steps):
    n = 30
    R, C = np.meshgrid(np.arange(n + 1), np.arange(n + 1), indexing="ij")
    hi, lo = -np.abs(R - C), np.maximum(-(R + C), R + C - 2 * n)
    start = np.stack([hi, lo, hi]).astype(np.int32)
    w = ts.SVWeights(1.0, 1.0, math.sqrt(2.0))
    h = SixVertexHandle(n, 3)
    h.set_weights(w)
    h.upload(start)
    h.walk([11], steps, step0=6, chain0=1)
    out = h.download()
    assert np.array_equal(out[0], start[0]) and np.array_equal(out[2], start[2])
    assert np.array_equal(out[1], oracle.sv_walk(start[1:2].copy(), [11], w.table(), steps, step0=6)[0])
