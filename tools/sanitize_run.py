"""Small-lattice workload for compute-sanitizer (tools/sanitize.sh): every
kernel family of libtsb.so, each result checked against the C oracle, with
no torch in the process (only libtsb's own kernels are launched).

    python tools/sanitize_run.py domino|cftp|heights|strips|sv|loz|domain

The TSB_* knobs in the environment select the kernel variant (the handle
reads them at creation / per walk)."""

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import paper_1804_07250_b200 as ts  # noqa: E402
from paper_1804_07250_b200.lattice import aztec_extremal_states  # noqa: E402
from paper_1804_07250_b200.sweeps import DominoHandle  # noqa: E402


def domino():
    for order, chains, steps in ((12, 3, 70), (70, 2, 67), (100, 1, 130)):
        d = ts.Domain.aztec(order)
        plan = ts.SweepPlan(d)
        t_max, t_min = aztec_extremal_states(order)
        start = np.stack([t_max, t_min] * chains)[:chains]
        seeds = np.arange(5, 5 + chains, dtype=np.uint64)
        out = ts.random_walk_batch(start, seeds, steps, plan)
        assert np.array_equal(out, oracle.domino_walk(start, seeds, plan.p_up, steps)), order
        fam = ts.seed_family(9, (d.n + 1, d.n + 1))
        t1 = ts.sweep(ts.Tiling(d, out[0]), fam, 3, ts.Color.WHITE, plan)
        assert np.array_equal(t1.states, oracle.domino_sweep(out[0], 9, plan.p_up, 3, 1))
    h = DominoHandle(ts.Domain.aztec(20), 41, 2)
    h.set_plan(ts.SweepPlan(ts.Domain.aztec(20)))
    h.upload(np.stack(aztec_extremal_states(20)))
    h.walk([1, 2], 40)
    h.sync()
    print("domino ok")


def cftp():
    d = ts.Domain.aztec(6)
    s = ts.cftp_sample_many(d, ts.SweepPlan(d), 0x5EED, 5)
    assert len(s) == 5
    print("cftp ok")


def heights():
    for relax in ("0", "1"):
        os.environ["TSB_HEIGHTS_RELAX"] = relax
        d = ts.Domain.aztec(30)
        t_max, _ = aztec_extremal_states(30)
        st = ts.random_walk(ts.Tiling(d, t_max), 3, 50, ts.SweepPlan(d)).states
        h = DominoHandle(d, d.n + 1, 1)
        h.upload(st[None])
        h.heights(0, d.reference_vertex)
        ext = ts.extremal_tilings(ts.Domain.rectangle(6, 8))
        assert ext is not None
        ld = ts.TriDomain.hexagon(5, 6, 7)
        lt = ts.loz_extremal(ld)[0]
        ts.loz_heights(lt)
    print("heights ok")


def strips():
    from paper_1804_07250_b200.strips import DeviceStripWalker, strip_bounds

    order, world, halo, steps = 60, 2, 8, 40
    d = ts.Domain.aztec(order)
    plan = ts.SweepPlan(d)
    t_max, _ = aztec_extremal_states(order)
    hs = []
    for _ in range(world):
        h = DominoHandle(d, d.n + 1, 1, device=0)
        h.set_plan(plan)
        h.upload(t_max[None])
        hs.append(h)
    ws = DeviceStripWalker.local(hs, strip_bounds(d.vertex_mask, world, min_rows=halo), halo)
    DeviceStripWalker.walk_lockstep(ws, 0x5EED, steps)
    got = np.concatenate([w.handle.download()[0][w.lo:w.hi] for w in ws])
    for w in ws:
        w.close()
    assert np.array_equal(got, oracle.domino_walk(t_max[None], [0x5EED], plan.p_up, steps)[0])
    print("strips ok")


def sv():
    from paper_1804_07250_b200.sixvertex import sv_random_walk_batch

    for n, chains in ((9, 2), (70, 3), (140, 1)):
        hi, lo = ts.sv_extremal(n, ts.dwbc(n))
        start = np.stack([hi.heights, lo.heights] * chains)[:chains]
        seeds = np.arange(3, 3 + chains, dtype=np.uint64)
        w = ts.SVWeights(1.0, 1.0, 1.5)
        out = sv_random_walk_batch(start, seeds, 37, w)
        assert np.array_equal(out, oracle.sv_walk(start, seeds, w.table(), 37)), n
    ts.sv_cftp(4, ts.dwbc(4), ts.SVWeights(1, 1, 1.2), 7, count=3)
    print("sv ok")


def loz():
    from paper_1804_07250_b200.lozenge import loz_p_up_grid, loz_random_walk_batch

    for abc, chains in (((3, 4, 5), 2), ((20, 25, 30), 3), ((60, 20, 40), 1)):
        d = ts.TriDomain.hexagon(*abc)
        t_max, t_min = ts.loz_extremal(d)
        start = np.stack([t_max.edges, t_min.edges] * chains)[:chains]
        seeds = np.arange(3, 3 + chains, dtype=np.uint64)
        w = ts.VolumeWeights(0.9)
        out = loz_random_walk_batch(start, seeds, 41, d, w)
        assert np.array_equal(out, oracle.loz_walk(start, seeds, loz_p_up_grid(d, w), 41)), abc
    ts.loz_cftp(ts.TriDomain.hexagon(2, 2, 2), ts.Uniform(), 5, count=3)
    print("loz ok")


def domain():
    import ctypes

    from paper_1804_07250_b200 import _native

    m = np.random.default_rng(1).random((300, 200)) < 0.6
    k = ctypes.c_int64()
    g = np.ascontiguousarray(m, dtype=np.uint8)
    _native.check(_native.lib().tsb_grid_components(0, _native.ptr(g), 300, 200, ctypes.byref(k)))
    u = np.ascontiguousarray(m, dtype=np.uint8)
    chi = ctypes.c_int64()
    _native.check(_native.lib().tsb_tri_check(0, _native.ptr(u), _native.ptr(u), 300, 200, ctypes.byref(k),
                                              ctypes.byref(chi)))
    print("domain ok")


if __name__ == "__main__":
    for name in sys.argv[1:]:
        globals()[name]()
