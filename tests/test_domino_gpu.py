"""Domino parity on the device: the CUDA path vs the reference's golden
outputs and vs the C oracle (bit-exact; integer/byte work)."""

import hashlib
import json
import os

import numpy as np
import pytest

import golden_cases as gc
import oracle
import paper_1804_07250_b200 as ts
from paper_1804_07250_b200.sweeps import DominoHandle

pytestmark = pytest.mark.gpu
G = os.path.join(os.path.dirname(__file__), "golden")


def load(name):
    return np.load(os.path.join(G, name))


def fp(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


def dom(faces):
    return ts.Domain(faces.shape[0], faces)


def test_c1_fingerprint():
    """BASELINE config 1: Aztec 64, T_max, seed 0x5EED, 1000 sweeps."""
    g = load("domino_c1.npz")
    d = ts.Domain.aztec(64)
    t = ts.random_walk(ts.Tiling(d, g["t_max"]), 0x5EED, 1000, ts.SweepPlan(d))
    assert fp(t.states) == "fe33268e95b1a840"
    assert np.array_equal(t.states, g["final"])


def test_golden_walk_cases():
    g = load("domino_walks.npz")
    for i, w in enumerate(gc.domino_walk_weights(ts)):
        d = dom(g[f"c{i}_faces"])
        plan = ts.SweepPlan(d, w)
        out = ts.random_walk_batch(g[f"c{i}_start"], g[f"c{i}_seeds"], int(g[f"c{i}_n_steps"]), plan)
        assert np.array_equal(out, g[f"c{i}_out"]), f"case {i}"


def test_golden_single_sweeps():
    g = load("domino_walks.npz")
    for j, (_, seed, step, color) in enumerate(gc.SWEEP_CASES):
        d = dom(g[f"s{j}_faces"])
        t0 = ts.Tiling(d, g[f"s{j}_in"])
        fam = ts.seed_family(seed, (d.n + 1, d.n + 1))
        t1, rot = ts.sweep(t0, fam, step, ts.Color(color), ts.SweepPlan(d), return_rotated=True)
        assert np.array_equal(t1.states, g[f"s{j}_out"])
        assert np.array_equal(rot, g[f"s{j}_rot"])


def test_uniform_grid_device():
    g = load("rng_grids.npz")
    for name in g.files:
        seed, r, c, step = (int(x) for x in name.split("_"))
        assert np.array_equal(ts.seed_family(seed, (r, c)).uniform_grid(step), g[name])


@pytest.mark.parametrize("order,steps,seed", [(50, 400, 1), (97, 333, 2**63 + 5), (130, 257, 0x5EED)])
def test_walk_vs_oracle_aztec(order, steps, seed):
    """Seeded parity vs the C oracle beyond the golden sizes (odd orders give
    side % 32 != 0, several warps per row and partially covered words)."""
    g = load("domino_c1.npz")
    d = ts.Domain.aztec(order)
    ext = ts.extremal_tilings(d)
    plan = ts.SweepPlan(d)
    start = np.stack([ext[0].states, ext[1].states])
    seeds = np.array([seed, seed + 1], dtype=np.uint64)
    out = ts.random_walk_batch(start, seeds, steps, plan)
    ref = oracle.domino_walk(start, seeds, plan.p_up, steps, threads=4)
    assert np.array_equal(out, ref)


def test_walk_vs_oracle_multi_chunk():
    """Rows wider than one warp tile (62 words = 1984 columns): tile seams,
    per-site thresholds (mode 2) and the graph + remainder launch path."""
    d = ts.Domain.aztec(1100)
    plan = ts.SweepPlan(d, ts.VolumeWeights(1.01, {(1100, 1100): 5.0, (1100, 1985): 0.2}))
    t_max, _ = ts.lattice.aztec_extremal_states(1100)
    out = ts.random_walk_batch(t_max[None], [77], 75, plan)
    ref = oracle.domino_walk(t_max[None], [77], plan.p_up, 75, threads=8)
    assert np.array_equal(out, ref)
    # a mixed start (coins active across the seams)
    out2 = ts.random_walk_batch(out, [78], 70, ts.SweepPlan(d))
    ref2 = oracle.domino_walk(ref, [78], np.full_like(plan.p_up, 0.5), 70, threads=8)
    assert np.array_equal(out2, ref2)


def test_walk_vs_oracle_weighted_square():
    d = ts.Domain.square(70)
    w = ts.VolumeWeights(0.8, {(5, 5): 3.0, (69, 1): 0.1})
    plan = ts.SweepPlan(d, w)
    ext = ts.extremal_tilings(d)
    start = np.stack([ext[1].states])
    out = ts.random_walk_batch(start, [12345], 500, plan)
    assert np.array_equal(out, oracle.domino_walk(start, [12345], plan.p_up, 500))


def test_split_walk_equals_one_walk():
    d = ts.Domain.aztec(40)
    plan = ts.SweepPlan(d)
    ext = ts.extremal_tilings(d)
    h = DominoHandle(d, d.n + 1, 2)
    h.set_p_up(plan.p_up)
    start = np.stack([ext[0].states, ext[1].states])
    h.upload(start)
    h.walk([7, 8], 37)
    h.walk([7, 8], 100, step0=37)
    a = h.download()
    b = ts.random_walk_batch(start, [7, 8], 137, plan)
    assert np.array_equal(a, b)
    # subset walks keep the other chain untouched
    h.upload(start)
    h.walk([9], 11, chain0=1)
    c = h.download()
    assert np.array_equal(c[0], start[0])
    assert np.array_equal(c[1], ts.random_walk_batch(start[1:], [9], 11, plan)[0])


def test_batch_matches_single_chain_runs():
    d = ts.Domain.rectangle(2, 3)
    plan = ts.SweepPlan(d)
    t0 = ts.extremal_tilings(d)[0]
    seeds = np.array([5, 6, 7], dtype=np.uint64)
    batch = ts.random_walk_batch(np.repeat(t0.states[None], 3, axis=0), seeds, 40, plan)
    for i, s in enumerate(seeds):
        assert np.array_equal(batch[i], ts.random_walk(t0, int(s), 40, plan).states)


def test_zero_steps_and_errors():
    d = ts.Domain.rectangle(2, 3)
    plan = ts.SweepPlan(d)
    t0 = ts.extremal_tilings(d)[0]
    assert ts.random_walk(t0, 7, 0, plan) == t0
    with pytest.raises(ValueError):
        ts.random_walk(t0, 7, -1, plan)
    bad = t0.states.copy()
    bad[0, 0] ^= 2  # unmirrored edge bit
    with pytest.raises(ts.InconsistencyError):
        ts.random_walk_batch(bad[None], [1], 3, plan)
    bad = t0.states.copy()
    bad[1, 1] = 200
    with pytest.raises(ts.InconsistencyError):
        ts.random_walk_batch(bad[None], [1], 3, plan)


def test_extremal_and_heights_golden():
    g = load("domino_extremal.npz")
    for i, d in enumerate(gc.extremal_domains(ts)):
        ext = ts.extremal_tilings(d)
        if f"d{i}_none" in g.files:
            assert ext is None, f"domain {i} should be untileable"
            continue
        assert ext is not None, f"domain {i}"
        assert np.array_equal(ext[0].states, g[f"d{i}_tmax"]), f"tmax {i}"
        assert np.array_equal(ext[1].states, g[f"d{i}_tmin"]), f"tmin {i}"
        for key in ("max", "min", "mixed"):
            st = g[f"d{i}_t{key}"] if key != "mixed" else g[f"d{i}_mixed"]
            hf = ts.height_function(ts.Tiling(d, st))
            assert np.array_equal(hf.heights, g[f"d{i}_h{key}"]), f"heights {key} {i}"


def test_c1_heights():
    g = load("domino_c1.npz")
    d = ts.Domain.aztec(64)
    assert np.array_equal(ts.height_function(ts.Tiling(d, g["final"])).heights, g["heights"])
    assert np.array_equal(ts.height_function(ts.Tiling(d, g["t_max"])).heights, g["heights_tmax"])
    ext = ts.extremal_tilings(d)
    assert np.array_equal(ext[0].states, g["t_max"]) and np.array_equal(ext[1].states, g["t_min"])


def test_untileable():
    d = ts.Domain.from_faces(2, [(0, 0), (0, 1), (1, 0)])
    assert ts.extremal_tilings(d) is None
    with pytest.raises(ts.UntileableDomain):
        ts.cftp_sample(d, ts.SweepPlan(d), 1)


def test_cftp_golden():
    g = load("domino_cftp.npz")
    traces = json.load(open(os.path.join(G, "domino_cftp_traces.json")))
    weights = [ts.Uniform(), ts.Uniform(), ts.VolumeWeights(1.0, {(2, 3): 2.0}), ts.Uniform(), ts.Uniform()]
    masters = [999, 3, 271828, 271828, 0x5EED]
    counts = [7, 3, 4, 1, 2]
    for i in range(5):
        d = dom(g[f"k{i}_faces"])
        trace = ts.CftpTrace()
        samples = ts.cftp_sample_many(d, ts.SweepPlan(d, weights[i]), masters[i], counts[i], trace=trace)
        assert np.array_equal(np.stack([s.states for s in samples]), g[f"k{i}_samples"]), f"case {i}"
        assert [[list(p) for p in r] for r in trace.rounds] == traces[i]["rounds"]
        assert trace.collapsed_at == traces[i]["collapsed_at"]


def test_cftp_batching_and_progress():
    import io

    d = ts.Domain.rectangle(2, 3)
    plan = ts.SweepPlan(d)
    a = ts.cftp_sample_many(d, plan, 999, 7, batch_size=2)
    b = ts.cftp_sample_many(d, plan, 999, 7, batch_size=7)
    singles = [ts.cftp_sample_many(d, plan, 999, k + 1)[k] for k in range(7)]
    assert a == b == singles
    buf = io.StringIO()
    ts.cftp_sample(ts.Domain.square(4), ts.SweepPlan(ts.Domain.square(4)), 3, progress=buf)
    lines = buf.getvalue().strip().splitlines()
    assert lines[-1].endswith("collapsed=True")
    assert all(ln.endswith("collapsed=False") for ln in lines[:-1])
    with pytest.raises(ts.ConvergenceCapExceeded):
        ts.cftp_sample(ts.Domain.square(6), ts.SweepPlan(ts.Domain.square(6)), 1, max_doublings=2)
    one = ts.Domain.rectangle(1, 2)
    trace = ts.CftpTrace()
    ts.cftp_sample(one, ts.SweepPlan(one), 9, trace=trace)
    assert trace.rounds == []


def test_strip_windows_on_one_device():
    """Two 'ranks' in one process: windowed walks + device row exchange
    (the NCCL path of bench.py --gpus N without the network) reproduce the
    single-handle walk."""
    import torch

    from paper_1804_07250_b200.strips import DominoStripEngine, StripWalker, strip_bounds

    order, halo, steps = 300, 16, 150
    d = ts.Domain.aztec(order)
    t_max, _ = ts.lattice.aztec_extremal_states(order)
    plan = ts.SweepPlan(d)
    bounds = strip_bounds(d.vertex_mask, 2, min_rows=halo)
    engines, walkers = [], []
    for rank in range(2):
        h = DominoHandle(d, d.n + 1, 1)
        h.set_stream(torch.cuda.current_stream().cuda_stream)
        h.set_p_up(plan.p_up)
        h.upload(t_max[None])
        w = StripWalker(None, bounds, rank, 2, halo)
        w.engine = DominoStripEngine(h, w.window)
        walkers.append(w)
    s = 0
    while s < steps:
        k = min(halo, steps - s)
        for w in walkers:
            w.engine.walk(0x5EED, s, k)
        a, b = walkers
        up = a.engine.get_rows(a.hi - halo, halo)
        dn = b.engine.get_rows(b.lo, halo)
        b.engine.set_rows(b.lo - halo, halo, up)
        a.engine.set_rows(a.hi, halo, dn)
        s += k
    full = ts.random_walk_batch(t_max[None], [0x5EED], steps, plan)[0]
    got = np.concatenate([walkers[r].engine.h.download()[0][bounds[r]:bounds[r + 1]] for r in range(2)])
    assert np.array_equal(got, full)


def test_c4_size_walk_windows_vs_oracle():
    """BASELINE config 4's lattice (Aztec order 16384, 1.07e9 vertices) on one
    GPU: after 40 sweeps the whole state is edge-consistent and three row
    bands (top, middle, bottom) equal the oracle's walk of those bands plus a
    40-row margin (one sweep moves information by one row)."""
    import oracle
    from paper_1804_07250_b200.lattice import BIT_DOWN, BIT_LEFT, BIT_RIGHT, BIT_UP, aztec_extremal_states
    from paper_1804_07250_b200.sweeps import DominoHandle

    order, steps = 16384, 40
    d = ts.Domain.aztec(order)
    plan = ts.SweepPlan(d)
    side = d.n + 1
    t_max, _ = aztec_extremal_states(order)
    h = DominoHandle(d, side, 1)
    h.set_plan(plan)
    h.upload(t_max[None])
    h.walk([0x5EED], steps)
    out = h.download()[0]
    del h
    for r0 in range(0, side, 2048):  # every crossed edge is seen from both of its vertices
        blk = out[r0:r0 + 2049]
        assert np.array_equal((blk[:-1] & BIT_DOWN) != 0, (blk[1:] & BIT_UP) != 0)
        assert np.array_equal((blk[:, :-1] & BIT_RIGHT) != 0, (blk[:, 1:] & BIT_LEFT) != 0)
    assert not np.array_equal(out, t_max)
    mid = side // 2
    for a, b in ((0, 64), (mid - 32, mid + 32), (side - 64, side)):
        lo, hi = max(0, a - steps), min(side, b + steps)
        rows = np.ascontiguousarray(t_max[lo:hi])
        oracle.domino_walk_window(rows, lo, 0x5EED, np.full((hi - lo, side), 0.5), steps)
        assert np.array_equal(rows[a - lo:b - lo], out[a:b]), (a, b)


@pytest.mark.parametrize("wpl,pipe", [(1, 0), (2, 0), (2, 1)])
def test_golden_walks_both_tile_widths(monkeypatch, wpl, pipe):
    """Every golden walk case with the multi-sweep tiles forced to 1 and to 2
    words per lane, and with one block per tile or the persistent pipelined
    kernel (the library picks per lattice and launch size; all must be
    exact)."""
    monkeypatch.setenv("TSB_DOM_WPL", str(wpl))
    monkeypatch.setenv("TSB_DOM_PIPE", str(pipe))
    monkeypatch.setenv("TSB_DOM_RESIDENT", "0")  # the tiled kernels, even for the small cases
    g = np.load(os.path.join(G, "domino_walks.npz"))
    i = 0
    while f"c{i}_faces" in g:
        d = ts.Domain(g[f"c{i}_faces"].shape[0], g[f"c{i}_faces"])
        start = g[f"c{i}_start"]
        h = DominoHandle(d, d.n + 1, start.shape[0])
        h.set_p_up(g[f"c{i}_p_up"])
        h.upload(start)
        h.walk(g[f"c{i}_seeds"], int(g[f"c{i}_n_steps"]))
        assert np.array_equal(h.download(), g[f"c{i}_out"]), f"case {i} wpl {wpl}"
        i += 1
    for order, steps in ((200, 333), (700, 130)):
        d = ts.Domain.aztec(order)
        plan = ts.SweepPlan(d)
        t_max, t_min = ts.extremal_tilings(d)
        start = np.stack([t_max.states, t_min.states])
        h = DominoHandle(d, d.n + 1, 2)
        h.set_plan(plan)
        h.upload(start)
        h.walk([5, 6], steps)
        assert np.array_equal(h.download(), oracle.domino_walk(start, [5, 6], plan.p_up, steps)), (order, wpl, pipe)


@pytest.mark.parametrize("mode", ["0", "1"])
def test_resident_and_tiled_paths(monkeypatch, mode):
    """The shared-memory resident walk (one block per chain for the whole
    walk) and the tiled graph/multi-sweep kernels, each forced on every
    golden walk case, the C1 fingerprint and the CFTP goldens (weights of all
    three threshold modes: uniform, parity, per-site grid)."""
    monkeypatch.setenv("TSB_DOM_RESIDENT", mode)
    test_golden_walk_cases()
    test_c1_fingerprint()
    test_cftp_golden()
    d = ts.Domain.aztec(40)
    plan = ts.SweepPlan(d, ts.VolumeWeights(0.7))
    t_max, t_min = ts.extremal_tilings(d)
    start = np.stack([t_max.states, t_min.states] * 10)
    seeds = np.arange(1, 21, dtype=np.uint64)
    out = ts.random_walk_batch(start, seeds, 301, plan)
    assert np.array_equal(out, oracle.domino_walk(start, seeds, plan.p_up, 301))


@pytest.mark.parametrize("mode", ["0", "1"])
@pytest.mark.parametrize("rows,cols", [(1, 2), (2, 2), (2, 3), (4, 31), (3, 32), (2, 64)])
def test_tiny_rectangles_vs_oracle(monkeypatch, mode, rows, cols):
    """Rectangles down to a single domino and widths at 32-column word edges,
    through the resident walk (1) and the tiled kernels (0)."""
    monkeypatch.setenv("TSB_DOM_RESIDENT", mode)
    d = ts.Domain.rectangle(rows, cols)
    plan = ts.SweepPlan(d, ts.VolumeWeights(0.6))
    t_max, t_min = ts.extremal_tilings(d)
    start = np.stack([t_max.states, t_min.states])
    out = ts.random_walk_batch(start, [9, 10], 97, plan)
    assert np.array_equal(out, oracle.domino_walk(start, [9, 10], plan.p_up, 97))


@pytest.mark.parametrize("adapt", ["0", "1"])
def test_adaptive_dispatch_order_is_exact(monkeypatch, adapt):
    """Whole-domain walks long enough for several reorderings of the tile
    dispatch (one per 64-sweep graph replay, by measured block durations)
    equal the oracle, with the adaptive order on and off."""
    monkeypatch.setenv("TSB_DOM_ADAPT", adapt)
    monkeypatch.setenv("TSB_DOM_RESIDENT", "0")
    monkeypatch.setenv("TSB_DOM_WPL", "2")  # the adaptive order serves the 2-word kernel
    d = ts.Domain.aztec(300)
    plan = ts.SweepPlan(d)
    t_max, t_min = ts.extremal_tilings(d)
    start = t_max.states[None]
    out = ts.random_walk_batch(start, [0x5EED], 1000, plan)
    assert np.array_equal(out, oracle.domino_walk(start, [0x5EED], plan.p_up, 1000))


@pytest.mark.parametrize("weights", ["edge", "volume_site"])
def test_adaptive_order_with_per_site_thresholds(monkeypatch, weights):
    """Per-site threshold grids (EdgeWeights; VolumeWeights with face
    overrides) through whole-domain graph replays with the adaptive tile
    order, on a batch of 3 chains (2-word tiles forced: the adaptive order
    serves the one-block-per-tile 2-word kernel)."""
    monkeypatch.setenv("TSB_DOM_RESIDENT", "0")
    monkeypatch.setenv("TSB_DOM_WPL", "2")
    d = ts.Domain.aztec(60)
    if weights == "edge":
        w = ts.EdgeWeights(1.0, {((60, 60), (60, 61)): 3.0, ((30, 50), (31, 50)): 0.25})
    else:
        w = ts.VolumeWeights(0.95, {(60, 60): 3.0, (40, 70): 0.4})
    plan = ts.SweepPlan(d, w)
    t_max, t_min = ts.extremal_tilings(d)
    start = np.stack([t_max.states, t_min.states, t_max.states])
    seeds = np.array([1, 2, 3], dtype=np.uint64)
    out = ts.random_walk_batch(start, seeds, 530, plan)
    assert np.array_equal(out, oracle.domino_walk(start, seeds, plan.p_up, 530))


def test_bench_launch_count_matches_profiler():
    """bench.py's `gpu_launches` claim: the kernels one 1000-sweep walk of the
    headline workload launches (set_walk, 15 graph replays of 32 multi-sweep
    kernels + the replay tail, 20 remainder multi-sweep kernels), counted by
    the CUDA profiler (CUPTI activity records include graph kernel nodes)."""
    import sys

    import torch
    from torch.profiler import ProfilerActivity, profile

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench
    from paper_1804_07250_b200.lattice import aztec_extremal_states

    order = 4096  # bench.py's workload: whole-domain tiles with the adaptive order
    d = ts.Domain.aztec(order)
    h = DominoHandle(d, d.n + 1, 1)
    h.set_collapse(False)
    h.set_plan(ts.SweepPlan(d))
    h.upload(aztec_extremal_states(order)[0][None])
    h.walk([5], 1000)  # graphs captured outside the profiled walk
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        h.walk([5], 1000, step0=1000)
        h.sync()
        torch.cuda.synchronize()
    names = [e.name for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    ours = [n for n in names if "tsb::" in n or "domino" in n or "replay_tail" in n or "set_walk" in n]
    assert len(ours) == bench.launches_per_walk(1000), collections_summary(ours)


def collections_summary(names):
    import collections

    return dict(collections.Counter(n.split("(")[0] for n in names))
