"""Bit-exact parity at the BASELINE configs' own sizes and sweep counts.

The fingerprints in tests/golden/configs/*.json were produced by running the
UNMODIFIED reference in the dev container (tests/golden/make_golden_configs.py);
here the device recomputes the same arrays and compares sha256[:16].

* C2  lozenge hexagon 1000^3, VolumeWeights(0.999), from loz_extremal's T_min,
      10^4 sweeps (lozenge.py:600-622, extremal lozenge.py:762-775)
* C3  six-vertex DWBC 2048 from h_min, (1,1,1) and (1,1,sqrt 8), 10^4 sweeps
      (sixvertex.py:445-467)
* M   Aztec 4096 (the metric lattice) from T_max, 1000 sweeps (+ heights)
* C4  Aztec 16384 from T_max, 100 sweeps, on one GPU and strip-sharded over
      2 / 4 / 8 device-exchanging windows (_kernels.py:35-69)
* C5  CFTP on Aztec 512: top and bottom chains after each of the first 13
      rounds of samples 0 and 1 (cftp.py:86-139), read through the progress
      hook of tsb_domino_cftp.
"""

import hashlib
import json
import math
import os

import numpy as np
import pytest

import paper_1804_07250_b200 as ts
from paper_1804_07250_b200.cftp import chain_master_seed
from paper_1804_07250_b200.lattice import aztec_extremal_states

pytestmark = pytest.mark.gpu
G = os.path.join(os.path.dirname(__file__), "golden", "configs")
SEED = 0x5EED


def golden(name):
    with open(os.path.join(G, name + ".json")) as f:
        return json.load(f)


def fp(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


# ------------------------------------------------------------------- C2
def test_c2_lozenge_hexagon_1000():
    from paper_1804_07250_b200.lozenge import loz_random_walk_batch

    g = golden("c2")
    d = ts.TriDomain.hexagon(1000, 1000, 1000)
    t_max, t_min = ts.loz_extremal(d)
    assert fp(t_max.edges) == g["t_max"] and fp(t_min.edges) == g["t_min"]
    assert fp(ts.loz_heights(t_max).heights) == g["h_max"]
    assert fp(ts.loz_heights(t_min).heights) == g["h_min"]
    w = ts.VolumeWeights(g["q"])
    for n in (100, 10000):
        out = loz_random_walk_batch(t_min.edges[None], [SEED], n, d, w)[0]
        assert fp(out) == g[f"walk_{n}"], n
    assert fp(ts.loz_heights(ts.LozengeTiling(d, out)).heights) == g["heights_10000"]


# ------------------------------------------------------------------- C3
def sv_hmin(n):
    r = np.arange(n + 1)
    s = r[:, None] + r[None, :]
    return np.maximum(-s, s - 2 * n).astype(np.int32)


@pytest.mark.parametrize("name", ["c3_half", "c3_afe"])
def test_c3_sixvertex_dwbc_2048(name):
    from paper_1804_07250_b200.sixvertex import sv_random_walk_batch

    g = golden(name)
    n = g["n"]
    hi, lo = ts.sv_extremal(n, ts.dwbc(n))
    assert fp(lo.heights) == g["h_min"]
    assert np.array_equal(lo.heights, sv_hmin(n))
    w = ts.SVWeights(*g["weights"])
    for k in (100, 10000):
        out = sv_random_walk_batch(lo.heights[None], [SEED], k, w)[0]
        assert int(out.astype(np.int64).sum()) == g[f"sum_{k}"], k
        assert fp(out) == g[f"walk_{k}"], k


# -------------------------------------------------------------- metric M
def test_metric_aztec_4096():
    import oracle

    g = golden("m4096")
    d = ts.Domain.aztec(4096)
    plan = ts.SweepPlan(d)
    t_max, _ = aztec_extremal_states(4096)
    assert fp(t_max) == g["t_max"]
    for n in (7, 1000):
        t = ts.random_walk(ts.Tiling(d, t_max), SEED, n, plan)
        assert fp(t.states) == g[f"walk_{n}"], n
        assert int(((t.states == 3) | (t.states == 12)).sum()) == g[f"rotateable_{n}"]
    assert fp(ts.height_function(t).heights) == g["heights_1000"]
    # and the pinned oracle agrees at this size (16 host threads, ~5 s)
    ref = oracle.domino_walk(t_max[None], [SEED], plan.p_up, 1000, threads=os.cpu_count() or 1)[0]
    assert np.array_equal(ref, t.states)


# ------------------------------------------------------------------- C4
@pytest.fixture(scope="module")
def c4():
    g = golden("c4")
    d = ts.Domain.aztec(16384)
    t_max, _ = aztec_extremal_states(16384)
    assert fp(t_max) == g["t_max"]
    return g, d, t_max


def _bands(states):
    v = states.shape[0]
    cuts = np.linspace(0, v, 9).astype(int)
    return [fp(states[a:b]) for a, b in zip(cuts[:-1], cuts[1:])]


def test_c4_aztec_16384_one_gpu(c4):
    g, d, t_max = c4
    t = ts.random_walk(ts.Tiling(d, t_max), SEED, 100, ts.SweepPlan(d))
    assert _bands(t.states) == g["bands_100"]
    assert fp(t.states) == g["walk_100"]


@pytest.mark.parametrize("world,halo", [(2, 64), (4, 32), (8, 64)])
def test_c4_aztec_16384_strips(c4, world, halo):
    """One chain strip-sharded over `world` windows with the device push/pull
    exchange (csrc/strips.cu), host lockstep on one GPU: the concatenated
    strips equal the reference's single-chain walk."""
    from paper_1804_07250_b200.strips import DeviceStripWalker, strip_bounds
    from paper_1804_07250_b200.sweeps import DominoHandle

    g, d, t_max = c4
    plan = ts.SweepPlan(d)
    hs = []
    for _ in range(world):
        h = DominoHandle(d, d.n + 1, 1, device=0)
        h.set_plan(plan)
        h.upload(t_max[None])
        hs.append(h)
    ws = DeviceStripWalker.local(hs, strip_bounds(d.vertex_mask, world, min_rows=halo), halo)
    DeviceStripWalker.walk_lockstep(ws, SEED, 100)
    got = np.empty_like(t_max)
    for w in ws:
        got[w.lo:w.hi] = w.handle.download()[0][w.lo:w.hi]
        w.close()
    del hs, ws
    assert _bands(got) == g["bands_100"]
    assert fp(got) == g["walk_100"]


@pytest.mark.parametrize("world,halo", [(2, 64), (8, 64)])
def test_c4_aztec_16384_memory_sharded_strips(c4, world, halo):
    """C4 with memory-sharded strips: each window handle holds only its strip
    plus halo (tsb_domino_create_window), uploaded and read back by rows."""
    from paper_1804_07250_b200.strips import DeviceStripWalker, strip_bounds
    from paper_1804_07250_b200.sweeps import DominoHandle

    g, d, t_max = c4
    plan = ts.SweepPlan(d)
    bounds = strip_bounds(d.vertex_mask, world, min_rows=halo)
    hs = []
    for r in range(world):
        a, b = max(0, bounds[r] - halo), min(d.n + 1, bounds[r + 1] + halo)
        h = DominoHandle.window(d, a, b, device=0)
        h.set_plan(plan)
        h.upload_rows(a, t_max[a:b])
        hs.append(h)
    ws = DeviceStripWalker.local(hs, bounds, halo)
    DeviceStripWalker.walk_lockstep(ws, SEED, 100)
    got = np.empty_like(t_max)
    for w in ws:
        got[w.lo:w.hi] = w.handle.download_rows(w.lo, w.hi - w.lo)
        w.close()
    del hs, ws
    assert _bands(got) == g["bands_100"]
    assert fp(got) == g["walk_100"]


# ------------------------------------------------------------------- C5
def test_c5_cftp_aztec_512_early_rounds():
    """The device CFTP driver's top/bottom chains after rounds 1..13 equal the
    reference's round replays (run_cftp_batch's loop, cftp.py:111-120) for
    samples 0 and 1 of master 0x5EED."""
    from paper_1804_07250_b200.sweeps import DominoCftp

    g = golden("c5")
    rounds = len(g["chains"][0]["top"])
    d = ts.Domain.aztec(512)
    plan = ts.SweepPlan(d)
    t_max, t_min = aztec_extremal_states(512)
    assert fp(t_max) == g["t_max"] and fp(t_min) == g["t_min"]
    masters = np.array([chain_master_seed(SEED, k) for k in (0, 1)], dtype=np.uint64)
    assert [int(m) for m in masters] == [c["master"] for c in g["chains"]]
    run = DominoCftp(d, plan, t_max, t_min, 2)
    seen = []

    def progress(round_no, steps, collapsed, total):
        # hook: at the end of a round chains 2j / 2j+1 hold sample j's top / bottom
        st = run.handle.download(0, 4)
        seen.append([fp(st[0]), fp(st[1]), fp(st[2]), fp(st[3])])

    with pytest.raises(ts.ConvergenceCapExceeded):
        run.run(masters, rounds, progress=progress)
    assert len(seen) == rounds
    for r in range(rounds):
        for k in (0, 1):
            c = g["chains"][k]
            assert seen[r][2 * k] == c["top"][r], (r, k, "top")
            assert seen[r][2 * k + 1] == c["bot"][r], (r, k, "bot")
