"""Six-vertex parity on the device vs the reference's golden outputs and the
C oracle (bit-exact integer heights)."""

import math
import os

import numpy as np
import pytest

import golden_cases as gc
import oracle
import paper_1804_07250_b200 as ts
from paper_1804_07250_b200.sixvertex import SixVertexHandle, p_high_lut, sv_random_walk_batch

pytestmark = pytest.mark.gpu
G = os.path.join(os.path.dirname(__file__), "golden")


def load(name):
    return np.load(os.path.join(G, name))


def closed_form(n):
    R, C = np.meshgrid(np.arange(n + 1), np.arange(n + 1), indexing="ij")
    return -np.abs(R - C), np.maximum(-(R + C), R + C - 2 * n)


def test_golden_walks():
    g = load("sixvertex.npz")
    for i, (n, w, seed, steps, _) in enumerate(gc.SV_CASES):
        out = sv_random_walk_batch(g[f"v{i}_start"][None], [seed], steps, ts.SVWeights(*w))
        assert np.array_equal(out[0], g[f"v{i}_out"]), f"sv case {i}"


def test_golden_extremal():
    g = load("sixvertex.npz")
    for n in gc.SV_EXTREMAL_N:
        hi, lo = ts.sv_extremal(n, ts.dwbc(n))
        assert np.array_equal(hi.heights, g[f"e{n}_hi"]) and np.array_equal(lo.heights, g[f"e{n}_lo"])


@pytest.mark.parametrize("n", [64, 300, 2048])
def test_extremal_closed_form(n):
    hi, lo = ts.sv_extremal(n, ts.dwbc(n))
    chi, clo = closed_form(n)
    assert np.array_equal(hi.heights, chi) and np.array_equal(lo.heights, clo)


@pytest.mark.parametrize("n,w,steps", [(200, (1.0, 1.0, 1.0), 400), (257, (1.0, 1.0, math.sqrt(8.0)), 333),
                                       (97, (0.6, 1.4, 2.0), 500)])
def test_walk_vs_oracle(n, w, steps):
    hi, lo = closed_form(n)
    start = np.stack([lo, hi, lo]).astype(np.int32)
    seeds = np.array([1, 2, 2**63 + 3], dtype=np.uint64)
    weights = ts.SVWeights(*w)
    out = sv_random_walk_batch(start, seeds, steps, weights)
    ref = oracle.sv_walk(start, seeds, weights.table(), steps)
    assert np.array_equal(out, ref)
    # continuation: split walks equal one walk
    h = SixVertexHandle(n, 3)
    h.set_weights(weights)
    h.upload(start)
    h.walk(seeds, steps // 2)
    h.walk(seeds, steps - steps // 2, step0=steps // 2)
    assert np.array_equal(h.download(), ref)


def test_sweep_and_errors():
    n = 6
    hi, lo = ts.sv_extremal(n, ts.dwbc(n))
    cfg = ts.config_from_heights(lo)
    fam = ts.seed_family(5, (n + 1, n + 1))
    for k in range(4):
        out = ts.sv_sweep(cfg, fam, 3, k, ts.SVWeights())
        ts.heights_from_config(out)  # valid configuration
    bad = lo.heights.copy()
    bad[3, 3] += 5
    with pytest.raises(ts.InconsistencyError):
        sv_random_walk_batch(bad[None], [1], 1, ts.SVWeights())
    with pytest.raises(ts.NonMonotoneWeights):
        ts.sv_cftp(3, ts.dwbc(3), ts.SVWeights(2.0, 1.0, 1.0), 1)


def test_cftp_golden():
    g = load("sixvertex.npz")
    for j, (n, w, master, count) in enumerate(gc.SV_CFTP_CASES):
        trace = ts.CftpTrace()
        res = ts.sv_cftp(n, ts.dwbc(n), ts.SVWeights(*w), master, count=count, trace=trace)
        res = res if isinstance(res, list) else [res]
        hs = np.stack([ts.heights_from_config(c).heights for c in res])
        assert np.array_equal(hs, g[f"k{j}_h"]), f"cftp {j}"
        assert trace.collapsed_at == int(g[f"k{j}_collapsed"])


def test_sweep_stays_monotone_coupled():
    """Grand coupling: the walk from h_max stays above the walk from h_min."""
    n = 40
    hi, lo = closed_form(n)
    out = sv_random_walk_batch(np.stack([hi, lo]).astype(np.int32), [9, 9], 300, ts.SVWeights(1, 1, 1.5))
    assert (out[0] >= out[1]).all()


@pytest.mark.parametrize("n,steps", [(1100, 70), (2048, 40), (3500, 36), (4200, 34)])
def test_multi_tile_geometries(n, steps):
    """Temporally blocked graph replays at every tile width (1..4 words per
    lane, and the word-halo tiling beyond 128 words per row) vs the oracle."""
    hi, lo = closed_form(n)
    start = np.stack([lo, hi]).astype(np.int32)
    seeds = np.array([0x5EED, 77], dtype=np.uint64)
    weights = ts.SVWeights(1.0, 1.0, math.sqrt(8.0))
    h = SixVertexHandle(n, 2)
    h.set_weights(weights)
    h.upload(start)
    # a warm-up that leaves the state mixed near the corners, then the test walk
    h.walk(seeds, steps)
    mid = h.download()
    ref_mid = oracle.sv_walk(start, seeds, weights.table(), steps)
    assert np.array_equal(mid, ref_mid)


@pytest.mark.parametrize("K,NW,WPL,n", [(2, 8, 0, 300), (4, 8, 0, 300), (8, 16, 0, 300), (16, 16, 0, 300),
                                        (4, 16, 0, 300), (8, 16, 1, 300), (8, 16, 1, 1500), (4, 8, 2, 1500),
                                        (8, 16, 3, 1500)])
def test_multi_k_nw(monkeypatch, K, NW, WPL, n):
    """Every sweeps-per-launch / block-height / tile-width setting is bit-identical."""
    monkeypatch.setenv("TSB_SV_K", str(K))
    monkeypatch.setenv("TSB_SV_NW", str(NW))
    monkeypatch.setenv("TSB_SV_WPL", str(WPL))
    steps = 150 if n < 1000 else 70
    hi, lo = closed_form(n)
    start = np.stack([lo, hi, lo]).astype(np.int32)
    seeds = np.array([5, 6, 2**64 - 1], dtype=np.uint64)
    weights = ts.SVWeights(0.7, 1.2, 1.5)
    h = SixVertexHandle(n, 3)
    h.set_weights(weights)
    h.upload(start)
    h.walk(seeds, 70)
    h.walk(seeds, steps - 70, step0=70)
    assert np.array_equal(h.download(), oracle.sv_walk(start, seeds, weights.table(), steps))


def test_large_batch_uses_batch_geometry():
    """40 chains: the per-batch sweeps-per-launch choice (K = 4 once the batch
    fills two waves) is bit-identical to the oracle."""
    n, steps, B = 300, 150, 40
    hi, lo = closed_form(n)
    start = np.stack([lo if k % 2 else hi for k in range(B)]).astype(np.int32)
    seeds = np.arange(1000, 1000 + B, dtype=np.uint64)
    w = ts.SVWeights(1.0, 1.0, 1.25)
    h = SixVertexHandle(n, B)
    h.set_weights(w)
    h.upload(start)
    h.walk(seeds, steps)
    assert np.array_equal(h.download(), oracle.sv_walk(start, seeds, w.table(), steps))


@pytest.mark.parametrize("n", [1, 2, 3, 5, 31, 32, 33])
def test_tiny_and_word_edge_sizes_vs_oracle(n):
    """DWBC sizes with no interior face (n = 1), a single one, and face grids
    one word wide or straddling a word boundary (32 / 33 / 34 columns)."""
    hi, lo = closed_form(n)
    start = np.stack([lo, hi]).astype(np.int32)
    seeds = np.array([3, 4], dtype=np.uint64)
    w = ts.SVWeights(0.8, 1.1, 1.7)
    out = sv_random_walk_batch(start, seeds, 150, w)
    assert np.array_equal(out, oracle.sv_walk(start, seeds, w.table(), 150))
    if n == 1:
        assert np.array_equal(out, start)


def test_general_boundaries_golden():
    """Non-DWBC boundaries (sixvertex.py:83-120) through the device
    sv_extremal (534-562): extremal heights, both InfeasibleBoundary paths
    (ring not closing, 527; mutually incompatible ring, 557) with the
    reference's messages, walks from h_max / h_min and sv_cftp -- all against
    reference-generated goldens (make_golden.py make_sv_boundaries)."""
    import json

    from paper_1804_07250_b200.sixvertex import sv_random_walk_batch

    g = load("sv_boundaries.npz")
    with open(os.path.join(G, "sv_boundaries.json")) as f:
        meta = json.load(f)
    w = ts.SVWeights(*meta["weights"])
    bounds = []
    for i, m in enumerate(meta["cases"]):
        b = ts.Boundary(m["n"], *(g[f"b{i}_{k}"] for k in ("top", "bottom", "left", "right")))
        bounds.append(b)
        if m["error"]:
            with pytest.raises(ts.InfeasibleBoundary, match=m["message"]):
                ts.sv_extremal(b.n, b)
            continue
        hi, lo = ts.sv_extremal(b.n, b)
        assert np.array_equal(hi.heights, g[f"b{i}_hi"]), i
        assert np.array_equal(lo.heights, g[f"b{i}_lo"]), i
        start = np.stack([hi.heights, lo.heights])
        out = sv_random_walk_batch(start, np.array([7 + i, 7 + i], dtype=np.uint64), meta["walk_steps"], w)
        assert np.array_equal(out, g[f"b{i}_walk"]), i
    assert sum(m["error"] is None for m in meta["cases"]) >= 20
    assert {m.get("message") for m in meta["cases"]} >= {"boundary ring heights do not close up",
                                                         "ring heights are mutually incompatible"}
    for j, c in enumerate(meta["cftp"]):
        b = bounds[c["case"]]
        trace = ts.CftpTrace()
        res = ts.sv_cftp(b.n, b, w, c["master"], count=3, trace=trace)
        assert np.array_equal(np.stack([ts.heights_from_config(x).heights for x in res]), g[f"c{j}_h"]), j
        assert trace.collapsed_at == c["collapsed_at"]


@pytest.mark.parametrize("n,chains,steps", [(1024, 2, 60), (3072, 2, 36), (4096, 1, 30), (1024, 16, 40)])
def test_east_boundary_word_tiles(n, chains, steps):
    """n a multiple of 1024: rows of 32*WPL words plus the read-only east
    boundary word (WPL = 1, 3, 4; 16 chains take the 2-blocks-per-SM build)
    are bit-identical to the oracle."""
    hi, lo = closed_form(n)
    start = np.stack([lo if k % 2 == 0 else hi for k in range(chains)]).astype(np.int32)
    seeds = np.arange(31, 31 + chains, dtype=np.uint64)
    w = ts.SVWeights(1.0, 1.0, 1.0)
    h = SixVertexHandle(n, chains)
    h.set_weights(w)
    h.upload(start)
    h.walk(seeds, steps)
    out = h.download()
    assert np.array_equal(out, oracle.sv_walk(start, seeds, w.table(), steps))
