"""Pin the CPU oracle (oracle/tsb_oracle.c) to the reference's own outputs.

The golden fixtures were produced by running the unmodified reference
(tests/golden/make_golden.py).  Everything here runs on CPU.
"""

import hashlib
import json
import os

import numpy as np
import pytest

import oracle

G = os.path.join(os.path.dirname(__file__), "golden")


def load(name):
    return np.load(os.path.join(G, name))


def fp(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


def test_rng_kats():
    kats = json.load(open(os.path.join(G, "rng_kats.json")))
    for k in kats["kats"]:
        key = oracle.site_key(k["seed"], k["shape"], k["site"])
        assert key == k["key"]
        assert oracle.lib().orc_splitmix_at(key, k["step"]) == k["x"]
        assert oracle.uniform_from_key(key, k["step"]).hex() == k["u"]
        gkey = oracle.site_key(k["seed"], k["shape"], (0, 0), tag=1)
        assert oracle.uniform_from_key(gkey, k["step"]).hex() == k["global_u"]
    for d in kats["derive"]:
        assert oracle.derive_seed(d["seed"], d["index"], d["salt"]) == d["out"]
    for c in kats["chains"]:
        chain = oracle.derive_seed(c["master"], c["k"], 2)
        assert chain == c["chain"]
        assert oracle.derive_seed(chain, 1, 0x51ED2701) == c["round1"]


def test_rng_appendix_b():
    # SURVEY.md Appendix B (computed by the reference)
    assert oracle.site_key(0x5EED, (129, 129), (64, 64)) == 0xD717FD28C0741425
    assert oracle.lib().orc_splitmix_at(0xD717FD28C0741425, 0) == 0x1A47E55D561E7D93
    assert oracle.derive_seed(0x5EED, 0, 2) == 0x9F8F55FFA30E6838


def test_uniform_grids():
    g = load("rng_grids.npz")
    for name in g.files:
        seed, r, c, step = (int(x) for x in name.split("_"))
        assert np.array_equal(oracle.uniform_grid(seed, (r, c), step), g[name])


def test_domino_c1_fingerprint():
    g = load("domino_c1.npz")
    v = g["t_max"].shape[0]
    p = np.full((v, v), 0.5)
    out = oracle.domino_walk(g["t_max"], [0x5EED], p, 1000)[0]
    assert fp(out) == "fe33268e95b1a840"
    assert np.array_equal(out, g["final"])
    # threaded row bands are bit-identical
    out4 = oracle.domino_walk(g["t_max"], [0x5EED], p, 1000, threads=4)[0]
    assert np.array_equal(out4, g["final"])


def test_domino_walk_cases():
    g = load("domino_walks.npz")
    i = 0
    while f"c{i}_out" in g.files:
        out = oracle.domino_walk(g[f"c{i}_start"], g[f"c{i}_seeds"], g[f"c{i}_p_up"],
                                 int(g[f"c{i}_n_steps"]))
        assert np.array_equal(out, g[f"c{i}_out"]), f"case {i}"
        # split walk == one walk (step counter continuation)
        n = int(g[f"c{i}_n_steps"])
        a = oracle.domino_walk(g[f"c{i}_start"], g[f"c{i}_seeds"], g[f"c{i}_p_up"], n // 3)
        b = oracle.domino_walk(a, g[f"c{i}_seeds"], g[f"c{i}_p_up"], n - n // 3, step0=n // 3)
        assert np.array_equal(b, g[f"c{i}_out"])
        i += 1
    assert i >= 5


def test_sixvertex_cases():
    g = load("sixvertex.npz")
    import golden_cases as gc
    for i, (n, w, seed, steps, _) in enumerate(gc.SV_CASES):
        out = oracle.sv_walk(g[f"v{i}_start"], [seed], g[f"v{i}_table"], steps)[0]
        assert np.array_equal(out, g[f"v{i}_out"]), f"sv case {i}"


def test_lozenge_cases():
    g = load("lozenge.npz")
    i = 0
    import golden_cases as gc
    seeds = [0x5EED, 31337, 8]
    steps = [500, 200, 150]
    while f"l{i}_out" in g.files:
        out = oracle.loz_walk(g[f"l{i}_start"], [seeds[i]], g[f"l{i}_p_up"], steps[i])[0]
        assert np.array_equal(out, g[f"l{i}_out"]), f"loz case {i}"
        i += 1
    assert i == 3


def test_oracle_observables_match_reference():
    """The oracle's restated statistics equal the reference's stats.py outputs."""
    import paper_1804_07250_b200 as ts

    g = np.load(os.path.join(G, "observables.npz"))
    d = ts.Domain.aztec(32)
    grids = [oracle.domino_orientation(s, d.faces) for s in g["dom_states"]]
    assert np.array_equal(grids[0], g["dom_orient0"], equal_nan=True)
    assert np.allclose(np.mean(grids, axis=0), g["dom_density"], equal_nan=True, rtol=0, atol=1e-15)
    assert [oracle.aztec_y_intercept(x) for x in grids] == list(g["dom_yint"])
    he, ve, cv = zip(*[(*oracle.sv_edges(h), None) for h in g["sv_heights"]])
    cv = [oracle.sv_c_vertex(a, b) for a, b in zip(he, ve)]
    assert np.array_equal(np.mean(he, axis=0), g["sv_h_edge"])
    assert np.array_equal(np.mean(ve, axis=0), g["sv_v_edge"])
    assert np.array_equal(np.mean(cv, axis=0), g["sv_c_vertex"])
    assert [int(c.sum()) for c in cv] == list(g["sv_ccount"])


def test_sixvertex_general_boundaries():
    """The oracle's six-vertex walk on the reference's non-DWBC golden walks
    (make_golden.py make_sv_boundaries): the sweep does not depend on DWBC."""
    import json

    import paper_1804_07250_b200 as ts

    g = load("sv_boundaries.npz")
    with open(os.path.join(G, "sv_boundaries.json")) as f:
        meta = json.load(f)
    table = ts.SVWeights(*meta["weights"]).table()
    k = 0
    for i, m in enumerate(meta["cases"]):
        if m["error"]:
            continue
        start = np.stack([g[f"b{i}_hi"], g[f"b{i}_lo"]])
        out = oracle.sv_walk(start, [7 + i, 7 + i], table, meta["walk_steps"])
        assert np.array_equal(out, g[f"b{i}_walk"]), i
        k += 1
    assert k >= 20
