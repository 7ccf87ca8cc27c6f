"""Host side of the archive format against the reference's own dumps."""

import io
import os

import numpy as np

import paper_1804_07250_b200 as ts
from paper_1804_07250_b200.archive import SampleArchive
from paper_1804_07250_b200.lozenge import LozengeTiling

G = os.path.join(os.path.dirname(__file__), "golden")


def _cases():
    g = np.load(os.path.join(G, "archives.npz"))
    d = ts.Domain.aztec(12)
    n = 8
    dom = ts.TriDomain.hexagon(3, 4, 5)
    return {
        "domino": (d, [ts.Tiling(d, s) for s in g["dom_states"]]),
        "sixvertex": (ts.dwbc(n), [ts.config_from_heights(ts.FaceHeights(n, h)) for h in g["sv_heights"]]),
        "lozenge": (dom, [LozengeTiling(dom, e) for e in g["loz_edges"]]),
    }


def test_host_dump_and_load_match_reference():
    for model, (domain, states) in _cases().items():
        ref = open(os.path.join(G, f"archive_{model}.txt")).read()
        arc = SampleArchive.create(model, domain, "uniform", 0x5EED, "sequential", "mcmc steps=60")
        arc.extend(states)
        buf = io.StringIO()
        arc.dump(buf)
        assert buf.getvalue() == ref, model
        back = SampleArchive.load(io.StringIO(ref), domain)
        assert back.header == arc.header and back.records == states, model


def test_host_statistics_match_reference_goldens():
    """density_map / domino_orientation_grid / aztec_y_intercept /
    c_vertex_count host mirrors vs the reference's outputs."""
    g = np.load(os.path.join(G, "observables.npz"))
    d = ts.Domain.aztec(32)
    arc = SampleArchive("domino", {}, [ts.Tiling(d, s) for s in g["dom_states"]])
    assert np.array_equal(ts.domino_orientation_grid(arc.records[0]), g["dom_orient0"], equal_nan=True)
    assert np.allclose(ts.density_map(arc, "domino-orientation").grid, g["dom_density"], equal_nan=True, rtol=0,
                       atol=1e-15)
    assert [ts.aztec_y_intercept(t) for t in arc.records] == list(g["dom_yint"])
    n = g["sv_heights"].shape[1] - 1
    cfgs = [ts.config_from_heights(ts.FaceHeights(n, h)) for h in g["sv_heights"]]
    sv = SampleArchive("sixvertex", {}, cfgs)
    for name in ("h-edge", "v-edge", "c-vertex"):
        assert np.array_equal(ts.density_map(sv, name).grid, g["sv_" + name.replace("-", "_")]), name
    assert [ts.c_vertex_count(c) for c in cfgs] == list(g["sv_ccount"])
    h = ts.scalar_observable(sv, "c-vertex-count")
    assert h.samples == len(cfgs) and np.isclose((h.density * np.diff(h.edges)).sum(), 1.0)
    res = ts.chi_square_gof([10, 12, 9, 11])
    assert res.dof == 3 and res.passed
    assert ts.total_variation({1: 0.5, 2: 0.5}, {1: 1.0}) == 0.5
