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
