"""Archive records formatted on the device (csrc/archive.cu, tsb_*_serialize)
are byte-identical to the reference's SampleArchive.dump."""

import os

import numpy as np
import pytest

import paper_1804_07250_b200 as ts
from paper_1804_07250_b200.archive import ArchiveWriter, device_record, serialize_state
from paper_1804_07250_b200.lozenge import LozengeHandle, LozengeTiling, loz_p_up_grid
from paper_1804_07250_b200.sixvertex import SixVertexHandle
from paper_1804_07250_b200.sweeps import DominoHandle

pytestmark = pytest.mark.gpu
G = os.path.join(os.path.dirname(__file__), "golden")


def test_writer_matches_reference_dumps(tmp_path):
    g = np.load(os.path.join(G, "archives.npz"))
    d = ts.Domain.aztec(12)
    hd = DominoHandle(d, d.n + 1, 3)
    hd.upload(g["dom_states"])
    hs = SixVertexHandle(8, 3)
    hs.upload(g["sv_heights"])
    dom = ts.TriDomain.hexagon(3, 4, 5)
    hl = LozengeHandle(dom, 3)
    hl.upload(g["loz_edges"])
    for model, domain, h in (("domino", d, hd), ("sixvertex", ts.dwbc(8), hs), ("lozenge", dom, hl)):
        path = tmp_path / f"{model}.txt"
        with ArchiveWriter(str(path), model, domain, "uniform", 0x5EED, "sequential", "mcmc steps=60") as w:
            w.add(h)
        assert path.read_text() == open(os.path.join(G, f"archive_{model}.txt")).read(), model


def test_device_records_of_walked_chains():
    """Larger mixed states (two-digit tilestates included) vs the host format."""
    d = ts.Domain.aztec(150)
    plan = ts.SweepPlan(d)
    t_max, _ = ts.extremal_tilings(d)
    h = DominoHandle(d, d.n + 1, 2)
    h.set_plan(plan)
    h.upload(np.stack([t_max.states] * 2))
    h.walk([3, 4], 3000)
    st = h.download()
    assert (st >= 10).any()
    for c in range(2):
        assert device_record(h, c) == serialize_state(ts.Tiling(d, st[c]))
    n = 90
    R, C = np.meshgrid(np.arange(n + 1), np.arange(n + 1), indexing="ij")
    lo = np.maximum(-(R + C), R + C - 2 * n).astype(np.int32)
    hs = SixVertexHandle(n, 1)
    hs.set_weights(ts.SVWeights(1.0, 1.0, 1.1))
    hs.upload(lo[None])
    hs.walk([5], 500)
    cfg = ts.config_from_heights(ts.FaceHeights(n, hs.download()[0]))
    assert device_record(hs, 0) == serialize_state(cfg)
    dom = ts.TriDomain.hexagon(20, 30, 25)
    t_max_l, _ = ts.loz_extremal(dom)
    hl = LozengeHandle(dom, 1)
    hl.set_p_up(loz_p_up_grid(dom, ts.Uniform()))
    hl.upload(t_max_l.edges[None])
    hl.walk([6], 400)
    assert device_record(hl, 0) == serialize_state(LozengeTiling(dom, hl.download()[0]))
