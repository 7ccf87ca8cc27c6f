"""Error behaviour of the host-side API on CPU: each case raises the same
exception class the reference raises for it (tests of the reference:
test_lattice.py, test_rng.py, test_sixvertex.py, test_lozenge.py,
test_cftp.py, test_harness.py; classes from errors.py:4-69).  None of these
paths touches the device."""

import numpy as np
import pytest

import paper_1804_07250_b200 as ts
from paper_1804_07250_b200 import rng, stats
from paper_1804_07250_b200.lozenge import is_valid_lozenge_tiling
from paper_1804_07250_b200.sixvertex import flippable


@pytest.fixture
def square2():
    return ts.Domain.square(2)


def _brick(d, horizontal=True):
    """Brick tiling of a 2 x 2k domain from its domino list."""
    n = d.n
    if horizontal:
        return ts.tiling_from_dominoes(d, [((r, c), (r, c + 1)) for r in range(n) for c in range(0, n, 2)])
    return ts.tiling_from_dominoes(d, [((r, c), (r + 1, c)) for r in range(0, n, 2) for c in range(n)])


def test_domino_codec_errors(square2):
    # lattice.py:407-429 -- a face covered twice, a face left over, a face
    # outside the domain, two faces that do not share an edge
    with pytest.raises(ts.OverlapError):
        ts.tiling_from_dominoes(square2, [((0, 0), (0, 1)), ((0, 1), (1, 1))])
    with pytest.raises(ts.CoverageError):
        ts.tiling_from_dominoes(square2, [((1, 0), (1, 1))])
    with pytest.raises(ts.OutOfDomainError):
        ts.tiling_from_dominoes(square2, [((0, 0), (0, 1)), ((1, 1), (1, 2))])
    with pytest.raises(ts.OutOfDomainError):
        ts.tiling_from_dominoes(square2, [((0, 0), (1, 1)), ((0, 1), (1, 0))])
    assert ts.dominoes_from_tiling(_brick(square2)) == [((0, 0), (0, 1)), ((1, 0), (1, 1))]


def test_inconsistent_state_grid_raises(square2):
    grid = np.zeros((3, 3), dtype=np.uint8)
    grid[2, 1] = 12  # a vertex claims two crossings no neighbour mirrors
    with pytest.raises(ts.InconsistencyError):
        ts.dominoes_from_tiling(ts.Tiling(square2, grid))


def test_weights_reject_nonpositive():
    for bad in (0.0, -2.0):
        with pytest.raises(ValueError):
            ts.VolumeWeights(bad)
    with pytest.raises(ValueError):
        ts.EdgeWeights(1.0, {((1, 1), (1, 2)): 0.0})


def test_order_compare_domain_mismatch(square2):
    a = ts.HeightFunction(square2, np.zeros((3, 3), np.int32))
    b = ts.HeightFunction(ts.Domain.square(4), np.zeros((5, 5), np.int32))
    with pytest.raises(ts.DomainMismatchError):
        ts.order_compare(a, b)


def test_stream_family_capacity_and_bounds():
    # rng.py:77-80 (capacity 2^48 sites) and the per-site grid check
    with pytest.raises(ts.CapacityError):
        rng.seed_family(3, (1 << 24, 1 << 25))
    fam = rng.seed_family(3, (4, 5))
    with pytest.raises(ts.OutOfGridError):
        fam.uniform((0, 5), 1)
    with pytest.raises(ts.OutOfGridError):
        fam.uniform((-1, 0), 1)
    assert rng.uniform(fam, (3, 4), 9) == fam.uniform((3, 4), 9)


def test_sixvertex_config_errors():
    # ice rule at a vertex (sixvertex.py:236-239) and single-valued heights
    # (sixvertex.py:247-277)
    h = np.zeros((1, 2), dtype=bool)
    v = np.zeros((2, 1), dtype=bool)
    v[0, 0] = True  # a lone north edge
    with pytest.raises(ts.IceRuleViolation):
        ts.vertex_type(ts.SixVertexConfig(1, h, v), (0, 0))
    h = np.zeros((3, 4), dtype=bool)
    v = np.zeros((4, 3), dtype=bool)
    v[1, 1] = True
    with pytest.raises(ts.InconsistencyError):
        ts.heights_from_config(ts.SixVertexConfig(3, h, v))


def test_flippable_rejects_boundary_faces():
    n = 3
    heights = np.add.outer(np.arange(n + 1), np.arange(n + 1)).astype(np.int32)  # h = r + c
    fh = ts.FaceHeights(n, heights)
    for face in ((0, 1), (1, 0), (n, 2), (2, n)):
        with pytest.raises(ts.BoundaryFaceError):
            flippable(fh, face)
    assert flippable(fh, (1, 1)) == ts.FlipDirection.NONE  # a slope: neither min nor max


def test_lozenge_codec_overlap():
    d = ts.TriDomain.hexagon(1, 1, 1)
    loz = ts.lozenges_from_tiling(ts.LozengeTiling(d, _unit_hexagon_edges(d)))
    with pytest.raises(ts.OverlapError):
        ts.tiling_from_lozenges(d, [loz[0], loz[0], loz[1]])


def _unit_hexagon_edges(d):
    """One of the two tilings of the unit hexagon, found by trying the edge
    patterns of its three lozenges (host-side codec only)."""
    import itertools

    shape = (3, d.size[0] + 1, d.size[1] + 1)
    cells = [(k, x, y) for k in range(3) for x in range(shape[1]) for y in range(shape[2])]
    for combo in itertools.combinations(cells, 3):
        e = np.zeros(shape, dtype=bool)
        for c in combo:
            e[c] = True
        try:
            t = ts.LozengeTiling(d, e)
            if is_valid_lozenge_tiling(t):
                return e
        except ts.TileSamplerError:
            continue
    raise AssertionError("no tiling of the unit hexagon found")


def test_collapse_check_domain_mismatch():
    a = _brick(ts.Domain.square(4))
    b = _brick(ts.Domain.square(2))
    assert ts.collapse_check(a, a) and not ts.collapse_check(a, _brick(ts.Domain.square(4), False))
    with pytest.raises(ts.DomainMismatchError):
        ts.collapse_check(a, b)


def test_cftp_rejects_untileable_before_any_walk():
    d = ts.Domain.from_faces(2, [(0, 0), (0, 1), (1, 0)])  # odd face count
    with pytest.raises(ts.UntileableDomain):
        ts.cftp_sample(d, ts.SweepPlan(d), 1)


def test_negative_steps_and_empty_archive(square2):
    with pytest.raises(ValueError):
        ts.random_walk(_brick(square2), 1, -1, ts.SweepPlan(square2))

    class Empty:
        records = []

        def __len__(self):
            return 0

    with pytest.raises(ts.EmptyArchive):
        stats.density_map(Empty(), "domino-orientation")
