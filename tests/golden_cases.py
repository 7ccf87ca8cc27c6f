"""Case definitions shared by tests/golden/make_golden.py (run against the
reference) and the parity tests (run against this package).

Only plain data lives at module level; functions that build domains take the
API module (`ts`) as an argument so the same definition drives both sides.
"""

from __future__ import annotations

import math

import numpy as np

# (seed, grid shape, site, step) -- includes SURVEY.md Appendix B rows
RNG_KATS = [
    (0x5EED, (129, 129), (64, 64), 0),
    (0x5EED, (129, 129), (1, 2), 999),
    (0x1, (8193, 8193), (4096, 4096), 7),
    (0x8000000000000005, (2049, 2049), (1024, 3), 123456),
    (0, (1, 1), (0, 0), 0),
    (0xFFFFFFFFFFFFFFFF, (3, 5), (2, 4), 2**40),
    (12345, (32769, 32769), (32768, 32768), 10**6),
]
DERIVE_KATS = [(0x5EED, 0, 2), (0x5EED, 1, 0x51ED2701), (0, 0, 0), (2**64 - 1, 7, 3)]
CHAIN_KATS = [(0x5EED, 0), (0x5EED, 63), (42, 5)]
GRID_KATS = [(7, (5, 9), 0), (0x5EED, (33, 17), 12)]


def random_subdomain(ts, rng: np.random.Generator, n: int, target: int | None = None):
    """Randomized-BFS simply-connected face set (tests/helpers.py:11-39)."""
    target = target or int(rng.integers(2, n * n + 1))
    while True:
        grid = np.zeros((n, n), dtype=bool)
        start = (int(rng.integers(n)), int(rng.integers(n)))
        grid[start] = True
        frontier = [start]
        while grid.sum() < target and frontier:
            i = int(rng.integers(len(frontier)))
            r, c = frontier[i]
            nbrs = [
                (rr, cc)
                for rr, cc in ((r - 1, c), (r + 1, c), (r, c - 1), (r, c + 1))
                if 0 <= rr < n and 0 <= cc < n and not grid[rr, cc]
            ]
            if not nbrs:
                frontier.pop(i)
                continue
            f = nbrs[int(rng.integers(len(nbrs)))]
            grid[f] = True
            frontier.append(f)
        try:
            return ts.Domain(n, grid)
        except ts.DomainError:
            continue


def random_tileable_domain(ts, rng: np.random.Generator, n: int):
    while True:
        d = random_subdomain(ts, rng, n)
        if d.face_count % 2 == 0 and ts.extremal_tilings(d) is not None:
            return d


def _both(ts, d):
    ext = ts.extremal_tilings(d)
    return [ext[0].states, ext[1].states]


def domino_walk_weights(ts):
    """Weight spec of each domino_walk_cases entry, in order."""
    return ([ts.VolumeWeights(1.0, {(2, 3): 2.0})] + [ts.Uniform()] * 6
            + [ts.EdgeWeights(1.0, {((3, 4), (3, 5)): 3.0, ((7, 7), (8, 7)): 0.25, ((0, 0), (0, 1)): 5.0}),
               ts.VolumeWeights(0.9), ts.Uniform(), ts.Uniform(),
               ts.VolumeWeights(1.05, {(40, 40): 3.0, (10, 40): 0.5})])


def domino_walk_cases(ts=None):
    if ts is None:
        import tilesampler as ts  # reference, only when generating
    cases = []
    # sweeps.py fused==numpy test (tests/test_sweeps.py:160-168)
    d = ts.Domain.aztec(3)
    plan = ts.SweepPlan(d, ts.VolumeWeights(1.0, {(2, 3): 2.0}))
    cases.append(dict(domain=d, plan=plan, start=lambda d=d: [ts.extremal_tilings(d)[1].states] * 5,
                      seeds=list(range(11, 16)), n_steps=97))
    rng = np.random.default_rng(2024)
    for k in range(6):
        d = random_tileable_domain(ts, rng, 12)
        cases.append(dict(domain=d, plan=ts.SweepPlan(d), start=lambda d=d: _both(ts, d),
                          seeds=[1000 + k, 2000 + k], n_steps=150 + 7 * k))
    d = ts.Domain.square(16)
    w = ts.EdgeWeights(1.0, {((3, 4), (3, 5)): 3.0, ((7, 7), (8, 7)): 0.25, ((0, 0), (0, 1)): 5.0})
    cases.append(dict(domain=d, plan=ts.SweepPlan(d, w), start=lambda d=d: _both(ts, d),
                      seeds=[3, 2**63 + 9], n_steps=150))
    d = ts.Domain.aztec(20)
    cases.append(dict(domain=d, plan=ts.SweepPlan(d, ts.VolumeWeights(0.9)),
                      start=lambda d=d: _both(ts, d)[:1], seeds=[0x5EED], n_steps=300))
    d = ts.Domain.rectangle(2, 3)
    cases.append(dict(domain=d, plan=ts.SweepPlan(d), start=lambda d=d: _both(ts, d)[:1] * 3,
                      seeds=[5, 6, 7], n_steps=40))
    d = ts.Domain.rectangle(30, 70)  # non-square box, wide rows (> 64 columns)
    cases.append(dict(domain=d, plan=ts.SweepPlan(d), start=lambda d=d: _both(ts, d)[1:],
                      seeds=[99], n_steps=211))
    d = ts.Domain.aztec(40)
    w = ts.VolumeWeights(1.05, {(40, 40): 3.0, (10, 40): 0.5})
    cases.append(dict(domain=d, plan=ts.SweepPlan(d, w), start=lambda d=d: _both(ts, d),
                      seeds=[17, 18], n_steps=257))
    return cases


def _sq(n):
    def f():
        import tilesampler as ts
        return ts.Domain.square(n)
    return f


def _az(n):
    def f():
        import tilesampler as ts
        return ts.Domain.aztec(n)
    return f


def _rect(r, c):
    def f():
        import tilesampler as ts
        return ts.Domain.rectangle(r, c)
    return f


SWEEP_CASES = [(_sq(6), 5, 0, 0), (_az(5), 99, 17, 1), (_rect(4, 7), 2**62, 3, 0)]


def extremal_domains(ts=None):
    if ts is None:
        import tilesampler as ts
    out = [ts.Domain.aztec(k) for k in (1, 2, 3, 4, 5, 8, 13, 16)]
    out += [ts.Domain.square(k) for k in (2, 3, 4, 6)]
    out += [ts.Domain.rectangle(3, 8), ts.Domain.rectangle(5, 2), ts.Domain.rectangle(1, 2)]
    out.append(ts.Domain.from_faces(2, [(0, 0), (0, 1), (1, 0)]))  # untileable L
    rng = np.random.default_rng(7)
    for _ in range(10):
        out.append(random_subdomain(ts, rng, 10))
    return out


CFTP_CASES = []  # filled lazily: needs weights objects of the reference


def _cftp_cases():
    import tilesampler as ts
    return [
        (_rect(2, 3), ts.Uniform(), 999, 7, 40),
        (_sq(4), ts.Uniform(), 3, 3, 40),
        (_az(3), ts.VolumeWeights(1.0, {(2, 3): 2.0}), 271828, 4, 40),
        (_sq(6), ts.Uniform(), 271828, 1, 40),
        (_az(6), ts.Uniform(), 0x5EED, 2, 40),
    ]


class _Lazy(list):
    def __iter__(self):
        return iter(_cftp_cases())


CFTP_CASES = _Lazy()

# six-vertex: (n, (a, b, c), seed, n_steps, start)
SV_CASES = [
    (16, (1.0, 1.0, 1.0), 0x5EED, 500, "min"),
    (16, (1.0, 1.0, math.sqrt(8.0)), 0x5EED, 500, "min"),
    (9, (0.7, 1.3, 1.9), 123, 333, "max"),
    (24, (2.0, 0.5, 1.0), 4242, 200, "min"),
]
SV_EXTREMAL_N = [1, 2, 3, 5, 8, 13]
SV_LUT_WEIGHTS = [(1.0, 1.0, 1.0), (1.0, 1.0, math.sqrt(8.0)), (0.7, 1.3, 1.9), (2.0, 0.5, 1.0), (1.0, 1.0, 0.3)]
SV_CFTP_CASES = [(3, (1.0, 1.0, 1.0), 11, 5), (4, (1.0, 1.0, 1.5), 2024, 3)]

# lozenges: ((a, b, c), weights, seed, n_steps, start)
def _loz_cases():
    import tilesampler as ts
    from tilesampler.lozenge import LozEdgeWeights
    return [
        ((8, 8, 8), ts.VolumeWeights(0.9), 0x5EED, 500, "min"),
        ((3, 4, 5), ts.Uniform(), 31337, 200, "max"),
        ((5, 2, 6), LozEdgeWeights(1.0, {(("up", 3, 4), ("down", 3, 3)): 2.5}), 8, 150, "min"),
    ]


class _LazyLoz(list):
    def __iter__(self):
        return iter(_loz_cases())


LOZ_CASES = _LazyLoz()
LOZ_EXTREMAL = [(1, 1, 1), (2, 2, 2), (3, 4, 5), (6, 1, 3)]
LOZ_CFTP_CASES = [((1, 1, 1), 5, 4), ((2, 2, 2), 77, 3)]

# CLI runs (cli.py:128-255): name -> argv; "{g}" is the golden directory.
# `density` / `hist` read the archives the `cftp` cases wrote.
CLI_CASES = [
    ("sample_domino_aztec", ["sample", "--model", "domino", "--aztec", "6", "--steps", "100", "--samples", "3",
                             "--seed", "0x2a", "--weights", "q=0.9"]),
    ("sample_domino_square", ["sample", "--square", "4", "--steps", "64", "--samples", "10"]),
    ("sample_lozenge", ["sample", "--model", "lozenge", "--hexagon", "3,4,2", "--steps", "50", "--samples", "2",
                        "--weights", "q=0.8", "--seed", "7"]),
    ("sample_sixvertex", ["sample", "--model", "sixvertex", "--dwbc", "6", "--steps", "40", "--samples", "3",
                          "--weights", "a=1,b=1,c=1.5", "--backend", "threads"]),
    ("cftp_domino", ["cftp", "--aztec", "3", "--samples", "8", "--seed", "0x2a"]),
    ("cftp_lozenge", ["cftp", "--model", "lozenge", "--hexagon", "2,2,2", "--samples", "4", "--seed", "5",
                      "--weights", "q=1.2"]),
    ("cftp_sixvertex", ["cftp", "--model", "sixvertex", "--dwbc", "4", "--samples", "5", "--seed", "9",
                        "--weights", "a=1,b=1,c=2"]),
    ("density_domino", ["density", "--aztec", "3", "--in", "{g}/cli_cftp_domino.txt",
                        "--observable", "domino-orientation"]),
    ("density_sixvertex_csv", ["density", "--model", "sixvertex", "--dwbc", "4", "--in", "{g}/cli_cftp_sixvertex.txt",
                               "--observable", "c-vertex", "--format", "csv"]),
    ("hist_sixvertex", ["hist", "--model", "sixvertex", "--dwbc", "4", "--in", "{g}/cli_cftp_sixvertex.txt"]),
    ("hist_domino_y", ["hist", "--aztec", "3", "--in", "{g}/cli_cftp_domino.txt", "--observable", "y-intercept"]),
]
