"""On-device observables: the reference's density maps and scalar statistics
computed from device-resident chains without downloading states.

Reference (relative to /root/reference/pkg/src/tilesampler/):
  stats.py:174-184  DensityMap(observable, grid, samples)
  stats.py:187-200  domino_orientation_grid
  stats.py:213-245  density_map(archive, observable): "h-edge", "v-edge",
                    "c-vertex", "domino-orientation"
  stats.py:262-288  c_vertex_count, aztec_y_intercept

`DeviceDensity(handle, observable)` accumulates integer indicator counts in
GPU memory (libtsb: tsb_domino_orientation_add, tsb_sv_observe_add); after
S `add()` calls over B chains, `result().grid` equals the reference's
`density_map` of those S*B states (same counts, same division).  Torch only
provides the device buffer.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native

_SV_OBS = {"h-edge": 0, "v-edge": 1, "c-vertex": 2}


@dataclass(frozen=True)
class DensityMap:
    """Per-site empirical means of an indicator observable (stats.py:174-184)."""

    observable: str
    grid: np.ndarray
    samples: int

    def to_csv(self) -> str:
        lines = [",".join(f"{x:.6f}" for x in row) for row in self.grid]
        return "\n".join(lines) + "\n"


class DeviceDensity:
    """Accumulates an indicator observable of a handle's chains on the device.

    `handle` is a DominoHandle ("domino-orientation", or "height" for the
    mean height function of lattice.py:537-551), a SixVertexHandle ("h-edge",
    "v-edge", "c-vertex", "height") or a LozengeHandle ("height", the mean of
    loz_heights, lozenge.py:414-447).  Each `add(chain0, n)` adds the current
    states of chains [chain0, chain0 + n); heights are summed exactly in int64
    and divided once in `result()`.
    """

    def __init__(self, handle, observable: str):
        import torch

        from .lozenge import LozengeHandle
        from .sixvertex import SixVertexHandle
        from .sweeps import DominoHandle

        self.handle = handle
        self.observable = observable
        self.samples = 0
        dev = torch.device("cuda", handle.device)
        if isinstance(handle, DominoHandle):
            if observable == "height":
                if handle.domain is None:
                    raise ValueError("the mean height function needs the handle's domain")
                self.shape = (handle.side, handle.side)
                self._acc = torch.zeros(self.shape, dtype=torch.int64, device=dev)
            elif observable == "domino-orientation":
                nf = handle.side - 1
                self.shape = (nf, nf)
                self._acc = torch.zeros(self.shape, dtype=torch.int32, device=dev)
            else:
                raise KeyError(f"unknown domino observable {observable!r}; have ['domino-orientation', 'height']")
        elif isinstance(handle, LozengeHandle):
            if observable != "height":
                raise KeyError(f"unknown lozenge observable {observable!r}; have ['height']")
            self.shape = (handle.X, handle.Y)
            self._acc = torch.zeros(self.shape, dtype=torch.int64, device=dev)
        elif isinstance(handle, SixVertexHandle):
            n = handle.n
            shapes = {"h-edge": (n, n + 1), "v-edge": (n + 1, n), "c-vertex": (n, n), "height": (n + 1, n + 1)}
            if observable not in shapes:
                raise KeyError(f"unknown six-vertex observable {observable!r}; have {sorted(shapes)}")
            self.shape = shapes[observable]
            dt = torch.int64 if observable == "height" else torch.int32
            self._acc = torch.zeros(self.shape, dtype=dt, device=dev)
        else:
            raise TypeError(f"no device observables for {type(handle)!r}")
        torch.cuda.synchronize(dev)  # the zeroed buffer is visible to the handle's stream

    def add(self, chain0: int = 0, n: int | None = None) -> None:
        from .lozenge import LozengeHandle
        from .sweeps import DominoHandle

        h = self.handle
        n = h.nchains - chain0 if n is None else n
        L = _native.lib()
        p = self._acc.data_ptr()
        if isinstance(h, DominoHandle) and self.observable == "height":
            r, c = h.domain.reference_vertex
            _native.check(L.tsb_domino_height_sum_add(h._h, chain0, n, int(r), int(c), p))
        elif isinstance(h, DominoHandle):
            _native.check(L.tsb_domino_orientation_add(h._h, chain0, n, p))
        elif isinstance(h, LozengeHandle):
            x, y = h.domain.reference_vertex
            _native.check(L.tsb_loz_height_sum_add(h._h, chain0, n, int(x), int(y), p))
        elif self.observable == "height":
            _native.check(L.tsb_sv_height_sum_add(h._h, chain0, n, p))
        else:
            _native.check(L.tsb_sv_observe_add(h._h, chain0, n, _SV_OBS[self.observable], p))
        self.samples += n

    def counts(self) -> np.ndarray:
        """Raw accumulated counts (or height sums), after the handle's stream drains."""
        self.handle.sync()
        return self._acc.cpu().numpy()

    def result(self) -> DensityMap:
        if self.samples == 0:
            from .errors import EmptyArchive

            raise EmptyArchive("no states were added")
        grid = self.counts().astype(np.float64) / self.samples
        if self.observable == "domino-orientation" and self.handle.domain is not None:
            grid = np.where(self.handle.domain.faces, grid, np.nan)  # NaN outside (stats.py:193-194)
        return DensityMap(self.observable, grid, self.samples)


def aztec_y_intercept_from_density(grid: np.ndarray) -> float:
    """aztec_y_intercept (stats.py:270-288) evaluated on an orientation grid;
    applied to a single state's grid (samples == 1) it is the reference's
    per-sample statistic."""
    n = grid.shape[0]
    mid = n // 2
    col = grid[:, mid]
    rows = np.nonzero(~np.isnan(col))[0]
    boundary = rows[0]
    for r in rows:
        if col[r] == 1.0:
            boundary = r + 1
        else:
            break
    return float(boundary - mid)


# -- host mirrors of the reference's statistics API (stats.py:28-315) ----------
# Post-processing of host state objects, kept so that code written against
# the reference's `tilesampler.stats` runs unchanged; the device path above
# (DeviceDensity) computes the same density maps without downloading states.

C_VERTEX_CODES = (0b1001, 0b0110)


@dataclass(frozen=True)
class ChiSquareResult:
    statistic: float
    dof: int
    pvalue: float
    significance: float

    @property
    def passed(self) -> bool:
        return self.pvalue >= self.significance


def chi_square_gof(counts, probs=None, significance: float = 0.001) -> ChiSquareResult:
    """stats.py:40-60: chi-square goodness of fit (uniform when probs is None)."""
    from scipy import stats as sps

    counts = np.asarray(list(counts), dtype=float)
    n = counts.sum()
    if probs is None:
        expected = np.full(len(counts), n / len(counts))
    else:
        probs = np.asarray(list(probs), dtype=float)
        expected = probs / probs.sum() * n
    stat = float(((counts - expected) ** 2 / expected).sum())
    dof = len(counts) - 1
    return ChiSquareResult(stat, dof, float(sps.chi2.sf(stat, dof)), significance)


def total_variation(emp: dict, exact: dict) -> float:
    """stats.py:63-65."""
    keys = set(emp) | set(exact)
    return 0.5 * sum(abs(emp.get(k, 0.0) - exact.get(k, 0.0)) for k in keys)


def domino_orientation_grid(t) -> np.ndarray:
    """stats.py:187-200: 1.0 where a face is covered by a horizontal domino
    (its left or right edge is interior to a domino: tilestate bit 2 "down"
    of its top corners), 0.0 for a vertical one, NaN outside the domain."""
    s = np.asarray(t.states)
    horiz = ((s[:-1, :-1] & 2) | (s[:-1, 1:] & 2)) != 0
    return np.where(t.domain.faces, horiz.astype(float), np.nan)


def _c_vertex_grid(state) -> np.ndarray:
    from .sixvertex import vertex_type_codes

    codes = vertex_type_codes(state)
    return (codes == C_VERTEX_CODES[0]) | (codes == C_VERTEX_CODES[1])


_OBSERVABLES = {
    "h-edge": lambda st: st.h_edges.astype(float),
    "v-edge": lambda st: st.v_edges.astype(float),
    "c-vertex": lambda st: _c_vertex_grid(st).astype(float),
    "domino-orientation": domino_orientation_grid,
}


def density_map(archive, observable: str) -> DensityMap:
    """stats.py:231-245: per-site mean of the named indicator over an archive
    of host states (for device-resident chains use DeviceDensity)."""
    from .errors import EmptyArchive

    if len(archive) == 0:
        raise EmptyArchive("archive holds no records")
    fn = _OBSERVABLES.get(observable)
    if fn is None:
        raise KeyError(f"unknown observable {observable!r}; have {sorted(_OBSERVABLES)}")
    acc = None
    for state in archive.records:
        grid = fn(state)
        acc = grid if acc is None else acc + grid
    return DensityMap(observable, acc / len(archive), len(archive))


@dataclass(frozen=True)
class Histogram:
    observable: str
    edges: np.ndarray
    density: np.ndarray
    samples: int

    def to_csv(self) -> str:
        lines = ["left,right,density"]
        for lo, hi, d in zip(self.edges[:-1], self.edges[1:], self.density):
            lines.append(f"{lo:.6f},{hi:.6f},{d:.6f}")
        return "\n".join(lines) + "\n"


def c_vertex_count(state) -> float:
    """stats.py:262-264."""
    return float(_c_vertex_grid(state).sum())


def aztec_y_intercept(t) -> float:
    """stats.py:267-288."""
    return aztec_y_intercept_from_density(domino_orientation_grid(t))


def scalar_observable(archive, fn, bins=None) -> Histogram:
    """stats.py:291-315: normalised histogram of a scalar observable
    ('c-vertex-count', 'y-intercept' or a callable) over an archive."""
    from .errors import EmptyArchive

    if len(archive) == 0:
        raise EmptyArchive("archive holds no records")
    name = fn if isinstance(fn, str) else getattr(fn, "__name__", "scalar")
    if fn == "c-vertex-count":
        fn = c_vertex_count
    elif fn == "y-intercept":
        fn = aztec_y_intercept
    values = np.array([fn(s) for s in archive.records], dtype=float)
    lo, hi = values.min(), values.max()
    edges = np.array([lo - 0.5, lo + 0.5]) if lo == hi else np.histogram_bin_edges(values, bins=bins or "auto")
    density, edges = np.histogram(values, bins=edges, density=True)
    return Histogram(name, edges, density, len(values))
