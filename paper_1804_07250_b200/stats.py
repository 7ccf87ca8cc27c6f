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

    `handle` is a DominoHandle ("domino-orientation") or a SixVertexHandle
    ("h-edge", "v-edge", "c-vertex", or "height" for the mean height
    function).  Each `add(chain0, n)` adds the current states of chains
    [chain0, chain0 + n).
    """

    def __init__(self, handle, observable: str):
        import torch

        from .sixvertex import SixVertexHandle
        from .sweeps import DominoHandle

        self.handle = handle
        self.observable = observable
        self.samples = 0
        dev = torch.device("cuda", handle.device)
        if isinstance(handle, DominoHandle):
            if observable != "domino-orientation":
                raise KeyError(f"unknown domino observable {observable!r}; have ['domino-orientation']")
            nf = handle.side - 1
            self.shape = (nf, nf)
            self._acc = torch.zeros(self.shape, dtype=torch.int32, device=dev)
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
        from .sweeps import DominoHandle

        h = self.handle
        n = h.nchains - chain0 if n is None else n
        L = _native.lib()
        p = self._acc.data_ptr()
        if isinstance(h, DominoHandle):
            _native.check(L.tsb_domino_orientation_add(h._h, chain0, n, p))
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
