"""Counter-based splitmix64 streams (the reference's RNG contract, rng.py:1-167).

Every draw is a pure function of (seed, site, tag, step).  The per-site
draws of a sweep are generated on the device inside the sweep kernels
(csrc/domino.cu); this module keeps the host-side scalar pieces the API
needs (child-seed derivation for CFTP schedules, single-site queries) and
exposes full grids through the device kernel `tsb_uniform_grid`.
"""

from __future__ import annotations

import numpy as np

from . import _native
from .errors import CapacityError, OutOfGridError

_MASK = (1 << 64) - 1
_GOLDEN = 0x9E3779B97F4A7C15
_CAPACITY = 1 << 48

TAG_SITE = 0
TAG_GLOBAL = 1
TAG_DERIVE = 2


def _mix(z: int) -> int:
    """splitmix64 finaliser (rng.py:34-39)."""
    z &= _MASK
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _MASK
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _MASK
    return z ^ (z >> 31)


def _splitmix_at(state: int, counter: int) -> int:
    return _mix((state + (counter + 1) * _GOLDEN) & _MASK)


def derive_seed(seed: int, index: int, salt: int = 0) -> int:
    """Deterministic 64-bit child seed (rng.py:57-59)."""
    return _splitmix_at(_mix(seed ^ (salt * 0xD6E8FEB86659FD93)), index)


def _to_unit(x: int) -> float:
    return (x >> 11) * 2.0**-53


def family_base(seed: int) -> int:
    return _mix((seed & _MASK) ^ 0x6A09E667F3BCC909)


def global_key(seed: int) -> int:
    return _splitmix_at(family_base(seed), TAG_GLOBAL << 48)


def color_at(seed: int, step: int) -> int:
    """Colour (0 BLACK / 1 WHITE) a domino sweep uses at `step` (sweeps.py:266-269)."""
    return 1 if _to_unit(_splitmix_at(global_key(seed), step)) >= 0.5 else 0


class StreamFamily:
    """A grid of independent uniform streams keyed by one 64-bit seed (rng.py:66-123)."""

    def __init__(self, seed: int, shape: tuple[int, int]):
        rows, cols = shape
        if rows <= 0 or cols <= 0:
            raise ValueError(f"grid shape must be positive, got {shape}")
        if rows * cols >= _CAPACITY:
            raise CapacityError(f"grid of {rows * cols} sites exceeds the {_CAPACITY} stream capacity")
        self.seed = seed & _MASK
        self.shape = (rows, cols)
        self._base = family_base(self.seed)

    def _stream_index(self, site: tuple[int, int], tag: int) -> int:
        r, c = site
        rows, cols = self.shape
        if not (0 <= r < rows and 0 <= c < cols):
            raise OutOfGridError(f"site {site} outside grid {self.shape}")
        return (tag << 48) | (r * cols + c)

    def site_key(self, site: tuple[int, int], tag: int = TAG_SITE) -> int:
        return _splitmix_at(self._base, self._stream_index(site, tag))

    def uniform(self, site: tuple[int, int], step: int, tag: int = TAG_SITE) -> float:
        return _to_unit(_splitmix_at(self.site_key(site, tag), step))

    def global_uniform(self, step: int) -> float:
        return _to_unit(_splitmix_at(self.site_key((0, 0), TAG_GLOBAL), step))

    def uniform_grid(self, step: int, tag: int = TAG_SITE) -> np.ndarray:
        """All sites at one step, float64 (rows, cols); computed on the device."""
        rows, cols = self.shape
        out = np.empty((rows, cols), dtype=np.float64)
        L = _native.lib()
        _native.check(L.tsb_uniform_grid(_native.device(), self.seed, rows, cols,
                                         _native.u64(step), tag, _native.ptr(out)))
        return out


def seed_family(seed: int, shape: tuple[int, int]) -> StreamFamily:
    return StreamFamily(seed, shape)


def uniform(family: StreamFamily, site: tuple[int, int], step: int) -> float:
    return family.uniform(site, step)
