"""Cluster Glauber dynamics for domino tilings -- device-backed.

Drop-in mirror of the reference's `sweeps.py` (same names, signatures and
results, sweeps.py:1-362).  Every sweep runs in the sm_100a kernel
`domino_sweep_kernel` (csrc/domino.cu) through the C ABI; the `backend`
argument is accepted for signature compatibility and ignored (the device is
the backend).  There is no CPU fallback.
"""

from __future__ import annotations

import ctypes
import enum
from collections import OrderedDict
from dataclasses import dataclass, field
from functools import cached_property

import numpy as np

from . import _native, rng
from .lattice import (
    HORIZONTAL_PAIR,
    VERTICAL_PAIR,
    Domain,
    EdgeWeights,
    Tiling,
    Uniform,
    VolumeWeights,
    WeightSpec,
    rotation_height_delta,
)


class Color(enum.IntEnum):
    """Checkerboard vertex colours; BLACK is even coordinate sum (sweeps.py:40-44)."""

    BLACK = 0
    WHITE = 1


class Sequential:
    """Signature-compatible stand-in for the reference's CPU band executor
    (sweeps.py:47-56).  The device runs every sweep; no CPU bands exist."""

    workers = 1

    def run_bands(self, n_rows: int, fn) -> None:
        fn(0, n_rows)

    def __repr__(self):
        return "Sequential()"


class MultiThreaded(Sequential):
    """Signature-compatible stand-in for the reference's threaded backend
    (sweeps.py:59-93); results are identical by construction."""

    def __init__(self, workers: int):
        if workers < 1:
            raise ValueError("worker count must be positive")
        self.workers = workers

    def __repr__(self):
        return f"MultiThreaded({self.workers})"


Backend = Sequential | MultiThreaded


def rotate_kernel(s: int, u: float, p_up: float) -> int:
    """Scalar rotate semantics (sweeps.py:102-110)."""
    if u < p_up:
        return VERTICAL_PAIR if s == HORIZONTAL_PAIR else s
    return HORIZONTAL_PAIR if s == VERTICAL_PAIR else s


def update_kernel(t_self: np.ndarray, t_other: np.ndarray, i: int, j: int, color: Color) -> int:
    """Scalar update semantics on checkerboard sub-arrays (sweeps.py:113-131)."""
    par = i % 2 if color == Color.BLACK else (i + 1) % 2

    def other(a: int, b: int) -> int:
        if 0 <= a < t_other.shape[0] and 0 <= b < t_other.shape[1]:
            return int(t_other[a, b])
        return 0

    return (
        ((other(i - 1, j) & 2) >> 1)
        | ((other(i + 1, j) & 1) << 1)
        | ((other(i, j + par - 1) & 8) >> 1)
        | ((other(i, j + par) & 4) << 1)
    )


def heat_bath_p_up(vertex: tuple[int, int], w: WeightSpec) -> float:
    """W_up / (W_up + W_down) at one vertex (sweeps.py:134-150)."""
    if isinstance(w, Uniform):
        return 0.5
    if isinstance(w, VolumeWeights):
        ratio = w.q(vertex) ** rotation_height_delta(vertex)
        return ratio / (1.0 + ratio)
    if isinstance(w, EdgeWeights):
        r, c = vertex
        w_up = w.weight((r - 1, c - 1), (r, c - 1)) * w.weight((r - 1, c), (r, c))
        w_down = w.weight((r - 1, c - 1), (r - 1, c)) * w.weight((r, c - 1), (r, c))
        return w_up / (w_up + w_down)
    raise TypeError(f"unsupported weight spec {type(w)!r}")


def _p_up_grid(v: int, w: WeightSpec) -> np.ndarray:
    """Vectorised SweepPlan.p_up, bit-identical to the per-vertex loop
    (sweeps.py:170-179): powers are taken with Python floats on the few
    distinct q values, products/quotients are IEEE-exact in numpy too."""
    if isinstance(w, Uniform):
        return np.full((v, v), 0.5)
    if isinstance(w, VolumeWeights):
        par = (np.arange(v)[:, None] + np.arange(v)[None, :]) % 2
        grid = np.empty((v, v))
        for p in (0, 1):
            ratio = w.default ** (4 if p == 0 else -4)
            grid[par == p] = ratio / (1.0 + ratio)
        for (r, c) in w.overrides:
            if 0 <= r < v and 0 <= c < v:
                grid[r, c] = heat_bath_p_up((r, c), w)
        return grid
    if isinstance(w, EdgeWeights):
        d = float(w.default)
        a = np.full((v, v), d)  # w((r-1,c-1),(r,c-1))
        b = np.full((v, v), d)  # w((r-1,c),(r,c))
        c_ = np.full((v, v), d)  # w((r-1,c-1),(r-1,c))
        e = np.full((v, v), d)  # w((r,c-1),(r,c))
        touched = []
        for key, val in w.overrides.items():
            fa, fb = sorted(key)
            (ra, ca), (rb, cb) = fa, fb
            if ca == cb and rb == ra + 1:  # vertical face pair
                for (rr, cc, arr) in ((rb, ca + 1, a), (rb, ca, b)):
                    if 0 <= rr < v and 0 <= cc < v:
                        arr[rr, cc] = val
                        touched.append((rr, cc))
            elif ra == rb and cb == ca + 1:  # horizontal face pair
                for (rr, cc, arr) in ((ra + 1, cb, c_), (ra, cb, e)):
                    if 0 <= rr < v and 0 <= cc < v:
                        arr[rr, cc] = val
                        touched.append((rr, cc))
        w_up = a * b
        w_dn = c_ * e
        return w_up / (w_up + w_dn)
    raise TypeError(f"unsupported weight spec {type(w)!r}")


@dataclass(frozen=True)
class SweepPlan:
    """Frozen per-domain sweep data: colour classes and flip probabilities
    (sweeps.py:153-179)."""

    domain: Domain
    weights: WeightSpec = field(default_factory=Uniform)

    @cached_property
    def parity(self) -> np.ndarray:
        v = self.domain.n + 1
        r = np.arange(v)
        return ((r[:, None] + r[None, :]) % 2).astype(np.uint8)

    def color_class(self, color: Color) -> np.ndarray:
        return self.parity == int(color)

    @cached_property
    def p_up(self) -> np.ndarray:
        return _p_up_grid(self.domain.n + 1, self.weights)

    @cached_property
    def p_up_parity(self) -> tuple[float, float] | None:
        """(p_up at even, at odd vertices) when p_up depends only on the
        parity (Uniform; VolumeWeights without overrides), else None -- the
        same float64 values as p_up (_p_up_grid), without the V x V grid."""
        w = self.weights
        if isinstance(w, Uniform):
            return 0.5, 0.5
        if isinstance(w, VolumeWeights) and not w.overrides:
            out = []
            for p in (0, 1):
                ratio = w.default ** (4 if p == 0 else -4)
                out.append(ratio / (1.0 + ratio))
            return out[0], out[1]
        return None


# -- device handles ------------------------------------------------------------


class DominoHandle:
    """Owns a batch of device-resident domino chains (tsb_domino)."""

    def __init__(self, domain: Domain | None, side: int, nchains: int, device: int | None = None):
        L = _native.lib()
        self.side = side
        self.nchains = nchains
        self.device = _native.device() if device is None else device
        self.domain = domain
        self._p_up_id = None
        self._p_up_ref = None
        self._h = ctypes.c_void_p()
        faces = domain.faces_u8 if domain is not None else None
        _native.check(L.tsb_domino_create(self.device, side, nchains,
                                          None if faces is None else _native.ptr(faces),
                                          ctypes.byref(self._h)))

    @classmethod
    def window(cls, domain: Domain, row_lo: int, row_hi: int, device: int | None = None) -> "DominoHandle":
        """One chain holding only the global rows [row_lo, row_hi) of the
        domain's grid (tsb_domino_create_window): a strip rank's share of a
        lattice.  Rows keep their global indices; use upload_rows /
        download_rows (whole-grid operations raise ValueError)."""
        h = cls.__new__(cls)
        L = _native.lib()
        h.side = domain.n + 1
        h.nchains = 1
        h.device = _native.device() if device is None else device
        h.domain = domain
        h._p_up_id = None
        h._p_up_ref = None
        h._h = ctypes.c_void_p()
        h.rows = (row_lo, row_hi)
        _native.check(L.tsb_domino_create_window(h.device, h.side, row_lo, row_hi, _native.ptr(domain.faces_u8),
                                                 ctypes.byref(h._h)))
        return h

    def upload_rows(self, r0: int, rows: np.ndarray):
        """Rows [r0, r0 + len(rows)) of chain 0 from a (n, V) uint8 tilestate grid."""
        g = np.ascontiguousarray(rows, dtype=np.uint8)
        if g.ndim != 2 or g.shape[1] != self.side:
            raise ValueError(f"rows must have shape (n, {self.side})")
        _native.check(_native.lib().tsb_domino_upload_rows(self._h, int(r0), g.shape[0], _native.ptr(g)))

    def download_rows(self, r0: int, nrows: int, out: np.ndarray | None = None) -> np.ndarray:
        if out is None:
            out = np.empty((nrows, self.side), dtype=np.uint8)
        elif out.shape != (nrows, self.side) or out.dtype != np.uint8 or not out.flags.c_contiguous:
            raise ValueError(f"out must be a C-contiguous uint8 array of shape {(nrows, self.side)}")
        _native.check(_native.lib().tsb_domino_download_rows(self._h, int(r0), int(nrows), _native.ptr(out)))
        return out

    def __del__(self):
        try:
            if self._h:
                _native.lib().tsb_domino_destroy(self._h)
                self._h = ctypes.c_void_p()
        except Exception:  # interpreter shutdown
            pass

    def set_stream(self, stream_ptr: int):
        _native.check(_native.lib().tsb_domino_set_stream(self._h, ctypes.c_void_p(stream_ptr)))

    def set_collapse(self, on: bool):
        """Run collapsing (tsb_domino_set_collapse): skip sweeps followed by a
        sweep of the same colour; bit-identical results."""
        _native.check(_native.lib().tsb_domino_set_collapse(self._h, int(bool(on))))

    def set_p_up(self, p_up: np.ndarray):
        if self._p_up_ref is p_up:
            return
        p = np.ascontiguousarray(p_up, dtype=np.float64)
        if p.shape != (self.side, self.side):
            raise ValueError(f"p_up must be {(self.side, self.side)}")
        _native.check(_native.lib().tsb_domino_set_p_up(self._h, _native.ptr(p)))
        self._p_up_ref = p_up

    def set_plan(self, plan: "SweepPlan"):
        """Thresholds of a SweepPlan; parity-only p_up (the common case)
        never materialises the V x V grid (8.6 GB at Aztec 16384)."""
        if self._p_up_ref is plan:
            return
        par = plan.p_up_parity
        if par is None:
            self.set_p_up(plan.p_up)
        else:
            _native.check(_native.lib().tsb_domino_set_p_up_parity(self._h, float(par[0]), float(par[1])))
        self._p_up_ref = plan

    def upload(self, states: np.ndarray, chain0: int = 0):
        s = np.ascontiguousarray(states, dtype=np.uint8)
        _native.check(_native.lib().tsb_domino_upload(self._h, chain0, s.shape[0], _native.ptr(s)))

    def download(self, chain0: int = 0, n: int | None = None, out: np.ndarray | None = None) -> np.ndarray:
        """States of chains [chain0, chain0+n) as (n, V, V) uint8; `out` (e.g. a
        pinned host buffer) is filled in place when given."""
        n = self.nchains - chain0 if n is None else n
        if out is None:
            out = np.empty((n, self.side, self.side), dtype=np.uint8)
        elif out.shape != (n, self.side, self.side) or out.dtype != np.uint8 or not out.flags.c_contiguous:
            raise ValueError(f"out must be a C-contiguous uint8 array of shape {(n, self.side, self.side)}")
        _native.check(_native.lib().tsb_domino_download(self._h, chain0, n, _native.ptr(out)))
        return out

    def walk(self, seeds, n_steps: int, step0: int = 0, chain0: int = 0):
        s = np.ascontiguousarray(seeds, dtype=np.uint64)
        _native.check(_native.lib().tsb_domino_walk(self._h, chain0, s.shape[0], _native.ptr(s),
                                                    _native.u64(step0), int(n_steps)))

    def sweep(self, seeds, step: int, color: int, chain0: int = 0):
        s = np.ascontiguousarray(seeds, dtype=np.uint64)
        _native.check(_native.lib().tsb_domino_sweep(self._h, chain0, s.shape[0], _native.ptr(s),
                                                     _native.u64(step), int(color)))

    def sync(self):
        _native.check(_native.lib().tsb_domino_sync(self._h))

    def heights(self, chain: int, ref) -> np.ndarray:
        out = np.empty((self.side, self.side), dtype=np.int32)
        _native.check(_native.lib().tsb_domino_heights(self._h, chain, int(ref[0]), int(ref[1]),
                                                       _native.ptr(out)))
        return out

    def extremal(self, ref, chain_max: int = 0, chain_min: int = 1) -> bool:
        rc = _native.lib().tsb_domino_extremal(self._h, chain_max, chain_min, int(ref[0]), int(ref[1]))
        if rc == _native.E_UNTILEABLE:
            return False
        _native.check(rc)
        return True


_CACHE: "OrderedDict[tuple, DominoHandle]" = OrderedDict()
_CACHE_MAX = 8
_COLLAPSE: bool | None = None  # None: the library default (run collapsing on, env TSB_DOM_COLLAPSE)


def set_default_collapse(on: bool | None) -> None:
    """Run collapsing for the walks of the drop-in API (random_walk_batch,
    random_walk, CFTP); None restores the library default.  Results are
    bit-identical either way (tsb_domino_set_collapse)."""
    global _COLLAPSE
    _COLLAPSE = on


def _handle_for(domain: Domain | None, nchains: int, side: int | None = None, slot: int = 0) -> DominoHandle:
    side = domain.n + 1 if domain is not None else side
    key = (domain._key if domain is not None else None, side, nchains, _native.device(), slot)
    h = _CACHE.get(key)
    if h is None:
        h = DominoHandle(domain, side, nchains)
        _CACHE[key] = h
        while len(_CACHE) > _CACHE_MAX:
            _CACHE.popitem(last=False)
    else:
        _CACHE.move_to_end(key)
    if _COLLAPSE is not None:
        h.set_collapse(_COLLAPSE)
    return h


def random_walk_batch(
    states: np.ndarray,
    seeds: np.ndarray,
    n_steps: int,
    plan: SweepPlan,
    backend: Backend | None = None,
    use_fused: bool | None = None,
) -> np.ndarray:
    """Evolve a (B, V, V) batch for n_steps coupled cluster sweeps on the
    device (sweeps.py:278-316).  Chain b's result depends on seeds[b] only."""
    states = np.ascontiguousarray(states, dtype=np.uint8)  # no copy for a C-contiguous uint8 batch
    v = states.shape[-1]
    seeds = np.asarray(seeds, dtype=np.uint64)
    if n_steps <= 0 or states.shape[0] == 0:
        return states.copy()  # a new array, like the reference (sweeps.py:299)
    if states.shape[0] >= 2 and v * v >= _PIPELINE_MIN_BYTES:
        return _walk_pipelined(states, seeds, n_steps, plan)
    h = _handle_for(plan.domain, states.shape[0]) if plan.domain.n + 1 == v else _handle_for(None, states.shape[0], v)
    h.set_plan(plan)
    h.upload(states)
    h.walk(seeds, n_steps)
    return h.download()


_PIPELINE_MIN_BYTES = 1 << 22  # chains of at least 4 MB of tilestates: copies worth overlapping


def _walk_pipelined(states: np.ndarray, seeds: np.ndarray, n_steps: int, plan: "SweepPlan") -> np.ndarray:
    """random_walk_batch for large lattices: the chains alternate between two
    one-chain handles, each on its own CUDA stream, so chain i+1's upload runs
    while chain i walks and chain i's download while chain i+1 walks.  Every
    chain's result depends on its own seed only (sweeps.py:286-292), so the
    output equals the batched walk."""
    v = states.shape[-1]
    dom = plan.domain if plan.domain.n + 1 == v else None
    hs = [_handle_for(dom, 1, v, slot=k) for k in (1, 2)]
    for h in hs:
        h.set_plan(plan)
    out = np.empty_like(states)
    pending = [None, None]
    for i in range(states.shape[0]):
        k = i & 1
        if pending[k] is not None:
            j = pending[k]
            hs[k].download(out=out[j:j + 1])
        hs[k].upload(states[i:i + 1])
        hs[k].walk(seeds[i:i + 1], n_steps)
        pending[k] = i
    for k in (0, 1):
        if pending[k] is not None:
            j = pending[k]
            hs[k].download(out=out[j:j + 1])
    return out


def sweep(
    t: Tiling,
    f: rng.StreamFamily,
    step: int,
    color: Color,
    plan: SweepPlan,
    backend: Backend | None = None,
    return_rotated: bool = False,
):
    """One sweep of `color` at `step` with family f's coins (sweeps.py:322-342)."""
    h = _handle_for(plan.domain, 1)
    h.set_plan(plan)
    h.upload(t.states[None])
    h.sweep([f.seed], step, int(color))
    new = h.download()[0]
    result = Tiling(t.domain, new)
    if return_rotated:
        rotated = (new != t.states) & plan.color_class(color)
        return result, rotated
    return result


def random_walk(
    t: Tiling,
    seed: int,
    n_steps: int,
    plan: SweepPlan,
    backend: Backend | None = None,
) -> Tiling:
    """n_steps sweeps with the colour chosen per step (sweeps.py:345-362)."""
    if n_steps < 0:
        raise ValueError("step count must be non-negative")
    states = random_walk_batch(t.states[None, :, :], np.array([seed], dtype=np.uint64), n_steps, plan, backend)
    return Tiling(t.domain, states[0])


class DominoCftp:
    """Device CFTP runner for a batch of samples (csrc/cftp.cu, tsb_domino_cftp)."""

    def __init__(self, domain: Domain, plan: SweepPlan, top0: np.ndarray, bot0: np.ndarray, count: int):
        self.domain = domain
        self.count = count
        self.top0 = np.ascontiguousarray(top0, dtype=np.uint8)
        self.bot0 = np.ascontiguousarray(bot0, dtype=np.uint8)
        self.handle = _handle_for(domain, 2 * count + 2)
        self.handle.set_plan(plan)

    def run(self, masters, max_doublings: int, progress=None, trace=None) -> np.ndarray:
        masters = np.ascontiguousarray(masters, dtype=np.uint64)
        b = len(masters)
        v = self.domain.n + 1
        out = np.zeros((b, v, v), dtype=np.uint8)
        rounds = np.zeros(b, dtype=np.int32)
        cb = None
        if progress is not None:
            cb = _native.PROGRESS_FN(lambda r, s, c, t, u: progress(r, int(s), c, t))
        rc = _native.lib().tsb_domino_cftp(
            self.handle._h, _native.ptr(self.top0), _native.ptr(self.bot0), _native.ptr(masters), b,
            int(max_doublings), _native.ptr(out), _native.ptr(rounds),
            ctypes.cast(cb, ctypes.c_void_p) if cb is not None else None, None)
        if trace is not None and b > 0:
            from .cftp import schedule_seed

            last = int(rounds[0]) if rc == _native.OK else int(max_doublings)
            m0 = int(masters[0])
            seeds = [schedule_seed(m0, i) for i in range(1, last + 1)]
            for r in range(1, last + 1):
                trace.rounds.append([(seeds[i - 1], 2**i) for i in range(r, 0, -1)])
            if rc == _native.OK:
                trace.collapsed_at = last
        _native.check(rc)
        return out
