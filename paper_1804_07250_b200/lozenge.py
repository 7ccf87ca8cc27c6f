"""Lozenge tilings of triangular-lattice domains -- device-backed.

Drop-in mirror of the reference's `lozenge.py` (lozenge.py:1-827): same
axial geometry, edge codec, rotation masks, heights, extremal tilings and
CFTP, with sweeps / heights / extremal / CFTP in csrc/lozenge.cu.  Domain
checks are vectorised (scipy connected components + Euler characteristic)
instead of Python BFS over triangles.
"""

from __future__ import annotations

import ctypes
from collections import OrderedDict
from dataclasses import dataclass
from functools import cached_property
from itertools import permutations
from typing import Iterable, Optional

import numpy as np

from . import _native, rng
from .cftp import CftpTrace, _progress_writer, chain_master_seed
from .errors import CoverageError, DomainError, InconsistencyError, OutOfDomainError, OverlapError, UntileableDomain
from .lattice import Uniform, VolumeWeights
from .sweeps import Backend

_TRI_DEVICE_CELLS = 1 << 16  # TriDomain checks on the GPU above this many cells (when present)

Triangle = tuple[str, int, int]
Lozenge = tuple[Triangle, Triangle]

DIRS = ((1, 0), (0, 1), (-1, 1), (-1, 0), (0, -1), (1, -1))
CUBE_UNIT = 3
_STEPS = tuple((1, -2) if k % 2 == 0 else (-1, 2) for k in range(6))


def _up_edges(x: int, y: int):
    return (("a", x, y), ("b", x, y), ("c", x, y + 1))


def _down_edges(x: int, y: int):
    return (("b", x + 1, y), ("a", x, y + 1), ("c", x, y + 1))


def _edge_at(x: int, y: int, k: int):
    """The edge leaving vertex (x, y) in direction k (lozenge.py:58-70)."""
    return (("a", x, y), ("b", x, y), ("c", x - 1, y + 1), ("a", x - 1, y), ("b", x, y - 1), ("c", x, y))[k]


def _edge_triangles(kind: str, x: int, y: int):
    if kind == "a":
        return ("up", x, y), ("down", x, y - 1)
    if kind == "b":
        return ("up", x, y), ("down", x - 1, y)
    return ("up", x, y - 1), ("down", x, y - 1)


def _star_triangles(x: int, y: int):
    return [("up", x, y), ("up", x - 1, y), ("up", x, y - 1), ("down", x - 1, y), ("down", x, y - 1),
            ("down", x - 1, y - 1)]


def shared_edge(a: Triangle, b: Triangle):
    if a[0] == "down":
        a, b = b, a
    if a[0] != "up" or b[0] != "down":
        raise OutOfDomainError(f"a lozenge needs one up and one down triangle: {a}, {b}")
    common = set(_up_edges(a[1], a[2])) & set(_down_edges(b[1], b[2]))
    if len(common) != 1:
        raise OutOfDomainError(f"triangles {a} and {b} are not adjacent")
    return common.pop()


def _derive_rotation_masks() -> tuple[int, int]:
    """Enumerate the three-lozenge covers of a vertex star (lozenge.py:107-138)."""
    x = y = 1
    ups = [t for t in _star_triangles(x, y) if t[0] == "up"]
    downs = [t for t in _star_triangles(x, y) if t[0] == "down"]
    masks = []
    for perm in permutations(range(3)):
        try:
            edges = {shared_edge(ups[i], downs[perm[i]]) for i in range(3)}
        except OutOfDomainError:
            continue
        state = sum(1 << k for k in range(6) if _edge_at(x, y, k) in edges)
        if bin(state).count("1") == 3:
            masks.append(state)
    masks = sorted(set(masks))
    assert len(masks) == 2, masks
    hi, lo = sorted(masks, key=lambda s: -_STEPS[0][bool(s & 1)], reverse=True)
    return hi, lo


ROT_HIGH, ROT_LOW = _derive_rotation_masks()


@dataclass(frozen=True, eq=False)
class TriDomain:
    """A simply-connected union of up/down triangles (lozenge.py:144-282)."""

    size: tuple[int, int]
    up: np.ndarray
    down: np.ndarray

    def __post_init__(self):
        sx, sy = self.size
        up = np.asarray(self.up, dtype=bool)
        down = np.asarray(self.down, dtype=bool)
        if up.shape != (sx, sy) or down.shape != (sx, sy):
            raise DomainError(f"triangle grids must be {self.size}")
        object.__setattr__(self, "up", up)
        object.__setattr__(self, "down", down)
        if not (up.any() or down.any()):
            raise DomainError("domain has no triangles")
        if up.size > _TRI_DEVICE_CELLS and _native.has_device():
            self._check_device()
        else:
            self._check_connected()
            self._check_simply_connected()

    def _check_device(self):
        """Both checks of lozenge.py:185-210 on the GPU (tsb_tri_check:
        union-find over the triangle graph, Euler characteristic V - E + F)."""
        import ctypes

        sx, sy = self.size
        u = np.ascontiguousarray(self.up, dtype=np.uint8)
        d = np.ascontiguousarray(self.down, dtype=np.uint8)
        k, chi = ctypes.c_int64(), ctypes.c_int64()
        _native.check(_native.lib().tsb_tri_check(_native.device(), _native.ptr(u), _native.ptr(d), sx, sy,
                                                  ctypes.byref(k), ctypes.byref(chi)))
        if k.value != 1:
            raise DomainError("triangles are not edge-connected")
        if chi.value != 1:
            raise DomainError("triangle set is not simply connected")

    def triangle_in(self, tri: Triangle) -> bool:
        kind, x, y = tri
        sx, sy = self.size
        if not (0 <= x < sx and 0 <= y < sy):
            return False
        return bool((self.up if kind == "up" else self.down)[x, y])

    def triangles(self) -> list[Triangle]:
        out = [("up", int(x), int(y)) for x, y in np.argwhere(self.up)]
        out += [("down", int(x), int(y)) for x, y in np.argwhere(self.down)]
        return sorted(out, key=lambda t: (t[1], t[2], t[0] == "down"))

    def _check_connected(self):
        from scipy.sparse import coo_matrix
        from scipy.sparse.csgraph import connected_components

        sx, sy = self.size
        n = sx * sy
        uid = np.arange(n).reshape(sx, sy)
        rows, cols = [], []
        # up(x,y) ~ down(x,y), down(x-1,y), down(x,y-1)
        for dx, dy in ((0, 0), (-1, 0), (0, -1)):
            xs, ys = np.nonzero(self.up)
            xd, yd = xs + dx, ys + dy
            ok = (xd >= 0) & (yd >= 0) & (xd < sx) & (yd < sy)
            xs, ys, xd, yd = xs[ok], ys[ok], xd[ok], yd[ok]
            ok = self.down[xd, yd]
            rows.append(uid[xs[ok], ys[ok]])
            cols.append(n + uid[xd[ok], yd[ok]])
        r = np.concatenate(rows)
        c = np.concatenate(cols)
        g = coo_matrix((np.ones(len(r), dtype=np.int8), (r, c)), shape=(2 * n, 2 * n))
        _, labels = connected_components(g, directed=False)
        present = np.concatenate([self.up.ravel(), self.down.ravel()])
        if len(np.unique(labels[present])) != 1:
            raise DomainError("triangles are not edge-connected")

    def _check_simply_connected(self):
        """Euler characteristic of a disk: V - E + F = 1 (lozenge.py:197-210)."""
        sx, sy = self.size
        ea = np.zeros((sx + 2, sy + 2), bool)
        eb = np.zeros_like(ea)
        ec = np.zeros_like(ea)
        ux, uy = np.nonzero(self.up)
        dx, dy = np.nonzero(self.down)
        ea[ux, uy] = True
        eb[ux, uy] = True
        ec[ux, uy + 1] = True
        eb[dx + 1, dy] = True
        ea[dx, dy + 1] = True
        ec[dx, dy + 1] = True
        e = int(ea.sum() + eb.sum() + ec.sum())
        v = int(self.vertex_mask.sum())
        f = int(self.up.sum() + self.down.sum())
        if v - e + f != 1:
            raise DomainError("triangle set is not simply connected")

    @cached_property
    def triangle_count(self) -> int:
        return int(self.up.sum() + self.down.sum())

    @cached_property
    def vertex_mask(self) -> np.ndarray:
        sx, sy = self.size
        m = np.zeros((sx + 1, sy + 1), dtype=bool)
        u, d = self.up, self.down
        m[:-1, :-1] |= u
        m[1:, :-1] |= u
        m[:-1, 1:] |= u
        m[1:, :-1] |= d
        m[:-1, 1:] |= d
        m[1:, 1:] |= d
        return m

    @cached_property
    def reference_vertex(self) -> tuple[int, int]:
        xs, ys = np.nonzero(self.vertex_mask)
        i = np.lexsort((ys, xs))[0]
        return (int(xs[i]), int(ys[i]))

    @classmethod
    def hexagon(cls, a: int, b: int, c: int) -> "TriDomain":
        """Hexagon with side lengths (a, b, c, a, b, c) (lozenge.py:233-247)."""
        if min(a, b, c) < 1:
            raise DomainError("hexagon sides must be positive")
        sx, sy = a + c, b + c
        s = np.add.outer(np.arange(sx), np.arange(sy))
        up = (s >= c) & (s + 1 <= a + b + c)
        down = (s + 1 >= c) & (s + 2 <= a + b + c)
        return cls((sx, sy), up, down)

    @classmethod
    def from_text(cls, text: str) -> "TriDomain":
        lines = [ln.strip() for ln in text.strip().splitlines() if ln.strip()]
        try:
            sx, sy = (int(tok) for tok in lines[0].split())
        except (ValueError, IndexError) as exc:
            raise DomainError("triangle domain file must start with 'sx sy'") from exc
        if len(lines) != 1 + 2 * sx:
            raise DomainError(f"expected {2 * sx} grid rows, got {len(lines) - 1}")

        def parse(rows):
            grid = np.zeros((sx, sy), dtype=bool)
            for x, ln in enumerate(rows):
                if len(ln) != sy or set(ln) - {"0", "1"}:
                    raise DomainError(f"row {x} must be {sy} characters of 0/1")
                grid[x] = [ch == "1" for ch in ln]
            return grid

        return cls((sx, sy), parse(lines[1 : 1 + sx]), parse(lines[1 + sx :]))

    def to_text(self) -> str:
        rows = [f"{self.size[0]} {self.size[1]}"]
        for grid in (self.up, self.down):
            rows += ["".join("1" if v else "0" for v in row) for row in grid]
        return "\n".join(rows) + "\n"

    @cached_property
    def _key(self):
        return hash((self.size, self.up.tobytes(), self.down.tobytes()))

    def __eq__(self, other):
        return (isinstance(other, TriDomain) and self.size == other.size
                and np.array_equal(self.up, other.up) and np.array_equal(self.down, other.down))

    def __hash__(self):
        return self._key


@dataclass(frozen=True, eq=False)
class LozengeTiling:
    """Crossed-edge grids of a lozenge tiling (lozenge.py:285-330)."""

    domain: TriDomain
    edges: np.ndarray

    def __post_init__(self):
        sx, sy = self.domain.size
        e = np.asarray(self.edges, dtype=bool)
        if e.shape != (3, sx + 1, sy + 1):
            raise InconsistencyError("edge grids have the wrong shape")
        object.__setattr__(self, "edges", e)

    def edge_crossed(self, kind: str, x: int, y: int) -> bool:
        sx, sy = self.domain.size
        if not (0 <= x <= sx and 0 <= y <= sy):
            return False
        return bool(self.edges["abc".index(kind), x, y])

    def state(self, vertex) -> int:
        x, y = vertex
        return sum(1 << k for k in range(6) if self.edge_crossed(*_edge_at(x, y, k)))

    @property
    def states_grid(self) -> np.ndarray:
        return states_grid_batch(self.edges[None])[0]

    def __eq__(self, other):
        return isinstance(other, LozengeTiling) and self.domain == other.domain and np.array_equal(
            self.edges, other.edges)

    def __hash__(self):
        return hash((self.domain, self.edges.tobytes()))


@dataclass(frozen=True)
class LozengeHeights:
    domain: TriDomain
    heights: np.ndarray

    def __eq__(self, other):
        m = self.domain.vertex_mask
        return (isinstance(other, LozengeHeights) and self.domain == other.domain
                and np.array_equal(self.heights[m], other.heights[m]))

    def __hash__(self):
        return hash((self.domain, self.heights[self.domain.vertex_mask].tobytes()))


def tiling_from_lozenges(domain: TriDomain, lozenges: Iterable[Lozenge]) -> LozengeTiling:
    sx, sy = domain.size
    edges = np.zeros((3, sx + 1, sy + 1), dtype=bool)
    covered: set = set()
    for a, b in lozenges:
        for t in (a, b):
            if not domain.triangle_in(t):
                raise OutOfDomainError(f"triangle {t} not in domain")
            if t in covered:
                raise OverlapError(f"triangle {t} covered twice")
            covered.add(t)
        kind, x, y = shared_edge(a, b)
        edges["abc".index(kind), x, y] = True
    if len(covered) != domain.triangle_count:
        raise CoverageError("triangles left uncovered")
    return LozengeTiling(domain, edges)


def lozenges_from_tiling(t: LozengeTiling) -> list[Lozenge]:
    domain = t.domain
    covered: set = set()
    out = []
    for idx, kind in enumerate("abc"):
        for x, y in np.argwhere(t.edges[idx]):
            tri_u, tri_d = _edge_triangles(kind, int(x), int(y))
            for tri in (tri_u, tri_d):
                if not domain.triangle_in(tri):
                    raise OutOfDomainError(f"crossed edge {kind, x, y} leaves the domain")
                if tri in covered:
                    raise OverlapError(f"triangle {tri} covered twice")
                covered.add(tri)
            out.append((tri_u, tri_d))
    if len(covered) != domain.triangle_count:
        raise CoverageError("decoded lozenges do not cover the domain")
    return sorted(out)


def is_valid_lozenge_tiling(t: LozengeTiling) -> bool:
    try:
        lozenges_from_tiling(t)
        return True
    except (OverlapError, CoverageError, OutOfDomainError):
        return False


def loz_rotateable(s: int) -> str:
    if s == ROT_LOW:
        return "up"
    if s == ROT_HIGH:
        return "down"
    return "none"


def states_grid_batch(edges: np.ndarray) -> np.ndarray:
    """Vertex states for a batch of edge grids (lozenge.py:453-468)."""
    ea, eb, ec = edges[:, 0], edges[:, 1], edges[:, 2]
    s = ea.astype(np.uint8)
    s |= np.uint8(2) * eb
    d2 = np.zeros_like(ea)
    d2[:, 1:, :-1] = ec[:, :-1, 1:]
    s |= np.uint8(4) * d2
    d3 = np.zeros_like(ea)
    d3[:, 1:, :] = ea[:, :-1, :]
    s |= np.uint8(8) * d3
    d4 = np.zeros_like(ea)
    d4[:, :, 1:] = eb[:, :, :-1]
    s |= np.uint8(16) * d4
    s |= np.uint8(32) * ec
    return s


def star_covers(vertex):
    x, y = vertex
    high = [(("up", x, y), ("down", x, y - 1)), (("up", x - 1, y), ("down", x - 1, y)),
            (("up", x, y - 1), ("down", x - 1, y - 1))]
    low = [(("up", x, y), ("down", x - 1, y)), (("up", x - 1, y), ("down", x - 1, y - 1)),
           (("up", x, y - 1), ("down", x, y - 1))]
    return high, low


@dataclass(frozen=True)
class LozEdgeWeights:
    """Positive weight per lozenge placement (lozenge.py:525-542)."""

    default: float = 1.0
    overrides: dict = None  # type: ignore[assignment]

    def __post_init__(self):
        canon = {frozenset(k): float(v) for k, v in (self.overrides or {}).items()}
        if self.default <= 0 or any(w <= 0 for w in canon.values()):
            raise ValueError("lozenge edge weights must be strictly positive")
        object.__setattr__(self, "overrides", canon)

    def weight(self, tri_a: Triangle, tri_b: Triangle) -> float:
        return self.overrides.get(frozenset((tri_a, tri_b)), self.default)

    def __hash__(self):
        return hash((self.default, tuple(sorted((tuple(sorted(k)), v) for k, v in self.overrides.items()))))


def loz_p_up_grid(domain: TriDomain, weights) -> np.ndarray:
    """Static per-vertex probability of the high state (lozenge.py:545-566),
    bit-identical: powers on the few distinct q values with Python floats,
    edge-weight stars near overrides with the reference's own np.prod."""
    sx, sy = domain.size
    if isinstance(weights, Uniform):
        return np.full((sx + 1, sy + 1), 0.5)
    if isinstance(weights, VolumeWeights):
        ratio = weights.default ** CUBE_UNIT
        grid = np.full((sx + 1, sy + 1), ratio / (1.0 + ratio))
        for (x, y), q in weights.overrides.items():
            if 0 <= x <= sx and 0 <= y <= sy:
                r = q ** CUBE_UNIT
                grid[x, y] = r / (1.0 + r)
        return grid
    if isinstance(weights, LozEdgeWeights):
        grid = np.empty((sx + 1, sy + 1))
        d = weights.default
        w = np.prod([d, d, d])
        grid[:] = w / (w + w)
        touched = set()
        for key in weights.overrides:
            for kind, x, y in key:
                for dx in (-1, 0, 1):
                    for dy in (-1, 0, 1):
                        touched.add((x + dx, y + dy))
        for x, y in touched:
            if 0 <= x <= sx and 0 <= y <= sy:
                high, low = star_covers((x, y))
                w_hi = np.prod([weights.weight(*loz) for loz in high])
                w_lo = np.prod([weights.weight(*loz) for loz in low])
                grid[x, y] = w_hi / (w_hi + w_lo)
        return grid
    raise TypeError(f"unsupported lozenge weight spec {type(weights)!r}")


# -- device handles ----------------------------------------------------------------


class LozengeHandle:
    """A batch of device-resident lozenge chains (tsb_loz)."""

    def __init__(self, domain: TriDomain, nchains: int, device: int | None = None):
        self.domain = domain
        sx, sy = domain.size
        self.X, self.Y = sx + 1, sy + 1
        self.nchains = nchains
        self.device = _native.device() if device is None else device
        self._h = ctypes.c_void_p()
        self._p_ref = None
        up = np.ascontiguousarray(domain.up, dtype=np.uint8)
        dn = np.ascontiguousarray(domain.down, dtype=np.uint8)
        _native.check(_native.lib().tsb_loz_create(self.device, sx, sy, nchains, _native.ptr(up), _native.ptr(dn),
                                                   ctypes.byref(self._h)))

    def __del__(self):
        try:
            if self._h:
                _native.lib().tsb_loz_destroy(self._h)
                self._h = ctypes.c_void_p()
        except Exception:
            pass

    def set_stream(self, stream_ptr: int):
        _native.check(_native.lib().tsb_loz_set_stream(self._h, ctypes.c_void_p(stream_ptr)))

    def set_collapse(self, on: bool):
        """Class-run collapsing (tsb_loz_set_collapse); bit-identical results."""
        _native.check(_native.lib().tsb_loz_set_collapse(self._h, int(bool(on))))

    def set_p_up(self, p_up: np.ndarray):
        if self._p_ref is p_up:
            return
        p = np.ascontiguousarray(p_up, dtype=np.float64)
        _native.check(_native.lib().tsb_loz_set_p_up(self._h, _native.ptr(p)))
        self._p_ref = p_up

    def upload(self, edges: np.ndarray, chain0: int = 0):
        e = np.ascontiguousarray(edges, dtype=np.uint8)
        _native.check(_native.lib().tsb_loz_upload(self._h, chain0, e.shape[0], _native.ptr(e)))

    def download(self, chain0: int = 0, n: int | None = None) -> np.ndarray:
        n = self.nchains - chain0 if n is None else n
        out = np.empty((n, 3, self.X, self.Y), dtype=np.uint8)
        _native.check(_native.lib().tsb_loz_download(self._h, chain0, n, _native.ptr(out)))
        return out.astype(bool)

    def walk(self, seeds, n_steps: int, step0: int = 0, chain0: int = 0):
        s = np.ascontiguousarray(seeds, dtype=np.uint64)
        _native.check(_native.lib().tsb_loz_walk(self._h, chain0, s.shape[0], _native.ptr(s), _native.u64(step0),
                                                 int(n_steps)))

    def sweep(self, seeds, step: int, color: int, chain0: int = 0):
        s = np.ascontiguousarray(seeds, dtype=np.uint64)
        _native.check(_native.lib().tsb_loz_sweep(self._h, chain0, s.shape[0], _native.ptr(s), _native.u64(step),
                                                  int(color)))

    def sync(self):
        _native.check(_native.lib().tsb_loz_sync(self._h))

    def heights(self, chain: int, ref) -> np.ndarray:
        out = np.empty((self.X, self.Y), dtype=np.int32)
        _native.check(_native.lib().tsb_loz_heights(self._h, chain, int(ref[0]), int(ref[1]), _native.ptr(out)))
        return out

    def extremal(self, ref, chain_max: int = 0, chain_min: int = 1) -> bool:
        rc = _native.lib().tsb_loz_extremal(self._h, chain_max, chain_min, int(ref[0]), int(ref[1]))
        if rc == _native.E_UNTILEABLE:
            return False
        _native.check(rc)
        return True


_CACHE: "OrderedDict[tuple, LozengeHandle]" = OrderedDict()


def _loz_handle(domain: TriDomain, nchains: int) -> LozengeHandle:
    key = (domain._key, nchains, _native.device())
    h = _CACHE.get(key)
    if h is None:
        h = LozengeHandle(domain, nchains)
        _CACHE[key] = h
        while len(_CACHE) > 8:
            _CACHE.popitem(last=False)
    else:
        _CACHE.move_to_end(key)
    return h


def loz_heights(t: LozengeTiling) -> LozengeHeights:
    """Heights over the domain's vertex graph (lozenge.py:414-447), on the device."""
    h = _loz_handle(t.domain, 1)
    h.upload(t.edges[None])
    return LozengeHeights(t.domain, h.heights(0, t.domain.reference_vertex))


def loz_sweep_batch_device(edges, seeds, step, color, domain, weights):
    h = _loz_handle(domain, edges.shape[0])
    h.set_p_up(_p_up_cached(domain, weights))
    h.upload(edges)
    h.sweep(seeds, step, color)
    return h.download()


_P_CACHE: "OrderedDict[tuple, np.ndarray]" = OrderedDict()


def _p_up_cached(domain: TriDomain, weights) -> np.ndarray:
    key = (domain._key, weights)
    p = _P_CACHE.get(key)
    if p is None:
        p = loz_p_up_grid(domain, weights)
        _P_CACHE[key] = p
        while len(_P_CACHE) > 8:
            _P_CACHE.popitem(last=False)
    return p


def loz_random_walk_batch(edges: np.ndarray, seeds: np.ndarray, n_steps: int, domain: TriDomain, weights,
                          backend: Backend | None = None) -> np.ndarray:
    """Evolve a (B, 3, sx+1, sy+1) edge batch on the device (lozenge.py:600-622)."""
    edges = np.asarray(edges)
    if n_steps <= 0 or edges.shape[0] == 0:
        return edges.copy()
    h = _loz_handle(domain, edges.shape[0])
    h.set_p_up(_p_up_cached(domain, weights))
    h.upload(edges)
    h.walk(np.asarray(seeds, dtype=np.uint64), n_steps)
    return h.download()


def loz_sweep(t: LozengeTiling, f: rng.StreamFamily, step: int, color: int, weights=None,
              backend: Backend | None = None) -> LozengeTiling:
    """Rotate every vertex of one colour class (lozenge.py:625-646)."""
    weights = weights or Uniform()
    out = loz_sweep_batch_device(t.edges[None], [f.seed], step, color, t.domain, weights)
    return LozengeTiling(t.domain, out[0])


def loz_random_walk(t: LozengeTiling, seed: int, n_steps: int, weights=None,
                    backend: Backend | None = None) -> LozengeTiling:
    weights = weights or Uniform()
    out = loz_random_walk_batch(t.edges[None], np.array([seed], dtype=np.uint64), n_steps, t.domain, weights, backend)
    return LozengeTiling(t.domain, out[0])


def loz_extremal(domain: TriDomain) -> Optional[tuple[LozengeTiling, LozengeTiling]]:
    """Maximal and minimal tilings, or None when untileable (lozenge.py:762-775)."""
    if int(domain.up.sum()) != int(domain.down.sum()):
        return None
    h = _loz_handle(domain, 2)
    if not h.extremal(domain.reference_vertex):
        return None
    e = h.download()
    return LozengeTiling(domain, e[0]), LozengeTiling(domain, e[1])


def loz_cftp(domain: TriDomain, weights, master_seed: int, backend: Backend | None = None, max_doublings: int = 40,
             count: int = 1, progress=None, trace: CftpTrace | None = None, batch_size: int = 2048):
    """Exact samples of lozenge tilings via monotone CFTP (lozenge.py:778-827)."""
    weights = weights or Uniform()
    extremals = loz_extremal(domain)
    if extremals is None:
        raise UntileableDomain("triangle domain is not tileable")
    t_max, t_min = extremals
    cb = _progress_writer(progress)
    results: list[LozengeTiling] = []
    if np.array_equal(t_max.edges, t_min.edges):
        results = [t_max] * count
    else:
        for lo in range(0, count, batch_size):
            hi = min(lo + batch_size, count)
            masters = np.array([chain_master_seed(master_seed, k) for k in range(lo, hi)], dtype=np.uint64)
            out = _loz_cftp_device(domain, weights, t_max.edges, t_min.edges, masters, max_doublings, cb,
                                   trace if lo == 0 else None)
            results.extend(LozengeTiling(domain, e) for e in out)
    return results[0] if count == 1 else results


def loz_cftp_distributed(domain: TriDomain, weights, master_seed: int, count: int, group=None,
                         max_doublings: int = 40) -> list[LozengeTiling]:
    """loz_cftp(..., count=count) with the samples spread round-robin over the
    ranks of a torch.distributed group (cftp.distribute_samples); equal to
    the one-GPU result.  Every rank returns the full list."""
    from .cftp import distribute_samples

    weights = weights or Uniform()
    extremals = loz_extremal(domain)
    if extremals is None:
        raise UntileableDomain("triangle domain is not tileable")
    t_max, t_min = extremals
    if np.array_equal(t_max.edges, t_min.edges):
        return [t_max] * count

    def run(mine):
        masters = np.array([chain_master_seed(master_seed, k) for k in mine], dtype=np.uint64)
        return _loz_cftp_device(domain, weights, t_max.edges, t_min.edges, masters, max_doublings, None, None)

    return [LozengeTiling(domain, e) for e in distribute_samples(count, run, group)]


def _loz_cftp_device(domain, weights, top0, bot0, masters, max_doublings, progress, trace):
    from .sixvertex import _fill_trace

    b = len(masters)
    h = _loz_handle(domain, 2 * b + 2)
    h.set_p_up(_p_up_cached(domain, weights))
    sx, sy = domain.size
    out = np.zeros((b, 3, sx + 1, sy + 1), dtype=np.uint8)
    rounds = np.zeros(b, dtype=np.int32)
    cb = _native.PROGRESS_FN(lambda r, s, c, t, u: progress(r, int(s), c, t)) if progress else None
    top0 = np.ascontiguousarray(top0, dtype=np.uint8)
    bot0 = np.ascontiguousarray(bot0, dtype=np.uint8)
    rc = _native.lib().tsb_loz_cftp(h._h, _native.ptr(top0), _native.ptr(bot0), _native.ptr(masters), b,
                                    int(max_doublings), _native.ptr(out), _native.ptr(rounds),
                                    ctypes.cast(cb, ctypes.c_void_p) if cb else None, None)
    _fill_trace(trace, masters, rounds, rc, max_doublings)
    _native.check(rc)
    return out.astype(bool)
