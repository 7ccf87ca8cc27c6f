"""CPU parity oracle for the reference `tilesampler` hot path.

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference leg may import this package; the
product (`paper_1804_07250_b200`) never does and has no CPU fallback.

`tsb_oracle.c` restates the reference's splitmix64 streams and the three
Glauber sweeps (dominoes `_kernels.py:35-69`, six-vertex
`sixvertex.py:369-467`, lozenges `lozenge.py:453-622`) in plain C.  It is
pinned against golden vectors produced by the Python reference itself
(tests/golden/make_golden.py -> tests/golden/*.npz, checked by
tests/test_oracle_golden.py).

Heights and extremal states are checked directly against the reference's
own outputs stored in tests/golden/ (they are unique fixpoints).
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

_u64 = ctypes.c_uint64
_p = ctypes.c_void_p


def build() -> str:
    """Compile liboracle.so with the committed Makefile (gcc only)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(
            os.path.join(_HERE, "tsb_oracle.c")
        ):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        for name in ("orc_mix", "orc_base", "orc_global_key"):
            getattr(L, name).restype = _u64
            getattr(L, name).argtypes = [_u64]
        L.orc_splitmix_at.restype = _u64
        L.orc_splitmix_at.argtypes = [_u64, _u64]
        L.orc_derive_seed.restype = _u64
        L.orc_derive_seed.argtypes = [_u64, _u64, _u64]
        L.orc_site_key.restype = _u64
        L.orc_site_key.argtypes = [_u64, _u64, _u64, _u64, _u64]
        L.orc_uniform_from_key.restype = ctypes.c_double
        L.orc_uniform_from_key.argtypes = [_u64, _u64]
        L.orc_uniform_grid.argtypes = [_u64, ctypes.c_int, ctypes.c_int, _u64, _u64, _p]
        L.orc_domino_walk.argtypes = [_p, ctypes.c_int, ctypes.c_int, _p, _p, _u64, _u64, ctypes.c_int]
        L.orc_domino_walk_window.argtypes = [_p, ctypes.c_int, ctypes.c_int, ctypes.c_int, _u64, _p, _u64, _u64]
        L.orc_domino_sweep.argtypes = [_p, ctypes.c_int, _u64, _p, _u64, ctypes.c_int]
        L.orc_sv_walk.argtypes = [_p, ctypes.c_int, ctypes.c_int, _p, _p, _u64, _u64]
        L.orc_loz_walk.argtypes = [_p, ctypes.c_int, ctypes.c_int, ctypes.c_int, _p, _p, _u64, _u64]
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def mix(z: int) -> int:
    return int(lib().orc_mix(z & (2**64 - 1)))


def derive_seed(seed: int, index: int, salt: int = 0) -> int:
    m = 2**64 - 1
    return int(lib().orc_derive_seed(seed & m, index & m, salt & m))


def site_key(seed: int, shape, site, tag: int = 0) -> int:
    return int(lib().orc_site_key(seed, tag, site[0], site[1], shape[1]))


def uniform_from_key(key: int, step: int) -> float:
    return float(lib().orc_uniform_from_key(key, step))


def uniform_grid(seed: int, shape, step: int, tag: int = 0) -> np.ndarray:
    out = np.empty(shape, dtype=np.float64)
    lib().orc_uniform_grid(seed, shape[0], shape[1], step, tag, _ptr(out))
    return out


def domino_walk(states: np.ndarray, seeds, p_up: np.ndarray, n_steps: int,
                step0: int = 0, threads: int = 1) -> np.ndarray:
    """Returns a new (B, V, V) uint8 array (reference random_walk_batch)."""
    out = np.ascontiguousarray(states, dtype=np.uint8).copy()
    if out.ndim == 2:
        out = out[None]
    seeds = np.ascontiguousarray(seeds, dtype=np.uint64)
    p = np.ascontiguousarray(p_up, dtype=np.float64)
    lib().orc_domino_walk(_ptr(out), out.shape[0], out.shape[-1], _ptr(seeds), _ptr(p),
                          step0, n_steps, threads)
    return out


def domino_walk_window(rows: np.ndarray, row0: int, seed: int, p_up_rows: np.ndarray, n_steps: int,
                       step0: int = 0) -> None:
    """In place on a (nrows, V) window of rows [row0, row0+nrows)."""
    assert rows.flags.c_contiguous and rows.dtype == np.uint8
    p = np.ascontiguousarray(p_up_rows, dtype=np.float64)
    lib().orc_domino_walk_window(_ptr(rows), rows.shape[0], rows.shape[1], row0, seed, _ptr(p), step0, n_steps)


def domino_sweep(states: np.ndarray, seed: int, p_up: np.ndarray, step: int, color: int):
    out = np.ascontiguousarray(states, dtype=np.uint8).copy()
    p = np.ascontiguousarray(p_up, dtype=np.float64)
    lib().orc_domino_sweep(_ptr(out), out.shape[-1], seed, _ptr(p), step, color)
    return out


def sv_walk(h: np.ndarray, seeds, table: np.ndarray, n_steps: int, step0: int = 0):
    out = np.ascontiguousarray(h, dtype=np.int32).copy()
    if out.ndim == 2:
        out = out[None]
    seeds = np.ascontiguousarray(seeds, dtype=np.uint64)
    t = np.ascontiguousarray(table, dtype=np.float64)
    lib().orc_sv_walk(_ptr(out), out.shape[0], out.shape[-1], _ptr(seeds), _ptr(t), step0, n_steps)
    return out


def loz_walk(edges: np.ndarray, seeds, p_up: np.ndarray, n_steps: int, step0: int = 0):
    out = np.ascontiguousarray(edges, dtype=np.uint8).copy()
    if out.ndim == 3:
        out = out[None]
    seeds = np.ascontiguousarray(seeds, dtype=np.uint64)
    p = np.ascontiguousarray(p_up, dtype=np.float64)
    lib().orc_loz_walk(_ptr(out), out.shape[0], out.shape[2], out.shape[3], _ptr(seeds), _ptr(p),
                       step0, n_steps)
    return out.astype(bool)


# ---------------------------------------------------------------- observables
# numpy restatements of the reference's statistics (stats.py:187-288); pinned
# against tests/golden/observables.npz (make_golden.py make_observables).

def domino_orientation(states: np.ndarray, faces: np.ndarray) -> np.ndarray:
    """stats.py:187-200 domino_orientation_grid: 1.0 where the face is covered
    by a horizontal domino (its left or right edge is interior to a domino,
    tilestate bit 2 "down" of the face's top-left / top-right corner), 0.0 for
    a vertical one, NaN outside the domain."""
    s = np.asarray(states)
    horiz = ((s[:-1, :-1] & 2) | (s[:-1, 1:] & 2)) != 0
    return np.where(faces, horiz.astype(float), np.nan)


def aztec_y_intercept(orient: np.ndarray) -> float:
    """stats.py:270-288 on an orientation grid: end of the top frozen
    horizontal cluster on the central column, relative to the centre row."""
    n = orient.shape[0]
    mid = n // 2
    col = orient[:, mid]
    rows = np.nonzero(~np.isnan(col))[0]
    boundary = rows[0]
    for r in rows:
        if col[r] == 1.0:
            boundary = r + 1
        else:
            break
    return float(boundary - mid)


def sv_edges(heights: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """config_from_heights (sixvertex.py:270-277): (h_edges, v_edges)."""
    h = np.asarray(heights).astype(np.int64)
    return (h[:-1, :] - h[1:, :]) == 1, (h[:, 1:] - h[:, :-1]) == 1


def sv_c_vertex(h_edges: np.ndarray, v_edges: np.ndarray) -> np.ndarray:
    """c-vertex indicator (stats.py:225-228, vertex_type_codes sixvertex.py:236-239)."""
    hh, vv = h_edges.astype(np.int8), v_edges.astype(np.int8)
    codes = hh[:, :-1] + 2 * hh[:, 1:] + 4 * vv[:-1, :] + 8 * vv[1:, :]
    return (codes == 0b1001) | (codes == 0b0110)
