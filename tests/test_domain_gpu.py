"""Device domain validation (tsb_grid_components) vs
scipy labelling, and the Domain errors of lattice.py:99-132 on large grids."""

import ctypes

import numpy as np
import pytest

import paper_1804_07250_b200 as ts
from paper_1804_07250_b200 import _native
from paper_1804_07250_b200.lattice import _label_count

pytestmark = pytest.mark.gpu


def _gpu_components(mask):
    g = np.ascontiguousarray(mask, dtype=np.uint8)
    k = ctypes.c_int64()
    _native.check(_native.lib().tsb_grid_components(0, _native.ptr(g), g.shape[0], g.shape[1], ctypes.byref(k)))
    return k.value


@pytest.mark.parametrize("shape,p", [((1, 1), 1.0), ((7, 13), 0.5), ((300, 257), 0.45), ((1000, 999), 0.6),
                                     ((2048, 2048), 0.5), ((5000, 3000), 0.59)])
def test_components_match_scipy(shape, p):
    rng = np.random.default_rng(shape[0] * 7 + shape[1])
    mask = rng.random(shape) < p
    assert _gpu_components(mask) == _label_count(mask)[1]


def test_large_domains():
    assert _native.has_device()
    d = ts.Domain.aztec(2048)  # 16.8 M faces: the device check
    assert d.faces.sum() == 2 * 2048 * 2049
    faces = d.faces.copy()
    faces[2048, 2048] = False  # a hole in the middle
    with pytest.raises(ts.DomainError):
        ts.Domain(d.n, faces)
    faces = d.faces.copy()
    faces[2040:2056, :] = False  # cut into two pieces
    with pytest.raises(ts.DomainError):
        ts.Domain(d.n, faces)


def _tri_device(up, down):
    u = np.ascontiguousarray(up, dtype=np.uint8)
    d = np.ascontiguousarray(down, dtype=np.uint8)
    k, chi = ctypes.c_int64(), ctypes.c_int64()
    _native.check(_native.lib().tsb_tri_check(0, _native.ptr(u), _native.ptr(d), u.shape[0], u.shape[1],
                                              ctypes.byref(k), ctypes.byref(chi)))
    return k.value, chi.value


def _tri_host(up, down):
    """The host restatement's two checks (lozenge.py:185-210), as booleans."""
    from paper_1804_07250_b200.lozenge import TriDomain

    t = TriDomain.__new__(TriDomain)
    object.__setattr__(t, "size", up.shape)
    object.__setattr__(t, "up", up)
    object.__setattr__(t, "down", down)
    res = []
    for check in (t._check_connected, t._check_simply_connected):
        try:
            check()
            res.append(True)
        except ts.DomainError:
            res.append(False)
    return res


@pytest.mark.parametrize("shape,p,seed", [((5, 7), 0.7, 1), ((40, 33), 0.8, 2), ((200, 150), 0.9, 3),
                                          ((64, 64), 0.97, 4), ((300, 301), 0.995, 5)])
def test_tri_check_matches_host(shape, p, seed):
    """tsb_tri_check (device TriDomain validation) agrees with the host
    checks on random triangle sets, connected or not, with or without holes."""
    rng = np.random.default_rng(seed)
    for _ in range(6):
        up = rng.random(shape) < p
        down = rng.random(shape) < p
        if not (up.any() or down.any()):
            continue
        k, chi = _tri_device(up, down)
        conn, simple = _tri_host(up, down)
        assert (k == 1) == conn
        if conn:
            assert (chi == 1) == simple


def test_large_tri_domains():
    """hexagon(1000) is validated on the device; a hole and
    a cut raise DomainError exactly like the reference's checks."""
    d = ts.TriDomain.hexagon(1000, 1000, 1000)
    k, chi = _tri_device(d.up, d.down)
    assert (k, chi) == (1, 1)
    up, down = d.up.copy(), d.down.copy()
    up[1000, 700] = down[1000, 700] = False  # a hole of two triangles in the middle
    with pytest.raises(ts.DomainError, match="simply connected"):
        ts.TriDomain(d.size, up, down)
    up, down = d.up.copy(), d.down.copy()
    up[990:1010, :] = down[990:1010, :] = False
    with pytest.raises(ts.DomainError, match="edge-connected"):
        ts.TriDomain(d.size, up, down)
