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
