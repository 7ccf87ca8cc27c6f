"""The documented drop-in hook: `tsb_domino_walk_host` bound exactly as
INTEGRATION.md §1 shows (a fresh ctypes CDLL, in place on a C-contiguous
(B, V, V) uint8 batch, with and without `faces`), and called from a plain C
program linked against libtsb.so.  It replaces the reference's fused hook
`_fused_walk(out, site_keys, global_keys, p_up, n_steps)` (sweeps.py:272-275,
306-309; numba `domino_walk`, _kernels.py:35-69); results are compared with
the reference-generated goldens (tests/golden/domino_walks.npz)."""

import ctypes
import os
import subprocess

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_1804_07250_b200", "_lib", "libtsb.so")
G = os.path.join(os.path.dirname(__file__), "golden")


def _bind():
    # verbatim from INTEGRATION.md §1
    _tsb = ctypes.CDLL(LIB)
    _tsb.tsb_domino_walk_host.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                                          ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64]
    _tsb.tsb_last_error.restype = ctypes.c_char_p

    def _device_walk(out, seeds, p_up, n_steps, faces=None):
        """In place on a C-contiguous (B, V, V) uint8 batch (== domino_walk)."""
        seeds = np.ascontiguousarray(seeds, dtype=np.uint64)
        p_up = np.ascontiguousarray(p_up, dtype=np.float64)
        f = None if faces is None else np.ascontiguousarray(faces, dtype=np.uint8)
        rc = _tsb.tsb_domino_walk_host(0, out.ctypes.data, out.shape[0], out.shape[-1],
                                       seeds.ctypes.data, p_up.ctypes.data,
                                       None if f is None else f.ctypes.data, n_steps)
        if rc:
            raise RuntimeError(_tsb.tsb_last_error().decode())

    return _device_walk


def _cases():
    g = np.load(os.path.join(G, "domino_walks.npz"))
    i = 0
    while f"c{i}_faces" in g:
        yield i, g[f"c{i}_faces"], g[f"c{i}_start"], g[f"c{i}_seeds"], int(g[f"c{i}_n_steps"]), \
            g[f"c{i}_p_up"], g[f"c{i}_out"]
        i += 1


@pytest.mark.parametrize("with_faces", [True, False])
def test_walk_host_ctypes_matches_reference(with_faces):
    walk = _bind()
    n = 0
    for i, faces, start, seeds, n_steps, p_up, ref in _cases():
        out = np.array(start, dtype=np.uint8, order="C")  # states.astype(np.uint8, copy=True)
        walk(out, seeds, p_up, n_steps, faces if with_faces else None)
        assert np.array_equal(out, ref), f"case {i}"
        n += 1
    assert n >= 4


def test_walk_host_c1_config():
    """BASELINE config 1 through the hook: Aztec 64, T_max, 0x5EED, 1000 sweeps."""
    g = np.load(os.path.join(G, "domino_c1.npz"))
    walk = _bind()
    out = g["t_max"][None].copy()
    walk(out, [0x5EED], np.full(out.shape[1:], 0.5), 1000)
    assert np.array_equal(out[0], g["final"])


def test_walk_host_errors():
    walk = _bind()
    bad = np.full((1, 9, 9), 99, dtype=np.uint8)
    with pytest.raises(RuntimeError, match="< 16"):
        walk(bad, [1], np.full((9, 9), 0.5), 3)


def test_walk_host_from_c_program(tmp_path):
    """A C caller (no Python on the call path) walks every golden case."""
    root_inc = ROOT
    src = tmp_path / "walk.c"
    src.write_text(r'''
#include "include/tsb.h"
#include <stdio.h>
#include <stdlib.h>
/* usage: walk in.bin out.bin B V n_steps   (in.bin: states, seeds, p_up) */
int main(int argc, char **argv) {
    int B = atoi(argv[3]), V = atoi(argv[4]);
    unsigned long long n = strtoull(argv[5], 0, 10);
    size_t ns = (size_t)B * V * V;
    uint8_t *st = malloc(ns); uint64_t *seeds = malloc(8 * (size_t)B); double *p = malloc(8 * (size_t)V * V);
    FILE *f = fopen(argv[1], "rb");
    if (fread(st, 1, ns, f) != ns || fread(seeds, 8, B, f) != (size_t)B ||
        fread(p, 8, (size_t)V * V, f) != (size_t)V * V) return 3;
    fclose(f);
    int rc = tsb_domino_walk_host(0, st, B, V, seeds, p, NULL, n);
    if (rc) { fprintf(stderr, "%s\n", tsb_last_error()); return 1; }
    f = fopen(argv[2], "wb"); fwrite(st, 1, ns, f); fclose(f);
    return 0;
}
''')
    lib_dir = os.path.dirname(LIB)
    exe = tmp_path / "walk"
    subprocess.run(["gcc", "-std=c99", "-O1", "-I", root_inc, str(src), "-L", lib_dir, "-ltsb",
                    f"-Wl,-rpath,{lib_dir}", "-o", str(exe)], check=True)
    for i, faces, start, seeds, n_steps, p_up, ref in _cases():
        start = np.ascontiguousarray(start, dtype=np.uint8)
        b, v = start.shape[0], start.shape[-1]
        fin, fout = tmp_path / f"in{i}.bin", tmp_path / f"out{i}.bin"
        with open(fin, "wb") as f:
            f.write(start.tobytes())
            f.write(np.ascontiguousarray(seeds, dtype=np.uint64).tobytes())
            f.write(np.ascontiguousarray(p_up, dtype=np.float64).tobytes())
        subprocess.run([str(exe), str(fin), str(fout), str(b), str(v), str(n_steps)], check=True)
        out = np.fromfile(fout, dtype=np.uint8).reshape(start.shape)
        assert np.array_equal(out, ref), f"case {i}"
