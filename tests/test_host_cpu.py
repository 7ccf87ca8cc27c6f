"""Host-side logic that runs without a GPU: domain construction, p_up grids,
codecs, seed derivation, and the C-ABI library's exported symbols."""

import ctypes
import json
import os

import numpy as np
import pytest

import golden_cases as gc
import paper_1804_07250_b200 as ts
from paper_1804_07250_b200 import _native, rng
from paper_1804_07250_b200.cftp import chain_master_seed, schedule_seed

G = os.path.join(os.path.dirname(__file__), "golden")


def load(name):
    return np.load(os.path.join(G, name))


def test_library_exports_every_declared_symbol():
    path = _native.LIB_PATH
    if not os.path.exists(path):
        _native.build()
    lib = ctypes.CDLL(path)
    declared = _native.declared_symbols()
    assert "tsb_domino_walk" in declared and "tsb_domino_cftp" in declared
    for name in declared:
        if name == "tsb_progress_fn":
            continue
        assert hasattr(lib, name), name
    assert set(declared) - {"tsb_progress_fn"} <= set(_native._SIGS)


def test_no_cpu_fallback_without_device():
    try:
        import torch

        if torch.cuda.is_available():
            pytest.skip("device present")
    except ImportError:
        pass
    d = ts.Domain.square(2)
    with pytest.raises(RuntimeError, match="no CPU fallback|no CUDA device"):
        ts.random_walk_batch(np.zeros((1, 3, 3), np.uint8), [1], 1, ts.SweepPlan(d))


def test_rng_host_scalars_match_kats():
    kats = json.load(open(os.path.join(G, "rng_kats.json")))
    for k in kats["kats"]:
        fam = ts.seed_family(k["seed"], tuple(k["shape"]))
        assert fam.site_key(tuple(k["site"])) == k["key"]
        assert fam.uniform(tuple(k["site"]), k["step"]).hex() == k["u"]
        assert fam.global_uniform(k["step"]).hex() == k["global_u"]
    for d in kats["derive"]:
        assert rng.derive_seed(d["seed"], d["index"], d["salt"]) == d["out"]
    for c in kats["chains"]:
        assert chain_master_seed(c["master"], c["k"]) == c["chain"]
        assert schedule_seed(c["chain"], 1) == c["round1"]


def test_color_at_matches_global_uniform():
    fam = ts.seed_family(0x5EED, (5, 5))
    for step in range(50):
        assert rng.color_at(0x5EED, step) == (1 if fam.global_uniform(step) >= 0.5 else 0)


def test_domains_match_reference_faces():
    g = load("domino_extremal.npz")
    doms = gc.extremal_domains(ts)
    for i, d in enumerate(doms):
        assert np.array_equal(d.faces, g[f"d{i}_faces"])
        if f"d{i}_vmask" in g.files:
            assert np.array_equal(d.vertex_mask, g[f"d{i}_vmask"])
            assert tuple(g[f"d{i}_ref"]) == d.reference_vertex


def test_domain_errors():
    with pytest.raises(ts.DomainError):
        ts.Domain.from_faces(3, [(0, 0), (2, 2)])  # disconnected
    ring = np.ones((3, 3), bool)
    ring[1, 1] = False
    with pytest.raises(ts.DomainError):
        ts.Domain(3, ring)  # hole
    with pytest.raises(ts.DomainError):
        ts.Domain(2, np.zeros((2, 2), bool))
    with pytest.raises(ts.DomainError):
        ts.Domain.from_faces(2, [(5, 5)])
    d = ts.Domain.from_text(ts.Domain.aztec(3).to_text())
    assert d == ts.Domain.aztec(3)


def test_p_up_grids_match_reference():
    g = load("domino_walks.npz")
    for i, w in enumerate(gc.domino_walk_weights(ts)):
        f = g[f"c{i}_faces"]
        plan = ts.SweepPlan(ts.Domain(f.shape[0], f), w)
        assert np.array_equal(plan.p_up, g[f"c{i}_p_up"]), f"case {i}"
    assert f"c{i + 1}_p_up" not in g.files
    # scalar helper
    assert ts.heat_bath_p_up((1, 1), ts.VolumeWeights(1.0, {(1, 1): 2.0})) == pytest.approx(16 / 17)
    assert ts.heat_bath_p_up((1, 2), ts.VolumeWeights(1.0, {(1, 2): 2.0})) == pytest.approx(1 / 17)


def test_codec_roundtrip_on_golden_tilings():
    g = load("domino_extremal.npz")
    for i, d in enumerate(gc.extremal_domains(ts)):
        if f"d{i}_none" in g.files:
            continue
        for key in ("tmax", "tmin", "mixed"):
            t = ts.Tiling(d, g[f"d{i}_{key}"])
            pairs = ts.dominoes_from_tiling(t)
            assert ts.tiling_from_dominoes(d, pairs) == t
            assert ts.is_valid_tiling(t)
        # decode heights -> tiling (lattice.py:598-620)
        assert ts.tiling_from_heights(d, g[f"d{i}_hmax"]).states.tobytes() == g[f"d{i}_tmax"].tobytes()
        assert ts.tiling_from_heights(d, g[f"d{i}_hmin"]).states.tobytes() == g[f"d{i}_tmin"].tobytes()


def test_split_merge_checkerboard():
    g = load("domino_c1.npz")
    tb, tw = ts.split_checkerboard(g["final"])
    merged = ts.merge_checkerboard(tb, tw)
    assert np.array_equal(merged[:129, :129], g["final"])


def test_rotate_kernel_cases():
    assert ts.rotate_kernel(3, 0.1, 0.5) == 12
    assert ts.rotate_kernel(12, 0.9, 0.5) == 3
    assert ts.rotate_kernel(5, 0.1, 0.5) == 5


def test_cftp_schedule_prepends():
    sched = ts.CftpSchedule(master_seed=42, max_doublings=5)
    seen = []
    for _ in range(4):
        sched.grow()
        seen.append(list(sched.pairs))
    for earlier, later in zip(seen, seen[1:]):
        assert later[1:] == earlier
    assert [s for _, s in sched.pairs] == [16, 8, 4, 2]
    with pytest.raises(ts.ConvergenceCapExceeded):
        sched.grow()
        sched.grow()


def test_sixvertex_p_high_lut_matches_reference():
    from paper_1804_07250_b200.sixvertex import p_high_lut

    g = load("sixvertex.npz")
    for j, w in enumerate(gc.SV_LUT_WEIGHTS):
        assert np.array_equal(p_high_lut(ts.SVWeights(*w)), g[f"lut{j}"]), w


def test_sixvertex_codecs_and_ring():
    from paper_1804_07250_b200.sixvertex import _ring_heights

    g = load("sixvertex.npz")
    for n in gc.SV_EXTREMAL_N:
        for key in ("hi", "lo"):
            fh = ts.FaceHeights(n, g[f"e{n}_{key}"])
            cfg = ts.config_from_heights(fh)
            assert ts.heights_from_config(cfg) == fh
        ring = _ring_heights(ts.dwbc(n))
        hi = g[f"e{n}_hi"]
        assert np.array_equal(ring[0], hi[0]) and np.array_equal(ring[:, 0], hi[:, 0])
    bad = ts.Boundary(2, top=[1, 1], bottom=[0, 0], left=[0, 0], right=[0, 0])
    with pytest.raises(ts.InfeasibleBoundary):
        _ring_heights(bad)


def test_lozenge_host_side():
    from paper_1804_07250_b200.lozenge import ROT_HIGH, ROT_LOW, loz_p_up_grid

    assert (ROT_HIGH, ROT_LOW) == (0b010101, 0b101010)
    g = load("lozenge.npz")
    weights = [ts.VolumeWeights(0.9), ts.Uniform(),
               ts.LozEdgeWeights(1.0, {(("up", 3, 4), ("down", 3, 3)): 2.5})]
    abcs = [(8, 8, 8), (3, 4, 5), (5, 2, 6)]
    for i, (abc, w) in enumerate(zip(abcs, weights)):
        d = ts.TriDomain.hexagon(*abc)
        assert np.array_equal(loz_p_up_grid(d, w), g[f"l{i}_p_up"])
        assert g[f"l{i}_start"].shape == (3, d.size[0] + 1, d.size[1] + 1)
        t = ts.LozengeTiling(d, g[f"l{i}_start"])
        assert ts.tiling_from_lozenges(d, ts.lozenges_from_tiling(t)) == t
    with pytest.raises(ts.DomainError):
        up = np.ones((3, 3), bool)
        dn = np.ones((3, 3), bool)
        up[1, 1] = dn[1, 1] = dn[0, 1] = dn[1, 0] = False  # hole
        ts.TriDomain((3, 3), up, dn)
    with pytest.raises(ts.DomainError):
        up = np.zeros((4, 4), bool)
        dn = np.zeros((4, 4), bool)
        up[0, 0] = up[3, 3] = True
        ts.TriDomain((4, 4), up, dn)


def test_aztec_closed_form_matches_brick_runs():
    """The row-by-row Aztec extremal states equal the generic brick tilings."""
    import numpy as np

    from paper_1804_07250_b200.lattice import Domain, aztec_extremal_states, brick_tiling_states

    for order in (1, 2, 3, 8, 31, 64, 129):
        d = Domain.aztec(order)
        hb, vb = brick_tiling_states(d, True), brick_tiling_states(d, False)
        t_max, t_min = aztec_extremal_states(order)
        exp = (hb, vb) if order % 2 == 0 else (vb, hb)
        assert np.array_equal(t_max, exp[0]) and np.array_equal(t_min, exp[1]), order


def test_p_up_parity_matches_grid():
    """SweepPlan.p_up_parity gives the same float64 values as the p_up grid."""
    import numpy as np

    import paper_1804_07250_b200 as ts

    d = ts.Domain.aztec(6)
    for w in (ts.Uniform(), ts.VolumeWeights(0.7), ts.VolumeWeights(1.3)):
        plan = ts.SweepPlan(d, w)
        pe, po = plan.p_up_parity
        par = np.add.outer(np.arange(d.n + 1), np.arange(d.n + 1)) & 1
        assert (plan.p_up[par == 0] == pe).all() and (plan.p_up[par == 1] == po).all()
    assert ts.SweepPlan(d, ts.VolumeWeights(0.7, {(2, 3): 0.4})).p_up_parity is None
    assert ts.SweepPlan(d, ts.EdgeWeights(1.0, {((0, 0), (0, 1)): 2.0})).p_up_parity is None


def test_c_abi_header_is_plain_c(tmp_path):
    """include/tsb.h compiles as C99 and C++17 (the FFI boundary carries no
    C++ or torch types) and a C program links against libtsb.so."""
    import os
    import subprocess

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    src = tmp_path / "t.c"
    src.write_text('#include "include/tsb.h"\n#include <stdio.h>\n'
                   'int main(void) { printf("%d\\n", tsb_abi_version()); return 0; }\n')
    lib_dir = os.path.join(root, "paper_1804_07250_b200", "_lib")
    subprocess.run(["gcc", "-std=c99", "-Wall", "-Werror", "-I", root, str(src), "-L", lib_dir, "-ltsb",
                    f"-Wl,-rpath,{lib_dir}", "-o", str(tmp_path / "t")], check=True)
    subprocess.run(["g++", "-std=c++17", "-Wall", "-Werror", "-I", root, "-x", "c++", "-c", str(src), "-o",
                    str(tmp_path / "t.o")], check=True)
    out = subprocess.run([str(tmp_path / "t")], capture_output=True, text=True, check=True).stdout
    assert out.strip() == "1"


def test_bench_reference_arm_workload_is_package_free():
    """bench.py's reference arm builds the Aztec workload in numpy (no
    product import): its T_max, colour coins and per-colour vertex counts
    equal the package's (closed form, rng.color_at, vertex_mask parity)."""
    import subprocess
    import sys

    import numpy as np

    import bench
    from paper_1804_07250_b200 import rng
    from paper_1804_07250_b200.lattice import aztec_extremal_states

    for order in (1, 2, 3, 8, 63, 64, 257):
        n = 2 * order
        r = np.arange(n) + 0.5 - order
        faces = (np.abs(r)[:, None] + np.abs(r)[None, :]) <= order
        p = np.pad(faces, 1)
        vm = p[:-1, :-1] | p[:-1, 1:] | p[1:, :-1] | p[1:, 1:]
        rr = np.arange(n + 1)
        even = ((rr[:, None] + rr[None, :]) & 1) == 0
        assert bench.aztec_counts(order) == (int((vm & even).sum()), int((vm & ~even).sum()))
        assert np.array_equal(bench.aztec_tmax_host(order), aztec_extremal_states(order)[0])
    for s in (0x5EED, 1, 2**63 + 5):
        assert [bench._color_at(s, k) for k in range(64)] == [rng.color_at(s, k) for k in range(64)]
    # the reference arm's module-level imports do not pull in the product
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = ("import sys; sys.path.insert(0, %r); import bench; "
            "print(any(m.startswith('paper_1804_07250_b200') for m in sys.modules))" % root)
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, check=True).stdout
    assert out.strip() == "False"
