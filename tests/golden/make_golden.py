"""Generate the golden parity fixtures by running the REFERENCE implementation.

Run in the dev container (where /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Every array written here is an output of the unmodified reference package
(`tilesampler`, /root/reference/pkg/src/tilesampler).  The fixtures are
committed so that the GPU box (which has no /root/reference) can check the
CUDA library and the C oracle against them.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import tilesampler as ts  # noqa: E402
from tilesampler import rng  # noqa: E402
from tilesampler.cftp import chain_master_seed, schedule_seed  # noqa: E402
from tilesampler.lozenge import LozengeTiling, loz_random_walk_batch  # noqa: E402
from tilesampler.sixvertex import sv_random_walk_batch  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, ".."))
import golden_cases as gc  # noqa: E402  (shared case definitions)


def fp(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


def save(name: str, **arrays):
    path = os.path.join(HERE, name)
    np.savez_compressed(path, **arrays)
    print(f"wrote {name}: {os.path.getsize(path)} B")


# ---------------------------------------------------------------- RNG KATs
def make_rng():
    kats = []
    for seed, shape, site, step in gc.RNG_KATS:
        fam = ts.seed_family(seed, shape)
        key = fam.site_key(site)
        x = rng._splitmix_at(key, step)
        u = fam.uniform(site, step)
        g = fam.global_uniform(step)
        kats.append(
            dict(seed=seed, shape=list(shape), site=list(site), step=step,
                 key=key, x=x, u=u.hex(), global_u=g.hex())
        )
    derives = [
        dict(seed=s, index=i, salt=salt, out=rng.derive_seed(s, i, salt))
        for s, i, salt in gc.DERIVE_KATS
    ]
    sched = [dict(master=m, k=k, chain=chain_master_seed(m, k),
                  round1=schedule_seed(chain_master_seed(m, k), 1))
             for m, k in gc.CHAIN_KATS]
    grids = {}
    for seed, shape, step in gc.GRID_KATS:
        grids[f"{seed}_{shape[0]}_{shape[1]}_{step}"] = ts.seed_family(seed, shape).uniform_grid(step)
    with open(os.path.join(HERE, "rng_kats.json"), "w") as f:
        json.dump(dict(kats=kats, derive=derives, chains=sched), f, indent=1)
    save("rng_grids.npz", **grids)


# ----------------------------------------------------------- domino walks
def make_domino():
    # C1 (BASELINE config 1): Aztec order 64, T_max, seed 0x5EED, 1000 sweeps
    d = ts.Domain.aztec(64)
    t_max, t_min = ts.extremal_tilings(d)
    plan = ts.SweepPlan(d)
    out = ts.random_walk(t_max, 0x5EED, 1000, plan)
    h = ts.height_function(out).heights
    print("C1 states", fp(out.states), "heights", fp(h), "t_max", fp(t_max.states))
    save("domino_c1.npz", t_max=t_max.states, t_min=t_min.states, final=out.states,
         heights=h, heights_tmax=ts.height_function(t_max).heights)

    arrays = {}
    for i, case in enumerate(gc.domino_walk_cases()):
        d, plan, start = case["domain"], case["plan"], case["start"]()
        states = np.stack(start)
        seeds = np.asarray(case["seeds"], dtype=np.uint64)
        res = ts.random_walk_batch(states, seeds, case["n_steps"], plan)
        arrays[f"c{i}_faces"] = d.faces
        arrays[f"c{i}_start"] = states
        arrays[f"c{i}_seeds"] = seeds
        arrays[f"c{i}_n_steps"] = np.array(case["n_steps"])
        arrays[f"c{i}_p_up"] = plan.p_up
        arrays[f"c{i}_out"] = res
    # single sweeps with an explicit colour/step (sweeps.py:322-342)
    for j, (dom, seed, step, color) in enumerate(gc.SWEEP_CASES):
        d = dom()
        plan = ts.SweepPlan(d)
        t0 = ts.random_walk(ts.extremal_tilings(d)[0], 77 + j, 40, plan)
        fam = ts.seed_family(seed, (d.n + 1, d.n + 1))
        t1, rot = ts.sweep(t0, fam, step, ts.Color(color), plan, return_rotated=True)
        arrays[f"s{j}_faces"] = d.faces
        arrays[f"s{j}_in"] = t0.states
        arrays[f"s{j}_out"] = t1.states
        arrays[f"s{j}_rot"] = rot
    save("domino_walks.npz", **arrays)


# ------------------------------------------------ extremal tilings, heights
def make_extremal():
    arrays = {}
    for i, d in enumerate(gc.extremal_domains()):
        arrays[f"d{i}_faces"] = d.faces
        ext = ts.extremal_tilings(d)
        if ext is None:
            arrays[f"d{i}_none"] = np.array(1)
            continue
        t_max, t_min = ext
        arrays[f"d{i}_tmax"] = t_max.states
        arrays[f"d{i}_tmin"] = t_min.states
        arrays[f"d{i}_hmax"] = ts.height_function(t_max).heights
        arrays[f"d{i}_hmin"] = ts.height_function(t_min).heights
        arrays[f"d{i}_ref"] = np.array(d.reference_vertex)
        arrays[f"d{i}_vmask"] = d.vertex_mask
        # a mixed tiling and its heights
        mixed = ts.random_walk(t_max, 1000 + i, 60, ts.SweepPlan(d))
        arrays[f"d{i}_mixed"] = mixed.states
        arrays[f"d{i}_hmixed"] = ts.height_function(mixed).heights
    save("domino_extremal.npz", **arrays)


# ------------------------------------------------------------------- CFTP
def make_cftp():
    arrays = {}
    meta = []
    for i, (dom, weights, master, count, maxd) in enumerate(gc.CFTP_CASES):
        d = dom()
        plan = ts.SweepPlan(d, weights)
        trace = ts.CftpTrace()
        samples = ts.cftp_sample_many(d, plan, master, count, max_doublings=maxd, trace=trace)
        arrays[f"k{i}_faces"] = d.faces
        arrays[f"k{i}_samples"] = np.stack([s.states for s in samples])
        meta.append(dict(rounds=[[list(p) for p in r] for r in trace.rounds],
                         collapsed_at=trace.collapsed_at))
    save("domino_cftp.npz", **arrays)
    with open(os.path.join(HERE, "domino_cftp_traces.json"), "w") as f:
        json.dump(meta, f)


# ------------------------------------------------------------- six-vertex
def make_sixvertex():
    arrays = {}
    for i, (n, weights, seed, n_steps, start) in enumerate(gc.SV_CASES):
        b = ts.dwbc(n)
        hi, lo = ts.sv_extremal(n, b)
        h0 = (hi if start == "max" else lo).heights
        out = sv_random_walk_batch(h0[None], np.array([seed], dtype=np.uint64), n_steps,
                                   ts.SVWeights(*weights))
        arrays[f"v{i}_start"] = h0
        arrays[f"v{i}_out"] = out[0]
        arrays[f"v{i}_table"] = ts.SVWeights(*weights).table()
        print(f"sv case {i} n={n} w={weights} -> {fp(out[0])}")
    for n in gc.SV_EXTREMAL_N:
        hi, lo = ts.sv_extremal(n, ts.dwbc(n))
        arrays[f"e{n}_hi"] = hi.heights
        arrays[f"e{n}_lo"] = lo.heights
    # p_high of the 32 flippable 3x3 patterns via the reference's own
    # sv_heat_bath_p_up (sixvertex.py:318-337), for the LUT check
    from tilesampler.sixvertex import sv_heat_bath_p_up
    for j, weights in enumerate(gc.SV_LUT_WEIGHTS):
        lut = []
        for idx in range(32):
            s_ = -1 if idx >= 16 else 1
            h = np.zeros((3, 3), dtype=np.int32)
            h[0, 1] = h[2, 1] = h[1, 0] = h[1, 2] = s_
            for bit, (r, c) in zip((8, 4, 2, 1), ((0, 0), (0, 2), (2, 0), (2, 2))):
                h[r, c] = 2 * s_ if idx & bit else 0
            lut.append(sv_heat_bath_p_up(ts.FaceHeights(2, h), (1, 1), ts.SVWeights(*weights)))
        arrays[f"lut{j}"] = np.array(lut)
    # CFTP on DWBC 3 / 4
    for j, (n, weights, master, count) in enumerate(gc.SV_CFTP_CASES):
        trace = ts.CftpTrace()
        res = ts.sv_cftp(n, ts.dwbc(n), ts.SVWeights(*weights), master, count=count, trace=trace)
        res = res if isinstance(res, list) else [res]
        arrays[f"k{j}_h"] = np.stack([ts.heights_from_config(c).heights for c in res])
        arrays[f"k{j}_collapsed"] = np.array(trace.collapsed_at)
    save("sixvertex.npz", **arrays)


# ---------------------------------------------------------------- lozenges
def make_lozenge():
    arrays = {}
    for i, (abc, weights, seed, n_steps, start) in enumerate(gc.LOZ_CASES):
        dom = ts.TriDomain.hexagon(*abc)
        t_max, t_min = ts.loz_extremal(dom)
        t0 = t_max if start == "max" else t_min
        out = loz_random_walk_batch(t0.edges[None], np.array([seed], dtype=np.uint64),
                                    n_steps, dom, weights)
        tout = LozengeTiling(dom, out[0])
        arrays[f"l{i}_start"] = t0.edges
        arrays[f"l{i}_out"] = out[0]
        arrays[f"l{i}_heights"] = ts.loz_heights(tout).heights
        from tilesampler.lozenge import loz_p_up_grid
        arrays[f"l{i}_p_up"] = loz_p_up_grid(dom, weights)
        print(f"loz case {i} {abc} -> edges {fp(out[0])} heights {fp(arrays[f'l{i}_heights'])}")
    for abc in gc.LOZ_EXTREMAL:
        dom = ts.TriDomain.hexagon(*abc)
        t_max, t_min = ts.loz_extremal(dom)
        key = "x" + "_".join(map(str, abc))
        arrays[key + "_max"] = t_max.edges
        arrays[key + "_min"] = t_min.edges
        arrays[key + "_hmax"] = ts.loz_heights(t_max).heights
        arrays[key + "_hmin"] = ts.loz_heights(t_min).heights
    for j, (abc, master, count) in enumerate(gc.LOZ_CFTP_CASES):
        dom = ts.TriDomain.hexagon(*abc)
        res = ts.loz_cftp(dom, ts.Uniform(), master, count=count)
        res = res if isinstance(res, list) else [res]
        arrays[f"k{j}_edges"] = np.stack([t.edges for t in res])
    save("lozenge.npz", **arrays)


# ------------------------------------------------------------- observables
def make_observables():
    """density_map / domino_orientation_grid / aztec_y_intercept /
    c_vertex_count (stats.py:187-288) of reference-sampled states."""
    from tilesampler import stats

    arrays = {}
    # dominoes: Aztec 32, 6 chains from T_max after 300 and 600 sweeps
    d = ts.Domain.aztec(32)
    t_max, _ = ts.extremal_tilings(d)
    plan = ts.SweepPlan(d)
    seeds = np.array([1, 2, 3, 4, 5, 6], dtype=np.uint64)
    s1 = ts.random_walk_batch(np.stack([t_max.states] * 6), seeds, 300, plan)
    s2 = ts.random_walk_batch(s1, seeds + np.uint64(100), 300, plan)
    states = np.concatenate([s1, s2])
    arc = stats.SampleArchive("domino", {}, [ts.Tiling(d, s) for s in states])
    arrays["dom_states"] = states
    arrays["dom_density"] = stats.density_map(arc, "domino-orientation").grid
    arrays["dom_orient0"] = stats.domino_orientation_grid(ts.Tiling(d, states[0]))
    arrays["dom_yint"] = np.array([stats.aztec_y_intercept(ts.Tiling(d, s)) for s in states])
    # six-vertex: DWBC 24, 4 chains from h_min / h_max after 150 sweeps
    n = 24
    hi, lo = ts.sv_extremal(n, ts.dwbc(n))
    start = np.stack([lo.heights, hi.heights, lo.heights, hi.heights])
    hs = sv_random_walk_batch(start, np.array([7, 8, 9, 10], dtype=np.uint64), 150, ts.SVWeights(1.0, 1.0, 1.5))
    cfgs = [ts.config_from_heights(ts.FaceHeights(n, h)) for h in hs]
    arc = stats.SampleArchive("sixvertex", {}, cfgs)
    arrays["sv_heights"] = hs
    for name in ("h-edge", "v-edge", "c-vertex"):
        arrays["sv_" + name.replace("-", "_")] = stats.density_map(arc, name).grid
    arrays["sv_ccount"] = np.array([stats.c_vertex_count(c) for c in cfgs])
    save("observables.npz", **arrays)


# ------------------------------------------------------------- archives
def make_archives():
    """stats.SampleArchive text (create + extend + dump, stats.py:75-153) of
    reference-sampled states of each model, with the states themselves."""
    import io

    from tilesampler import stats

    arrays = {}
    d = ts.Domain.aztec(12)
    t_max, _ = ts.extremal_tilings(d)
    st = ts.random_walk_batch(np.stack([t_max.states] * 3), np.array([1, 2, 3], dtype=np.uint64), 60,
                              ts.SweepPlan(d))
    n = 8
    b = ts.dwbc(n)
    lo = ts.sv_extremal(n, b)[1]
    hs = sv_random_walk_batch(np.stack([lo.heights] * 3), np.array([4, 5, 6], dtype=np.uint64), 50,
                              ts.SVWeights(1.0, 1.0, 1.2))
    dom = ts.TriDomain.hexagon(3, 4, 5)
    t_max_l, _ = ts.loz_extremal(dom)
    es = loz_random_walk_batch(np.stack([t_max_l.edges] * 3), np.array([7, 8, 9], dtype=np.uint64), 50, dom,
                               ts.Uniform())
    cases = {
        "domino": (d, [ts.Tiling(d, s) for s in st]),
        "sixvertex": (b, [ts.config_from_heights(ts.FaceHeights(n, h)) for h in hs]),
        "lozenge": (dom, [LozengeTiling(dom, e) for e in es]),
    }
    arrays.update(dom_states=st, sv_heights=hs, loz_edges=es)
    for model, (domain, states) in cases.items():
        arc = stats.SampleArchive.create(model, domain, "uniform", 0x5EED, "sequential", "mcmc steps=60")
        arc.extend(states)
        buf = io.StringIO()
        arc.dump(buf)
        with open(os.path.join(HERE, f"archive_{model}.txt"), "w") as fh:
            fh.write(buf.getvalue())
        print(f"archive {model}: {len(buf.getvalue())} chars")
    save("archives.npz", **arrays)


def make_cli():
    """Outputs of the reference CLI (cli.py:128-255) for gc.CLI_CASES, written
    to cli_<name>.txt through its --out flag."""
    from tilesampler.cli import main

    for name, argv in gc.CLI_CASES:
        out = os.path.join(HERE, f"cli_{name}.txt")
        code = main([a.replace("{g}", HERE) for a in argv] + ["--out", out])
        assert code == 0, (name, code)
        print(f"cli {name}: {os.path.getsize(out)} B")


# ------------------------------------------ six-vertex non-DWBC boundaries
def _boundary_from_heights(h):
    dh = h[:-1, :] - h[1:, :]
    dv = h[:, 1:] - h[:, :-1]
    he, ve = dh == 1, dv == 1
    n = h.shape[0] - 1
    return ts.Boundary(n, top=ve[0, :], bottom=ve[n, :], left=he[:, 0], right=he[:, n])


def make_sv_boundaries():
    """General boundaries (sixvertex.py:83-120) through sv_extremal
    (534-562), including InfeasibleBoundary from _ring_heights (527) and
    from the compatibility check (557), a walk from each feasible h_max and
    h_min, and sv_cftp on small general boundaries."""
    from tilesampler.errors import InfeasibleBoundary

    rng_ = np.random.default_rng(20261017)
    arrays, meta = {}, []
    cases = []
    for n in (1, 2, 3, 5, 8, 13, 40, 97):
        for _ in range(3):
            # min of two separable +-1 walks: a valid height function
            hs = []
            for _ in range(2):
                f = np.concatenate([[0], np.cumsum(rng_.choice([-1, 1], n))])
                g = np.concatenate([[0], np.cumsum(rng_.choice([-1, 1], n))])
                hs.append(f[:, None] + g[None, :])
            cases.append(_boundary_from_heights(np.minimum(hs[0], hs[1] + 2 * rng_.integers(-2, 3))))
    # random occupancies (mostly infeasible: ring does not close or is incompatible)
    for n in (2, 3, 4, 6, 10, 31):
        for _ in range(4):
            b = [rng_.random(n) < 0.5 for _ in range(4)]
            cases.append(ts.Boundary(n, *b))
    # rings that close but are mutually incompatible (sixvertex.py:557): the
    # top ring peaks mid-row while the bottom ring dips, further apart in
    # height than in distance
    for n in (4, 6, 10, 17):
        half = np.arange(n) < n // 2
        ones = np.ones(n, bool)
        cases.append(ts.Boundary(n, top=half, bottom=~half, left=ones, right=ones))
        cases.append(ts.Boundary(n, top=~half, bottom=half, left=~ones, right=~ones))
    w = ts.SVWeights(1.0, 1.0, 1.5)
    for i, b in enumerate(cases):
        for k in ("top", "bottom", "left", "right"):
            arrays[f"b{i}_{k}"] = getattr(b, k)
        try:
            hi, lo = ts.sv_extremal(b.n, b)
        except InfeasibleBoundary as e:
            meta.append(dict(n=b.n, error=type(e).__name__, message=str(e)))
            continue
        arrays[f"b{i}_hi"] = hi.heights
        arrays[f"b{i}_lo"] = lo.heights
        start = np.stack([hi.heights, lo.heights])
        out = sv_random_walk_batch(start, np.array([7 + i, 7 + i], dtype=np.uint64), 60, w)
        arrays[f"b{i}_walk"] = out
        meta.append(dict(n=b.n, error=None))
    # CFTP on small general boundaries
    cftp = []
    for j, i in enumerate([k for k, m in enumerate(meta) if m["error"] is None and 3 <= m["n"] <= 8][:4]):
        b = cases[i]
        trace = ts.CftpTrace()
        res = ts.sv_cftp(b.n, b, w, 0x5EED + j, count=3, trace=trace)
        arrays[f"c{j}_h"] = np.stack([ts.heights_from_config(c).heights for c in res])
        cftp.append(dict(case=i, master=0x5EED + j, collapsed_at=trace.collapsed_at))
    save("sv_boundaries.npz", **arrays)
    with open(os.path.join(HERE, "sv_boundaries.json"), "w") as f:
        json.dump(dict(cases=meta, cftp=cftp, weights=[1.0, 1.0, 1.5], walk_steps=60), f, indent=1)
    print("sv boundaries:", sum(m["error"] is None for m in meta), "feasible of", len(meta),
          sorted(set(m.get("message", "") for m in meta)))


if __name__ == "__main__":
    which = sys.argv[1:] or ["rng", "domino", "extremal", "cftp", "sixvertex", "lozenge", "observables", "archives",
                             "cli", "sv_boundaries"]
    for w in which:
        globals()[f"make_{w}"]()
