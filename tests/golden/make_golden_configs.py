"""Reference fingerprints at the BASELINE configs' own sizes and sweep counts.

Run in the dev container (where /root/reference exists), one job per config
(each is minutes to an hour of single-core numpy/numba):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_configs.py JOB

JOB is one of c2, c3_half, c3_afe, m4096, c4, c5.  Each writes
tests/golden/configs/JOB.json holding sha256[:16] fingerprints of the arrays
the UNMODIFIED reference (`tilesampler`) produced.  The lattices are too large
to commit, so the GPU tests (tests/test_configs_gpu.py) recompute the same
arrays on the device and compare fingerprints.

Start states where the reference's own constructor is infeasible at the size
(SURVEY.md §8(c)): Aztec T_max is the closed form of SURVEY Appendix C (all
horizontal bricks for even order), built here in numpy and checked against the
reference's `extremal_tilings` at small orders before use; the six-vertex
DWBC h_min is the closed form `max(-(R+C), R+C-2n)` checked against
`sv_extremal` at small n.  `random_walk_batch` reads only `plan.p_up`
(sweeps.py:294-309), so at orders 4096/16384 a duck-typed plan carrying the
reference's uniform p_up grid (sweeps.py:171-173) replaces the O(n^2)
pure-Python `Domain` validation.
"""

from __future__ import annotations

import hashlib
import json
import math
import os
import sys
import time
import types

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import tilesampler as ts  # noqa: E402
from tilesampler.cftp import chain_master_seed, schedule_seed  # noqa: E402
from tilesampler.lozenge import LozengeTiling, loz_random_walk_batch  # noqa: E402
from tilesampler.sixvertex import sv_random_walk_batch  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "configs")
SEED = 0x5EED


def fp(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


def write(name: str, rec: dict) -> None:
    os.makedirs(OUT, exist_ok=True)
    with open(os.path.join(OUT, name + ".json"), "w") as f:
        json.dump(rec, f, indent=1)
    print(name, json.dumps(rec), flush=True)


def aztec_tmax_closed(order: int) -> np.ndarray:
    """every row (odd order: column) of the diamond is an
    even run of faces paired from its first face."""
    n = 2 * order
    v = n + 1
    r = np.arange(n, dtype=float) + 0.5 - order
    faces = (np.abs(r)[:, None] + np.abs(r)[None, :]) <= order
    st = np.zeros((v, v), dtype=np.uint8)
    f = faces if order % 2 == 0 else faces.T
    s = np.zeros((v, v), dtype=np.uint8)
    for i in range(n):
        cols = np.flatnonzero(f[i])
        a = cols[0]
        x = np.arange(a + 1, cols[-1] + 1, 2)  # interior edge at vertex column x
        s[i, x] |= 2   # down from (i, x)
        s[i + 1, x] |= 1  # up from (i+1, x)
    if order % 2 == 0:
        st = s
    else:  # transpose: vertical bricks; up/down bits become left/right
        t = s.T
        st = (((t & 1) << 2) | ((t & 2) << 2)).astype(np.uint8)
    return st


def check_closed_forms() -> None:
    for order in (1, 2, 3, 8, 9, 32):
        t_max, _ = ts.extremal_tilings(ts.Domain.aztec(order))
        assert np.array_equal(aztec_tmax_closed(order), t_max.states), order
    for n in (1, 2, 5, 16, 33):
        _, lo = ts.sv_extremal(n, ts.dwbc(n))
        assert np.array_equal(sv_hmin_closed(n), lo.heights), n


def sv_hmin_closed(n: int) -> np.ndarray:
    r = np.arange(n + 1)
    s = r[:, None] + r[None, :]
    return np.maximum(-s, s - 2 * n).astype(np.int32)


def uniform_plan(order: int):
    v = 2 * order + 1
    return types.SimpleNamespace(p_up=np.full((v, v), 0.5))


# --------------------------------------------------------------------- jobs
def job_m4096():
    """Metric lattice: Aztec 4096 from T_max, seed 0x5EED, 1000 sweeps (fused
    numba path, the reference default)."""
    order, steps = 4096, 1000
    t0 = aztec_tmax_closed(order)
    rec = dict(order=order, seed=SEED, t_max=fp(t0))
    plan = uniform_plan(order)
    for n_steps in (7, steps):
        t = time.time()
        out = ts.random_walk_batch(t0[None], np.array([SEED], np.uint64), n_steps, plan)[0]
        rec[f"walk_{n_steps}"] = fp(out)
        rec[f"rotateable_{n_steps}"] = int(((out == 3) | (out == 12)).sum())
        rec[f"seconds_{n_steps}"] = round(time.time() - t, 1)
        write("m4096", rec)
    d = ts.Domain.aztec(order)
    t = time.time()
    rec["heights_" + str(steps)] = fp(ts.height_function(ts.Tiling(d, out)).heights)
    rec["heights_seconds"] = round(time.time() - t, 1)
    write("m4096", rec)


def job_c4():
    """C4: Aztec 16384 from T_max, seed 0x5EED (fused numba path)."""
    order = 16384
    t0 = aztec_tmax_closed(order)
    rec = dict(order=order, seed=SEED, t_max=fp(t0))
    plan = uniform_plan(order)
    for n_steps in (100,):
        t = time.time()
        out = ts.random_walk_batch(t0[None], np.array([SEED], np.uint64), n_steps, plan)[0]
        rec[f"walk_{n_steps}"] = fp(out)
        # per-strip fingerprints (8 equal row bands) to localise a mismatch
        v = out.shape[0]
        cuts = np.linspace(0, v, 9).astype(int)
        rec[f"bands_{n_steps}"] = [fp(out[a:b]) for a, b in zip(cuts[:-1], cuts[1:])]
        rec[f"rotateable_{n_steps}"] = int(((out == 3) | (out == 12)).sum())
        rec[f"seconds_{n_steps}"] = round(time.time() - t, 1)
        write("c4", rec)


def job_c3(name: str, weights: tuple):
    """C3: six-vertex DWBC 2048 from h_min, seed 0x5EED, 10^4 sweeps."""
    n = 2048
    h0 = sv_hmin_closed(n)
    w = ts.SVWeights(*weights)
    rec = dict(n=n, seed=SEED, weights=list(weights), h_min=fp(h0))
    for n_steps in (100, 10000):
        t = time.time()
        out = sv_random_walk_batch(h0[None], np.array([SEED], np.uint64), n_steps, w)[0]
        rec[f"walk_{n_steps}"] = fp(out)
        rec[f"sum_{n_steps}"] = int(out.astype(np.int64).sum())
        rec[f"seconds_{n_steps}"] = round(time.time() - t, 1)
        write(name, rec)


def job_c2():
    """C2: lozenge hexagon 1000^3, VolumeWeights(0.999), from loz_extremal's
    T_min, seed 0x5EED, 10^4 sweeps."""
    a = 1000
    q = 0.999
    t = time.time()
    dom = ts.TriDomain.hexagon(a, a, a)
    rec = dict(abc=[a, a, a], q=q, seed=SEED, domain_seconds=round(time.time() - t, 1))
    t = time.time()
    t_max, t_min = ts.loz_extremal(dom)
    rec.update(t_max=fp(t_max.edges), t_min=fp(t_min.edges),
               extremal_seconds=round(time.time() - t, 1))
    write("c2", rec)
    t = time.time()
    rec.update(h_max=fp(ts.loz_heights(t_max).heights),
               h_min=fp(ts.loz_heights(t_min).heights),
               heights_seconds=round(time.time() - t, 1))
    write("c2", rec)
    w = ts.VolumeWeights(q)
    for n_steps in (100, 10000):
        t = time.time()
        out = loz_random_walk_batch(t_min.edges[None], np.array([SEED], np.uint64),
                                    n_steps, dom, w)[0]
        rec[f"walk_{n_steps}"] = fp(out)
        rec[f"seconds_{n_steps}"] = round(time.time() - t, 1)
        write("c2", rec)
    rec[f"heights_{n_steps}"] = fp(ts.loz_heights(LozengeTiling(dom, out)).heights)
    write("c2", rec)


def job_c5():
    """C5: CFTP on Aztec 512 -- the reference's own run_cftp_batch round
    structure (cftp.py:111-120) replayed with the reference's walk for the
    first R rounds of chains k = 0, 1 of master 0x5EED; fingerprints of top and
    bottom after every round."""
    order, rounds = 512, 13
    t = time.time()
    d = ts.Domain.aztec(order)
    t_max, t_min = ts.extremal_tilings(d)
    plan = ts.SweepPlan(d)
    rec = dict(order=order, master=SEED, t_max=fp(t_max.states), t_min=fp(t_min.states),
               setup_seconds=round(time.time() - t, 1), chains=[])
    assert np.array_equal(t_max.states, aztec_tmax_closed(order))
    for k in (0, 1):
        m = chain_master_seed(SEED, k)
        seeds = [schedule_seed(m, r) for r in range(1, rounds + 1)]
        ch = dict(k=k, master=m, top=[], bot=[], differ=[])
        for r in range(1, rounds + 1):
            top = t_max.states[None].copy()
            bot = t_min.states[None].copy()
            for i in range(r, 0, -1):
                s = np.array([seeds[i - 1]], np.uint64)
                top = ts.random_walk_batch(top, s, 2**i, plan)
                bot = ts.random_walk_batch(bot, s, 2**i, plan)
            ch["top"].append(fp(top[0]))
            ch["bot"].append(fp(bot[0]))
            ch["differ"].append(int((top[0] != bot[0]).sum()))
            print(k, r, ch["differ"][-1], round(time.time() - t, 1), flush=True)
        rec["chains"].append(ch)
        write("c5", rec)


JOBS = {
    "m4096": job_m4096,
    "c4": job_c4,
    "c3_half": lambda: job_c3("c3_half", (1.0, 1.0, 1.0)),
    "c3_afe": lambda: job_c3("c3_afe", (1.0, 1.0, math.sqrt(8.0))),
    "c2": job_c2,
    "c5": job_c5,
}

if __name__ == "__main__":
    check_closed_forms()
    for name in sys.argv[1:]:
        JOBS[name]()
