#!/usr/bin/env python
"""Throughput of the BASELINE.json configs other than the headline metric
(reported in DESIGN.md; bench.py is the contract line).  Device-resident
states, CUDA-event timing on the handle's stream after warm-up.

    python tools/bench_configs.py [--only c1,c2,c3,c4,c5,mixed] [--quick]
"""

from __future__ import annotations

import argparse
import json
import math
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def timed(torch, stream, fn):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record(stream)
    fn()
    b.record(stream)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / 1e3


def c1(torch, stream, quick):
    import hashlib

    import paper_1804_07250_b200 as ts
    from paper_1804_07250_b200 import rng
    from paper_1804_07250_b200.lattice import aztec_extremal_states
    from paper_1804_07250_b200.sweeps import DominoHandle

    d = ts.Domain.aztec(64)
    t_max, _ = aztec_extremal_states(64)
    h = DominoHandle(d, d.n + 1, 1)
    h.set_stream(stream.cuda_stream)
    h.set_plan(ts.SweepPlan(d))
    h.upload(t_max[None])
    h.walk([0x5EED], 1000)
    fp = hashlib.sha256(h.download()[0].tobytes()).hexdigest()[:16]
    h.upload(t_max[None])
    dt = timed(torch, stream, lambda: h.walk([0x5EED], 1000))
    mask = d.vertex_mask
    par = np.add.outer(np.arange(d.n + 1), np.arange(d.n + 1)) & 1
    counts = (int((mask & (par == 0)).sum()), int((mask & (par == 1)).sum()))
    att = sum(counts[rng.color_at(0x5EED, s)] for s in range(1000))
    return {"config": "C1 aztec64 T_max 1000 sweeps seed 0x5EED", "fingerprint": fp,
            "seconds": dt, "us_per_sweep": dt * 1e3, "attempts_per_s": att / dt}


def c2(torch, stream, quick):
    import paper_1804_07250_b200 as ts
    from paper_1804_07250_b200.lozenge import LozengeHandle, loz_p_up_grid

    a = 300 if quick else 1000
    d = ts.TriDomain.hexagon(a, a, a)
    t0 = time.perf_counter()
    t_max, t_min = ts.loz_extremal(d)
    t_ext = time.perf_counter() - t0
    w = ts.VolumeWeights(0.999)
    h = LozengeHandle(d, 1)
    h.set_stream(stream.cuda_stream)
    h.set_p_up(loz_p_up_grid(d, w))
    h.upload(t_min.edges[None])
    steps = 10_000
    h.walk([0x5EED], 320)
    dt = timed(torch, stream, lambda: h.walk([0x5EED], steps, step0=320))
    nv = int(d.vertex_mask.sum())
    return {"config": f"C2 lozenge hexagon {a},{a},{a} VolumeWeights(0.999) from T_min, {steps} sweeps",
            "extremal_s": t_ext, "us_per_sweep": dt / steps * 1e6, "attempts_per_s": nv / 3 * steps / dt,
            "domain_vertices": nv}


def c3(torch, stream, quick):
    import paper_1804_07250_b200 as ts
    from paper_1804_07250_b200.sixvertex import SixVertexHandle

    n = 512 if quick else 2048
    t0 = time.perf_counter()
    hi, lo = ts.sv_extremal(n, ts.dwbc(n))
    t_ext = time.perf_counter() - t0
    out = []
    for w, label in (((1.0, 1.0, 1.0), "Delta=1/2 (disordered)"), ((1.0, 1.0, math.sqrt(8.0)), "Delta=-3 (antiferroelectric)")):
        h = SixVertexHandle(n, 1)
        h.set_stream(stream.cuda_stream)
        h.set_weights(ts.SVWeights(*w))
        h.upload(lo.heights[None])
        steps = 10_000
        h.walk([0x5EED], 200)
        dt = timed(torch, stream, lambda: h.walk([0x5EED], steps, step0=200))
        faces = (n - 1) ** 2
        out.append({"config": f"C3 six-vertex DWBC n={n} {label} from h_min, {steps} sweeps",
                    "extremal_s": t_ext, "us_per_sweep": dt / steps * 1e6,
                    "attempts_per_s": faces / 4 * steps / dt})
    return out


def c5(torch, stream, quick):
    """CFTP order 512: time the first rounds of a 64-sample batch (a full
    sample needs ~21 rounds); reports coupled chain-sweeps per second."""
    import paper_1804_07250_b200 as ts
    from paper_1804_07250_b200.cftp import chain_master_seed
    from paper_1804_07250_b200.lattice import aztec_extremal_states
    from paper_1804_07250_b200.sweeps import DominoHandle
    import ctypes

    from paper_1804_07250_b200 import _native

    order, count, rounds = (128, 16, 8) if quick else (512, 64, 10)
    d = ts.Domain.aztec(order)
    t_max, t_min = aztec_extremal_states(order)
    h = DominoHandle(d, d.n + 1, 2 * count + 2)
    h.set_stream(stream.cuda_stream)
    h.set_plan(ts.SweepPlan(d))
    masters = np.array([chain_master_seed(0x5EED, k) for k in range(count)], dtype=np.uint64)
    out = np.zeros((count, d.n + 1, d.n + 1), dtype=np.uint8)
    rr = np.zeros(count, dtype=np.int32)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rc = _native.lib().tsb_domino_cftp(h._h, _native.ptr(t_max), _native.ptr(t_min), _native.ptr(masters), count,
                                       rounds, _native.ptr(out), _native.ptr(rr), None, None)
    dt = time.perf_counter() - t0
    chain_sweeps = 2 * count * sum(2 ** (r + 1) - 2 for r in range(1, rounds + 1))
    return {"config": f"C5 CFTP aztec {order}, {count} samples, first {rounds} rounds",
            "status": "coalesced" if rc == 0 else "cap (expected: not all samples coalesce this early)",
            "collapsed": int((rr > 0).sum()), "seconds": dt, "chain_sweeps": chain_sweeps,
            "chain_sweeps_per_s": chain_sweeps / dt,
            "attempts_per_s": chain_sweeps * int(d.vertex_mask.sum()) / 2 / dt}


def _domino_counts(d):
    """(BLACK, WHITE) in-domain vertices, row blocks (no n^2 integer temporaries)."""
    mask = d.vertex_mask
    black = 0
    cols = np.arange(d.n + 1)
    for r0 in range(0, d.n + 1, 2048):
        rows = np.arange(r0, min(d.n + 1, r0 + 2048))
        even = ((rows[:, None] + cols[None, :]) & 1) == 0
        black += int((mask[r0:r0 + 2048] & even).sum())
    return black, int(mask.sum()) - black


def c4(torch, stream, quick):
    """Aztec order 16384 on one GPU (the per-GPU share of BASELINE config 4
    at N=1): 536,969,217 domain vertices, 2 x 277 MB of planes, HBM-resident."""
    import paper_1804_07250_b200 as ts
    from paper_1804_07250_b200 import rng
    from paper_1804_07250_b200.lattice import aztec_extremal_states
    from paper_1804_07250_b200.sweeps import DominoHandle

    order = 4096 if quick else 16384
    d = ts.Domain.aztec(order)
    t_max, _ = aztec_extremal_states(order)
    h = DominoHandle(d, d.n + 1, 1)
    h.set_stream(stream.cuda_stream)
    h.set_plan(ts.SweepPlan(d))
    h.upload(t_max[None])
    del t_max
    steps = 1024
    h.walk([0x5EED], 64)
    dt = timed(torch, stream, lambda: h.walk([0x5EED], steps, step0=64))
    counts = _domino_counts(d)
    att = sum(counts[rng.color_at(0x5EED, s)] for s in range(64, 64 + steps))
    nv = counts[0] + counts[1]
    gbs = nv * steps / dt / 1e9
    return {"config": f"C4 aztec {order} T_max on 1 GPU, {steps} sweeps", "us_per_sweep": dt / steps * 1e6,
            "attempts_per_s": att / dt, "domain_vertices": nv, "algorithmic_GBps": gbs}


def mixed(torch, stream, quick):
    """The headline workload after a long warm-up (Aztec 4096 from T_max,
    2^21 sweeps), so the timed sweeps see a mixed state with many rotateable
    sites (RNG-heavy), next to the fraction of rotateable vertices."""
    import paper_1804_07250_b200 as ts
    from paper_1804_07250_b200 import rng
    from paper_1804_07250_b200.lattice import aztec_extremal_states
    from paper_1804_07250_b200.sweeps import DominoHandle

    order, warm = (1024, 1 << 20) if quick else (4096, 1 << 21)
    d = ts.Domain.aztec(order)
    t_max, _ = aztec_extremal_states(order)
    h = DominoHandle(d, d.n + 1, 1)
    h.set_stream(stream.cuda_stream)
    h.set_plan(ts.SweepPlan(d))
    h.upload(t_max[None])
    tw = timed(torch, stream, lambda: h.walk([0x5EED], warm))
    st = h.download()[0]
    rot = float(((st == 3) | (st == 12))[d.vertex_mask].mean())
    steps = 1024
    dt = timed(torch, stream, lambda: h.walk([0x5EED], steps, step0=warm))
    counts = _domino_counts(d)
    att = sum(counts[rng.color_at(0x5EED, s)] for s in range(warm, warm + steps))
    return {"config": f"aztec {order} after {warm} warm-up sweeps from T_max, {steps} timed sweeps",
            "rotateable_fraction": rot, "warm_us_per_sweep": tw / warm * 1e6, "us_per_sweep": dt / steps * 1e6,
            "attempts_per_s": att / dt}


def batched(torch, stream, quick):
    """C2 and C3 lattices with 32 independent chains per launch (chains are
    the multi-GPU replica unit): the single-chain configs are latency-bound,
    the batch shows the kernels' throughput at the same lattice size."""
    import paper_1804_07250_b200 as ts
    from paper_1804_07250_b200.lozenge import LozengeHandle, loz_p_up_grid
    from paper_1804_07250_b200.sixvertex import SixVertexHandle

    B = 8 if quick else 32
    out = []
    a = 300 if quick else 1000
    d = ts.TriDomain.hexagon(a, a, a)
    t_max, t_min = ts.loz_extremal(d)
    h = LozengeHandle(d, B)
    h.set_stream(stream.cuda_stream)
    h.set_p_up(loz_p_up_grid(d, ts.VolumeWeights(0.999)))
    h.upload(np.stack([t_min.edges] * B))
    seeds = np.arange(1, B + 1, dtype=np.uint64)
    h.walk(seeds, 256)
    steps = 2048
    dt = timed(torch, stream, lambda: h.walk(seeds, steps, step0=256))
    nv = int(d.vertex_mask.sum())
    att = B * nv / 3 * steps / dt
    out.append({"config": f"C2 lattice x{B} chains: lozenge hexagon {a}^3 q=0.999 from T_min, {steps} sweeps",
                "us_per_sweep_all_chains": dt / steps * 1e6, "attempts_per_s": att,
                "roofline_frac": att * 2.25 / 1e9 / 6463.7})
    n = 512 if quick else 2048
    hi, lo = ts.sv_extremal(n, ts.dwbc(n))
    h = SixVertexHandle(n, B)
    h.set_stream(stream.cuda_stream)
    h.set_weights(ts.SVWeights(1.0, 1.0, 1.0))
    h.upload(np.stack([lo.heights] * B))
    h.walk(seeds, 256)
    dt = timed(torch, stream, lambda: h.walk(seeds, steps, step0=256))
    att = B * (n - 1) ** 2 / 4 * steps / dt
    out.append({"config": f"C3 lattice x{B} chains: six-vertex DWBC n={n} Delta=1/2 from h_min, {steps} sweeps",
                "us_per_sweep_all_chains": dt / steps * 1e6, "attempts_per_s": att,
                "roofline_frac": att * 2.0 / 1e9 / 6463.7})
    return out


def c5full(torch, stream, quick):
    """C5 to completion: exact CFTP samples of the Aztec diamond of order 512
    (cftp_sample_many, coupled T_max / T_min chains, doubling rounds) for a
    small batch; reports the round each sample coalesced in and the time."""
    import paper_1804_07250_b200 as ts
    from paper_1804_07250_b200.cftp import chain_master_seed
    from paper_1804_07250_b200.lattice import aztec_extremal_states
    from paper_1804_07250_b200.sweeps import DominoHandle
    from paper_1804_07250_b200 import _native

    order, count = (64, 4) if quick else (512, int(os.environ.get("TSB_C5_COUNT", "8")))
    d = ts.Domain.aztec(order)
    t_max, t_min = aztec_extremal_states(order)
    h = DominoHandle(d, d.n + 1, 2 * count + 2)
    h.set_stream(stream.cuda_stream)
    h.set_plan(ts.SweepPlan(d))
    masters = np.array([chain_master_seed(0x5EED, k) for k in range(count)], dtype=np.uint64)
    out = np.zeros((count, d.n + 1, d.n + 1), dtype=np.uint8)
    rr = np.zeros(count, dtype=np.int32)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rc = _native.lib().tsb_domino_cftp(h._h, _native.ptr(t_max), _native.ptr(t_min), _native.ptr(masters), count,
                                       40, _native.ptr(out), _native.ptr(rr), None, None)
    dt = time.perf_counter() - t0
    _native.check(rc)
    sweeps = [2 * (2 ** (int(r) + 1) - 2) for r in rr]  # coupled chain-sweeps per sample (cftp.py:115-119)
    return {"config": f"C5 CFTP aztec {order}, {count} exact samples to coalescence", "seconds": dt,
            "collapsed_rounds": rr.tolist(), "chain_sweeps_per_sample": sweeps,
            "seconds_per_sample": dt / count}


def strips(torch, stream, quick):
    """Per-rank compute of strip-sharded Aztec walks (the strong-scaling
    share of one GPU): for N = 2, 4, 8 the busiest rank's window (its strip +
    32 halo rows per side) is swept alone on this GPU with the exchange
    kernels disabled -- the pool has one GPU, so NVLink time is not included."""
    import paper_1804_07250_b200 as ts
    from paper_1804_07250_b200 import _native
    from paper_1804_07250_b200.lattice import aztec_extremal_states
    from paper_1804_07250_b200.strips import strip_bounds
    from paper_1804_07250_b200.sweeps import DominoHandle

    out = []
    for order in ((1024,) if quick else (4096, 16384)):
        d = ts.Domain.aztec(order)
        t_max, _ = aztec_extremal_states(order)
        h = DominoHandle(d, d.n + 1, 1)
        h.set_stream(stream.cuda_stream)
        h.set_plan(ts.SweepPlan(d))
        h.upload(t_max[None])
        del t_max
        steps = 1024 if order <= 4096 else 256
        base = None
        for world in (1, 2, 4, 8):
            b = strip_bounds(d.vertex_mask, world, min_rows=32)
            times = []
            for r in range(world):
                lo, hi = max(0, b[r] - 32), min(d.n + 1, b[r + 1] + 32)
                _native.check(_native.lib().tsb_domino_set_window(h._h, lo, hi))
                h.walk([0x5EED], 64)
                times.append(timed(torch, stream, lambda: h.walk([0x5EED], steps, step0=64)) / steps)
            _native.check(_native.lib().tsb_domino_set_window(h._h, 0, -1))
            t = max(times)
            base = base or t
            out.append({"config": f"strips aztec {order}: busiest of {world} rank windows (halo 32), compute only",
                        "us_per_sweep": t * 1e6, "compute_speedup": base / t})
    return out


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--only", default="c1,c2,c3,c4,c5,mixed")
    p.add_argument("--quick", action="store_true")
    args = p.parse_args()
    import torch

    torch.cuda.set_device(0)
    stream = torch.cuda.current_stream()
    for name in args.only.split(","):
        r = globals()[name](torch, stream, args.quick)
        for x in r if isinstance(r, list) else [r]:
            print(json.dumps(x), flush=True)


if __name__ == "__main__":
    main()
