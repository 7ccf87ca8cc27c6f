#!/usr/bin/env python
"""Wall time of exact CFTP samples on small domains of the three models."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1804_07250_b200 as ts  # noqa: E402

for a in (8, 16, 32):
    d = ts.Domain.aztec(a)
    ts.cftp_sample_many(d, ts.SweepPlan(d), 1, 2)
    t0 = time.perf_counter()
    ts.cftp_sample_many(d, ts.SweepPlan(d), 7, 64)
    print(f"domino aztec {a}: 64 samples {time.perf_counter() - t0:.3f} s", flush=True)
for a in (4, 8, 16):
    d = ts.TriDomain.hexagon(a, a, a)
    ts.loz_cftp(d, ts.Uniform(), 1, count=2)
    t0 = time.perf_counter()
    ts.loz_cftp(d, ts.Uniform(), 7, count=64)
    print(f"lozenge hexagon {a}: 64 samples {time.perf_counter() - t0:.3f} s", flush=True)
for n in (8, 16, 32):
    b = ts.dwbc(n)
    w = ts.SVWeights(1.0, 1.0, 1.0)
    ts.sv_cftp(n, b, w, 1, count=2)
    t0 = time.perf_counter()
    ts.sv_cftp(n, b, w, 7, count=64)
    print(f"six-vertex dwbc {n}: 64 samples {time.perf_counter() - t0:.3f} s", flush=True)
