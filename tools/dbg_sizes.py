#!/usr/bin/env python
"""µs per sweep of one domino chain on Aztec diamonds of several orders, from
T_max (run under different TSB_* settings to compare kernel variants)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1804_07250_b200 as ts  # noqa: E402
from paper_1804_07250_b200.lattice import aztec_extremal_states  # noqa: E402
from paper_1804_07250_b200.sweeps import DominoHandle  # noqa: E402

tag = " ".join(f"{k}={v}" for k, v in os.environ.items() if k.startswith("TSB_")) or "default"
orders = [int(x) for x in (sys.argv[1:] or ["2048", "4096", "8192", "12288", "16384"])]
for order in orders:
    d = ts.Domain.aztec(order)
    t_max, _ = aztec_extremal_states(order)
    h = DominoHandle(d, d.n + 1, 1)
    h.set_plan(ts.SweepPlan(d))
    h.upload(t_max[None])
    h.walk([7], 256)
    S = 512
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    h.sync()
    e0.record()
    h.walk([7], S, step0=256)
    h.sync()
    e1.record()
    torch.cuda.synchronize()
    print(f"{tag} aztec {order}: {1000 * e0.elapsed_time(e1) / S:.3f} us/sweep", flush=True)
    del h
