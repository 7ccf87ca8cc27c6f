#!/usr/bin/env python
"""µs per sweep of domino walks on small Aztec diamonds (resident vs tiled:
run once with TSB_DOM_RESIDENT=0 and once without)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1804_07250_b200 as ts  # noqa: E402
from paper_1804_07250_b200.lattice import aztec_extremal_states  # noqa: E402
from paper_1804_07250_b200.sweeps import DominoHandle  # noqa: E402

mode = os.environ.get("TSB_DOM_RESIDENT", "auto")
for order in (16, 32, 64, 128, 256):
    for nch in (1, 128):
        d = ts.Domain.aztec(order)
        t_max, _ = aztec_extremal_states(order)
        h = DominoHandle(d, d.n + 1, nch)
        h.set_plan(ts.SweepPlan(d))
        h.upload(t_max[None].repeat(nch, 0))
        seeds = list(range(1, nch + 1))
        h.walk(seeds, 2048)
        h.sync()
        S = 4096
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        h.walk(seeds, S, step0=2048)
        h.sync()
        e1.record()
        torch.cuda.synchronize()
        print(f"mode={mode} aztec {order} chains {nch}: {1000 * e0.elapsed_time(e1) / S:.3f} us/sweep", flush=True)
