"""Time domino walks restricted to row windows of the Aztec 4096 diamond."""
import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
import paper_1804_07250_b200 as ts
from paper_1804_07250_b200 import _native
from paper_1804_07250_b200.lattice import aztec_extremal_states
from paper_1804_07250_b200.sweeps import DominoHandle
order = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
d = ts.Domain.aztec(order); t_max, _ = aztec_extremal_states(order)
h = DominoHandle(d, d.n + 1, 1); h.set_plan(ts.SweepPlan(d)); h.upload(t_max[None])
mid = (d.n + 1) // 2
for rows in (8193, 4096, 2048, 1024, 512, 256, 128, 64, 24):
    lo, hi = max(0, mid - rows // 2), min(d.n + 1, mid + rows // 2)
    _native.check(_native.lib().tsb_domino_set_window(h._h, lo, hi))
    h.walk([1], 64); h.sync()
    torch.cuda.synchronize()
    t = time.perf_counter(); h.walk([1], 1024, step0=64); h.sync(); dt = time.perf_counter() - t
    print(f"rows {rows:5d}  us/sweep {dt / 1024 * 1e6:7.2f}", flush=True)
