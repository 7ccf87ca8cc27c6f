"""Per-rank window times of strip-sharded Aztec walks (TSB_DOM_ADAPT=0/1 A/B)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1804_07250_b200 as ts  # noqa: E402
from paper_1804_07250_b200 import _native  # noqa: E402
from paper_1804_07250_b200.lattice import aztec_extremal_states  # noqa: E402
from paper_1804_07250_b200.strips import strip_bounds  # noqa: E402
from paper_1804_07250_b200.sweeps import DominoHandle  # noqa: E402

order, world = int(sys.argv[1]), int(sys.argv[2])
d = ts.Domain.aztec(order)
t_max, _ = aztec_extremal_states(order)
h = DominoHandle(d, d.n + 1, 1)
h.set_plan(ts.SweepPlan(d))
h.upload(t_max[None])
b = strip_bounds(d.vertex_mask, world, min_rows=32)
for r in range(world):
    lo, hi = max(0, b[r] - 32), min(d.n + 1, b[r + 1] + 32)
    _native.check(_native.lib().tsb_domino_set_window(h._h, lo, hi))
    h.walk([0x5EED], 64)
    h.sync()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    h.walk([0x5EED], 1024, step0=64)
    h.sync()
    e1.record()
    torch.cuda.synchronize()
    print(f"adapt={os.environ.get('TSB_DOM_ADAPT', '1')} rank {r} rows [{lo},{hi}): {1000 * e0.elapsed_time(e1) / 1024:.3f} us/sweep")
