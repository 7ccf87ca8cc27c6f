"""Debug driver for the device strip exchange on one GPU (handles in one process)."""
import sys, time
import numpy as np
sys.path.insert(0, '.')
import oracle
import paper_1804_07250_b200 as ts
from paper_1804_07250_b200.lattice import aztec_extremal_states
from paper_1804_07250_b200.strips import DeviceStripWalker, strip_bounds
from paper_1804_07250_b200.sweeps import DominoHandle

world, halo, steps, order = (int(x) for x in sys.argv[1:5])
d = ts.Domain.aztec(order); plan = ts.SweepPlan(d); t_max, _ = aztec_extremal_states(order)
hs = []
for _ in range(world):
    h = DominoHandle(d, d.n + 1, 1, device=0); h.set_plan(plan); h.upload(t_max[None]); hs.append(h)
bounds = strip_bounds(d.vertex_mask, world, min_rows=halo)
print('bounds', bounds, flush=True)
ws = DeviceStripWalker.local(hs, bounds, halo)
t = time.time()
for w in ws:
    w.walk(0x5EED, steps, step0=5)
print('enqueued', time.time() - t, flush=True)
for i, w in enumerate(ws):
    try:
        print('status', i, w.status(), time.time() - t, flush=True)
    except Exception as e:
        print('status', i, 'ERR', e, flush=True)
got = np.concatenate([w.handle.download()[0][w.lo:w.hi] for w in ws])
ref = oracle.domino_walk(t_max[None].copy(), [0x5EED], plan.p_up, steps, step0=5)[0]
print('equal', np.array_equal(got, ref), flush=True)
