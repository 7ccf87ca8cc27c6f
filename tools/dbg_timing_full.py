"""Per-block timeline of whole-domain multi-sweep launches at Aztec 4096 in
the bench's state (TSB_TIMING build):
TSB_LIB=paper_1804_07250_b200/_lib/libtsb_timing.so python tools/dbg_timing_full.py [warm sweeps]"""
import ctypes
import sys

sys.path.insert(0, '.')
import numpy as np

import paper_1804_07250_b200 as ts
from paper_1804_07250_b200 import _native
from paper_1804_07250_b200.lattice import aztec_extremal_states
from paper_1804_07250_b200.sweeps import DominoHandle

warm = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
order = 4096
d = ts.Domain.aztec(order)
t_max, _ = aztec_extremal_states(order)
h = DominoHandle(d, d.n + 1, 1)
h.set_plan(ts.SweepPlan(d))
h.upload(t_max[None])
h.walk([1], warm)
h.sync()
h.walk([1], 512, step0=warm)  # graph replays: the adaptive order settles
warm += 512
h.sync()
L = _native.lib()
L.tsb_debug_timing.argtypes = [ctypes.c_void_p]
h.walk([1], 32, step0=warm)  # 16 direct multi-sweep launches (< one graph replay)
h.sync()
tt = np.zeros((16, 2048, 6), dtype=np.uint64)
L.tsb_debug_timing(tt.ctypes.data)
nb = int((tt[0, :, 5] > 0).sum())
print("blocks per launch", nb)
for l in range(1, 16):
    x = tt[l, :nb].astype(np.int64)
    t0 = x[:, 0].min()
    x = x - t0
    dur = x[:, 5] - x[:, 2]
    prev_end = (tt[l - 1, :nb, 5].astype(np.int64) - t0).max()
    q = np.percentile(dur, [10, 50, 90, 99, 100]).astype(int)
    last_start = x[:, 2].max()
    heavy = np.argsort(dur)[-3:]
    print(f"launch {l:2d}: prev grid end {prev_end:6d}  waits done {x[:,2].min():6d}..{last_start:6d}  end {x[:,5].max():6d}"
          f"  block ns p10/50/90/99/max {q.tolist()}  slowest blocks {heavy.tolist()}")
