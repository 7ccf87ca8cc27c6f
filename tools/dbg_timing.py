"""Per-block phase timestamps of the multi-sweep kernel (TSB_TIMING build):
TSB_LIB=.../libtsb_timing.so python tools/dbg_timing.py <window rows>"""
import ctypes, sys
sys.path.insert(0, '.')
import numpy as np
import paper_1804_07250_b200 as ts
from paper_1804_07250_b200 import _native
from paper_1804_07250_b200.lattice import aztec_extremal_states
from paper_1804_07250_b200.sweeps import DominoHandle
rows = int(sys.argv[1]); order = 4096
d = ts.Domain.aztec(order); t_max, _ = aztec_extremal_states(order)
h = DominoHandle(d, d.n + 1, 1); h.set_plan(ts.SweepPlan(d)); h.upload(t_max[None])
mid = (d.n + 1) // 2
_native.check(_native.lib().tsb_domino_set_window(h._h, mid - rows // 2, mid + rows // 2))
h.walk([1], 64); h.sync()
L = _native.lib(); L.tsb_debug_timing.argtypes = [ctypes.c_void_p]
h.walk([1], 32, step0=64); h.sync()
tt = np.zeros((16, 2048, 6), dtype=np.uint64)
L.tsb_debug_timing(tt.ctypes.data)
nb = int((tt[0, :, 5] > 0).sum())
t0 = tt[0, :nb, 0].min()
print("blocks", nb)
for l in range(16):
    x = tt[l, :nb].astype(np.int64) - int(t0)
    print(f"launch {l:2d}: start {x[:,0].min():7d}..{x[:,0].max():7d}  wait_done {x[:,2].min():7d}..{x[:,2].max():7d}"
          f"  sweep0 {np.median(x[:,3]-x[:,2]):6.0f}  sweep1 {np.median(x[:,4]-x[:,3]):6.0f}  end {x[:,5].max():7d}")
print("per-block phases of launch 5 (ns from its first start): start, launched_dep, wait_done, sweep0_end, sweep1_end, end")
x = tt[5, :nb].astype(np.int64)
x = x - x[:, 0].min()
for b in range(min(nb, 20)):
    print(b, list(x[b]))
