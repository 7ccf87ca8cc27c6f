import os, sys, numpy as np
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import oracle, paper_1804_07250_b200 as ts
from paper_1804_07250_b200.sweeps import DominoHandle
g = np.load('/root/repo/tests/golden/domino_cftp.npz')
d = ts.Domain(g["k0_faces"].shape[0], g["k0_faces"]); plan = ts.SweepPlan(d)
t_max, t_min = ts.extremal_tilings(d)
print("side", d.n + 1)
for steps in (2, 3, 5, 64, 200):
    st = np.stack([t_max.states, t_min.states, t_max.states, t_min.states])
    seeds = np.array([5, 5, 9, 9], dtype=np.uint64)
    h = DominoHandle(d, d.n + 1, 4); h.set_plan(plan); h.upload(st); h.walk(seeds, steps)
    ref = oracle.domino_walk(st, seeds, plan.p_up, steps)
    print(steps, [bool(np.array_equal(a, b)) for a, b in zip(h.download(), ref)])
