"""Debug: device CFTP (tsb_domino_cftp) top/bottom chains after every round
vs oracle replays of run_cftp_batch's round loop (cftp.py:111-120)."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle
import paper_1804_07250_b200 as ts
from paper_1804_07250_b200.cftp import chain_master_seed, schedule_seed
from paper_1804_07250_b200.sweeps import DominoCftp

g = np.load(os.path.join(ROOT, "tests", "golden", "domino_cftp.npz"))
case, master, count = int(sys.argv[1]) if len(sys.argv) > 1 else 0, 999, 7
d = ts.Domain(g[f"k{case}_faces"].shape[0], g[f"k{case}_faces"])
plan = ts.SweepPlan(d)
t_max, t_min = ts.extremal_tilings(d)
masters = np.array([chain_master_seed(master, k) for k in range(count)], dtype=np.uint64)
run = DominoCftp(d, plan, t_max.states, t_min.states, count)
seen = []
def progress(r, steps, collapsed, total):
    seen.append(run.handle.download(0, 2 * count))
try:
    run.run(masters, 3, progress=progress)
except Exception as e:
    print("run:", type(e).__name__, e)
for r in range(1, len(seen) + 1):
    for k in range(count):
        seeds = [schedule_seed(int(masters[k]), i) for i in range(1, r + 1)]
        top, bot = t_max.states[None].copy(), t_min.states[None].copy()
        for i in range(r, 0, -1):
            top = oracle.domino_walk(top, [seeds[i - 1]], plan.p_up, 2 ** i)
            bot = oracle.domino_walk(bot, [seeds[i - 1]], plan.p_up, 2 ** i)
        st = seen[r - 1]
        ok_t, ok_b = np.array_equal(st[2 * k], top[0]), np.array_equal(st[2 * k + 1], bot[0])
        if not (ok_t and ok_b) or r == 1:
            print(f"round {r} sample {k}: top {'ok' if ok_t else 'DIFF'} bottom {'ok' if ok_b else 'DIFF'}"
                  f" ref_coalesced {np.array_equal(top, bot)} dev_top==T_max {np.array_equal(st[2*k], t_max.states)}"
                  f" ref_top==T_max {np.array_equal(top[0], t_max.states)} dev_top==ref_bot {np.array_equal(st[2*k], bot[0])}")
        if r > 1 and k > 0: break
