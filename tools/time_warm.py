"""Device time per sweep at Aztec 4096 from the committed warm state
(bench_data/aztec4096_warm.npz) vs from T_max: CUDA events on the handle's
stream, 1000-sweep steps after a 1000-sweep warm-up.  One JSON line."""

import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import torch  # noqa: E402

import paper_1804_07250_b200 as ts  # noqa: E402
from make_warm_state import load  # noqa: E402
from paper_1804_07250_b200.lattice import aztec_extremal_states  # noqa: E402
from paper_1804_07250_b200.sweeps import DominoHandle  # noqa: E402

d = ts.Domain.aztec(4096)
nv = int(d.vertex_mask.sum())
out = {}
for name, st in (("warm", load(os.path.join(ROOT, "bench_data", "aztec4096_warm.npz"))),
                 ("tmax", aztec_extremal_states(4096)[0])):
    h = DominoHandle(d, d.n + 1, 1)
    stream = torch.cuda.current_stream()
    h.set_stream(stream.cuda_stream)
    h.set_plan(ts.SweepPlan(d))
    h.upload(st[None])
    h.walk([7], 1000)
    ts_ = []
    for k in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        h.walk([7], 1000, step0=1000 * (k + 1))
        b.record(stream)
        torch.cuda.synchronize()
        ts_.append(a.elapsed_time(b))
    s = h.download()[0]
    out[name] = {"us_per_sweep": min(ts_), "us_per_sweep_all": [round(x, 3) for x in ts_],
                 "rotateable_frac": float(((s == 3) | (s == 12)).sum() / nv),
                 "frac_of_roofline": nv / (min(ts_) * 1e-6) / 1e9 / 6463.7}
print(json.dumps(out))
