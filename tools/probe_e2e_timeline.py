"""Host timeline of random_walk_batch's two-handle pipeline at Aztec 4096
(B = 2, 1000 sweeps, every sweep executed): upload A, walk A, upload B,
walk B, download A, download B, with chain B's walk either free to share
the GPU with chain A's or ordered after it (event wait between the two
handles' torch streams)."""

import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1804_07250_b200 as ts  # noqa: E402
from paper_1804_07250_b200.lattice import aztec_extremal_states  # noqa: E402
from paper_1804_07250_b200.sweeps import DominoHandle  # noqa: E402

d = ts.Domain.aztec(4096)
plan = ts.SweepPlan(d)
t_max, t_min = aztec_extremal_states(4096)
states = np.stack([t_max, t_min])
streams = [torch.cuda.Stream(), torch.cuda.Stream()]
hs = []
for s in streams:
    h = DominoHandle(d, d.n + 1, 1)
    h.set_collapse(False)
    h.set_stream(s.cuda_stream)
    h.set_plan(plan)
    hs.append(h)
out = np.empty_like(states)
res = {}
for rep in range(4):
    for order in (False, True):
        torch.cuda.synchronize()
        t = [time.perf_counter()]
        hs[0].upload(states[0:1]); t.append(time.perf_counter())
        hs[0].walk([11], 1000); t.append(time.perf_counter())
        hs[1].upload(states[1:2]); t.append(time.perf_counter())
        if order:
            ev = torch.cuda.Event()
            ev.record(streams[0])
            streams[1].wait_event(ev)
        hs[1].walk([12], 1000); t.append(time.perf_counter())
        hs[0].download(out=out[0:1]); t.append(time.perf_counter())
        hs[1].download(out=out[1:2]); t.append(time.perf_counter())
        if rep:
            key = "ordered" if order else "shared"
            res.setdefault(key, []).append([round(1e3 * (b - a), 2) for a, b in zip(t, t[1:])] + [round(1e3 * (t[-1] - t[0]), 2)])
print(json.dumps({"columns": ["upload A", "walk A", "upload B", "walk B", "download A", "download B", "total"], **res}))
