"""Where the time of a pageable `random_walk` call goes at Aztec 4096:
upload / walk / download of the reference's uint8 tilestates through the
handle, pageable vs pinned, fresh vs pre-faulted output arrays."""

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


def t(fn, reps=5):
    best = 1e9
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        best = min(best, time.perf_counter() - t0)
    return 1e3 * best


order = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
d = ts.Domain.aztec(order)
plan = ts.SweepPlan(d)
t_max, _ = aztec_extremal_states(order)
side = d.n + 1
h = DominoHandle(d, side, 1)
h.set_plan(plan)
pageable = t_max[None].copy()
pinned = torch.empty((1, side, side), dtype=torch.uint8, pin_memory=True).numpy()
pinned[:] = pageable
out_pre = np.empty_like(pageable)
out_pre[:] = 1
res = {
    "order": order, "bytes": int(pageable.nbytes),
    "upload_pageable_ms": t(lambda: h.upload(pageable)),
    "upload_pinned_ms": t(lambda: h.upload(pinned)),
    "walk1000_ms": t(lambda: (h.walk([1], 1000), h.sync())),
    "download_pageable_prefaulted_ms": t(lambda: h.download(out=out_pre)),
    "download_pinned_ms": t(lambda: h.download(out=pinned)),
    "download_fresh_ms": t(lambda: h.download()),
    "np_empty_fill_ms": t(lambda: np.empty_like(pageable).fill(0)),
    "np_copy_ms": t(lambda: pageable.copy()),
    "random_walk_1000_ms": t(lambda: ts.random_walk(ts.Tiling(d, pageable[0]), 5, 1000, plan), 3),
    "cpus": os.cpu_count(),
    "thp": open("/sys/kernel/mm/transparent_hugepage/enabled").read().strip()
    if os.path.exists("/sys/kernel/mm/transparent_hugepage/enabled") else None,
}
print(json.dumps(res))
