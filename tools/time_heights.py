"""Time the domino height export (row scan vs relaxation) and the mean-height
accumulator at Aztec 4096 / 16384 after a short walk from T_max; one JSON line
per case on stdout (profiles/round2_heights.jsonl)."""

import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1804_07250_b200 as ts  # noqa: E402
from paper_1804_07250_b200.lattice import aztec_extremal_states  # noqa: E402
from paper_1804_07250_b200.stats import DeviceDensity  # noqa: E402
from paper_1804_07250_b200.sweeps import DominoHandle  # noqa: E402


def run(order, relax, sweeps=200, reps=3):
    os.environ["TSB_HEIGHTS_RELAX"] = "1" if relax else "0"
    d = ts.Domain.aztec(order)
    t_max, _ = aztec_extremal_states(order)
    h = DominoHandle(d, d.n + 1, 1)
    h.set_plan(ts.SweepPlan(d))
    h.upload(t_max[None])
    h.walk([0x5EED], sweeps)
    h.sync()
    ref = d.reference_vertex
    out = h.heights(0, ref)  # classify + warm
    ts_ = []
    for _ in range(reps):
        t0 = time.perf_counter()
        out = h.heights(0, ref)
        ts_.append(time.perf_counter() - t0)
    acc = DeviceDensity(h, "height")
    acc.add()
    torch.cuda.synchronize()
    ta = []
    for _ in range(reps):
        t0 = time.perf_counter()
        acc.add()
        h.sync()
        ta.append(time.perf_counter() - t0)
    ok = bool(np.array_equal(acc.counts(), (1 + reps) * out.astype(np.int64)))
    return {"order": order, "path": "relax" if relax else "row-scan", "sweeps": sweeps,
            "heights_ms": 1e3 * min(ts_), "sum_add_ms": 1e3 * min(ta), "acc_consistent": ok,
            "note": "heights_ms includes the (side^2 int32) D2H copy to pageable host memory; "
                    "sum_add_ms is device-only (accumulator stays on the GPU)"}


if __name__ == "__main__":
    for order, relax in ((4096, False), (4096, True), (16384, False)):
        print(json.dumps(run(order, relax)), flush=True)
