#!/usr/bin/env python
"""Small fixed workloads for ncu captures of one kernel family.

    python tools/prof_driver.py sv   [--n 2048] [--warm 2000] [--sweeps 64]
    python tools/prof_driver.py lz   [--n 1000] ...
    python tools/prof_driver.py dom  [--n 4096] ...

Warms the chain up (so the captured launches see a mixed state), then runs
`--sweeps` more sweeps; run under `ncu -k regex:<kernel> -s <skip> -c <count>`.
"""

from __future__ import annotations

import argparse
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    p = argparse.ArgumentParser()
    p.add_argument("model", choices=["sv", "lz", "dom"])
    p.add_argument("--n", type=int, default=0)
    p.add_argument("--warm", type=int, default=2000)
    p.add_argument("--sweeps", type=int, default=64)
    p.add_argument("--state", default="", help="dom: start from this warm-state npz (tools/make_warm_state.py)")
    a = p.parse_args()
    import torch

    import paper_1804_07250_b200 as ts

    if a.model == "sv":
        from paper_1804_07250_b200.sixvertex import SixVertexHandle

        n = a.n or 2048
        hi, lo = ts.sv_extremal(n, ts.dwbc(n))
        h = SixVertexHandle(n, 1)
        h.set_weights(ts.SVWeights(1.0, 1.0, 1.0))
        h.upload(lo.heights[None])
    elif a.model == "lz":
        from paper_1804_07250_b200.lozenge import LozengeHandle, loz_p_up_grid

        n = a.n or 1000
        d = ts.TriDomain.hexagon(n, n, n)
        t_max, t_min = ts.loz_extremal(d)
        h = LozengeHandle(d, 1)
        h.set_p_up(loz_p_up_grid(d, ts.VolumeWeights(0.999)))
        h.upload(t_min.edges[None])
    else:
        from paper_1804_07250_b200.lattice import aztec_extremal_states
        from paper_1804_07250_b200.sweeps import DominoHandle

        n = a.n or 4096
        d = ts.Domain.aztec(n)
        t_max, _ = aztec_extremal_states(n)
        h = DominoHandle(d, d.n + 1, 1)
        h.set_plan(ts.SweepPlan(d))
        if a.state:
            sys.path.insert(0, os.path.join(ROOT, "tools"))
            from make_warm_state import load

            h.upload(load(a.state)[None])
        else:
            h.upload(t_max[None])
    h.walk([0x5EED], a.warm)
    h.walk([0x5EED], a.sweeps, step0=a.warm)
    torch.cuda.synchronize()
    print("done", a.model, n, math.nan if False else a.sweeps)


if __name__ == "__main__":
    main()
