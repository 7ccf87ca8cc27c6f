"""Equilibrated Aztec-4096 start state for bench.py's warm sub-record.

T_max (closed form) walked for 2^26 = 67 M = 4 n^2 sweeps (order 4096) of
seed 0xA11CE on the device; the rotateable fraction is printed every 2^22
sweeps to show how far it has settled.  `--from old.npz` continues a shorter
walk of the same seed (steps old.sweeps .. SWEEPS - 1): counter-based coins
make that identical to one walk from T_max.  The state is stored as its two edge planes
bit-packed (numpy packbits of the V / H crossed-edge grids, 2 bits/vertex)
and compressed, with the sha256[:16] of the reference-layout uint8 tilestates
so bench.py can check what it loads.  Deterministic: the same seed and sweep
count reproduce the file bit for bit.

    python tools/make_warm_state.py [out.npz] [--from old.npz]   (GPU; ~15 min from T_max)
"""

import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

ORDER, SEED, SWEEPS, CHUNK = 4096, 0xA11CE, 1 << 26, 1 << 22


def planes_of(states: np.ndarray):
    """V[r, c] = edge (r,c)-(r+1,c) crossed (bit 2), H[r, c] = (r,c)-(r,c+1) (bit 8)."""
    return (states & 2) != 0, (states & 8) != 0


def states_of(v: np.ndarray, h: np.ndarray) -> np.ndarray:
    """Inverse of planes_of (lattice.py:51-53 tilestate bits)."""
    s = np.zeros(v.shape, dtype=np.uint8)
    s |= v.astype(np.uint8) << 1
    s[1:] |= v[:-1].astype(np.uint8)
    s |= h.astype(np.uint8) << 3
    s[:, 1:] |= h[:, :-1].astype(np.uint8) << 2
    return s


def load(path: str) -> np.ndarray:
    z = np.load(path)
    side = int(z["side"])
    v = np.unpackbits(z["v"], count=side * side).reshape(side, side).astype(bool)
    h = np.unpackbits(z["h"], count=side * side).reshape(side, side).astype(bool)
    s = states_of(v, h)
    fp = hashlib.sha256(s.tobytes()).hexdigest()[:16]
    if fp != str(z["sha"]):
        raise ValueError(f"warm state {path}: fingerprint {fp} != {z['sha']}")
    return s


def main(out, start=None):
    import paper_1804_07250_b200 as ts
    from paper_1804_07250_b200.lattice import aztec_extremal_states
    from paper_1804_07250_b200.sweeps import DominoHandle

    d = ts.Domain.aztec(ORDER)
    h = DominoHandle(d, d.n + 1, 1)
    h.set_plan(ts.SweepPlan(d))
    done, trace = 0, []
    if start:
        z = np.load(start)
        assert int(z["order"]) == ORDER and int(z["seed"]) == SEED and int(z["sweeps"]) < SWEEPS
        done, trace = int(z["sweeps"]), [list(x) for x in z["trace"]]
        h.upload(load(start)[None])
    else:
        h.upload(aztec_extremal_states(ORDER)[0][None])
    nv = int(d.vertex_mask.sum())
    t0 = time.time()
    while done < SWEEPS:
        n = min(CHUNK - done % CHUNK, SWEEPS - done)
        h.walk([SEED], n, step0=done)
        done += n
        s = h.download()[0]
        rot = int(((s == 3) | (s == 12)).sum())
        trace.append([done, rot / nv])
        print(json.dumps({"sweeps": done, "rotateable_frac": rot / nv,
                          "seconds": round(time.time() - t0, 1)}), flush=True)
    v, hz = planes_of(s)
    assert np.array_equal(states_of(v, hz), s)
    fp = hashlib.sha256(s.tobytes()).hexdigest()[:16]
    np.savez_compressed(out, v=np.packbits(v.ravel()), h=np.packbits(hz.ravel()), side=s.shape[0], sha=fp,
                        order=ORDER, seed=SEED, sweeps=SWEEPS, trace=np.array(trace))
    print(json.dumps({"out": out, "sha": fp, "bytes": os.path.getsize(out)}))


if __name__ == "__main__":
    import argparse

    ap = argparse.ArgumentParser()
    ap.add_argument("out", nargs="?", default=os.path.join(ROOT, "bench_data", "aztec4096_warm.npz"))
    ap.add_argument("--from", dest="start", default=None, help="continue this shorter walk of the same seed")
    a = ap.parse_args()
    main(a.out, a.start)
