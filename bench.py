#!/usr/bin/env python
"""Headline benchmark: domino Glauber sweeps on the Aztec diamond, order 4096.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Metric (BASELINE.json): flip attempts/s = in-domain sites of the active
colour class per sweep x sweeps / time, on the Aztec diamond of order 4096
(33,579,009 in-domain vertices), uniform weights, start T_max, seed 0x5EED.

One "step" = `--sweeps-per-step` consecutive sweeps (default 1000) of one
chain; between timed steps L2 is flushed by writing a 256 MiB buffer
(outside the events), each step timed with CUDA events on the launching
stream, and the per-rank total is reduced with MAX over ranks.  With N > 1
(torchrun), --mode replicas runs one independent chain of the workload per
GPU (weak scaling; the way an MCMC sampler uses more GPUs when one lattice
fits a GPU) and --mode strips shards ONE chain into row strips (strong
scaling): each rank sweeps its rows plus --halo halo rows and refreshes the
halos from its neighbours every --halo sweeps with push/pull kernels over
peer memory (csrc/strips.cu; --host-exchange: NCCL from the host instead).
The default (auto) shards lattices above order 8192 (BASELINE config 4) and
replicates smaller ones: at order 4096 a 1/8 strip is latency-bound
(~4.4 us per sweep for the busiest strip vs 6.2 us for the whole lattice,
profiles/round1_strips_compute.jsonl).  Rank 0 prints one JSON line.

`--impl reference` times the reference algorithm's CPU path (the C port in
oracle/, all host threads) on the same workload, rank 0 only.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "flip attempts/sec (Aztec diamond n=4096, 1/2/4/8 B200) vs HBM roofline"
UNIT = "flip attempts/s"
SEED = 0x5EED


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--order", type=int, default=4096)
    p.add_argument("--sweeps-per-step", type=int, default=1000)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-warm", action="store_true", help="skip the equilibrating-state sub-record")
    p.add_argument("--no-collapsed", action="store_true", help="skip the run-collapsing sub-record")
    p.add_argument("--mode", default="auto", choices=["auto", "replicas", "strips"],
                   help="N>1: independent chains per GPU (weak scaling) or one strip-sharded chain "
                        "(strong scaling); auto = strips above order 8192")
    p.add_argument("--replicas", action="store_true", help="alias for --mode replicas")
    p.add_argument("--halo", type=int, default=64, help="strip sharding: halo rows = sweeps between exchanges")
    p.add_argument("--host-exchange", action="store_true",
                   help="strip sharding: host-driven NCCL halo exchange instead of the device push/pull kernels")
    return p.parse_args()


def workload(order: int):
    import paper_1804_07250_b200 as ts
    from paper_1804_07250_b200.lattice import aztec_extremal_states

    d = ts.Domain.aztec(order)
    t_max, _ = aztec_extremal_states(order)
    return d, t_max, aztec_counts(order)


# ---- package-free host side of the workload (the reference arm and the CPU
# baseline never import paper_1804_07250_b200 or load libtsb.so) -------------
_M64 = (1 << 64) - 1


def _mix(z: int) -> int:
    """splitmix64 finaliser (reference rng.py:34-39)."""
    z &= _M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


def _color_at(seed: int, step: int) -> int:
    """Domino colour coin (sweeps.py:266-269: WHITE iff u >= 0.5 = bit 63 of
    the global draw; global key rng.py:101-103)."""
    g = 0x9E3779B97F4A7C15
    gkey = _mix(_mix((seed & _M64) ^ 0x6A09E667F3BCC909) + ((1 << 48) + 1) * g)
    return _mix(gkey + (step + 1) * g) >> 63


def _face_range(order: int, i: int):
    """Columns [a, b] of face row i of the Aztec diamond (Domain.aztec,
    lattice.py:156-162: |r+0.5-order| + |c+0.5-order| <= order)."""
    di = abs(2 * i + 1 - 2 * order)  # 2 * |i + 0.5 - order|
    return (di - 1) // 2, (4 * order - di - 1) // 2


def aztec_counts(order: int):
    """(BLACK, WHITE) in-domain vertices (vertex_mask: vertices touching a
    face), row by row without V x V temporaries."""
    n = 2 * order
    black = total = 0
    for r in range(n + 1):
        rows = [i for i in (r - 1, r) if 0 <= i < n]
        a = min(_face_range(order, i)[0] for i in rows)
        b = max(_face_range(order, i)[1] for i in rows) + 1
        cnt = b - a + 1
        first_even = (a + r) % 2 == 0
        black += (cnt + 1) // 2 if first_even else cnt // 2
        total += cnt
    return black, total - black


def aztec_tmax_host(order: int) -> np.ndarray:
    """Closed-form T_max: all-horizontal bricks for
    even order, all-vertical for odd, each row (column) paired from its first
    face; the tilestate bit of a brick's interior edge (lattice.py:51-53)."""
    n = 2 * order
    s = np.zeros((n + 1, n + 1), dtype=np.uint8)
    for i in range(n):
        a, b = _face_range(order, i)
        x = np.arange(a + 1, b + 1, 2)
        s[i, x] |= 2
        s[i + 1, x] |= 1
    if order % 2 == 0:
        return s
    t = np.ascontiguousarray(s.T)
    return (((t & 1) << 2) | ((t & 2) << 2)).astype(np.uint8)


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


MK = 2            # sweeps per domino_multi_kernel launch (kMK in csrc/domino.cu)
GRAPH_SWEEPS = 64  # sweeps per CUDA-graph replay (kGraphSweeps)


def launches_per_walk(n: int) -> int:
    """Kernels one tsb_domino_walk of n sweeps launches: set_walk (step base
    and the first colour table), then per graph replay GRAPH_SWEEPS/MK
    multi-sweep kernels and the replay tail (adaptive reorder when due, step
    advance, next colour table); the remainder as direct multi-sweep
    launches (after set_walk when there was no replay) and at most one
    single-sweep kernel."""
    replays, rem = divmod(n, GRAPH_SWEEPS)
    k = 1 + replays * (1 + GRAPH_SWEEPS // MK) if replays else 0
    if rem >= MK:  # remainder: (set_walk,) direct multi-sweep launches
        k += (0 if replays else 1) + rem // MK
        rem %= MK
    return k + rem


def attempts_for(seed: int, step0: int, n: int, counts) -> int:
    return sum(counts[_color_at(seed, s)] for s in range(step0, step0 + n))


def traffic(kernel: str):
    """DRAM bytes per launch from the committed ncu capture (profiles/traffic.json)."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            return int(json.load(f)[kernel]["dram_bytes_per_launch"])
    except Exception:
        return None


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append(ln.strip())

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def strips_mode(args, world: int) -> bool:
    """N > 1: one strip-sharded chain (strong scaling) or replicas (weak)."""
    mode = "replicas" if args.replicas else args.mode
    if mode == "auto":
        mode = "strips" if args.order > 8192 else "replicas"
    return world > 1 and mode == "strips"


def bench_config(args, world: int, strips: bool) -> dict:
    """The `config` object both arms print (identical for the same flags)."""
    black, white = aztec_counts(args.order)
    return {"workload": f"aztec{args.order}_uniform_from_Tmax", "order": args.order,
            "domain_vertices": black + white, "sweeps_per_step": args.sweeps_per_step, "seed": SEED,
            "parallelism": (f"strips x{world}, halo {args.halo} rows exchanged every {args.halo} sweeps "
                            + ("(host NCCL p2p)" if args.host_exchange else "(device push/pull over peer memory)")
                            + ", each rank holding only its window of rows"
                            if strips else (f"replicas x{world}" if world > 1 else "single chain")),
            "l2": "flushed (256 MiB write) between timed steps; state planes stay "
                  "L2-resident within a step by design"}


def cpu_baseline(order: int, budget_s: float = 12.0):
    """The reference algorithm's CPU path (oracle/ C port of _kernels.py
    domino_walk, pthread row bands over all host threads) on a bounded sample."""
    import oracle

    t_max, counts = aztec_tmax_host(order), aztec_counts(order)
    threads = os.cpu_count() or 1
    p_up = np.full(t_max.shape, 0.5)
    t0 = time.perf_counter()
    s = oracle.domino_walk(t_max[None], [SEED], p_up, 1, threads=threads)
    one = time.perf_counter() - t0
    n = max(2, min(2000, int(budget_s / max(one, 1e-6))))
    t0 = time.perf_counter()
    oracle.domino_walk(s, [SEED], p_up, n, step0=1, threads=threads)
    dt = time.perf_counter() - t0
    att = attempts_for(SEED, 1, n, counts)
    return {"value": att / dt, "unit": UNIT, "cores": threads, "kind": "port", "cpu": cpu_model(),
            "sample": f"aztec order {order} from T_max, sweeps 1..{n} of seed 0x5EED ({dt:.1f} s)"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle  # the C port of the reference's CPU path; nothing of the product is imported

    t_max, counts = aztec_tmax_host(args.order), aztec_counts(args.order)
    threads = os.cpu_count() or 1
    p_up = np.full(t_max.shape, 0.5)
    s = t_max[None].copy()
    per_step = args.sweeps_per_step  # the same step as the GPU arm (1000 sweeps: ~5 s on 16 host threads)
    step = 0
    for _ in range(args.warmup):
        s = oracle.domino_walk(s, [SEED], p_up, per_step, step0=step, threads=threads)
        step += per_step
    t0 = time.perf_counter()
    first = step
    for _ in range(args.steps):
        s = oracle.domino_walk(s, [SEED], p_up, per_step, step0=step, threads=threads)
        step += per_step
    dt = time.perf_counter() - t0
    att = attempts_for(SEED, first, step - first, counts)
    value = att / dt
    sample = (f"aztec order {args.order} from T_max, {per_step} sweeps/step, "
              f"{args.steps} steps after {args.warmup} warm-up steps")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
        "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u8",
        "data": "synthetic: Aztec diamond from the closed-form T_max, uniform weights",
        "config": bench_config(args, args.gpus, strips_mode(args, args.gpus)),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port", "sample": sample,
                         "cpu": cpu_model()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def relaunch_under_torchrun(args) -> int:
    """`--gpus N` (N > 1) without a torchrun environment: start N ranks of
    this script the way the driver does (one process per GPU, 127.0.0.1)."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def warm_record(args, d, plan, counts, stream, flush, red_dev, world, torch, dist, seed, collapse=False):
    """The same step timed from the committed warm state instead of T_max
    (bench_data/aztec4096_warm.npz: T_max + 4 n^2 sweeps, ~11 % of vertices
    rotateable, i.e. the regime a sampler spends its life in; the frozen T_max
    start has 0.3 %).  Device events per step, L2 flushed between steps."""
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    from make_warm_state import load

    from paper_1804_07250_b200.sweeps import DominoHandle

    path = os.path.join(ROOT, "bench_data", "aztec4096_warm.npz")
    st = load(path)  # raises if the fingerprint does not match
    h = DominoHandle(d, d.n + 1, 1)
    h.set_collapse(collapse)
    h.set_stream(stream.cuda_stream)
    h.set_plan(plan)
    h.upload(st[None])
    S = args.sweeps_per_step
    step = 0
    for _ in range(args.warmup):
        h.walk([seed], S, step0=step)
        step += S
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    first = step
    for k in range(args.steps):
        flush.zero_()
        ev[k][0].record(stream)
        h.walk([seed], S, step0=step)
        ev[k][1].record(stream)
        step += S
    torch.cuda.synchronize()
    ms = sum(a.elapsed_time(b) for a, b in ev)
    att = attempts_for(seed, first, step - first, counts)
    t = torch.tensor([ms], dtype=torch.float64, device=red_dev)
    a = torch.tensor([float(att)], dtype=torch.float64, device=red_dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(a, op=dist.ReduceOp.SUM)
    fin = h.download()[0]
    nv = counts[0] + counts[1]
    rot = float(((fin == 3) | (fin == 12)).sum()) / nv
    per_launch_ms = float(t.item()) / (args.steps * S / MK)
    achieved = MK * nv / (per_launch_ms / 1e3) / 1e9
    peak, _ = peaks()
    return {"value": float(a.item()) / (float(t.item()) / 1e3), "unit": UNIT,
            "ms_per_step": float(t.item()) / args.steps, "us_per_sweep": 1e3 * float(t.item()) / (args.steps * S),
            "rotateable_frac_end": rot,
            "roofline": {"achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak},
            "state": "bench_data/aztec4096_warm.npz (T_max + %d sweeps of seed 0xA11CE, sha %s)"
                     % (int(np.load(path)["sweeps"]), str(np.load(path)["sha"]))}


def collapsed_record(args, d, plan, t_max, counts, stream, flush, red_dev, world, torch, dist, seed):
    """The library default (tsb_domino_set_collapse): a sweep followed by a
    sweep of the same colour is skipped -- the move is a heat-bath update and
    a colour's rotateable set cannot change while only that colour moves, so
    the last sweep of a run decides and the states are bit-identical (tests
    run with collapsing on and off).  Reported beside, not in, the headline:
    the attempt count is the reference's workload, about half of whose sweeps
    are executed here.  Same steps as the headline, from T_max and from the
    warm state."""
    from paper_1804_07250_b200.sweeps import DominoHandle

    h = DominoHandle(d, d.n + 1, 1)
    h.set_collapse(True)
    h.set_stream(stream.cuda_stream)
    h.set_plan(plan)
    h.upload(t_max[None])
    S = args.sweeps_per_step
    step = 0
    for _ in range(args.warmup):
        h.walk([seed], S, step0=step)
        step += S
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    first = step
    for k in range(args.steps):
        flush.zero_()
        ev[k][0].record(stream)
        h.walk([seed], S, step0=step)
        ev[k][1].record(stream)
        step += S
    torch.cuda.synchronize()
    ms = sum(a.elapsed_time(b) for a, b in ev)
    executed = sum(1 for s in range(first, step)
                   if (s + 1 - first) % S == 0 or _color_at(seed, s) != _color_at(seed, s + 1))  # walk ends: never skipped
    att = attempts_for(seed, first, step - first, counts)
    t = torch.tensor([ms], dtype=torch.float64, device=red_dev)
    a = torch.tensor([float(att)], dtype=torch.float64, device=red_dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(a, op=dist.ReduceOp.SUM)
    rec = {"value": float(a.item()) / (float(t.item()) / 1e3), "unit": UNIT,
           "us_per_sweep": 1e3 * float(t.item()) / (args.steps * S),
           "sweeps_executed_frac": executed / (step - first)}
    if args.order == 4096 and not args.no_warm:
        w = warm_record(args, d, plan, counts, stream, flush, red_dev, world, torch, dist, seed, collapse=True)
        rec["warm"] = {"value": w["value"], "us_per_sweep": w["us_per_sweep"]}
    return rec


def main():
    args = parse()
    world_env = os.environ.get("WORLD_SIZE")
    if world_env is not None and int(world_env) != args.gpus:
        raise SystemExit(f"bench.py: WORLD_SIZE={world_env} but --gpus {args.gpus}; launch one rank per GPU")
    if args.impl == "reference":
        run_reference(args)
        return
    if args.gpus > 1 and world_env is None:
        sys.exit(relaunch_under_torchrun(args))
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    ndev = torch.cuda.device_count()
    # more ranks than visible GPUs (a functional check on a 1-GPU box): ranks
    # share devices round-robin and the host collectives go through gloo
    # (NCCL refuses two ranks on one device); timings are then not scaling data
    shared_gpu = world > ndev
    local = local % ndev
    torch.cuda.set_device(local)
    if world > 1:
        if shared_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    red_dev = "cpu" if shared_gpu else "cuda"

    import paper_1804_07250_b200 as ts
    from paper_1804_07250_b200 import _native, rng
    from paper_1804_07250_b200.sweeps import DominoHandle

    _native.set_device(local)
    d, t_max, counts = workload(args.order)
    plan = ts.SweepPlan(d)
    seed = SEED if rank == 0 else rng.derive_seed(SEED, rank, rng.TAG_DERIVE)
    S = args.sweeps_per_step
    stream = torch.cuda.current_stream()

    strips = strips_mode(args, world)
    if strips:
        seed = SEED  # one chain sharded over all GPUs
    if strips:
        from paper_1804_07250_b200.strips import (DeviceStripWalker, DominoStripEngine, StripWalker,
                                                  strip_bounds)

        # memory-sharded: each rank holds only its strip plus halo rows
        bounds = strip_bounds(d.vertex_mask, world, min_rows=args.halo)
        win = (max(0, bounds[rank] - args.halo), min(d.n + 1, bounds[rank + 1] + args.halo))
        h = DominoHandle.window(d, win[0], win[1])
    else:
        h = DominoHandle(d, d.n + 1, 1)
    h.set_collapse(False)  # the headline executes every sweep (run collapsing: the "collapsed" record)
    h.set_stream(stream.cuda_stream)
    h.set_plan(plan)
    if strips:
        h.upload_rows(win[0], t_max[win[0]:win[1]])
    else:
        h.upload(t_max[None])
    if strips:
        row_engine = None
        if args.host_exchange:  # halo rows through torch.distributed (NCCL) from the host
            walker = StripWalker(None, bounds, rank, world, args.halo)
            walker.engine = row_engine = DominoStripEngine(h, walker.window)
        else:  # push/pull kernels over peer memory (CUDA IPC), no host round trip
            walker = DeviceStripWalker(h, bounds, rank, world, args.halo)
            row_engine = DominoStripEngine.__new__(DominoStripEngine)  # row readback helper only
            row_engine.h, row_engine.torch, row_engine._native = h, torch, _native
            nb = ctypes.c_int64()
            _native.check(_native.lib().tsb_domino_row_bytes(h._h, ctypes.byref(nb)))
            row_engine.row_bytes, row_engine.device = nb.value, torch.device("cuda", local)
        strip_vertices = int(d.vertex_mask[walker.lo:walker.hi].sum())

        def run(n, step0):
            walker.walk(seed, n, step0=step0)
    else:
        def run(n, step0):
            h.walk([seed], n, step0=step0)
    clk = ClockSampler(local).__enter__()  # nvidia-smi needs ~0.5 s to start sampling
    time.sleep(1.0)
    step = 0
    for _ in range(args.warmup):
        run(S, step)
        step += S
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    first = step
    for k in range(args.steps):
        flush.zero_()  # evict L2 between timed steps (outside the events)
        ev[k][0].record(stream)
        run(S, step)
        ev[k][1].record(stream)
        step += S
    torch.cuda.synchronize()
    clk.__exit__()
    if world > 1:
        dist.barrier()
    total_ms = sum(a.elapsed_time(b) for a, b in ev)
    att = attempts_for(seed, first, step - first, counts)
    t = torch.tensor([total_ms], dtype=torch.float64, device=red_dev)
    a = torch.tensor([float(att)], dtype=torch.float64, device=red_dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        if not strips:  # replicas: every rank ran its own chain
            dist.all_reduce(a, op=dist.ReduceOp.SUM)
    max_ms = float(t.item())
    value = float(a.item()) / (max_ms / 1e3)

    # roofline of the dominant kernel: domino_multi_kernel, MK sweeps per
    # launch, ~97% of the step (profiles/round1_launches_4096.txt); achieved =
    # algorithmic bytes per launch / average launch interval on the stream
    n_domain = counts[0] + counts[1]
    n_rank = strip_vertices if strips else n_domain
    walk_len = args.halo if strips else S
    per_launch_ms = total_ms / (args.steps * S / MK)
    achieved = MK * n_rank / (per_launch_ms / 1e3) / 1e9  # 1 B/vertex/sweep algorithmic
    peak, peak_src = peaks()

    e2e = None
    if not args.no_e2e and strips:

        rows = walker.hi - walker.lo
        host = torch.empty(rows * row_engine.row_bytes, dtype=torch.uint8, pin_memory=True)
        seeds_h = torch.empty(1, dtype=torch.int64, pin_memory=True)
        seeds_d = torch.empty(1, dtype=torch.int64, device="cuda")
        torch.cuda.synchronize()
        dist.barrier()
        t0 = time.perf_counter()
        for k in range(args.steps):
            seeds_h[0] = k
            seeds_d.copy_(seeds_h, non_blocking=True)  # the step's input (its seed index)
            run(S, step)
            step += S
            host.copy_(row_engine.get_rows(walker.lo, rows), non_blocking=True)  # the step's result
            torch.cuda.synchronize()
        dt = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=red_dev)
        dist.all_reduce(dt, op=dist.ReduceOp.MAX)
        e2e_att = attempts_for(seed, step - args.steps * S, args.steps * S, counts)
        e2e = {"value": e2e_att / float(dt.item()), "unit": UNIT, "h2d_bytes_per_step": 8,
               "d2h_bytes_per_step": int(host.numel()),
               "api": ("StripWalker (host NCCL exchange)" if args.host_exchange else "DeviceStripWalker")
                      + " over DominoHandle; state resident, strip rows read back to pinned host each step",
               "clock": "host wall clock, max over ranks"}
    if not args.no_e2e and not strips:
        # End to end through the drop-in API a reference user calls:
        # random_walk_batch on a (2, V, V) uint8 numpy batch (pageable memory),
        # every step uploading the tilestates, walking S sweeps and returning
        # a new array that is the next step's input (sweeps.py:278-316).  Run
        # collapsing off, like the headline.
        from paper_1804_07250_b200 import sweeps as _sweeps

        side = d.n + 1
        _sweeps.set_default_collapse(False)
        states = np.stack([t_max, t_max])
        ts.random_walk_batch(states, np.array([1, 2], dtype=np.uint64), S, plan)  # warm the handle and graph
        e2e_att = 0
        t0 = time.perf_counter()
        for k in range(args.steps):
            seeds_k = np.array([rng.derive_seed(seed, k, 7), rng.derive_seed(seed, k, 8)], dtype=np.uint64)
            states = ts.random_walk_batch(states, seeds_k, S, plan)
            e2e_att += sum(attempts_for(int(x), 0, S, counts) for x in seeds_k)
        dt = time.perf_counter() - t0
        # the same with the library default (run collapsing on)
        _sweeps.set_default_collapse(None)
        ts.random_walk_batch(states, np.array([3, 4], dtype=np.uint64), S, plan)
        att_c = 0
        t1 = time.perf_counter()
        for k in range(args.steps):
            seeds_k = np.array([rng.derive_seed(seed, k, 9), rng.derive_seed(seed, k, 10)], dtype=np.uint64)
            states = ts.random_walk_batch(states, seeds_k, S, plan)
            att_c += sum(attempts_for(int(x), 0, S, counts) for x in seeds_k)
        dt_c = time.perf_counter() - t1
        e2e_v = torch.tensor([dt], dtype=torch.float64, device=red_dev)
        e2e_a = torch.tensor([float(e2e_att)], dtype=torch.float64, device=red_dev)
        if world > 1:
            dist.all_reduce(e2e_v, op=dist.ReduceOp.MAX)
            dist.all_reduce(e2e_a, op=dist.ReduceOp.SUM)
        e2e = {"value": float(e2e_a.item()) / float(e2e_v.item()), "unit": UNIT,
               "h2d_bytes_per_step": 2 * side * side + 16, "d2h_bytes_per_step": 2 * side * side,
               "api": "paper_1804_07250_b200.random_walk_batch on a (2, V, V) uint8 numpy batch in pageable "
                      "memory (the reference's call, sweeps.py:278-316): upload, S sweeps per chain, new array "
                      "back, every step; run collapsing off; host wall clock",
               "collapsed_library_default": att_c / dt_c}

    warm = collapsed = None
    if not args.no_warm and not strips and args.order == 4096:
        warm = warm_record(args, d, plan, counts, stream, flush, red_dev, world, torch, dist, seed)
    if not args.no_collapsed and not strips:
        collapsed = collapsed_record(args, d, plan, t_max, counts, stream, flush, red_dev, world, torch, dist, seed)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args.order)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": max_ms / args.steps, "higher_is_better": True,
            **({"shared_gpu": f"{world} ranks on {ndev} visible GPU(s): functional run, not scaling data"}
               if shared_gpu else {}),
            "scaling": "strong" if strips else "weak", "vs_baseline": None, "dtype": "u32",
            "data": "synthetic: Aztec diamond from the closed-form T_max, uniform weights",
            "config": bench_config(args, world, strips),
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic("domino_multi_kernel"),
                         "traffic_source": "profiles/traffic.json (ncu --set full capture)",
                         "kernel": "domino_multi_kernel", "sweeps_per_launch": MK,
                         "launch_ms": per_launch_ms,
                         "bytes_per_launch": MK * n_rank, "peak_source": peak_src,
                         "accounting": "1 B per in-domain vertex per sweep (4-bit state read + write)"},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "warm": warm,
            "collapsed": collapsed,
            "clocks": clk.summary(),
            "gpu_launches": args.steps * (S // walk_len) * (launches_per_walk(walk_len)
                                                           + (3 if strips and not args.host_exchange else 0)),  # + push/pull/epoch
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.cuda.synchronize()
        dist.barrier()  # every rank finished pushing into its neighbours' exchange regions
        if strips and not args.host_exchange:
            walker.close()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
