"""Strip sharding with the CUDA engine: 2 processes share cuda:0 over gloo
(host-staged rows; on a multi-GPU box the same walker runs over NCCL) and
must reproduce the single-GPU walk bit for bit."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu
ORDER, SEED, STEPS, HALO = 700, 0x5EED, 300, 24


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_dir):
    import paper_1804_07250_b200 as ts
    from paper_1804_07250_b200.lattice import aztec_extremal_states
    from paper_1804_07250_b200.strips import DominoStripEngine, StripWalker, strip_bounds
    from paper_1804_07250_b200.sweeps import DominoHandle

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    d = ts.Domain.aztec(ORDER)
    t_max, _ = aztec_extremal_states(ORDER)
    h = DominoHandle(d, d.n + 1, 1, device=0)
    h.set_stream(torch.cuda.current_stream().cuda_stream)
    h.set_p_up(ts.SweepPlan(d).p_up)
    h.upload(t_max[None])
    bounds = strip_bounds(d.vertex_mask, world, min_rows=HALO)
    w = StripWalker(None, bounds, rank, world, HALO, stage_cpu=True)
    w.engine = DominoStripEngine(h, w.window)
    w.walk(SEED, STEPS)
    np.save(os.path.join(out_dir, f"strip{rank}.npy"), h.download()[0][w.lo:w.hi])
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_strips_two_processes_one_gpu(tmp_path, world):
    import paper_1804_07250_b200 as ts
    from paper_1804_07250_b200.lattice import aztec_extremal_states

    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    d = ts.Domain.aztec(ORDER)
    t_max, _ = aztec_extremal_states(ORDER)
    ref = ts.random_walk_batch(t_max[None], [SEED], STEPS, ts.SweepPlan(d))[0]
    got = np.concatenate([np.load(tmp_path / f"strip{r}.npy") for r in range(world)])
    assert np.array_equal(got, ref)


@pytest.mark.parametrize("world,halo,steps", [(2, 32, 300), (3, 24, 250), (4, 16, 97)])
def test_device_strips_local(world, halo, steps):
    """Device-driven halo exchange (csrc/strips.cu: walk + peer push, flag wait
    + pull) between handles of one process on one GPU, in host lockstep:
    bit-identical to one walk."""
    import paper_1804_07250_b200 as ts
    from paper_1804_07250_b200.lattice import aztec_extremal_states
    from paper_1804_07250_b200.strips import DeviceStripWalker, strip_bounds
    from paper_1804_07250_b200.sweeps import DominoHandle

    order = 300
    d = ts.Domain.aztec(order)
    plan = ts.SweepPlan(d)
    t_max, _ = aztec_extremal_states(order)
    hs = []
    for _ in range(world):
        h = DominoHandle(d, d.n + 1, 1, device=0)
        h.set_p_up(plan.p_up)
        h.upload(t_max[None])
        hs.append(h)
    bounds = strip_bounds(d.vertex_mask, world, min_rows=halo)
    ws = DeviceStripWalker.local(hs, bounds, halo)
    DeviceStripWalker.walk_lockstep(ws, SEED, steps, step0=5)
    for w in ws:
        assert w.status() == -(-steps // halo)
    got = np.concatenate([w.handle.download()[0][w.lo:w.hi] for w in ws])
    for w in ws:
        w.close()
    ref = oracle_walk(t_max, plan.p_up, steps, 5)
    assert np.array_equal(got, ref)


def oracle_walk(start, p_up, steps, step0):
    import oracle

    return oracle.domino_walk(start[None].copy(), [SEED], p_up, steps, step0=step0)[0]


def _ipc_worker(rank, world, port, out_dir, halo, steps):
    import paper_1804_07250_b200 as ts
    from paper_1804_07250_b200.lattice import aztec_extremal_states
    from paper_1804_07250_b200.strips import DeviceStripWalker, strip_bounds
    from paper_1804_07250_b200.sweeps import DominoHandle

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    d = ts.Domain.aztec(ORDER)
    t_max, _ = aztec_extremal_states(ORDER)
    h = DominoHandle(d, d.n + 1, 1, device=0)
    h.set_p_up(ts.SweepPlan(d).p_up)
    h.upload(t_max[None])
    w = DeviceStripWalker(h, strip_bounds(d.vertex_mask, world, min_rows=halo), rank, world, halo)
    w.walk(SEED, steps)
    assert w.status() == -(-steps // halo)
    np.save(os.path.join(out_dir, f"dstrip{rank}.npy"), h.download()[0][w.lo:w.hi])
    dist.barrier()
    w.close()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,halo", [(2, 64), (3, 32), (2, 16)])
def test_device_strips_ipc_processes(tmp_path, world, halo):
    """The same exchange across processes through CUDA IPC handles (here all
    processes share cuda:0; on the 8-GPU box each has its own GPU).  halo 64
    (= kGraphSweeps) runs the rounds as graph replays with the exchange
    captured as their tail, halo 32 / 16 as explicit per-round launches."""
    import paper_1804_07250_b200 as ts
    from paper_1804_07250_b200.lattice import aztec_extremal_states

    steps = 200
    mp.spawn(_ipc_worker, args=(world, _free_port(), str(tmp_path), halo, steps), nprocs=world, join=True)
    d = ts.Domain.aztec(ORDER)
    t_max, _ = aztec_extremal_states(ORDER)
    ref = oracle_walk(t_max, ts.SweepPlan(d).p_up, steps, 0)
    got = np.concatenate([np.load(tmp_path / f"dstrip{r}.npy") for r in range(world)])
    assert np.array_equal(got, ref)


def _cftp_worker(rank, world, port, out_dir):
    import paper_1804_07250_b200 as ts
    from paper_1804_07250_b200.cftp import cftp_sample_many_distributed

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    d = ts.Domain.aztec(10)
    res = cftp_sample_many_distributed(d, ts.SweepPlan(d), 0xC0FFEE, 7)
    if rank == 0:
        np.save(os.path.join(out_dir, "cftp.npy"), np.stack([t.states for t in res]))
    dist.barrier()
    dist.destroy_process_group()


def test_cftp_samples_spread_over_processes(tmp_path):
    """CFTP samples distributed round-robin over ranks equal the one-GPU run."""
    import paper_1804_07250_b200 as ts

    mp.spawn(_cftp_worker, args=(3, _free_port(), str(tmp_path)), nprocs=3, join=True)
    d = ts.Domain.aztec(10)
    ref = np.stack([t.states for t in ts.cftp_sample_many(d, ts.SweepPlan(d), 0xC0FFEE, 7)])
    assert np.array_equal(np.load(tmp_path / "cftp.npy"), ref)


def _cftp_models_worker(rank, world, port, out_dir):
    import paper_1804_07250_b200 as ts

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    loz = ts.loz_cftp_distributed(ts.TriDomain.hexagon(3, 2, 4), ts.VolumeWeights(0.8), 77, 5)
    sv = ts.sv_cftp_distributed(6, ts.dwbc(6), ts.SVWeights(1.0, 1.0, 1.5), 2024, 5)
    if rank == 0:
        np.save(os.path.join(out_dir, "loz.npy"), np.stack([t.edges for t in loz]))
        np.save(os.path.join(out_dir, "sv.npy"), np.stack([np.concatenate([c.h_edges.ravel(), c.v_edges.ravel()])
                                                           for c in sv]))
    dist.barrier()
    dist.destroy_process_group()


def test_lozenge_and_sixvertex_cftp_spread_over_processes(tmp_path):
    """loz_cftp / sv_cftp samples spread round-robin over 2 ranks equal the
    one-GPU runs (replicas: coupled pairs never leave their GPU)."""
    import paper_1804_07250_b200 as ts

    mp.spawn(_cftp_models_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    loz = ts.loz_cftp(ts.TriDomain.hexagon(3, 2, 4), ts.VolumeWeights(0.8), 77, count=5)
    sv = ts.sv_cftp(6, ts.dwbc(6), ts.SVWeights(1.0, 1.0, 1.5), 2024, count=5)
    assert np.array_equal(np.load(tmp_path / "loz.npy"), np.stack([t.edges for t in loz]))
    assert np.array_equal(np.load(tmp_path / "sv.npy"),
                          np.stack([np.concatenate([c.h_edges.ravel(), c.v_edges.ravel()]) for c in sv]))


def _window_walkers(d, plan, t_max, world, halo):
    from paper_1804_07250_b200.strips import DeviceStripWalker, strip_bounds
    from paper_1804_07250_b200.sweeps import DominoHandle

    bounds = strip_bounds(d.vertex_mask, world, min_rows=halo)
    hs = []
    for r in range(world):
        a, b = max(0, bounds[r] - halo), min(d.n + 1, bounds[r + 1] + halo)
        h = DominoHandle.window(d, a, b, device=0)
        h.set_plan(plan)
        h.upload_rows(a, t_max[a:b])
        hs.append(h)
    return hs, DeviceStripWalker.local(hs, bounds, halo)


@pytest.mark.parametrize("world,halo,steps", [(2, 32, 300), (3, 24, 250), (4, 16, 97)])
def test_device_strips_row_windows(world, halo, steps):
    """Memory-sharded strips: every rank's handle holds only its window
    (tsb_domino_create_window); the concatenated strips equal one walk."""
    import paper_1804_07250_b200 as ts
    from paper_1804_07250_b200.lattice import aztec_extremal_states

    order = 300
    d = ts.Domain.aztec(order)
    plan = ts.SweepPlan(d)
    t_max, _ = aztec_extremal_states(order)
    hs, ws = _window_walkers(d, plan, t_max, world, halo)
    from paper_1804_07250_b200.strips import DeviceStripWalker

    DeviceStripWalker.walk_lockstep(ws, SEED, steps, step0=5)
    got = np.concatenate([w.handle.download_rows(w.lo, w.hi - w.lo) for w in ws])
    for w in ws:
        w.close()
    assert np.array_equal(got, oracle_walk(t_max, plan.p_up, steps, 5))


def test_row_window_handle_api():
    """Row windows: whole-grid operations raise, rows round-trip, and a
    window walked alone equals the full walk on rows far from its edges."""
    import paper_1804_07250_b200 as ts
    from paper_1804_07250_b200.lattice import aztec_extremal_states
    from paper_1804_07250_b200.sweeps import DominoHandle

    order = 200
    d = ts.Domain.aztec(order)
    plan = ts.SweepPlan(d)
    t_max, _ = aztec_extremal_states(order)
    a, b = 100, 260
    h = DominoHandle.window(d, a, b, device=0)
    h.set_plan(plan)
    h.upload_rows(a, t_max[a:b])
    # the window's first row has no row above it: its "up" bits read back as 0
    assert np.array_equal(h.download_rows(a + 1, b - a - 1), t_max[a + 1:b])
    with pytest.raises(ValueError):
        h.download()
    with pytest.raises(ValueError):
        h.upload(t_max[None])
    with pytest.raises(ValueError):
        h.heights(0, d.reference_vertex)
    with pytest.raises(ValueError):
        h.upload_rows(a - 40, t_max[a - 40:a])  # outside the window
    steps = 20
    h.walk([SEED], steps)
    ref = oracle_walk(t_max, plan.p_up, steps, 0)
    # rows at least `steps` away from the window edges are exact
    assert np.array_equal(h.download_rows(a + steps, b - a - 2 * steps), ref[a + steps:b - steps])
    full = DominoHandle(d, d.n + 1, 1, device=0)
    full.upload(t_max[None])
    assert np.array_equal(full.download_rows(7, 50), t_max[7:57])
