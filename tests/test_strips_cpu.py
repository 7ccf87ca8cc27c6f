"""Multi-rank strip sharding on CPU: the StripWalker halo
protocol over torch.distributed gloo (world_size 2 and 3), with the C oracle
as the per-rank sweep engine, must reproduce the single-process walk bit for
bit.  The GPU engine runs the same protocol over NCCL (bench.py --gpus N)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_1804_07250_b200.lattice import Domain, aztec_extremal_states
from paper_1804_07250_b200.strips import StripWalker, strip_bounds

ORDER, SEED, STEPS = 30, 0x5EED, 257


class OracleWindowEngine:
    """Holds rows [w0, w1) of the grid; walks them with the oracle."""

    def __init__(self, full: np.ndarray, window, p_up: np.ndarray):
        self.w0, self.w1 = window
        self.rows = np.ascontiguousarray(full[self.w0:self.w1]).copy()
        self.p = np.ascontiguousarray(p_up[self.w0:self.w1])
        self.v = full.shape[1]

    def walk(self, seed, step0, n):
        oracle.domino_walk_window(self.rows, self.w0, seed, self.p, n, step0=step0)

    def empty_rows(self, n):
        return torch.empty(n * self.v, dtype=torch.uint8)

    def get_rows(self, r0, n):
        return torch.from_numpy(self.rows[r0 - self.w0:r0 - self.w0 + n].reshape(-1).copy())

    def set_rows(self, r0, n, buf):
        self.rows[r0 - self.w0:r0 - self.w0 + n] = buf.numpy().reshape(n, self.v)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, halo, out_dir):
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    d = Domain.aztec(ORDER)
    t_max, _ = aztec_extremal_states(ORDER)
    p_up = np.full(t_max.shape, 0.5)
    bounds = strip_bounds(d.vertex_mask, world, min_rows=halo)
    walker = StripWalker(None, bounds, rank, world, halo)
    walker.engine = OracleWindowEngine(t_max, walker.window, p_up)
    n_ex = walker.walk(SEED, 100)
    n_ex += walker.walk(SEED, STEPS - 100, step0=100)  # continuation across calls
    eng = walker.engine
    strip = eng.rows[walker.lo - eng.w0:walker.hi - eng.w0]
    np.save(os.path.join(out_dir, f"strip{rank}.npy"), strip)
    np.save(os.path.join(out_dir, f"ex{rank}.npy"), np.array(n_ex))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,halo", [(2, 4), (3, 7), (2, 1)])
def test_strip_walk_matches_single_process(tmp_path, world, halo):
    mp.spawn(_worker, args=(world, _free_port(), halo, str(tmp_path)), nprocs=world, join=True)
    t_max, _ = aztec_extremal_states(ORDER)
    ref = oracle.domino_walk(t_max[None], [SEED], np.full(t_max.shape, 0.5), STEPS)[0]
    got = np.concatenate([np.load(tmp_path / f"strip{r}.npy") for r in range(world)])
    assert got.shape == ref.shape
    assert np.array_equal(got, ref)
    expected_ex = -(-100 // halo) + -(-(STEPS - 100) // halo)
    assert int(np.load(tmp_path / "ex0.npy")) == expected_ex


def test_strip_bounds_balance():
    d = Domain.aztec(64)
    b = strip_bounds(d.vertex_mask, 8, min_rows=8)
    assert b[0] == 0 and b[-1] == d.n + 1 and all(x < y for x, y in zip(b, b[1:]))
    per = [int(d.vertex_mask[b0:b1].sum()) for b0, b1 in zip(b, b[1:])]
    assert max(per) - min(per) <= 2 * (d.n + 1)  # within one row of perfect balance
    with pytest.raises(ValueError):
        strip_bounds(d.vertex_mask, 200, min_rows=8)


def _replica_worker(rank, world, port, out_dir):
    from paper_1804_07250_b200.cftp import distribute_samples

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    seen = []

    def run(mine):
        seen.extend(mine)
        return [np.full(3, k * k, dtype=np.int64) for k in mine]

    out = distribute_samples(7, run)
    np.save(os.path.join(out_dir, f"rep{rank}.npy"), np.stack(out))
    np.save(os.path.join(out_dir, f"mine{rank}.npy"), np.array(seen))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_cftp_replicas_round_robin(tmp_path, world):
    """distribute_samples (the CFTP replica layer of all three models): rank r
    runs samples r, r + world, ...; every rank gets all results in order."""
    mp.spawn(_replica_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    want = np.stack([np.full(3, k * k, dtype=np.int64) for k in range(7)])
    for r in range(world):
        assert np.array_equal(np.load(tmp_path / f"rep{r}.npy"), want)
        assert list(np.load(tmp_path / f"mine{r}.npy")) == list(range(r, 7, world))
