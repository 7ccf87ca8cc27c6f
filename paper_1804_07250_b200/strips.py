"""Strip sharding of one large lattice across GPUs.

Rows are split into contiguous strips, one per rank, with equal numbers of
in-domain vertices.  Each rank keeps the whole grid allocated but sweeps only
its strip plus `halo` rows above and below (tsb_domino_set_window).  One sweep
moves information by one row, so after k <= halo sweeps the strip rows are
still exact although the outer halo rows have gone stale; the ranks then
swap their `halo` boundary rows with their neighbours (NCCL point-to-point
over NVLink) and continue.  Coins are pure in (seed, site, step) and the
colour coin is chain-global, so every rank computes them locally and the
sharded walk is bit-identical to the single-GPU walk; no all-reduce is
needed.

The walker is engine-agnostic: `DominoStripEngine` drives the CUDA library;
tests/test_strips_cpu.py drives the same protocol with the C oracle over
the gloo backend.
"""

from __future__ import annotations

import ctypes

import numpy as np


def strip_bounds(vertex_mask: np.ndarray, world: int, min_rows: int = 1) -> list[int]:
    """Row boundaries b_0 = 0 < ... < b_world = rows splitting the in-domain
    vertices as evenly as possible (the Aztec diamond's rows are uneven)."""
    rows = vertex_mask.shape[0]
    if world < 1 or world * min_rows > rows:
        raise ValueError(f"cannot split {rows} rows into {world} strips of >= {min_rows} rows")
    per_row = vertex_mask.sum(axis=1).astype(np.int64)
    cum = np.concatenate([[0], np.cumsum(per_row)])
    total = int(cum[-1])
    b = [0]
    for i in range(1, world):
        target = total * i / world
        r = int(np.searchsorted(cum, target))
        r = max(r, b[-1] + min_rows)
        r = min(r, rows - (world - i) * min_rows)
        b.append(r)
    b.append(rows)
    return b


class StripWalker:
    """Runs a walk on rank `rank` of `world`, exchanging halos every `halo`
    sweeps.  `engine` provides walk(seed, step0, n), get_rows(r0, n),
    set_rows(r0, n, buf) and empty_rows(n)."""

    def __init__(self, engine, bounds: list[int], rank: int, world: int, halo: int, group=None,
                 stage_cpu: bool = False):
        self.engine = engine
        self.rank = rank
        self.world = world
        self.lo, self.hi = bounds[rank], bounds[rank + 1]
        self.rows = bounds[-1]
        if halo < 1:
            raise ValueError("halo must be >= 1")
        if world > 1 and min(b1 - b0 for b0, b1 in zip(bounds, bounds[1:])) < halo:
            raise ValueError("every strip needs at least `halo` rows")
        self.halo = halo
        self.group = group
        self.stage_cpu = stage_cpu  # gloo: move device rows through host memory
        self.window = (max(0, self.lo - halo), min(self.rows, self.hi + halo))

    def exchange(self):
        if self.world == 1:
            return
        import torch.distributed as dist

        k = self.halo
        st = (lambda t: t.cpu()) if self.stage_cpu else (lambda t: t)
        empty = (lambda n: self.engine.empty_rows(n).cpu()) if self.stage_cpu else self.engine.empty_rows
        ops = []
        recv_up = recv_dn = None
        if self.rank > 0:
            ops.append(dist.P2POp(dist.isend, st(self.engine.get_rows(self.lo, k)), self.rank - 1, self.group))
            recv_up = empty(k)
            ops.append(dist.P2POp(dist.irecv, recv_up, self.rank - 1, self.group))
        if self.rank < self.world - 1:
            ops.append(dist.P2POp(dist.isend, st(self.engine.get_rows(self.hi - k, k)), self.rank + 1, self.group))
            recv_dn = empty(k)
            ops.append(dist.P2POp(dist.irecv, recv_dn, self.rank + 1, self.group))
        for w in dist.batch_isend_irecv(ops):
            w.wait()
        dev = (lambda t: t.to(self.engine.device)) if self.stage_cpu else (lambda t: t)
        if recv_up is not None:
            self.engine.set_rows(self.lo - k, k, dev(recv_up))
        if recv_dn is not None:
            self.engine.set_rows(self.hi, k, dev(recv_dn))

    def walk(self, seed: int, n_steps: int, step0: int = 0) -> int:
        """n_steps sweeps; returns the number of halo exchanges."""
        s = 0
        exchanges = 0
        while s < n_steps:
            k = min(self.halo, n_steps - s)
            self.engine.walk(seed, step0 + s, k)
            self.exchange()
            exchanges += 1
            s += k
        return exchanges


class DominoStripEngine:
    """Strip engine over a device DominoHandle (chain 0) with torch rows."""

    def __init__(self, handle, window: tuple[int, int]):
        import torch

        from . import _native

        self.h = handle
        self.torch = torch
        self._native = _native
        L = _native.lib()
        _native.check(L.tsb_domino_set_window(handle._h, int(window[0]), int(window[1])))
        nb = ctypes.c_int64()
        _native.check(L.tsb_domino_row_bytes(handle._h, ctypes.byref(nb)))
        self.row_bytes = nb.value
        self.device = torch.device("cuda", handle.device)

    def walk(self, seed: int, step0: int, n: int):
        self.h.walk([seed], n, step0=step0)

    def empty_rows(self, n: int):
        return self.torch.empty(n * self.row_bytes, dtype=self.torch.uint8, device=self.device)

    def get_rows(self, r0: int, n: int):
        t = self.empty_rows(n)
        self._native.check(self._native.lib().tsb_domino_get_rows(self.h._h, 0, r0, n, ctypes.c_void_p(t.data_ptr())))
        return t

    def set_rows(self, r0: int, n: int, buf):
        self._native.check(self._native.lib().tsb_domino_set_rows(self.h._h, 0, r0, n,
                                                                  ctypes.c_void_p(buf.data_ptr())))


class DeviceStripWalker:
    """Strip walk with the halo exchange in device code (csrc/strips.cu).

    Each rank's `DominoHandle` (chain 0 = the whole lattice) sweeps rows
    [lo, hi) plus `halo` rows per side; every `halo` sweeps the boundary rows
    are pushed into the neighbours' exchange regions over peer memory
    (NVLink / NVSwitch; CUDA IPC between processes) and pulled after a flag
    wait, all in the handle's stream.  `walk` only enqueues work: the host
    never waits on a neighbour.  Bit-identical to the single-GPU walk.

    Across processes the 64-byte IPC handles are exchanged once through
    `torch.distributed` (any backend); `DeviceStripWalker.local(handles, ...)`
    links handles of one process directly (tests on one GPU).
    """

    def __init__(self, handle, bounds: list[int], rank: int, world: int, halo: int, group=None,
                 connect: bool = True):
        from . import _native

        self.handle = handle
        self.rank, self.world = rank, world
        self.lo, self.hi = bounds[rank], bounds[rank + 1]
        self.halo = halo
        if world > 1 and min(b1 - b0 for b0, b1 in zip(bounds, bounds[1:])) < halo:
            raise ValueError("every strip needs at least `halo` rows")
        self.window = (max(0, self.lo - halo), min(bounds[-1], self.hi + halo))
        self._ipc = ctypes.create_string_buffer(64)
        L = _native.lib()
        _native.check(L.tsb_domino_strip_init(handle._h, self.lo, self.hi, halo, self._ipc))
        if connect and world > 1:
            import torch.distributed as dist

            handles = [None] * world
            dist.all_gather_object(handles, bytes(self._ipc.raw), group=group)
            up = ctypes.create_string_buffer(handles[rank - 1], 64) if rank > 0 else None
            dn = ctypes.create_string_buffer(handles[rank + 1], 64) if rank < world - 1 else None
            _native.check(L.tsb_domino_strip_connect(handle._h, up, dn))
            dist.barrier(group=group)  # every region is mapped before the first push

    @staticmethod
    def walk_lockstep(walkers: list["DeviceStripWalker"], seed: int, n_steps: int, step0: int = 0) -> None:
        """Walk handles of ONE process round by round: every rank's sweeps and
        push, then every rank's pull (the flag waits never spin), with a host
        synchronisation between the halves.  For several strips on one GPU."""
        from . import _native

        L = _native.lib()
        for w in walkers:
            _native.check(L.tsb_domino_strip_seed(w.handle._h, _native.u64(seed)))
        done = 0
        while done < n_steps:
            k = min(walkers[0].halo, n_steps - done)
            for w in walkers:
                _native.check(L.tsb_domino_strip_step(w.handle._h, _native.u64(step0 + done), _native.u64(k), 0))
            for w in walkers:
                w.handle.sync()
            for w in walkers:
                _native.check(L.tsb_domino_strip_step(w.handle._h, _native.u64(0), _native.u64(0), 1))
            for w in walkers:
                w.handle.sync()
            done += k

    @classmethod
    def local(cls, handles, bounds: list[int], halo: int) -> list["DeviceStripWalker"]:
        """One walker per handle of this process, linked without IPC."""
        from . import _native

        ws = [cls(h, bounds, r, len(handles), halo, connect=False) for r, h in enumerate(handles)]
        L = _native.lib()
        for r, w in enumerate(ws):
            up = handles[r - 1]._h if r > 0 else None
            dn = handles[r + 1]._h if r < len(handles) - 1 else None
            _native.check(L.tsb_domino_strip_connect_local(w.handle._h, up, dn))
        return ws

    def walk(self, seed: int, n_steps: int, step0: int = 0) -> None:
        from . import _native

        _native.check(_native.lib().tsb_domino_strip_walk(self.handle._h, _native.u64(seed), _native.u64(step0),
                                                          int(n_steps)))

    def status(self) -> int:
        """Wait for the enqueued work; raises if a neighbour flag wait timed out.
        Returns the number of exchanges so far."""
        from . import _native

        e = ctypes.c_uint64()
        _native.check(_native.lib().tsb_domino_strip_status(self.handle._h, ctypes.byref(e), None))
        return e.value

    def close(self) -> None:
        """Release the exchange region (after every rank finished walking)."""
        from . import _native

        _native.check(_native.lib().tsb_domino_strip_close(self.handle._h))
