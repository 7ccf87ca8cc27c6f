"""Sample archives: the reference's line-delimited
text format, with records formatted on the device from live chains.

Reference (relative to /root/reference/pkg/src/tilesampler/):
  stats.py:75-143   SampleArchive(model, header, records): create / append /
                    extend / dump / load; header lines "# key: value" in the
                    order model, domain_hash, weights, seed, backend, sampler,
                    samples, then one record per line
  stats.py:146-153  _serialize_state: domino tilestates in decimal joined by
                    spaces; six-vertex h_edges then v_edges, lozenge edges,
                    as '0'/'1'
  stats.py:156-168  _parse_state

`device_record(handle, chain)` returns the record of a device-resident chain
(libtsb tsb_*_serialize: the text is produced by a CUDA kernel from the bit
planes, the host only receives it), so `ArchiveWriter` streams thousands of
samples to disk without materialising host states.  The output is
byte-identical to the reference's `SampleArchive.dump` of the same states
(tests/test_archive_gpu.py against tests/golden/archive_*.txt).
"""

from __future__ import annotations

import ctypes
import hashlib
import os
import tempfile
from dataclasses import dataclass, field

import numpy as np

from . import _native
from .errors import InconsistencyError


def _domain_hash(text: str) -> str:
    return hashlib.sha256(text.encode()).hexdigest()[:16]


def serialize_state(state) -> str:
    """Host-side record of a state object (stats.py:146-153)."""
    from .lattice import Tiling
    from .lozenge import LozengeTiling
    from .sixvertex import SixVertexConfig

    if isinstance(state, Tiling):
        return " ".join(str(int(x)) for x in state.states.ravel())
    if isinstance(state, SixVertexConfig):
        bits = np.concatenate([state.h_edges.ravel(), state.v_edges.ravel()])
        return "".join("1" if b else "0" for b in bits)
    if isinstance(state, LozengeTiling):
        return "".join("1" if b else "0" for b in state.edges.ravel())
    raise TypeError(f"unknown state type {type(state)!r}")


def parse_state(model: str, domain, line: str):
    """stats.py:156-168."""
    from .lattice import Tiling
    from .lozenge import LozengeTiling
    from .sixvertex import Boundary, SixVertexConfig

    if model == "domino":
        v = domain.n + 1
        grid = np.array(line.split(), dtype=np.uint8).reshape(v, v)
        return Tiling(domain, grid)
    if model == "sixvertex":
        n = domain.n if isinstance(domain, Boundary) else domain
        bits = np.frombuffer(line.encode(), dtype=np.uint8) == ord("1")
        nh = n * (n + 1)
        return SixVertexConfig(n, bits[:nh].reshape(n, n + 1), bits[nh:].reshape(n + 1, n))
    if model == "lozenge":
        sx, sy = domain.size
        bits = np.frombuffer(line.encode(), dtype=np.uint8) == ord("1")
        return LozengeTiling(domain, bits.reshape(3, sx + 1, sy + 1))
    raise InconsistencyError(f"unknown archive model {model!r}")


def device_record(handle, chain: int = 0) -> str:
    """The archive record of chain `chain` of a DominoHandle, SixVertexHandle
    or LozengeHandle, formatted on the device."""
    from .lozenge import LozengeHandle
    from .sixvertex import SixVertexHandle
    from .sweeps import DominoHandle

    L = _native.lib()
    fn = {DominoHandle: L.tsb_domino_serialize, SixVertexHandle: L.tsb_sv_serialize,
          LozengeHandle: L.tsb_loz_serialize}.get(type(handle))
    if fn is None:
        raise TypeError(f"no device records for {type(handle)!r}")
    n = ctypes.c_size_t()
    _native.check(fn(handle._h, chain, None, 0, ctypes.byref(n)))
    buf = ctypes.create_string_buffer(n.value)
    _native.check(fn(handle._h, chain, buf, n.value, ctypes.byref(n)))
    return buf.raw[:n.value].decode("ascii")


@dataclass
class SampleArchive:
    """Header metadata plus serialized states, one record per line (stats.py:75-143)."""

    model: str
    header: dict = field(default_factory=dict)
    records: list = field(default_factory=list)

    @classmethod
    def create(cls, model: str, domain, weights_text: str, seed: int, backend: str, sampler: str) -> "SampleArchive":
        header = {"model": model, "domain_hash": _domain_hash(domain.to_text()), "weights": weights_text,
                  "seed": hex(seed), "backend": backend, "sampler": sampler, "samples": "0"}
        arc = cls(model, header)
        arc._domain = domain
        return arc

    def append(self, state) -> None:
        self.records.append(state)
        self.header["samples"] = str(len(self.records))

    def extend(self, states) -> None:
        for s in states:
            self.append(s)

    def __len__(self):
        return len(self.records)

    def dump(self, fh) -> None:
        for k, v in self.header.items():
            fh.write(f"# {k}: {v}\n")
        for state in self.records:
            fh.write((state if isinstance(state, str) else serialize_state(state)) + "\n")

    @classmethod
    def load(cls, fh, domain) -> "SampleArchive":
        header, records = {}, []
        for line in fh:
            line = line.rstrip("\n")
            if not line.strip():
                continue
            if line.startswith("#"):
                k, _, v = line[1:].partition(":")
                header[k.strip()] = v.strip()
                continue
            records.append(parse_state(header.get("model", ""), domain, line))
        arc = cls(header.get("model", ""), header, records)
        arc._domain = domain
        return arc


class ArchiveWriter:
    """Streams device-resident chains into a SampleArchive text file.

    Records are spooled to a temporary file as they are added (one device
    formatting pass per record); `close()` writes the header with the final
    sample count followed by the records, byte-identical to
    `SampleArchive.dump` of the same states.
    """

    def __init__(self, path: str, model: str, domain, weights_text: str, seed: int, backend: str, sampler: str):
        self.path = path
        self.header = SampleArchive.create(model, domain, weights_text, seed, backend, sampler).header
        self.count = 0
        fd, self._spool_path = tempfile.mkstemp(prefix="tsb_archive_", dir=os.path.dirname(os.path.abspath(path)))
        self._spool = os.fdopen(fd, "w")

    def add(self, handle, chains=None) -> None:
        for c in range(handle.nchains) if chains is None else chains:
            self._spool.write(device_record(handle, c) + "\n")
            self.count += 1

    def close(self) -> None:
        self._spool.close()
        self.header["samples"] = str(self.count)
        with open(self.path, "w") as out, open(self._spool_path) as spool:
            for k, v in self.header.items():
                out.write(f"# {k}: {v}\n")
            while True:
                chunk = spool.read(1 << 24)
                if not chunk:
                    break
                out.write(chunk)
        os.unlink(self._spool_path)

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()
