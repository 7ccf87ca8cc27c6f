"""Command-line sampling on the device.

Mirrors the reference CLI's sampling and archive commands
(/root/reference/pkg/src/tilesampler/cli.py):
  cli.py:53-67     common flags (--model --domain --aztec --square --hexagon
                   --dwbc --weights --seed --samples --steps --backend
                   --threads --out --format)
  cli.py:128-167   _sample_states: CFTP (cftp_sample_many / loz_cftp /
                   sv_cftp) or `--steps` MCMC sweeps from the minimal state,
                   chain k seeded derive_seed(seed, k, TAG_DERIVE)
  cli.py:170-200   `sample` / `cftp`: a SampleArchive with sampler
                   "mcmc steps=S" / "cftp"
  cli.py:230-255   `density` / `hist` over an archive
  cli.py:356-371   exit codes: 2 invalid input, 3 untileable or infeasible,
                   4 non-monotone six-vertex weights, 5 CFTP cap

The archive bytes equal the reference's for the same arguments.  MCMC
chains walk on the device in batches and every record is formatted on the
device (archive.device_record); `--backend` / `--threads` are accepted and
recorded in the header as the reference does, the sweeps always run on the
GPU.  The reference's enumeration / exact-distribution / rendering commands
are outside the hot path and are not provided.
"""

from __future__ import annotations

import argparse
import sys

import numpy as np

from . import rng
from .archive import SampleArchive, device_record
from .errors import (
    ConvergenceCapExceeded,
    InfeasibleBoundary,
    NonMonotoneWeights,
    TileSamplerError,
    UntileableDomain,
)

# device memory per MCMC batch of chains (uint8 staging of the reference layout)
_BATCH_BYTES = 1 << 30


def _add_common(p: argparse.ArgumentParser):
    p.add_argument("--model", choices=("domino", "lozenge", "sixvertex"), default="domino")
    p.add_argument("--domain", help="domain file (domino: 0/1 grid, lozenge: triangle grids)")
    p.add_argument("--aztec", type=int, help="Aztec diamond order")
    p.add_argument("--square", type=int, help="square side (faces)")
    p.add_argument("--hexagon", help="lozenge hexagon sides A,B,C")
    p.add_argument("--dwbc", type=int, help="six-vertex domain-wall size")
    p.add_argument("--weights", default="", help="e.g. q=20 or a=1,b=1,c=2")
    p.add_argument("--seed", default="1", help="decimal or 0x-hex master seed")
    p.add_argument("--samples", type=int, default=1)
    p.add_argument("--steps", type=int, help="sweeps per MCMC sample (required for `sample`)")
    p.add_argument("--backend", choices=("seq", "threads"), default="seq")
    p.add_argument("--threads", type=int, default=None)
    p.add_argument("--out", help="output path (default stdout)")
    p.add_argument("--format", choices=("txt", "csv", "svg"), default="txt")


def _parse_seed(text: str) -> int:
    return int(text, 0)


def _parse_weights(model: str, text: str):
    from .lattice import Uniform, VolumeWeights
    from .sixvertex import SVWeights

    fields = {}
    if text:
        for part in text.split(","):
            key, _, val = part.partition("=")
            if not val:
                raise ValueError(f"bad weight entry {part!r}")
            fields[key.strip()] = float(val)
    if model == "sixvertex":
        return SVWeights(fields.get("a", 1.0), fields.get("b", 1.0), fields.get("c", 1.0))
    if "q" in fields:
        return VolumeWeights(fields["q"])
    return Uniform()


def _build_domain(args):
    from .lattice import Domain
    from .lozenge import TriDomain
    from .sixvertex import dwbc

    model = args.model
    if model == "domino":
        if args.aztec:
            return Domain.aztec(args.aztec)
        if args.square:
            return Domain.square(args.square)
        if args.domain:
            with open(args.domain) as fh:
                return Domain.from_text(fh.read())
        raise ValueError("domino model needs --aztec, --square, or --domain")
    if model == "lozenge":
        if args.hexagon:
            a, b, c = (int(x) for x in args.hexagon.split(","))
            return TriDomain.hexagon(a, b, c)
        if args.domain:
            with open(args.domain) as fh:
                return TriDomain.from_text(fh.read())
        raise ValueError("lozenge model needs --hexagon or --domain")
    if args.dwbc:
        return dwbc(args.dwbc)
    raise ValueError("sixvertex model needs --dwbc")


class _Output:
    """--out file or stdout."""

    def __init__(self, path):
        self.path = path
        self.fh = open(path, "w") if path else sys.stdout

    def write(self, text: str):
        self.fh.write(text)

    def close(self):
        if self.path:
            self.fh.close()


def _header(args, domain, sampler: str, count: int) -> dict:
    header = SampleArchive.create(args.model, domain, args.weights or "uniform", _parse_seed(args.seed),
                                  args.backend, sampler).header
    header["samples"] = str(count)
    return header


def _write_header(out: _Output, header: dict):
    for k, v in header.items():
        out.write(f"# {k}: {v}\n")


def _mcmc_setup(args, domain, weights):
    """The model's minimal state and a factory of device handles of n chains
    holding it (cli.py:145-167)."""
    model = args.model
    if model == "domino":
        from .lattice import extremal_tilings
        from .sweeps import SweepPlan, _handle_for

        ext = extremal_tilings(domain)
        if ext is None:
            raise UntileableDomain("domain is not tileable")
        plan = SweepPlan(domain, weights)
        start = ext[1].states

        def make(n):
            h = _handle_for(domain, n)
            h.set_plan(plan)
            return h
    elif model == "lozenge":
        from .lozenge import _loz_handle, _p_up_cached, loz_extremal

        ext = loz_extremal(domain)
        if ext is None:
            raise UntileableDomain("triangle domain is not tileable")
        start = ext[1].edges.astype(np.uint8)

        def make(n):
            h = _loz_handle(domain, n)
            h.set_p_up(_p_up_cached(domain, weights))
            return h
    else:
        from .sixvertex import SVWeights, _sv_handle, sv_extremal

        if not isinstance(weights, SVWeights):
            raise ValueError("sixvertex model needs a=,b=,c= weights")
        start = sv_extremal(domain.n, domain)[1].heights

        def make(n):
            h = _sv_handle(domain.n, n)
            h.set_weights(weights)
            return h
    return np.asarray(start), make


def _state_bytes(args, domain) -> int:
    if args.model == "domino":
        return (domain.n + 1) ** 2
    if args.model == "lozenge":
        sx, sy = domain.size
        return 3 * (sx + 1) * (sy + 1)
    return 4 * (domain.n + 1) ** 2


def _cmd_sample(args) -> int:
    domain = _build_domain(args)
    weights = _parse_weights(args.model, args.weights)
    if args.steps is None:
        raise ValueError("MCMC sampling requires an explicit --steps")
    if args.steps < 0:
        raise ValueError("steps must be non-negative")
    seed = _parse_seed(args.seed)
    count = args.samples
    seeds = np.array([rng.derive_seed(seed, k, rng.TAG_DERIVE) for k in range(count)], dtype=np.uint64)
    batch = max(1, min(count, _BATCH_BYTES // max(1, _state_bytes(args, domain))))
    header = _header(args, domain, f"mcmc steps={args.steps}", count)
    start, make = _mcmc_setup(args, domain, weights)  # errors surface before any output
    out = _Output(args.out)
    try:
        _write_header(out, header)
        for c0 in range(0, count, batch):
            n = min(batch, count - c0)
            h = make(n)
            h.upload(np.repeat(start[None], n, axis=0))
            if args.steps > 0:
                h.walk(seeds[c0:c0 + n], args.steps)
            for c in range(n):
                out.write(device_record(h, c) + "\n")
    finally:
        out.close()
    return 0


def _cftp_states(args, domain, weights):
    from .cftp import cftp_sample_many
    from .lozenge import loz_cftp
    from .sixvertex import sv_cftp
    from .sweeps import SweepPlan

    seed = _parse_seed(args.seed)
    count = args.samples
    if args.model == "domino":
        return cftp_sample_many(domain, SweepPlan(domain, weights), seed, count)
    if args.model == "lozenge":
        res = loz_cftp(domain, weights, seed, count=count)
        return res if isinstance(res, list) else [res]
    res = sv_cftp(domain.n, domain, weights, seed, count=count)
    return res if isinstance(res, list) else [res]


def _cmd_cftp(args) -> int:
    domain = _build_domain(args)
    weights = _parse_weights(args.model, args.weights)
    states = _cftp_states(args, domain, weights)
    out = _Output(args.out)
    try:
        _write_header(out, _header(args, domain, "cftp", len(states)))
        from .archive import serialize_state

        for s in states:
            out.write(serialize_state(s) + "\n")
    finally:
        out.close()
    return 0


def _load_archive(args, domain):
    if not getattr(args, "infile", None):
        raise ValueError("this command needs --in ARCHIVE")
    with open(args.infile) as fh:
        return SampleArchive.load(fh, domain)


def _cmd_density(args) -> int:
    from .stats import density_map

    domain = _build_domain(args)
    dm = density_map(_load_archive(args, domain), args.observable)
    out = _Output(args.out)
    try:
        if args.format == "csv":
            out.write(dm.to_csv())
        else:
            out.write("\n".join(" ".join(f"{x:.4f}" for x in row) for row in dm.grid) + "\n")
    finally:
        out.close()
    return 0


def _cmd_hist(args) -> int:
    from .stats import scalar_observable

    domain = _build_domain(args)
    h = scalar_observable(_load_archive(args, domain), args.observable, bins=args.bins)
    out = _Output(args.out)
    try:
        out.write(h.to_csv())
    finally:
        out.close()
    return 0


def build_parser() -> argparse.ArgumentParser:
    parser = argparse.ArgumentParser(
        prog="tilesampler",
        description="Exact and MCMC sampling of dominoes, lozenges, and six-vertex states on a B200",
    )
    sub = parser.add_subparsers(dest="command", required=True)
    for name, fn in (("sample", _cmd_sample), ("cftp", _cmd_cftp), ("density", _cmd_density),
                     ("hist", _cmd_hist)):
        p = sub.add_parser(name)
        _add_common(p)
        p.set_defaults(fn=fn)
        if name in ("density", "hist"):
            p.add_argument("--in", dest="infile", help="input archive")
        if name == "density":
            p.add_argument("--observable", default="h-edge",
                           choices=("h-edge", "v-edge", "c-vertex", "domino-orientation"))
        if name == "hist":
            p.add_argument("--observable", default="c-vertex-count", choices=("c-vertex-count", "y-intercept"))
            p.add_argument("--bins", type=int, default=None)
    return parser


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    try:
        return args.fn(args)
    except (UntileableDomain, InfeasibleBoundary) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 3
    except NonMonotoneWeights as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 4
    except ConvergenceCapExceeded as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 5
    except (TileSamplerError, ValueError, OSError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())
