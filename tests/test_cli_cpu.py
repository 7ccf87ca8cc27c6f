"""CLI archive commands on the host (cli.py:230-255, 356-371): `density` and
`hist` over the reference-written archives reproduce the reference CLI's
output bytes, and argument errors map to the reference's exit codes."""

import os

import pytest

from golden_cases import CLI_CASES
from paper_1804_07250_b200.cli import main

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def run(capsys, argv):
    code = main(argv)
    out = capsys.readouterr()
    return code, out.out, out.err


@pytest.mark.parametrize("name,argv", [c for c in CLI_CASES if c[1][0] in ("density", "hist")],
                         ids=[c[0] for c in CLI_CASES if c[1][0] in ("density", "hist")])
def test_archive_commands_match_reference(name, argv, capsys):
    code, out, _ = run(capsys, [a.replace("{g}", GOLDEN) for a in argv])
    assert code == 0
    with open(os.path.join(GOLDEN, f"cli_{name}.txt")) as fh:
        assert out == fh.read()


def test_archive_commands_write_out_file(tmp_path, capsys):
    name, argv = next(c for c in CLI_CASES if c[0] == "density_domino")
    path = tmp_path / "d.txt"
    assert main([a.replace("{g}", GOLDEN) for a in argv] + ["--out", str(path)]) == 0
    with open(os.path.join(GOLDEN, f"cli_{name}.txt")) as fh:
        assert path.read_text() == fh.read()


def test_sample_requires_steps(capsys):
    code, _, err = run(capsys, ["sample", "--model", "domino", "--square", "2"])
    assert code == 2 and "steps" in err


def test_invalid_input_exit_codes(capsys):
    assert run(capsys, ["cftp", "--model", "lozenge", "--hexagon", "nope"])[0] == 2
    assert run(capsys, ["sample", "--model", "domino", "--steps", "3"])[0] == 2  # no domain
    assert run(capsys, ["density", "--aztec", "2"])[0] == 2  # no --in
    code, _, err = run(capsys, ["sample", "--aztec", "2", "--steps", "3", "--weights", "q"])
    assert code == 2 and "bad weight" in err
