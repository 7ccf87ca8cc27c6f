"""CLI sampling on the device (cli.py:128-200): `sample` and `cftp` write the
same archive bytes as the reference CLI for the same arguments
(tests/golden/cli_*.txt, written by the reference's own `main`), and the
domain / weight errors map to its exit codes (cli.py:356-371)."""

import os

import pytest

from golden_cases import CLI_CASES
from paper_1804_07250_b200.cli import main

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
pytestmark = pytest.mark.gpu
_SAMPLING = [c for c in CLI_CASES if c[1][0] in ("sample", "cftp")]


@pytest.mark.parametrize("name,argv", _SAMPLING, ids=[c[0] for c in _SAMPLING])
def test_sampling_archives_match_reference(name, argv, tmp_path):
    path = tmp_path / "arc.txt"
    assert main(argv + ["--out", str(path)]) == 0
    with open(os.path.join(GOLDEN, f"cli_{name}.txt")) as fh:
        assert path.read_text() == fh.read()


def test_sample_to_stdout_batches(capsys, monkeypatch):
    """Records are identical when the chains walk in several device batches."""
    import paper_1804_07250_b200.cli as cli

    name, argv = next(c for c in CLI_CASES if c[0] == "sample_domino_square")
    monkeypatch.setattr(cli, "_BATCH_BYTES", 3 * 25)  # 3 chains of a 5x5 vertex grid per batch
    assert main(argv) == 0
    with open(os.path.join(GOLDEN, f"cli_{name}.txt")) as fh:
        assert capsys.readouterr().out == fh.read()


def test_untileable_exit_code(tmp_path, capsys):
    path = tmp_path / "odd.txt"
    path.write_text("2\n11\n10\n")
    code = main(["cftp", "--model", "domino", "--domain", str(path), "--samples", "1"])
    assert code == 3 and "tileable" in capsys.readouterr().err
    code = main(["sample", "--model", "domino", "--domain", str(path), "--steps", "5"])
    assert code == 3 and "tileable" in capsys.readouterr().err


def test_non_monotone_exit_code(capsys):
    code = main(["cftp", "--model", "sixvertex", "--dwbc", "3", "--weights", "a=2,b=1,c=1"])
    assert code == 4 and "a <= c" in capsys.readouterr().err


def test_threads_backend_header(capsys):
    assert main(["cftp", "--model", "domino", "--square", "2", "--samples", "2", "--backend", "threads"]) == 0
    assert "# backend: threads" in capsys.readouterr().out
