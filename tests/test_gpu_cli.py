"""The CLI's reports are the reference CLI's, character for character
(SURVEY 8f row 4): `run` reports (probabilities, amplitudes, maxcut) under
several rank/state layouts, noise-ensemble CSVs, and bench-gate's
message/byte columns (tests/golden/cli, made by make_golden.py gen_cli)."""
import contextlib
import io
import json
import os

import pytest

from paper_2001_10554_b200 import cli

from conftest import GOLDEN

pytestmark = pytest.mark.gpu
CLI_DIR = os.path.join(GOLDEN, "cli")
CASES = json.load(open(os.path.join(CLI_DIR, "cases.json")))


def run_cli(argv):
    buf = io.StringIO()
    cwd = os.getcwd()
    os.chdir(CLI_DIR)
    try:
        with contextlib.redirect_stdout(buf):
            rc = cli.main(argv)
    finally:
        os.chdir(cwd)
    return rc, buf.getvalue()


@pytest.mark.parametrize("name", sorted(k for k in CASES if k != "bench_gate"))
def test_report_matches_reference(name):
    rc, text = run_cli(CASES[name])
    assert rc == 0
    assert text == open(os.path.join(CLI_DIR, name + ".txt")).read()


def test_bench_gate_columns_match_reference():
    rc, text = run_cli(CASES["bench_gate"])
    assert rc == 0
    rows = [r.split(",") for r in text.splitlines()]
    assert rows[0] == ["qubit", "mean_seconds", "messages", "bytes", "ranks", "n", "min_seconds"]
    got = "\n".join(",".join(r[i] for i in (0, 2, 3, 4, 5)) for r in rows) + "\n"
    assert got == open(os.path.join(CLI_DIR, "bench_gate.txt")).read()
    for r in rows[1:]:
        assert 0 < float(r[6]) <= float(r[1])


def test_unbound_slot_is_a_usage_error(capsys):
    rc, _ = run_cli(["run", "qaoa6.qc"])
    assert rc == cli.EXIT_USAGE
    assert "unbound" in capsys.readouterr().err
