"""Circuit and graph text formats (circuit.py:130-237, graphs.py:53-88) and
the CLI's pre-device usage errors; no GPU needed."""
import os

import pytest

from paper_2001_10554_b200 import cli
from paper_2001_10554_b200.circuit import (CircuitParseError, load_circuit, parse_circuit,
                                            serialize_circuit)
from paper_2001_10554_b200.graphs import load_graph, parse_graph, serialize_graph

from conftest import GOLDEN

CLI_DIR = os.path.join(GOLDEN, "cli")


def test_golden_files_round_trip():
    for name in ("mix.qc", "qaoa6.qc", "layers12.qc"):
        text = open(os.path.join(CLI_DIR, name)).read()
        c = load_circuit(os.path.join(CLI_DIR, name))
        assert serialize_circuit(c) == text
    for name in ("ring.graph", "cubic6.graph"):
        text = open(os.path.join(CLI_DIR, name)).read()
        assert serialize_graph(load_graph(os.path.join(CLI_DIR, name))) == text


def test_circuit_contents():
    c = load_circuit(os.path.join(CLI_DIR, "mix.qc"))
    kinds = [g.kind for g in c.gates]
    assert kinds == ["h"] * 4 + ["noise", "diagcost", "cx", "rz", "noise", "ry", "cz"]
    assert c.gates[4].duration == 1.5 and c.gates[5].param == 0.61
    assert c.gates[5].graph.edges == ((0, 1), (1, 2), (2, 3), (3, 0))
    q = load_circuit(os.path.join(CLI_DIR, "qaoa6.qc"))
    assert q.slots == ("gamma1", "beta1", "gamma2", "beta2")


@pytest.mark.parametrize("text,msg", [
    ("h 0\n", "line 1: gate before qubits header"),
    ("qubits 2\nqubits 2\n", "line 2: repeated qubits header"),
    ("qubits 2\nfoo 1\n", "line 2: unknown mnemonic 'foo'"),
    ("qubits 2\nrx 0\n", "line 2: expected 'rx <q> <angle|$slot>'"),
    ("qubits 2\nrx 0 abc\n", "line 2: bad number 'abc'"),
    ("qubits 2\nrx 0 $\n", "line 2: empty slot name"),
    ("qubits 2\nnoise 0 -1\n", "line 2: negative noise duration"),
    ("qubits 2\ncx 1 1\n", "line 2: cx needs two distinct qubits"),
    ("# only a comment\n", "line 0: missing 'qubits <n>' header"),
    ("qubits 2\nh 5\n", "line 0: h on qubit 5 out of range"),
])
def test_parse_errors(text, msg):
    with pytest.raises(CircuitParseError) as e:
        parse_circuit(text)
    assert str(e.value) == msg


def test_graph_parse_errors():
    for text in ("edge 0 1\n", "vertices 3\nvertices 3\n", "vertices 3\nedge 0\n",
                 "vertices 3\nloop 0 1\n", "vertices 3\nedge 0 0\n", "vertices 3\nedge 0 1\n"
                 "edge 1 0\n", ""):
        with pytest.raises(ValueError):
            parse_graph(text)
    assert parse_graph("vertices 3 # c\n\nedge 0 2\n").edges == ((0, 2),)


def test_cli_usage_errors_exit_2(capsys):
    qc = os.path.join(CLI_DIR, "mix.qc")
    assert cli.main(["run", qc, "--bind", "nope"]) == cli.EXIT_USAGE
    assert cli.main(["run", qc, "--transport", "socket"]) == cli.EXIT_USAGE
    assert cli.main(["bench-gate", "--n", "4", "--repetitions", "0"]) == cli.EXIT_USAGE
    assert cli.main(["noise-ensemble", qc, "--t1", "1", "--t2", "1", "--trajectories", "0"]) \
        == cli.EXIT_USAGE
    assert cli.main(["noise-ensemble", qc, "--t1", "1", "--t2", "1",
                     "--observable", "energy"]) == cli.EXIT_USAGE
    assert cli.main(["noise-ensemble", qc, "--t1", "1", "--t2", "3"]) == cli.EXIT_USAGE
    err = capsys.readouterr().err
    assert "error: --bind expects NAME=VALUE" in err
