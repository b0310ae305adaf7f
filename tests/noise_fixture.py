"""Decode tests/golden/golden_noise.npz (made by make_golden.py gen_noise)."""
from conftest import golden

KINDS = {0: "h", 1: "rx", 2: "ry", 3: "cx", 4: "noise"}


def load():
    g = golden("golden_noise.npz")
    glist = []
    for kind, q0, q1, param, dur in g["gates"]:
        k = KINDS[int(kind)]
        if k == "cx":
            glist.append({"kind": k, "qubits": (int(q0), int(q1))})
        elif k == "noise":
            glist.append({"kind": k, "qubits": (int(q0),), "duration": float(dur)})
        elif k == "h":
            glist.append({"kind": k, "qubits": (int(q0),)})
        else:
            glist.append({"kind": k, "qubits": (int(q0),), "param": float(param)})
    return glist, g["states"], float(g["t1"]), float(g["t2"]), int(g["seed"])


def to_circuit(glist, n=12, with_noise=True):
    from paper_2001_10554_b200.circuit import Circuit, GateSpec

    specs = []
    for g in glist:
        if g["kind"] == "noise":
            if with_noise:
                specs.append(GateSpec("noise", g["qubits"], duration=g["duration"]))
        else:
            specs.append(GateSpec(g["kind"], g["qubits"], g.get("param")))
    return Circuit(n, tuple(specs))
