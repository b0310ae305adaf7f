"""Record the reference's public call signatures (run in the build container,
the only place /root/reference exists):

    python tests/golden/make_signatures.py

Writes ref_signatures.json: for every public function / class of the
reference modules on the drop-in surface, its parameters (name, kind,
default repr).  tests/test_signatures.py compares the shim against it with
inspect.signature, so the comparison needs no reference at test time.
"""
from __future__ import annotations

import importlib
import inspect
import json
import os
import sys

REF = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "ref_signatures.json")
MODULES = ["statevector", "distribution", "runtime", "pool", "gates", "graphs", "circuit",
           "noise", "optimize"]


def describe(obj):
    try:
        sig = inspect.signature(obj)
    except (TypeError, ValueError):
        return None
    out = []
    for p in sig.parameters.values():
        default = "<required>" if p.default is inspect.Parameter.empty else repr(p.default)
        out.append([p.name, p.kind.name, default])
    return out


def main():
    sys.path.insert(0, REF)
    table = {}
    for name in MODULES:
        mod = importlib.import_module(f"qpool.{name}")
        entries = {}
        for attr, obj in vars(mod).items():
            if attr.startswith("_"):
                continue
            if not (inspect.isfunction(obj) or inspect.isclass(obj)):
                continue
            if getattr(obj, "__module__", None) != mod.__name__:
                continue
            entries[attr] = {"kind": "class" if inspect.isclass(obj) else "function",
                             "params": describe(obj)}
        table[name] = entries
    pkg = importlib.import_module("qpool")
    table["__init__"] = sorted(n for n in getattr(pkg, "__all__", dir(pkg)) if not n.startswith("_"))
    with open(OUT, "w") as fh:
        json.dump(table, fh, indent=1, sort_keys=True)
    print("wrote", OUT, {k: len(v) for k, v in table.items()})


if __name__ == "__main__":
    main()
