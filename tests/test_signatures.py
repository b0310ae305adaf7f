"""The drop-in boundary: every public function and class of the reference's
modules exists in the shim with the reference's positional signature
(parameter names, order, kinds and defaults, reference
pkg/src/qpool/*.py).  Shim-only parameters are allowed only after the
reference's ones and must have defaults, so a reference caller's positional
and keyword arguments mean the same thing here.  The reference side was
recorded by tests/golden/make_signatures.py (ref_signatures.json)."""
import importlib
import inspect
import json
import os

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
with open(os.path.join(HERE, "golden", "ref_signatures.json")) as fh:
    REF = json.load(fh)

# dataclass fields the shim adds after the reference's (all defaulted) are
# fine; these reference classes have constructor parameters that are pure
# host plumbing and are compared too.
CASES = [(mod, name) for mod in REF if mod != "__init__" for name in sorted(REF[mod])]


def shim_params(obj):
    sig = inspect.signature(obj)
    return [(p.name, p.kind.name,
             "<required>" if p.default is inspect.Parameter.empty else repr(p.default))
            for p in sig.parameters.values()]


@pytest.mark.parametrize("mod,name", CASES)
def test_signature_matches_reference(mod, name):
    entry = REF[mod][name]
    m = importlib.import_module(f"paper_2001_10554_b200.{mod}")
    assert hasattr(m, name), f"{mod}.{name} missing from the shim"
    obj = getattr(m, name)
    if entry["params"] is None:
        return
    got = shim_params(obj)
    ref = entry["params"]
    assert len(got) >= len(ref), (mod, name, got, ref)
    for (gname, gkind, gdef), (rname, rkind, rdef) in zip(got, ref):
        assert gname == rname, (mod, name, gname, rname)
        if rkind in ("POSITIONAL_OR_KEYWORD", "POSITIONAL_ONLY"):
            assert gkind in ("POSITIONAL_OR_KEYWORD", "POSITIONAL_ONLY"), (mod, name, gname)
        else:
            assert gkind == rkind, (mod, name, gname, gkind, rkind)
        assert gdef == rdef, (mod, name, gname, gdef, rdef)
    for gname, gkind, gdef in got[len(ref):]:
        assert gkind in ("KEYWORD_ONLY", "VAR_KEYWORD") or gdef != "<required>", (
            mod, name, "extra parameter without default", gname)


def test_package_exports_reference_names():
    import paper_2001_10554_b200 as qs
    missing = [n for n in REF["__init__"] if not hasattr(qs, n)]
    assert not missing, missing
