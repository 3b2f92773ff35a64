"""pytest plugin (-p refshim): makes ``import rnscope`` resolve to the drop-in package, so that the
reference's OWN hot-path test files (a travelling, git-ignored copy under baseline/_ref/ref_tests,
made by __graft_entry__.build() from /root/reference/pkg/tests) run unchanged against the CUDA
engine.  Only the module API the drop-in mirrors is aliased; the analytical cost
model the reference's conftest imports is the reference's own pure-Python file."""
import importlib
import importlib.util
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

import paper_2512_18345_b200 as _pkg  # noqa: E402

sys.modules["rnscope"] = _pkg
for _name in ("rns", "transform", "baseconv", "keyswitch", "params", "vectors", "instrument"):
    _mod = importlib.import_module(f"paper_2512_18345_b200.{_name}")
    sys.modules[f"rnscope.{_name}"] = _mod
    setattr(_pkg, _name, _mod)

_cm = ROOT / "baseline" / "_ref" / "rnscope" / "costmodel.py"
if _cm.exists():
    _spec = importlib.util.spec_from_file_location("rnscope.costmodel", _cm)
    _module = importlib.util.module_from_spec(_spec)
    _module.__package__ = "rnscope"
    sys.modules["rnscope.costmodel"] = _module
    _spec.loader.exec_module(_module)
    _pkg.costmodel = _module
