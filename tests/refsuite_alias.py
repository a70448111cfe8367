"""pytest plugin: run the REFERENCE's own unit tests against the drop-in.

``python -m pytest -p refsuite_alias oracle/_ref/tests`` (see
tests/test_reference_suite.py) makes ``import fmm2d`` and its submodules
resolve to ``paper_1205_4611_b200``, so the reference's tests
(pkg/tests/*.py, staged by oracle/build_ref.sh) exercise the GPU package
unmodified.  Test infrastructure only.
"""

import importlib
import sys

import paper_1205_4611_b200 as _pkg

_SUBMODULES = {
    "tree": "tree",
    "connectivity": "connectivity",
    "engine": "engine",
    "operators": "operators",
    "geometry": "geometry",
    "datasets": "datasets",
    "fileio": "fileio",
    "bench": "experiments",     # the reference's experiment runners (bench.py)
}

sys.modules["fmm2d"] = _pkg
for _ref_name, _ours in _SUBMODULES.items():
    _mod = importlib.import_module(f"paper_1205_4611_b200.{_ours}")
    sys.modules[f"fmm2d.{_ref_name}"] = _mod
    setattr(_pkg, _ref_name, _mod)
