"""Alias shim for running the reference's own test suite against the drop-in
(test infrastructure).

Staged by oracle/stage_ref_suite.py as ``conftest.py`` next to copies of the
reference's test files (oracle/_ref/pkg_tests/, git-ignored).  Before the
reference's tests import ``implicitrk``, every module name they use is bound
to the B200 package, so ``from implicitrk.sparsela import fgmres`` resolves to
paper_2403_08084_b200.sparsela.fgmres, and so on.  Nothing of the
reference's implementation is imported: the tests exercise only the drop-in.
"""

import importlib
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[3]
sys.path.insert(0, str(ROOT))

_pkg = importlib.import_module("paper_2403_08084_b200")
sys.modules["implicitrk"] = _pkg
for _sub in ("bcs", "cli", "precond", "problems", "sparsela", "stepper", "tableaux"):
    sys.modules[f"implicitrk.{_sub}"] = importlib.import_module(f"paper_2403_08084_b200.{_sub}")
