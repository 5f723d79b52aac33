"""The reference's own test suite run against the drop-in (gpu).

oracle/stage_ref_suite.py (called by __graft_entry__.build() in the build
container) stages /root/reference/pkg/tests with an alias conftest that binds
``implicitrk`` and its submodules to paper_2403_08084_b200; this test runs
that suite in a subprocess on the GPU and parses its JUnit report.  Every
failure must be a documented deviation (DEVIATIONS, with the reason); the
per-file tally is printed (profiles/r02/reference_suite.txt keeps a run).
"""

import os
import subprocess
import sys
import xml.etree.ElementTree as ET
from collections import Counter
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]
SUITE = ROOT / "oracle" / "_ref" / "pkg_tests"

# nodeid -> why the drop-in deliberately differs.  Test names are the
# reference's (pkg/tests/...).
DEVIATIONS = {
    "test_acceptance::test_criterion_08_preconditioner_scaling":
        "fails in the reference itself, by design (pkg/test_output.txt:371; SPEC.md criterion "
        "8).  The drop-in reproduces the reference's iteration counts exactly (rana-ld 1,4,5,6; "
        "jacobi 1,9,13,16; gs-lower 1,6,7,9), so it fails the same assertion",
    "test_cli.TestPrecondBench::test_solver_failure_exit_3":
        "relies on modified Gram-Schmidt's stagnation: with rtol 1e-30 the reference's MGS "
        "recurrence residual stalls at 1.5e-30 > target 5.5e-31 and exhausts maxit.  north_star "
        "(3) prescribes classical Gram-Schmidt with fused multi-dots; CGS (and CGS2) keep "
        "reducing the recurrence residual and converge, so the CLI exits 0.  Exit code 3 on "
        "maxit is covered by tests/test_mms_cli.py::test_cli_solver_failure_exit_3",
}

MIN_PASSED = 300


def _cases(xml_path):
    root = ET.parse(xml_path).getroot()
    for tc in root.iter("testcase"):
        cls = tc.get("classname", "")
        name = tc.get("name", "")
        outcome = "passed"
        for child in tc:
            if child.tag in ("failure", "error"):
                outcome = "failed"
            elif child.tag == "skipped":
                outcome = "skipped"
        yield cls, name, outcome


def test_reference_suite_against_drop_in(cuda, tmp_path):
    if not (SUITE / "conftest.py").exists():
        pytest.skip("reference suite not staged (oracle/stage_ref_suite.py runs in the build "
                    "container, where /root/reference exists)")
    xml = tmp_path / "ref.xml"
    env = dict(os.environ, PYTHONDONTWRITEBYTECODE="1")
    proc = subprocess.run([sys.executable, "-m", "pytest", str(SUITE), "-q", "-p",
                           "no:cacheprovider", f"--junitxml={xml}", "-o",
                           "junit_family=xunit1"],
                          cwd=str(SUITE), env=env, capture_output=True, text=True, timeout=3000)
    assert xml.exists(), proc.stdout[-3000:] + proc.stderr[-3000:]
    tally = Counter()
    per_file = {}
    failed = []
    for cls, name, outcome in _cases(xml):
        mod = cls.split(".")[0] if cls else "?"
        per_file.setdefault(mod, Counter())[outcome] += 1
        tally[outcome] += 1
        if outcome == "failed":
            failed.append(f"{cls}::{name}")
    for mod in sorted(per_file):
        c = per_file[mod]
        print(f"{mod}: {c['passed']} passed, {c['failed']} failed, {c['skipped']} skipped")
    print(f"total: {dict(tally)}")
    for f in failed:
        print("FAILED", f, "--", DEVIATIONS.get(f, "UNDOCUMENTED"))
    undocumented = [f for f in failed if f not in DEVIATIONS]
    assert not undocumented, "\n".join(undocumented) + "\n" + proc.stdout[-6000:]
    assert tally["passed"] >= MIN_PASSED
