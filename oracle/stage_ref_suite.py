"""Stage the reference's own test suite for the alias-shim run (test
infrastructure, build container only).

Copies /root/reference/pkg/tests/test_*.py into oracle/_ref/pkg_tests/ (git-
ignored like every oracle/_ref output, NOT gpurun-ignored, so the staged
suite travels to the GPU box with the built libirk.so) and adds the alias
conftest (oracle/ref_suite_conftest.py).  tests/test_reference_suite.py runs
it there against paper_2403_08084_b200.  The reference's implementation is
never copied: only its tests, which import ``implicitrk`` -> the drop-in.
"""

from __future__ import annotations

import shutil
from pathlib import Path

HERE = Path(__file__).resolve().parent
SRC = Path("/root/reference/pkg/tests")
DST = HERE / "_ref" / "pkg_tests"


def stage() -> Path | None:
    if not SRC.is_dir():
        return DST if DST.is_dir() else None
    DST.mkdir(parents=True, exist_ok=True)
    for p in DST.glob("*.py"):
        p.unlink()
    for p in sorted(SRC.glob("test_*.py")):
        shutil.copyfile(p, DST / p.name)
    shutil.copyfile(HERE / "ref_suite_conftest.py", DST / "conftest.py")
    # keep the staged suite out of the repo's own collection
    (DST / "pytest.ini").write_text("[pytest]\naddopts = -p no:cacheprovider\n")
    return DST


if __name__ == "__main__":
    print(stage())
