"""CPU checks of the C-ABI boundary: libirk.so loads, exports every symbol
include/irk.h declares, and the Python binding covers exactly that set."""

import ctypes
import re

import pytest

from conftest import ROOT


def header_symbols():
    text = (ROOT / "include" / "irk.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|size_t|const char\*)\s+(irk_\w+)\s*\(", text, re.M)))


def test_header_declares_core_entry_points():
    syms = header_symbols()
    for name in ("irk_stage_apply", "irk_pcg", "irk_cocg", "irk_multidot", "irk_orth_update",
                 "irk_mat_assemble_p1", "irk_stage_update", "irk_semilinear_residual"):
        assert name in syms


def test_library_exports_every_header_symbol():
    from paper_2403_08084_b200 import _build

    lib_path = _build.build()
    lib = ctypes.CDLL(str(lib_path))
    missing = [s for s in header_symbols() if not hasattr(lib, s)]
    assert not missing, f"symbols declared in irk.h but not exported: {missing}"


def test_binding_matches_header():
    from paper_2403_08084_b200 import _lib

    assert sorted(_lib.EXPORTED) == header_symbols()


def test_version_without_gpu():
    from paper_2403_08084_b200 import _lib

    assert b"sm_100a" in _lib.load().irk_version()


def test_built_for_sm100a():
    import subprocess

    from paper_2403_08084_b200 import _build

    out = subprocess.run(["cuobjdump", "--list-elf", str(_build.build())],
                         capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_context_needs_a_device():
    import torch

    if torch.cuda.is_available():
        pytest.skip("device present")
    from paper_2403_08084_b200 import _lib

    with pytest.raises(_lib.LibraryUnavailable):
        _lib.ctx()
