"""The C-ABI library loads and exports exactly the symbols include/btp.h declares (no GPU
work is launched here)."""

import re
import subprocess
from pathlib import Path

import pytest

from paper_2512_12131_b200 import _native

ROOT = Path(__file__).resolve().parent.parent


def _declared():
    hdr = (ROOT / "include" / "btp.h").read_text()
    return set(re.findall(r"^\s*(?:int|const char\*)\s+(btp_\w+)\s*\(", hdr, flags=re.M))


def test_header_and_binding_agree():
    assert _declared() == set(_native.EXPORTED_SYMBOLS)


def test_library_exports_every_symbol():
    lib = _native.library_path()
    if not lib.exists():
        pytest.skip("libbtp.so not built (run __graft_entry__.build())")
    out = subprocess.run(["nm", "-D", "--defined-only", str(lib)], capture_output=True, text=True, check=True).stdout
    exported = {ln.split()[-1] for ln in out.splitlines() if " T " in ln}
    assert _declared() <= exported
    handle = _native.load()
    for name in _native.EXPORTED_SYMBOLS:
        assert getattr(handle, name) is not None
    assert b"sm_100a" in handle.btp_version()


def test_sass_has_tcgen05_and_tma():
    lib = _native.library_path()
    if not lib.exists():
        pytest.skip("libbtp.so not built")
    sass = subprocess.run(["cuobjdump", "-sass", str(lib)], capture_output=True, text=True).stdout
    if not sass:
        pytest.skip("cuobjdump unavailable")
    assert "UTCHMMA" in sass and "UTMALDG" in sass and "LDTM" in sass


def test_gemm_problem_layout_matches_header_and_docs():
    """The ctypes GemmProblem, the btp_gemm_problem struct of include/btp.h and the binding example
    in INTEGRATION.md list the same fields in the same order (a mismatch silently corrupts calls)."""
    hdr = (ROOT / "include" / "btp.h").read_text()
    body = hdr[hdr.index("typedef struct btp_gemm_problem {"):hdr.index("} btp_gemm_problem;")]
    body = re.sub(r"/\*.*?\*/", "", body, flags=re.S)
    hdr_fields = []
    for decl in re.findall(r"^\s*([^;{}]+);", body.split("{", 1)[1], flags=re.M):
        first, *rest = [t.strip() for t in decl.split(",")]
        hdr_fields += [first.split()[-1].lstrip("*")] + [r.lstrip("*") for r in rest]
    ctypes_fields = [f[0] for f in _native.GemmProblem._fields_]
    doc = (ROOT / "INTEGRATION.md").read_text()
    doc = doc[doc.index("class btp_gemm_problem"):doc.index("lib.btp_gemm.argtypes")]
    doc_fields = re.findall(r'\("(\w+)", ctypes\.c_\w+\)', doc)
    assert hdr_fields == ctypes_fields == doc_fields
