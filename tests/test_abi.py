"""C-ABI checks that need no GPU: libhga.so loads and exports every symbol
include/hga.h declares; the ctypes table matches the header."""

from __future__ import annotations

import ctypes
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "hga.h"
LIB = ROOT / "paper_2208_14961_b200" / "libhga.so"


def header_functions() -> set[str]:
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return set(re.findall(r"\b(hga_[a-z0-9_]+)\s*\(", text))


def test_header_parses():
    fns = header_functions()
    assert "hga_fitness_i8" in fns and "hga_run" in fns and len(fns) >= 20


@pytest.mark.skipif(not LIB.exists(), reason="libhga.so not built")
def test_library_exports_every_header_symbol():
    dll = ctypes.CDLL(str(LIB))
    missing = [f for f in sorted(header_functions()) if not hasattr(dll, f)]
    assert not missing, missing


def test_ctypes_table_covers_header():
    from paper_2208_14961_b200._lib import SIGNATURES

    assert header_functions() == set(SIGNATURES)


@pytest.mark.skipif(not LIB.exists(), reason="libhga.so not built")
def test_host_side_validation_without_gpu():
    from paper_2208_14961_b200._lib import lib

    assert lib.hga_abi_version() == 1
    assert lib.hga_strerror(1) == b"invalid argument"
    # argument errors are detected on the host before any launch
    assert lib.hga_fitness_i8(None, -1, 4, 1, None, None, None, None, None, None, 0, None) == 1
    assert lib.hga_fitness_i8(None, 4, 4, 0, None, None, None, None, None, None, 0, None) == 1
    assert lib.hga_ref_uniform(1, 2, 0, 5, 3, 4, None, None) == 1
    assert lib.hga_run_ws_bytes(1000, 20) > 16000
    assert lib.hga_select_max_range() == 1 << 22


def test_product_has_no_oracle_dependency():
    pkg = ROOT / "paper_2208_14961_b200"
    for f in pkg.rglob("*.py"):
        src = f.read_text()
        assert "import oracle" not in src and "from oracle" not in src, f
