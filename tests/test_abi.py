"""The C-ABI library loads on a CPU host and exports every declared symbol
(no compute calls: there is no GPU here), and fails loudly without a GPU."""

import ctypes
import os
import re

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols(header: str) -> set[str]:
    text = open(os.path.join(REPO, "include", header)).read()
    return set(re.findall(r"^\s*(?:[\w\s\*]+?)\b(gs_\w+)\s*\(", text, re.M))


def test_libgs_exports_every_declared_symbol():
    from paper_2107_08538_b200 import _native

    lib = _native.lib()
    names = declared_symbols("gs.h")
    assert len(names) >= 25
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    assert set(_native.SIGNATURES) == names
    assert lib.gs_abi_version() == 1


def test_struct_layouts_match_header():
    from paper_2107_08538_b200 import _native as nat

    assert ctypes.sizeof(nat.GsProbe) == 64
    assert ctypes.sizeof(nat.GsLedger) == 64
    assert ctypes.sizeof(nat.GsDecision) == 32
    assert ctypes.sizeof(nat.GsResidency) == 48
    assert ctypes.sizeof(nat.GsSpec) == 48


@pytest.mark.skipif(__import__("torch").cuda.is_available(), reason="GPU host")
def test_engine_refuses_without_gpu():
    from paper_2107_08538_b200 import _native

    with pytest.raises(RuntimeError, match="no CPU fallback|unavailable"):
        _native.Engine(0)
