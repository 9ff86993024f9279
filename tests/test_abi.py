"""CPU-side checks of the boundary (-m "not gpu"): the C-ABI library builds for sm_100a,
loads, exports every symbol include/gwdp.h declares, and its host-only entry points
behave (no compute calls without a GPU)."""

import ctypes as C
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "gwdp.h")


def _declared():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    names = re.findall(r"^\s*(?:gw_status|const char|int)\s+\**\s*(\w+)\s*\(", txt, flags=re.M)
    return sorted(set(names))


@pytest.fixture(scope="module")
def lib():
    import __graft_entry__ as ge
    ge.build()
    from paper_2404_08970_b200 import _lib
    return _lib.load()


def test_header_declares_the_hot_path():
    names = _declared()
    for n in ["gw_grad_dp", "sinkhorn_solve", "entropic_gw_solve", "fgw_solve", "ugw_solve"]:
        assert n in names


def test_library_exports_every_declared_symbol(lib):
    from paper_2404_08970_b200 import _lib
    names = _declared()
    assert sorted(names) == sorted(_lib.SYMBOLS)
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\s[TW]\s+(\w+)$", out, flags=re.M))
    for n in names:
        assert n in exported, n
        assert hasattr(lib, n)


def test_library_is_sm100a(lib):
    from paper_2404_08970_b200 import _lib
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_host_only_entry_points(lib):
    assert lib.gw_abi_version() == 2
    # null-argument validation of ugw_solve happens before any device work
    from paper_2404_08970_b200 import _lib
    st = lib.ugw_solve(None, None, 1.0, None, None, None, 0, None, None, None, None)
    assert _lib.STATUS[st] == "GW_ERR_INVALID_ARG"
    # null-argument validation happens before any device work
    assert _lib.STATUS[lib.gw_grad_dp(None, None, None, 0, None, 0, None)] == "GW_ERR_INVALID_ARG"
    assert _lib.STATUS[lib.gw_solve_set_export(None, 1, None, None, 0)] == "GW_ERR_INVALID_ARG"


def test_product_path_has_no_oracle_or_fallback():
    """The product package never imports the oracle and has no CPU fallback."""
    pkg = os.path.join(ROOT, "paper_2404_08970_b200")
    for fn in os.listdir(pkg):
        if fn.endswith(".py"):
            src = open(os.path.join(pkg, fn)).read()
            assert "import oracle" not in src and "from oracle" not in src, fn
