"""CPU checks of the boundary: libprohd.so loads and exports every symbol include/prohd.h declares;
pure-host entry points behave; the ctypes structs match the header's layout. No compute calls."""
import ctypes as C
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_2511_18207_b200.build import build
    build()
    from paper_2511_18207_b200 import _lib
    return _lib.load()


def _declared():
    with open(os.path.join(ROOT, "include", "prohd.h")) as f:
        src = f.read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?(?:int|size_t|char\s*\*|const char\s*\*)\s*\**\s*([a-z_0-9]+)\s*\(", src, re.M)
    return sorted(set(names))


def test_header_declares_expected(lib):
    from paper_2511_18207_b200 import _lib
    assert set(_declared()) == set(_lib.EXPORTED)


def test_exports_every_declared_symbol(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", os.path.join(ROOT, "paper_2511_18207_b200", "libprohd.so")],
                         capture_output=True, text=True, check=True).stdout
    exported = {ln.split()[-1] for ln in out.splitlines() if " T " in ln}
    for name in _declared():
        assert name in exported, name
        assert getattr(lib, name) is not None


def test_sm100a_only(lib):
    out = subprocess.run(["cuobjdump", "--list-elf", os.path.join(ROOT, "paper_2511_18207_b200", "libprohd.so")],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_host_entry_points(lib):
    assert lib.prohd_version().decode().startswith("prohd-b200")
    assert lib.prohd_workspace_bytes(0, 10, 4, 0, 1, 0) == 0
    small = lib.prohd_workspace_bytes(2000, 2000, 16, 4, 20, 0)
    host = lib.prohd_workspace_bytes(2000, 2000, 16, 4, 20, 1)
    assert 0 < small < host
    assert host - small >= 2 * 2000 * 16 * 4
    big = lib.prohd_workspace_bytes(2_000_000, 2_000_000, 256, 16, 1000, 0)
    assert big > 4 * 2_000_000 * 256 * 4  # hi/lo operands of both sets


def test_null_context_errors(lib):
    from paper_2511_18207_b200 import _lib as L
    assert lib.prohd_set_workspace(None, None, 0) == L.PROHD_E_INVALID
    assert lib.prohd_set_stream(None, None) == L.PROHD_E_INVALID
    assert lib.prohd_last_error(None) == b"null context"
    out = L.Directed()
    assert lib.directed_hd(None, None, 1, None, 1, 1, C.byref(out)) == L.PROHD_E_INVALID


def test_struct_sizes():
    from paper_2511_18207_b200 import _lib as L
    assert C.sizeof(L.Directed) == 40
    assert C.sizeof(L.HD) == 88
    assert C.sizeof(L.Est) == 8 + 80 + 16 + 8
    assert C.sizeof(L.Timings) == 9 * 8 + 8
