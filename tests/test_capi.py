"""The C-ABI library (the drop-in boundary) loads and exports every symbol that
include/shouji_b200.h declares. No compute calls here (no GPU in CI)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "shouji_b200.h")
LIB = os.path.join(ROOT, "paper_1809_07858_b200", "libshouji_b200.so")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(pf_[a-z_0-9]+)\s*\(", src)))


def test_header_declares_entry_points():
    names = declared_functions()
    for must in ("pf_shouji_filter_batch", "pf_shouji_filter_device", "pf_shouji_filter_one",
                 "pf_ctx_create", "pf_ctx_destroy", "pf_status_string"):
        assert must in names


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(LIB)
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing
    from paper_1809_07858_b200 import _lib
    assert sorted(_lib.EXPORTED) == declared_functions()


def test_exports_are_plain_c():
    out = subprocess.run(["nm", "-D", "--defined-only", LIB], capture_output=True, text=True).stdout
    exported = {l.split()[-1] for l in out.splitlines() if " T " in l}
    for n in declared_functions():
        assert n in exported  # unmangled extern "C"


def test_library_is_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", LIB], capture_output=True, text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_status_strings_and_pitch():
    from paper_1809_07858_b200 import _lib
    assert _lib.lib.pf_status_string(2) == b"illegal character"
    assert _lib.lib.pf_status_string(7) == b"invalid parameters"
    assert _lib.lib.pf_device_pitch(100) == 100
    assert _lib.lib.pf_device_pitch(250) == 252
    assert _lib.lib.pf_device_pitch(150) == 152
    assert _lib.lib.pf_device_pitch(1) == 4


def test_no_device_fails_loudly():
    from paper_1809_07858_b200 import _lib
    if _lib.lib.pf_device_count() > 0:
        pytest.skip("a device is present")
    import paper_1809_07858_b200 as pf
    with pytest.raises(pf.device_error):
        pf.Context()
    with pytest.raises(pf.device_error):
        pf.shouji_filter(pf.seq("ACGT"), pf.seq("ACGT"), 1)
