"""The C-ABI library builds for sm_100a, loads, and exports every symbol the
public header declares (CPU-only: no compute calls)."""

import ctypes
import os
import re
import subprocess

from paper_2403_11166_b200 import _build, _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "pencil_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(pb_[a-z0-9_]+)\s*\(", src)))


def test_library_builds_and_exports_header_symbols():
    path = _build.build()
    assert os.path.exists(path)
    lib = ctypes.CDLL(path)
    names = _declared()
    assert len(names) >= 30
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    # python binding covers every declared entry point
    assert set(names) <= set(_lib.SIGNATURES), set(names) - set(_lib.SIGNATURES)


def test_library_is_sm100a_native():
    path = _build.build()
    out = subprocess.run(["cuobjdump", "--list-elf", path], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_abi_version_and_error_channel():
    lib = _lib.load()
    assert lib.pb_abi_version() == _lib.ABI_VERSION == 2
    # argument validation runs host-side, before any device work
    st = lib.pb_ring_binary(99, None, None, None, 0, 1, 59, None)
    assert st == 8
    assert "null" in _lib.last_error() or "bad" in _lib.last_error()
