"""CPU-side checks of the C-ABI library (-m "not gpu"): libwn.so builds for
sm_100a, loads, and exports every symbol include/wn.h declares; no compute
calls are made without a GPU."""
import ctypes
import os
import re
import subprocess

import pytest

import paper_2510_25159_b200 as wn
from paper_2510_25159_b200 import _build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "wn.h")).read()
    return sorted(set(re.findall(r"\b(wn_[a-z_]+)\s*\(", src)))


def test_header_declares_expected_api():
    d = _declared()
    for name in ["wn_build_faces", "wn_query", "wn_faces_info", "wn_free_faces", "wn_last_error"]:
        assert name in d


def test_library_builds_and_exports_every_symbol():
    path = _build.build()
    lib = ctypes.CDLL(path)
    for name in _declared():
        assert hasattr(lib, name), name
    assert sorted(wn.EXPORTS) == sorted(_declared())


def test_sass_is_sm100a():
    path = _build.build()
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", path], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_last_error_without_calls():
    wn.load()
    assert isinstance(wn.last_error(), str)


def test_query_without_handle_fails_loudly():
    L = wn.load()
    rc = L.wn_query(None, 10, None, None, None, None, None)
    assert rc == 1 and "NULL" in wn.last_error()
