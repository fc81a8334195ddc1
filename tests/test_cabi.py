"""The C-ABI library loads without a GPU and exports every symbol include/coex_b200.h
declares; the Python binding's signature table covers the same set."""

import ctypes
import os
import re

from paper_2201_09210_b200 import b200

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared():
    hdr = open(os.path.join(ROOT, "include", "coex_b200.h")).read()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    return set(re.findall(r"\b(coex_[a-z0-9_]+)\s*\(", hdr))


def test_header_symbols_exported():
    lib = ctypes.CDLL(b200.lib_path())
    names = declared()
    assert len(names) >= 30
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_binding_covers_header():
    assert declared() == set(b200.SIGNATURES)


def test_load_library_and_version():
    lib = b200.load_library()
    assert b"sm_100a" in lib.coex_version()


def test_no_cpu_fallback_without_device():
    import pytest
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(Exception):
        b200.B200Backend()
