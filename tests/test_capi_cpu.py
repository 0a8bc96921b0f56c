"""The C-ABI library loads without a GPU and exports every symbol include/hdgb200.h declares."""

import ctypes
import os
import re

from conftest import ROOT


def declared_symbols():
    hdr = open(os.path.join(ROOT, "include", "hdgb200.h")).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[\w\s\*]+?\b(hdg_\w+)\s*\(", hdr, re.M)))


def test_header_symbols_exported():
    import paper_1705_09907_b200._lib as L
    names = declared_symbols()
    assert len(names) >= 20
    raw = ctypes.CDLL(L.LIB_PATH)
    for n in names:
        assert hasattr(raw, n), n
    assert sorted(L.exported_symbols()) == names


def test_error_reporting_without_gpu():
    import paper_1705_09907_b200._lib as L
    h = ctypes.c_void_p()
    rc = L.lib.hdg_level_create_shared(4, 4, 0, None, ctypes.byref(h))
    assert rc != 0
    assert L.lib.hdg_last_error()
