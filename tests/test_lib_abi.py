"""The C-ABI library loads and exports every symbol include/spanpipe.h
declares (no compute calls: this runs without a GPU)."""

import ctypes
import os
import re

from conftest import ROOT


def _declared():
    src = open(os.path.join(ROOT, "include", "spanpipe.h")).read()
    return sorted(set(re.findall(r"\b(sp_[a-z0-9_]+)\s*\(", src)))


def test_header_and_binding_agree():
    from paper_2312_08361_b200 import _lib
    assert sorted(_lib.EXPORTS) == _declared()


def test_library_exports_every_declared_symbol():
    from paper_2312_08361_b200 import _lib
    lib = ctypes.CDLL(_lib.LIB_PATH)
    for name in _declared():
        assert hasattr(lib, name), name
    lib2 = _lib.load()
    assert lib2.sp_version() == 1
    # host-only entry points are callable without a GPU
    assert lib2.sp_fnv1a64(ctypes.c_char_p(b""), 0) == 0xCBF29CE484222325
    assert lib2.sp_fnv1a64(ctypes.c_char_p(b"a"), 1) == 0xAF63DC4C8601EC8C
    from oracle import model as om
    assert lib2.sp_stream_seed(1, 3, 5) == om.stream_seed(1, 3, "w1")


def test_config_struct_layout():
    from paper_2312_08361_b200 import _lib
    assert ctypes.sizeof(_lib.SpConfig) == 10 * 4 + 8 + 8
