"""The C-ABI library loads and exports every symbol include/tbgemm.h
declares (no compute calls: runs without a GPU)."""

import ctypes
import re
from pathlib import Path

from paper_1705_05249_b200.kernels import native

HEADER = Path(__file__).resolve().parent.parent / "include" / "tbgemm.h"


def declared_functions():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(tb_[a-z0-9_]+)\s*\(", text)))


def test_header_and_binding_agree():
    assert declared_functions() == sorted(native.EXPORTED_SYMBOLS)


def test_library_exports_every_symbol():
    so = native.lib()
    for name in declared_functions():
        assert hasattr(so, name), name
    assert so.tb_abi_version() == native.ABI_VERSION == 2
    assert so.tb_status_str(0) == b"ok"
    assert so.tb_status_str(3) == b"unsupported"


def test_struct_layouts():
    assert ctypes.sizeof(native.TbGemmConfig) == 7 * 4
    assert [f for f, _ in native.TbGemmConfig._fields_] == list(native.B200_PARAM_NAMES)
    assert ctypes.sizeof(native.TbLaunchRecord) == 64 + 24 + 12 + 12 + 4 + 4 + 8


def test_library_has_sm100a_code():
    data = native.library_path().read_bytes()
    assert b"sm_100a" in data or b"sm_100" in data
