"""ctypes binding of libtbgemm.so — the C-ABI declared in include/tbgemm.h.

The native library is the ONLY compute path: there is no CPU fallback.  If
the shared object is missing or fails to load, every routine call raises
:class:`NativeLibraryError` (loudly), mirroring how the reference's
``run_kernel`` (pkg/src/tunedblas/kernels/compute.py:116-130) is the single
place arithmetic happens.
"""

from __future__ import annotations

import ctypes
import os
import threading
from collections.abc import Mapping
from pathlib import Path

from ..errors import TunedBlasError

__all__ = [
    "NativeLibraryError",
    "TbGemmConfig",
    "B200_PARAM_NAMES",
    "TbLaunchRecord",
    "lib",
    "library_path",
    "EXPORTED_SYMBOLS",
    "PREC_H",
    "PREC_S",
    "COL_MAJOR",
    "ROW_MAJOR",
    "FLAG_TF32",
    "FLAG_NO_TMA",
    "FLAG_SIMT_GENERAL",
    "FLAG_NO_PACK",
    "FLAG_NO_2SM",
    "FLAG_NO_SPLITK",
    "FLAG_WAVE_SYNC",
]

PREC_H, PREC_S = 0, 1
COL_MAJOR, ROW_MAJOR = 0, 1
NO_TRANS, TRANS, CONJ_TRANS = 0, 1, 2
XF_COPY, XF_SYMMETRIZE, XF_TRIANGULARIZE, XF_TRI_COPY = 0, 1, 2, 3
FLAG_TF32, FLAG_NO_TMA, FLAG_SIMT_GENERAL, FLAG_NO_PACK, FLAG_NO_2SM, FLAG_NO_SPLITK = 1, 2, 4, 8, 16, 32
FLAG_WAVE_SYNC = 64
TB_OK = 0

#: Every symbol include/tbgemm.h declares (checked by tests/test_native_abi.py).
EXPORTED_SYMBOLS = (
    "tb_gemm",
    "tb_convgemm",
    "tb_im2col",
    "tb_transform",
    "tb_convert_f32",
    "tb_trsm_block",
    "tb_gemm_strided_batched",
    "tb_gemm_batched",
    "tb_last_launch",
    "tb_status_str",
    "tb_last_error",
    "tb_abi_version",
    "tb_device_sm_count",
    "tb_prepare_device",
)

#: Expected TBGEMM_ABI_VERSION (include/tbgemm.h).
ABI_VERSION = 2


class NativeLibraryError(TunedBlasError, RuntimeError):
    """The CUDA library could not be loaded or a kernel launch failed."""


#: The "gemm_b200" tuning family (include/tbgemm.h tb_gemm_config;
#: kernels/params.py), in struct order.
B200_PARAM_NAMES = ("MWG", "NWG", "KWG", "STAGES", "CTA_GROUP", "SPLIT_K", "GROUP_M")


class TbGemmConfig(ctypes.Structure):
    _fields_ = [(name, ctypes.c_int32) for name in B200_PARAM_NAMES]

    @classmethod
    def from_dict(cls, values: dict) -> "TbGemmConfig":
        return cls(*(int(values[name]) for name in B200_PARAM_NAMES))


class TbLaunchRecord(ctypes.Structure):
    _fields_ = [
        ("kernel", ctypes.c_char * 64),
        ("grid", ctypes.c_int64 * 3),
        ("block", ctypes.c_int32 * 3),
        ("cluster", ctypes.c_int32 * 3),
        ("smem_bytes", ctypes.c_int32),
        ("launches", ctypes.c_int32),
        ("tiles", ctypes.c_int64),
    ]

    def to_dict(self) -> dict:
        return {
            "kernel": self.kernel.decode(),
            "grid": tuple(self.grid),
            "block": tuple(self.block),
            "cluster": tuple(self.cluster),
            "smem_bytes": int(self.smem_bytes),
            "launches": int(self.launches),
            "tiles": int(self.tiles),
        }


def library_path() -> Path:
    override = os.environ.get("TBGEMM_LIB")
    if override:
        return Path(override)
    return Path(__file__).resolve().parent.parent / "_lib" / "libtbgemm.so"


_lock = threading.Lock()
_lib = None

_i32, _i64, _f32, _vp = ctypes.c_int, ctypes.c_int64, ctypes.c_float, ctypes.c_void_p
_P = ctypes.POINTER


def _declare(so) -> None:
    so.tb_gemm.restype = _i32
    so.tb_gemm.argtypes = [_i32, _i32, _i32, _i32, _i64, _i64, _i64, _f32,
                           _vp, _i64, _i64, _vp, _i64, _i64, _f32,
                           _vp, _i64, _i64, _P(TbGemmConfig), _i32, _vp]
    so.tb_gemm_strided_batched.restype = _i32
    so.tb_gemm_strided_batched.argtypes = [
        _i32, _i32, _i32, _i32, _i64, _i64, _i64, _f32,
        _vp, _i64, _i64, _i64, _vp, _i64, _i64, _i64, _f32,
        _vp, _i64, _i64, _i64, _i64, _P(TbGemmConfig), _i32, _vp]
    so.tb_gemm_batched.restype = _i32
    so.tb_gemm_batched.argtypes = [
        _i32, _i32, _i32, _i32, _i64, _i64, _i64, _vp,
        _vp, _vp, _i64, _vp, _vp, _i64, _vp,
        _vp, _vp, _i64, _i64, _i32, _P(TbGemmConfig), _i32, _vp]
    so.tb_convgemm.restype = _i32
    so.tb_convgemm.argtypes = [_i32] + [_i64] * 13 + [_vp, _i64, _vp, _i64, _vp, _i64, _i32, _vp]
    so.tb_im2col.restype = _i32
    so.tb_im2col.argtypes = [_i32] + [_i64] * 11 + [_vp, _i64, _vp, _i64, _vp]
    so.tb_transform.restype = _i32
    so.tb_transform.argtypes = [_i32, _i32, _i64, _i64, _vp, _i64, _i64, _vp, _i64, _i64, _i32, _i32, _vp]
    so.tb_convert_f32.restype = _i32
    so.tb_convert_f32.argtypes = [_i32, _i32, _i64, _i64, _f32, _vp, _i64, _i64, _i32, _vp, _i64, _i64, _vp]
    so.tb_trsm_block.restype = _i32
    so.tb_trsm_block.argtypes = [_i64, _i64, _vp, _i64, _i64, _vp, _i64, _i64, _i32, _i32, _vp]
    so.tb_last_launch.restype = _i32
    so.tb_last_launch.argtypes = [_P(TbLaunchRecord)]
    so.tb_status_str.restype = ctypes.c_char_p
    so.tb_status_str.argtypes = [_i32]
    so.tb_last_error.restype = ctypes.c_char_p
    so.tb_last_error.argtypes = []
    so.tb_abi_version.restype = _i32
    so.tb_abi_version.argtypes = []
    so.tb_device_sm_count.restype = _i32
    so.tb_device_sm_count.argtypes = []
    so.tb_prepare_device.restype = _i32
    so.tb_prepare_device.argtypes = []


def lib():
    """The loaded library (raises NativeLibraryError when unavailable)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            path = library_path()
            if not path.exists():
                raise NativeLibraryError(
                    f"CUDA library {path} is missing; run __graft_entry__.build() "
                    "(there is no CPU fallback)")
            try:
                so = ctypes.CDLL(str(path))
            except OSError as exc:
                raise NativeLibraryError(f"cannot load {path}: {exc}") from exc
            _declare(so)
            ver = so.tb_abi_version()
            if ver != ABI_VERSION:
                raise NativeLibraryError(
                    f"{path} has ABI version {ver}, this package needs {ABI_VERSION}; "
                    "rebuild with __graft_entry__.build()")
            _lib = so
    return _lib


def check(status: int, what: str) -> None:
    if status != TB_OK:
        so = lib()
        raise NativeLibraryError(
            f"{what} failed: {so.tb_status_str(status).decode()} "
            f"({so.tb_last_error().decode()})")


class NativeLaunch(Mapping):
    """Read-only view of one ``tb_launch_record`` (copied at call time,
    decoded to a dict on first access)."""

    __slots__ = ("_rec", "_d")

    def __init__(self, rec: TbLaunchRecord):
        self._rec = rec
        self._d = None

    def _dict(self) -> dict:
        d = self._d
        if d is None:
            d = self._d = self._rec.to_dict()
        return d

    def __getitem__(self, key):
        return self._dict()[key]

    def __iter__(self):
        return iter(self._dict())

    def __len__(self):
        return len(self._dict())

    def __eq__(self, other):
        return dict(self._dict()) == (dict(other) if isinstance(other, Mapping) else other)

    def __repr__(self):
        return repr(self._dict())


def last_launch() -> NativeLaunch:
    rec = TbLaunchRecord()
    st = lib().tb_last_launch(ctypes.byref(rec))
    if st != TB_OK:
        check(st, "tb_last_launch")
    return NativeLaunch(rec)
