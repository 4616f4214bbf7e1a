"""ctypes binding of the sm_100a TCEC library (libtcec.so, C ABI in include/tcec.h).

This is the only way the package reaches compute: there is no CPU fallback.
If the library is missing or the device is not an sm_100 GPU, every compute
call raises.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

_HERE = os.path.dirname(os.path.abspath(__file__))
# TCEC_LIB may point at another build of the same library
LIB_PATH = os.environ.get("TCEC_LIB") or os.path.join(_HERE, "libtcec.so")
CSRC = os.path.join(_HERE, "csrc")

# constants mirrored from include/tcec.h
TCEC_FP16, TCEC_TF32 = 0, 1
ROUND_DEFAULT, ROUND_RN, ROUND_RNA, ROUND_RZ = -1, 0, 1, 2
FLAG_OVERFLOW, FLAG_OUT_OF_RANGE, FLAG_NONFINITE_INPUT = 1, 2, 4
OK, ERR_ARG, ERR_ALIGN, ERR_UNSUPPORTED, ERR_CUDA, ERR_ARCH = 0, -1, -2, -3, -4, -5

# every symbol include/tcec.h declares (checked by the CPU test-suite)
EXPORTS = (
    "tcec_version",
    "tcec_status_str",
    "tcec_sgemm",
    "tcec_sgemm_host",
    "tcec_sgemm_multi",
    "tcec_split",
    "tcec_split_census",
    "tcec_launch_count",
    "tcec_host_release",
)


class TcecOpts(ctypes.Structure):
    _fields_ = [
        ("split_rounding", ctypes.c_int32),
        ("scale_log2", ctypes.c_int32),
        ("drain_k", ctypes.c_int32),
        ("block_n", ctypes.c_int32),
        ("group_m", ctypes.c_int32),
        ("split_mode", ctypes.c_int32),
        ("scheme", ctypes.c_int32),
        ("host_row_blocks", ctypes.c_int32),
        ("host_col_blocks", ctypes.c_int32),
        ("split_k", ctypes.c_int32),
        ("kernel_variant", ctypes.c_int32),
        ("reserved", ctypes.c_int32 * 2),
    ]


class TcecError(RuntimeError):
    def __init__(self, status: int, what: str):
        self.status = status
        super().__init__(f"{what}: {status_str(status)} (status {status})")


_lib = None


def build(force: bool = False) -> str:
    """Compile libtcec.so in place (nvcc, sm_100a)."""
    if force or not os.path.exists(LIB_PATH):
        subprocess.run(["make", "-s", "-C", CSRC], check=True)
    return LIB_PATH


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"TCEC CUDA library not built: {LIB_PATH} is missing "
            "(run `python -c 'import __graft_entry__ as g; g.build()'` or `make -C "
            f"{CSRC}`); there is no CPU fallback")
    L = ctypes.CDLL(LIB_PATH)
    i64, i32, p, u64 = ctypes.c_int64, ctypes.c_int, ctypes.c_void_p, ctypes.c_uint64
    L.tcec_version.restype = i32
    L.tcec_status_str.restype = ctypes.c_char_p
    L.tcec_status_str.argtypes = [i32]
    L.tcec_sgemm.restype = i32
    L.tcec_sgemm.argtypes = [i32, i64, i64, i64, p, i64, p, i64, p, i64, p, p, p]
    L.tcec_sgemm_multi.restype = i32
    L.tcec_sgemm_multi.argtypes = [i32, i64, i64, i64, p, i64, p, i64, p, i32, i64, p, p, p]
    L.tcec_sgemm_host.restype = i32
    L.tcec_sgemm_host.argtypes = [i32, i64, i64, i64, p, i64, p, i64, p, i64, p, p, p]
    L.tcec_split_census.restype = i32
    L.tcec_split_census.argtypes = [i32, i32, i32, p, p]
    L.tcec_split.restype = i32
    L.tcec_split.argtypes = [i32, i32, i32, p, i64, p, p, p, p]
    L.tcec_launch_count.restype = u64
    if hasattr(L, "tcec_host_release"):  # (absent from round-1 builds used in A/B runs)
        L.tcec_host_release.restype = i32
    _lib = L
    return L


def status_str(status: int) -> str:
    try:
        return lib().tcec_status_str(status).decode()
    except Exception:  # pragma: no cover - library missing
        return "unknown"


def check(status: int, what: str) -> None:
    if status != OK:
        raise TcecError(status, what)


def make_opts(split_rounding: int = ROUND_DEFAULT, scale_log2: int = -1, drain_k: int = 0,
              block_n: int = 0, group_m: int = 0, kernel_variant: int = 0,
              split_mode: int = 0, scheme: int = 0, host_blocks: tuple = (0, 0),
              split_k: int = 0) -> TcecOpts:
    o = TcecOpts()
    o.split_k = split_k
    o.host_row_blocks, o.host_col_blocks = host_blocks
    o.split_mode = split_mode
    o.scheme = scheme
    o.kernel_variant = kernel_variant
    o.split_rounding = split_rounding
    o.scale_log2 = scale_log2
    o.drain_k = drain_k
    o.block_n = block_n
    o.group_m = group_m
    return o


def launch_count() -> int:
    return int(lib().tcec_launch_count())
