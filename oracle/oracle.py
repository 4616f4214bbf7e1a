"""ctypes front-end of the CPU parity oracle -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this module; the product package never does (the
product path is the sm_100a library and fails loudly without it).

The C restatement (oracle/tcec_oracle.c) follows
/root/reference/pkg/src/tcgemm/{formats,splitting,mma,schemes}.py line by line
and is pinned bit-for-bit against golden vectors generated from the reference
(tests/golden/make_golden.py).
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libtcec_oracle.so")
_lib = None

FMT_FP16, FMT_TF32, FMT_FP32 = 0, 1, 2
RM_RN, RM_RNA, RM_RZ = 0, 1, 2
FLAG_OVERFLOW, FLAG_OUT_OF_RANGE = 1, 2

# variant name -> (format, residual scale, default split rounding); mirrors
# splitting.py:43-67 (scaled_halfhalf: FP16, s=11, RN; tf32tf32: TF32, s=0, RNA)
VARIANTS = {
    "fp16": (FMT_FP16, 11, RM_RN),
    "tf32": (FMT_TF32, 0, RM_RNA),
    "fp16u": (FMT_FP16, 0, RM_RN),  # markidis_halfhalf (splitting.py:70-71), unscaled
}


def build() -> str:
    """Compile the oracle in place (gcc via oracle/Makefile)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        i64, i32, p = ctypes.c_int64, ctypes.c_int, ctypes.c_void_p
        L.tcec_oracle_round.argtypes = [i32, i32, i64, p, p]
        L.tcec_oracle_split.argtypes = [i32, i32, i32, i64, p, p, p]
        L.tcec_oracle_classify.argtypes = [i32, i32, i64, p, p]
        L.tcec_oracle_corrected3.argtypes = [
            i32, i32, i32, i64, i64, i64, p, i64, p, i64, p, i64,
            i32, i32, i32, i32, i32, p,
        ]
        L.tcec_oracle_inunit.argtypes = [
            i32, i32, i32, i32, i32, i64, i64, i64, p, i64, p, i64, p, i64, i32, i32, p,
        ]
        L.tcec_oracle_hw.argtypes = [
            i32, i32, i32, i32, i64, i64, i64, p, i64, p, i64, p, i64, i32, i32, p,
        ]
        L.tcec_oracle_fp32_simt.argtypes = [i64, i64, i64, p, i64, p, i64, p, i64, i32]
        L.tcec_oracle_fp64_ref.argtypes = [i64, i64, i64, p, i64, p, i64, p, i64]
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data)


def round_to_format(x, fmt: int, mode: int) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.float64)
    out = np.empty_like(x)
    lib().tcec_oracle_round(fmt, mode, x.size, _ptr(x), _ptr(out))
    return out


def split(x, variant: str = "fp16", rounding: int | None = None):
    """Elementwise (hi, lo) of splitting.py:_split_arrays as float64 arrays."""
    fmt, s, rm = VARIANTS[variant]
    if rounding is not None:
        rm = rounding
    x = np.ascontiguousarray(x, dtype=np.float32)
    hi = np.empty(x.shape, np.float64)
    lo = np.empty(x.shape, np.float64)
    lib().tcec_oracle_split(fmt, s, rm, x.size, _ptr(x), _ptr(hi), _ptr(lo))
    return hi, lo


def classify(x, variant: str = "fp16") -> np.ndarray:
    fmt, s, _ = VARIANTS[variant]
    x = np.ascontiguousarray(x, dtype=np.float32)
    out = np.empty(x.shape, np.int8)
    lib().tcec_oracle_classify(fmt, s, x.size, _ptr(x), _ptr(out))
    return out


def corrected3(a, b, variant: str = "fp16", block_k: int = 16, drain_k: int | None = None,
               acc_bits: int = 25, include_dd: bool = False, rounding: int | None = None,
               nthreads: int = 0):
    """schemes.py:gemm(corrected3) restated; returns (C float32, flags int)."""
    fmt, s, rm = VARIANTS[variant]
    if rounding is not None:
        rm = rounding
    a = np.ascontiguousarray(a, dtype=np.float32)
    b = np.ascontiguousarray(b, dtype=np.float32)
    m, k = a.shape
    k2, n = b.shape
    if k2 != k:
        raise ValueError(f"inner dimensions differ: {k} vs {k2}")
    c = np.empty((m, n), np.float32)
    flags = ctypes.c_uint32(0)
    rc = lib().tcec_oracle_corrected3(
        fmt, s, rm, m, n, k, _ptr(a), k, _ptr(b), n, _ptr(c), n,
        block_k, drain_k or block_k, acc_bits, int(include_dd), nthreads,
        ctypes.byref(flags))
    if rc != 0:
        raise ValueError(f"oracle rejected arguments (rc={rc})")
    return c, int(flags.value)


# MMA k-step (products per tcgen05.mma instruction) and the kernels' default
# drain interval in k, per variant
MMA_K = {"fp16": 16, "fp16u": 16, "tf32": 8}
DEFAULT_DRAIN_K = {"fp16": 128, "fp16u": 128, "tf32": 64}


def _hw(sched: int, a, b, fmt: int, s: int, rm: int, drain_ksteps: int, nthreads: int):
    a = np.ascontiguousarray(a, dtype=np.float32)
    b = np.ascontiguousarray(b, dtype=np.float32)
    m, k = a.shape
    k2, n = b.shape
    if k2 != k:
        raise ValueError(f"inner dimensions differ: {k} vs {k2}")
    c = np.empty((m, n), np.float32)
    flags = ctypes.c_uint32(0)
    rc = lib().tcec_oracle_hw(sched, fmt, s, rm, m, n, k, _ptr(a), k, _ptr(b), n, _ptr(c), n,
                              drain_ksteps, nthreads, ctypes.byref(flags))
    if rc != 0:
        raise ValueError(f"oracle rejected arguments (rc={rc})")
    return c, int(flags.value)


def corrected3_hw(a, b, variant: str = "fp16", drain_k: int | None = None,
                  include_dd: bool = False, rounding: int | None = None, nthreads: int = 0):
    """The GPU kernels' corrected3 (tcec_oracle_hw): the reference's split and
    product order with the B200 tensor core's measured MMA arithmetic and the
    kernels' drain schedule (drain_k in k, a multiple of the MMA k-step;
    default the kernels' 128 FP16 / 64 TF32).  Returns (C float32, flags int);
    the GPU must match it bit for bit."""
    fmt, s, rm = VARIANTS[variant]
    if rounding is not None:
        rm = rounding
    d = drain_k or DEFAULT_DRAIN_K[variant]
    if d % MMA_K[variant]:
        raise ValueError("drain_k must be a multiple of the MMA k-step")
    return _hw(1 if include_dd else 0, a, b, fmt, s, rm, d // MMA_K[variant], nthreads)


def corrected3_hw_split_k(a, b, variant: str, parts: int, drain_k: int | None = None,
                          nthreads: int = 0):
    """The split-K path (opts.split_k) with the hardware model: k in `parts`
    contiguous ranges of whole operand stages (part p: stages
    [p nop / S, (p + 1) nop / S), as tcec_gemm_pers_kernel<kSplitK> walks
    them), each part's main-term sum and raw dC from the hardware model, then
    tcec_splitk_reduce_kernel's fixed-order combine: c = RN(..RN(c_0 + c_1)..),
    d likewise, C = RN(c + d 2^-s).  Returns (C float32, flags int)."""
    fmt, s, rm = VARIANTS[variant]
    d = drain_k or DEFAULT_DRAIN_K[variant]
    de = d // MMA_K[variant]
    stage = 64 if fmt == FMT_FP16 else 32
    k = a.shape[1]
    nop = -(-k // stage)
    parts = min(parts, nop)
    c = dc = None
    flags = 0
    for p in range(parts):
        k0 = min(k, p * nop // parts * stage)
        k1 = min(k, (p + 1) * nop // parts * stage)
        cp, f1 = _hw(5, a[:, k0:k1], b[k0:k1], fmt, s, rm, de, nthreads)
        dp, _ = _hw(6, a[:, k0:k1], b[k0:k1], fmt, s, rm, de, nthreads)
        flags |= f1
        c = cp if c is None else (c + cp).astype(np.float32)
        dc = dp if dc is None else (dc + dp).astype(np.float32)
    with np.errstate(all="ignore"):
        # RN(c + dC 2^-s): the float64 sum is exact or far below FP32's half-ulp
        out = (c.astype(np.float64) + dc.astype(np.float64) * 2.0 ** -s).astype(np.float32)
    if not np.all(np.isfinite(out)):
        flags |= FLAG_OVERFLOW
    return out, flags


def inunit_hw(a, b, scheme: str, block_k: int = 16, nthreads: int = 0):
    """The GPU kernels' in-unit comparator schedules with the hardware MMA model
    (tcec_oracle_hw): tc_plain_fp16 / tc_plain_tf32, markidis4 / markidis4_tf32
    / corrected4_rz (one accumulator), corrected4_rn / corrected4_rn_tf32 (a
    block of block_k per product, RN folds).  Returns (C float32, flags int)."""
    kinds = {"tc_plain_fp16": (2, FMT_FP16, RM_RN), "tc_plain_tf32": (2, FMT_TF32, RM_RNA),
             "markidis4": (3, FMT_FP16, RM_RN), "markidis4_tf32": (3, FMT_TF32, RM_RNA),
             "corrected4_rz": (3, FMT_FP16, RM_RN), "corrected4_rn": (4, FMT_FP16, RM_RN),
             "corrected4_rn_tf32": (4, FMT_TF32, RM_RNA)}
    sched, fmt, rm = kinds[scheme]
    kstep = 16 if fmt == FMT_FP16 else 8
    if block_k % kstep:
        raise ValueError("block_k must be a multiple of the MMA k-step")
    return _hw(sched, a, b, fmt, 0, rm, block_k // kstep, nthreads)


def inunit(a, b, scheme: str, block_k: int = 16, acc_bits: int = 25):
    """schemes.py:gemm for the in-unit comparators restated (tcec_oracle_inunit):
    scheme in tc_plain_fp16, tc_plain_tf32, markidis4, markidis4_tf32,
    corrected4_rn, corrected4_rz, corrected4_rn_tf32 (RN terminal, TF32 split).  Returns (C float32, flags int)."""
    kinds = {"tc_plain_fp16": (0, 0, 0, 0, 2), "tc_plain_tf32": (0, 1, 0, 1, 2),
             "markidis4": (1, 0, 0, 0, 2), "markidis4_tf32": (1, 1, 0, 1, 2),
             "corrected4_rn": (1, 0, 0, 0, 0), "corrected4_rz": (1, 0, 0, 0, 2),
             "corrected4_rn_tf32": (1, 1, 0, 1, 0)}
    kind, fmt, s, rm, term = kinds[scheme]
    a = np.ascontiguousarray(a, dtype=np.float32)
    b = np.ascontiguousarray(b, dtype=np.float32)
    m, k = a.shape
    k2, n = b.shape
    if k2 != k:
        raise ValueError(f"inner dimensions differ: {k} vs {k2}")
    c = np.empty((m, n), np.float32)
    flags = ctypes.c_uint32(0)
    rc = lib().tcec_oracle_inunit(kind, fmt, s, rm, term, m, n, k, _ptr(a), k, _ptr(b), n,
                                  _ptr(c), n, block_k, acc_bits, ctypes.byref(flags))
    if rc != 0:
        raise ValueError(f"oracle rejected arguments (rc={rc})")
    return c, int(flags.value)


def fp32_simt(a, b, block_k: int = 16) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.float32)
    b = np.ascontiguousarray(b, dtype=np.float32)
    m, k = a.shape
    n = b.shape[1]
    c = np.empty((m, n), np.float32)
    lib().tcec_oracle_fp32_simt(m, n, k, _ptr(a), k, _ptr(b), n, _ptr(c), n, block_k)
    return c


def fp64_ref(a, b) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.float32)
    b = np.ascontiguousarray(b, dtype=np.float32)
    m, k = a.shape
    n = b.shape[1]
    c = np.empty((m, n), np.float64)
    lib().tcec_oracle_fp64_ref(m, n, k, _ptr(a), k, _ptr(b), n, _ptr(c), n)
    return c


def relative_residual(c_test, c_ref) -> float:
    """analysis.py:175-192 (Eq. 7): ||ref - test||_F / ||ref||_F in float64."""
    test = np.asarray(c_test, dtype=np.float64)
    ref = np.asarray(c_ref, dtype=np.float64)
    if test.shape != ref.shape:
        raise ValueError("shapes differ")
    num = float(np.linalg.norm(ref - test))
    den = float(np.linalg.norm(ref))
    if den == 0.0:
        if num == 0.0:
            return 0.0
        raise ValueError("zero reference norm with nonzero residual")
    return num / den


# ---- input generators: genmat.py restated (Philox, counter based) ---------

_SEED_MIX = 0x9E3779B97F4A7C15


def pair_seed(seed: int) -> int:
    """genmat.py:22-24."""
    return (int(seed) + _SEED_MIX) % (1 << 64)


def _rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.Philox(key=np.uint64(seed % (1 << 64))))


def urand(rows: int, cols: int, lo: float, hi: float, seed: int) -> np.ndarray:
    """genmat.py:75-82 (Urand on the open interval)."""
    rng = _rng(seed)
    u = rng.random((rows, cols))
    vals = (lo + u * (hi - lo)).astype(np.float32)
    vals = np.where(vals <= lo, np.nextafter(np.float32(lo), np.float32(hi)), vals)
    vals = np.where(vals >= hi, np.nextafter(np.float32(hi), np.float32(lo)), vals)
    return vals.astype(np.float32)


def exprand(rows: int, cols: int, a: int, b: int, seed: int) -> np.ndarray:
    """genmat.py:83-89 (ExpRand, Eq. 25)."""
    rng = _rng(seed)
    shape = (rows, cols)
    e = rng.integers(a, b + 1, size=shape)
    mant = rng.integers(0, 1 << 23, size=shape)
    s = rng.integers(0, 2, size=shape)
    m = 1.0 + np.ldexp(mant.astype(np.float64), -23)
    vals = (2.0 * s - 1.0) * np.ldexp(m, e)
    return vals.astype(np.float32)


_BANDS = {"high": (-15, 14), "low": (-35, -15), "out": (-100, -35)}


def type_pair(type_id: int, m: int, n: int, k: int, seed: int):
    """genmat.py:100-121 (Types 1-4, list variant of Type 2)."""
    da, db = {1: ("high", "high"), 2: ("high", "out"), 3: ("low", "low"),
              4: ("out", "out")}[type_id]
    a = exprand(m, k, *_BANDS[da], seed)
    b = exprand(k, n, *_BANDS[db], pair_seed(seed))
    return a, b
