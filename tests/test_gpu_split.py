"""GPU split kernel vs the reference split, bit for bit.

The GPU split runs the same device functions as the fused GEMM's split warps
(csrc/split.cuh).  Checked against the reference's own outputs (golden
fixtures made by importing the reference, tests/golden/make_golden.py) and
against the CPU oracle on random bit patterns and the edge set."""

import os

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden")

MODES = [  # (golden name, scheme factory args, oracle variant, oracle rounding)
    ("fp16_rn", ("scaled_halfhalf", "rn"), "fp16", O.RM_RN),
    ("fp16_rz", ("scaled_halfhalf", "rz"), "fp16", O.RM_RZ),
    ("tf32_rna", ("tf32tf32", "rna"), "tf32", O.RM_RNA),
    ("tf32_rn", ("tf32tf32", "rn"), "tf32", O.RM_RN),
    ("tf32_rz", ("tf32tf32", "rz"), "tf32", O.RM_RZ),
]


def _scheme(kind, rnd):
    import paper_2203_03341_b200 as T

    return {"scaled_halfhalf": T.scaled_halfhalf, "tf32tf32": T.tf32tf32,
            "markidis_halfhalf": T.markidis_halfhalf}[kind](T.RoundingMode(rnd))


def _gpu_split(x, scheme):
    import torch

    import paper_2203_03341_b200 as T

    xt = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).cuda()
    fl = torch.zeros(1, dtype=torch.int32, device="cuda")
    hi, lo = T.split_device(xt, scheme, fl)
    return (hi.cpu().numpy().astype(np.float64), lo.cpu().numpy().astype(np.float64),
            int(fl.item()))


def _bits_equal(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    assert a.shape == b.shape
    assert np.array_equal(np.isnan(a), np.isnan(b))
    m = ~np.isnan(a)
    bad = np.nonzero(a[m].view(np.uint64) != b[m].view(np.uint64))[0]
    assert bad.size == 0, (bad[:5], a[m][bad[:5]], b[m][bad[:5]])


@pytest.mark.parametrize("gname,sargs,variant,rm", MODES)
def test_split_matches_reference_goldens(gname, sargs, variant, rm):
    g = np.load(os.path.join(GOLD, "split_golden.npz"))
    x = g["x"]
    hi, lo, fl = _gpu_split(x, _scheme(*sargs))
    _bits_equal(hi, g[gname + "_hi"])
    _bits_equal(lo, g[gname + "_lo"])
    cls = g[gname + "_class"]
    ovf = bool(np.any(np.isinf(g[gname + "_hi"])))
    assert bool(fl & 2) == bool(np.any(cls == 2)), gname
    assert bool(fl & 1) == ovf, gname


@pytest.mark.parametrize("gname,sargs,variant,rm", MODES)
def test_split_random_bit_patterns_vs_oracle(gname, sargs, variant, rm):
    rng = np.random.default_rng(7)
    bits = rng.integers(0, 1 << 32, size=1 << 21, dtype=np.uint64).astype(np.uint32)
    x = bits.view(np.float32)
    x = x[np.isfinite(x)]
    hi, lo, _ = _gpu_split(x, _scheme(*sargs))
    ohi, olo = O.split(x, variant, rm)
    _bits_equal(hi, ohi)
    _bits_equal(lo, olo)


def test_split_unscaled_fp16_vs_oracle():
    rng = np.random.default_rng(8)
    x = np.concatenate([rng.uniform(-1, 1, 1 << 18).astype(np.float32),
                        O.exprand(1, 1 << 18, -40, 17, 3).ravel()])
    hi, lo, fl = _gpu_split(x, _scheme("markidis_halfhalf", "rn"))
    ohi, olo = O.split(x, "fp16u")
    _bits_equal(hi, ohi)
    _bits_equal(lo, olo)
    cls = O.classify(x, "fp16u")
    assert bool(fl & 2) == bool(np.any(cls == 2))


def test_split_flags_per_band():
    """classify_array bands (splitting.py:187-215) on single-value inputs."""
    T_FP16 = _scheme("scaled_halfhalf", "rn")
    T_TF32 = _scheme("tf32tf32", "rna")
    cases = [  # value, fp16 flags, tf32 flags
        (0.0, 0, 0), (1.0, 0, 0), (2.0 ** -34, 0, 0), (2.0 ** -35, 2, 0),
        (np.float32(2.0 ** -35 * 1.999), 2, 0), (65504.0, 0, 0), (65519.0, 0, 0),
        (65520.0, 1, 0), (65535.0, 1, 0), (65536.0, 3, 0), (2.0 ** -126, 2, 0),
        (2.0 ** -127, 2, 2), (2.0 ** -149, 2, 2), (3.4028235e38, 3, 1),
        (np.float32(3.3e38), 3, 0),
    ]
    for v, f16, f32 in cases:
        x = np.array([v, 0.5], np.float32)
        assert _gpu_split(x, T_FP16)[2] == f16, (v, "fp16")
        assert _gpu_split(x, T_TF32)[2] == f32, (v, "tf32")


def test_split_nonfinite_input_flag():
    for v in (np.inf, -np.inf, np.nan):
        x = np.array([1.0, v, 2.0], np.float32)
        assert _gpu_split(x, _scheme("scaled_halfhalf", "rn"))[2] & 4
        assert _gpu_split(x, _scheme("tf32tf32", "rna"))[2] & 4


@pytest.mark.slow
@pytest.mark.parametrize("variant", ["fp16", "tf32"])
def test_split_exhaustive_all_fp32(variant):
    """All 2^32 bit patterns (finite ones), default rounding, vs the oracle.
    Chunked; the oracle runs on all host threads (ctypes releases the GIL)."""
    import concurrent.futures as cf

    import torch

    import paper_2203_03341_b200 as T

    scheme = T.scaled_halfhalf() if variant == "fp16" else T.tf32tf32()
    chunk = 1 << 26
    sub = chunk // (os.cpu_count() or 1)
    pool = cf.ThreadPoolExecutor(max_workers=os.cpu_count() or 1)

    def oracle_part(xp):
        return O.split(xp, variant)

    for start in range(0, 1 << 32, chunk):
        bits = torch.arange(start, start + chunk, dtype=torch.int64, device="cuda")
        x = bits.to(torch.int32).view(torch.float32)
        hi, lo = T.split_device(x, scheme)
        xh = x.cpu().numpy()
        fin = np.isfinite(xh)
        hh = hi.cpu().numpy().astype(np.float64)[fin]
        ll = lo.cpu().numpy().astype(np.float64)[fin]
        xf = xh[fin]
        parts = [xf[i:i + sub] for i in range(0, xf.size, sub)]
        res = list(pool.map(oracle_part, parts))
        ohi = np.concatenate([r[0] for r in res])
        olo = np.concatenate([r[1] for r in res])
        _bits_equal(hh, ohi)
        _bits_equal(ll, olo)
