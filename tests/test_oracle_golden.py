"""Pin the CPU oracle (test infrastructure) to the reference, bit for bit.

The fixtures in tests/golden/ were produced by importing the reference package
(tests/golden/make_golden.py); here the C restatement must reproduce every one
of them exactly.  No GPU needed.
"""

import os

import numpy as np
import pytest

from oracle import oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def split_gold():
    return np.load(os.path.join(GOLD, "split_golden.npz"))


@pytest.fixture(scope="module")
def gemm_gold():
    return np.load(os.path.join(GOLD, "gemm_golden.npz"))


def _same(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    assert a.shape == b.shape
    # bit-exact including signed zeros and NaN positions
    assert np.array_equal(np.isnan(a), np.isnan(b))
    m = ~np.isnan(a)
    assert np.array_equal(a[m].view(np.uint64), b[m].view(np.uint64))


@pytest.mark.parametrize("name,variant,rm", [
    ("fp16_rn", "fp16", O.RM_RN), ("fp16_rz", "fp16", O.RM_RZ),
    ("tf32_rna", "tf32", O.RM_RNA), ("tf32_rn", "tf32", O.RM_RN), ("tf32_rz", "tf32", O.RM_RZ),
])
def test_split_matches_reference(split_gold, name, variant, rm):
    x = split_gold["x"]
    hi, lo = O.split(x, variant, rm)
    _same(hi, split_gold[name + "_hi"])
    _same(lo, split_gold[name + "_lo"])
    assert np.array_equal(O.classify(x, variant), split_gold[name + "_class"])


@pytest.mark.parametrize("fmt", ["fp16", "tf32", "fp32"])
@pytest.mark.parametrize("mode", ["rn", "rna", "rz"])
def test_round_to_format_matches_reference(split_gold, fmt, mode):
    f = {"fp16": O.FMT_FP16, "tf32": O.FMT_TF32, "fp32": O.FMT_FP32}[fmt]
    m = {"rn": O.RM_RN, "rna": O.RM_RNA, "rz": O.RM_RZ}[mode]
    _same(O.round_to_format(split_gold["round_x"], f, m), split_gold[f"round_{fmt}_{mode}"])


def test_eq10_worked_example():
    # SPEC.md:136-137 / PAPER Eq. 10: 0x3F801003 under RN -> hi = 1 + 2^-10,
    # (scaled) lo = -4092 * 2^-23 * 2^11
    x = np.array([0x3F801003], np.uint32).view(np.float32)
    hi, lo = O.split(x, "fp16", O.RM_RN)
    assert hi[0] == 1.0 + 2.0 ** -10
    assert lo[0] == -4092 * 2.0 ** -23 * 2.0 ** 11
    hi, lo = O.split(x, "fp16", O.RM_RZ)
    assert hi[0] == 1.0 and lo[0] == 2.0 ** -11 * 2.0 ** 11


def _cases(g):
    return [str(n) for n in g["names"]]


def test_gemm_corrected3_matches_reference(gemm_gold):
    for tag in _cases(gemm_gold):
        a, b = gemm_gold[f"{tag}__A"], gemm_gold[f"{tag}__B"]
        for sname, variant in (("corrected3_halfhalf", "fp16"), ("corrected3_tf32", "tf32")):
            c, flags = O.corrected3(a, b, variant)
            _same(c, gemm_gold[f"{tag}__{sname}__C"])
            ov, oor = gemm_gold[f"{tag}__{sname}__flags"]
            assert bool(flags & O.FLAG_OVERFLOW) == bool(ov), (tag, sname)
            assert bool(flags & O.FLAG_OUT_OF_RANGE) == bool(oor), (tag, sname)


def test_gemm_baselines_match_reference(gemm_gold):
    for tag in _cases(gemm_gold):
        a, b = gemm_gold[f"{tag}__A"], gemm_gold[f"{tag}__B"]
        _same(O.fp32_simt(a, b), gemm_gold[f"{tag}__fp32_simt__C"])
        _same(O.fp64_ref(a, b), gemm_gold[f"{tag}__fp64_ref__C"])


def test_drain_interval_restatement(gemm_gold):
    a, b = gemm_gold["drain__A"], gemm_gold["drain__B"]
    for variant, bk in (("fp16", 16), ("tf32", 8)):
        for d in (bk, 64, 128):
            c, _ = O.corrected3(a, b, variant, block_k=bk, drain_k=d)
            _same(c, gemm_gold[f"drain__{variant}__bk{bk}__d{d}"])


def test_four_term_sibling(gemm_gold):
    a, b = gemm_gold["dd__A"], gemm_gold["dd__B"]
    c3, _ = O.corrected3(a, b, "fp16")
    c4, _ = O.corrected3(a, b, "fp16", include_dd=True)
    _same(c3, gemm_gold["dd__C3"])
    _same(c4, gemm_gold["dd__C4"])


def test_identity_gives_b(gemm_gold):
    b = gemm_gold["identity_16__B"]
    for v in ("fp16", "tf32"):
        c, flags = O.corrected3(np.eye(16, dtype=np.float32), b, v)
        assert np.array_equal(c, b) and flags == 0


def test_threads_do_not_change_bits():
    a = O.urand(37, 300, -1, 1, 4)
    b = O.urand(300, 19, -1, 1, O.pair_seed(4))
    c1, _ = O.corrected3(a, b, "fp16", nthreads=1)
    c8, _ = O.corrected3(a, b, "fp16", nthreads=8)
    assert np.array_equal(c1, c8)


def test_row_column_separable():
    # gemm(A[r], B[:, c]) == gemm(A, B)[r, c] bit-exactly
    a = O.urand(24, 160, -1, 1, 8)
    b = O.urand(160, 20, -1, 1, O.pair_seed(8))
    c, _ = O.corrected3(a, b, "tf32")
    cs, _ = O.corrected3(a[5:11], b[:, 3:17], "tf32")
    assert np.array_equal(cs, c[5:11, 3:17])


def test_generators_match_reference():
    g = np.load(os.path.join(GOLD, "genmat_golden.npz"))
    assert np.array_equal(O.urand(4, 5, -1, 1, 0), g["urand_s0"])
    assert np.array_equal(O.urand(5, 3, -1, 1, O.pair_seed(0)), g["urand_pair_s0"])
    assert np.array_equal(O.exprand(6, 4, -15, 14, 3), g["exprand_s3"])
    for t in (1, 2, 3, 4):
        a, b = O.type_pair(t, 3, 4, 5, 9)
        assert np.array_equal(a, g[f"type{t}_A"]) and np.array_equal(b, g[f"type{t}_B"])


def test_inunit_comparators_match_reference_goldens():
    """oracle.inunit (tc_plain, markidis4, corrected4 RN/RZ; schemes.py:343-364)
    equals the reference's gemm bit for bit, flags included."""
    g = np.load(os.path.join(GOLD, "inunit_golden.npz"))
    for tag in g["names"]:
        a, b = g[f"{tag}__A"], g[f"{tag}__B"]
        for sname in g["schemes"]:
            c, fl = O.inunit(a, b, str(sname))
            _same(c, g[f"{tag}__{sname}__C"])
            ov, oor = g[f"{tag}__{sname}__flags"]
            assert (bool(fl & 1), bool(fl & 2)) == (bool(ov), bool(oor)), (tag, sname, fl)


# ---------------------------------------------------------------------------
# The oracle's HARDWARE model (tcec_oracle_hw) against outputs recorded on the
# B200: tests/golden/hw_probe_golden.npz (tests/golden/make_hw_fixture.py, from
# scripts/probe_accumulator.py).  tc_plain datasets are raw tensor-core
# accumulations (one instruction and chains, crafted / random / subnormal /
# overflowing / non-finite operands); c3* datasets are the corrected3
# kernels' outputs at the default and the reference's drain intervals.


@pytest.fixture(scope="module")
def hw_gold():
    return np.load(os.path.join(GOLD, "hw_probe_golden.npz"))


def _hw_cases(g):
    return sorted({k.split("__")[0] for k in g.files})


def test_hw_model_reproduces_tensor_core_outputs(hw_gold):
    n = 0
    for nm in _hw_cases(hw_gold):
        a, b, c = hw_gold[nm + "__A"], hw_gold[nm + "__B"], hw_gold[nm + "__C"]
        if nm.startswith("c3"):
            continue
        scheme = "tc_plain_fp16" if nm.startswith("f16") else "tc_plain_tf32"
        oc, _ = O.inunit_hw(a, b, scheme)
        _same(oc, c)
        n += c.size
    assert n > 15000


def test_hw_model_reproduces_corrected3_kernel_outputs(hw_gold):
    for nm in _hw_cases(hw_gold):
        if not nm.startswith("c3"):
            continue
        variant = "fp16" if nm.startswith("c3f16") else "tf32"
        drain = int(nm.split("_d")[1]) if "_d" in nm else 0
        oc, _ = O.corrected3_hw(hw_gold[nm + "__A"], hw_gold[nm + "__B"], variant,
                                drain_k=drain or None)
        _same(oc, hw_gold[nm + "__C"])


def test_hw_model_nonfinite_outputs_match_reference(gemm_gold):
    """Where the reference's output is non-finite (hi overflow), the hardware
    model gives the same value: +-inf with the same sign, or NaN."""
    seen = 0
    for tag in _cases(gemm_gold):
        a, b = gemm_gold[f"{tag}__A"], gemm_gold[f"{tag}__B"]
        for sname, variant in (("corrected3_halfhalf", "fp16"), ("corrected3_tf32", "tf32")):
            ref = gemm_gold[f"{tag}__{sname}__C"]
            bad = ~np.isfinite(ref)
            if not bad.any():
                continue
            oc, fl = O.corrected3_hw(a, b, variant)
            _same(oc[bad], ref[bad])
            assert np.array_equal(np.isfinite(oc), ~bad)
            ov, oor = gemm_gold[f"{tag}__{sname}__flags"]
            assert (bool(fl & 1), bool(fl & 2)) == (bool(ov), bool(oor))
            seen += int(bad.sum())
    assert seen > 0
