"""Input generators (product restatement of genmat.py) against the reference's
own outputs, and the accuracy harness CLI (CPU parts + one GPU run)."""

import os

import numpy as np
import pytest

from paper_2203_03341_b200 import accuracy as ACC
from paper_2203_03341_b200 import genmat as G

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_generators_match_reference_fixtures():
    g = np.load(os.path.join(GOLD, "genmat_golden.npz"))
    assert np.array_equal(G.generate(G.MatrixSpec(4, 5, G.Urand(-1, 1), 0)), g["urand_s0"])
    assert np.array_equal(G.generate(G.MatrixSpec(5, 3, G.Urand(-1, 1), G.pair_seed(0))),
                          g["urand_pair_s0"])
    assert np.array_equal(G.generate(G.MatrixSpec(6, 4, G.ExpRand(-15, 14), 3)), g["exprand_s3"])
    for t in (1, 2, 3, 4):
        a, b = G.type_pair(t, 3, 4, 5, 9)
        assert np.array_equal(a, g[f"type{t}_A"]) and np.array_equal(b, g[f"type{t}_B"])


def test_generators_match_reference_gemm_inputs():
    """The GEMM goldens were drawn by the reference's generate(): same bits here."""
    g = np.load(os.path.join(GOLD, "gemm_golden.npz"))
    a = G.generate(G.MatrixSpec(16, 1024, G.Urand(-1, 1), 0))
    b = G.generate(G.MatrixSpec(1024, 16, G.Urand(-1, 1), G.pair_seed(0)))
    assert np.array_equal(a, g["urand_s0_16x16x1024__A"])
    assert np.array_equal(b, g["urand_s0_16x16x1024__B"])


def test_spec_validation():
    with pytest.raises(ValueError):
        G.Urand(1, 1)
    with pytest.raises(ValueError):
        G.ExpRand(3, 2)
    with pytest.raises(ValueError):
        G.MatrixSpec(0, 3, G.Urand(0, 1), 1)
    with pytest.raises(ValueError):
        G.type_pair(5, 2, 2, 2, 0)


def test_parse_dist_and_cli_errors(capsys):
    assert ACC.parse_dist("urand:-1,1") == G.Urand(-1.0, 1.0)
    assert ACC.parse_dist("exprand:-15,14") == G.ExpRand(-15, 14)
    assert ACC.parse_dist("type:3") == ("type", 3)
    for bad in ("urand:1", "type:7", "gauss:0,1"):
        with pytest.raises(ValueError):
            ACC.parse_dist(bad)
    assert ACC.main(["gemm-accuracy", "--scheme", "fp32_simt"]) == 1
    assert "error:" in capsys.readouterr().err


@pytest.mark.gpu
def test_gemm_accuracy_csv_on_gpu(tmp_path):
    out = tmp_path / "acc.csv"
    rc = ACC.main(["--out", str(out), "gemm-accuracy", "--m", "16", "--n", "16", "--k", "1024",
                   "--seeds", "0,1,2,3", "--scheme",
                   "corrected3_halfhalf,corrected3_tf32,cublas_sgemm"])
    assert rc == 0
    lines = out.read_text().strip().splitlines()
    assert lines[0] == "m,n,k,scheme,seed,residual,flags"
    avg = {ln.split(",")[3]: float(ln.split(",")[5]) for ln in lines if ",avg," in ln}
    assert set(avg) == {"corrected3_halfhalf", "corrected3_tf32", "cublas_sgemm"}
    for name in ("corrected3_halfhalf", "corrected3_tf32"):
        assert avg[name] < 4e-7
    rc = ACC.main(["--out", str(out), "gemm-accuracy", "--k", "256", "--seeds", "0",
                   "--scheme", "corrected3_halfhalf", "--dist", "type:4"])
    assert rc == 0
    assert "out_of_range" in out.read_text()


def test_ablation_cli_rejects_type_distributions(capsys):
    assert ACC.main(["ablate-delta", "--dist", "type:2"]) == 1
    assert ACC.main(["rounding-ablation", "--dist", "type:2"]) == 1
    assert "error:" in capsys.readouterr().err


@pytest.mark.gpu
def test_ablation_csvs_on_gpu(tmp_path):
    """The paper's two ablations on the tensor core (cli.py:173-214 analogues)."""
    out = tmp_path / "abl.csv"
    assert ACC.main(["--out", str(out), "ablate-delta", "--k", "16,1024", "--seeds", "0,1"]) == 0
    lines = out.read_text().strip().splitlines()
    assert lines[0] == "m,n,k,seed,residual_3term,residual_4term,max_ulp_diff"
    for ln in lines[1:]:
        r3, r4 = (float(x) for x in ln.split(",")[4:6])
        assert r3 < 1e-6 and r4 < 1e-6 and abs(r3 - r4) <= 0.1 * r4
    assert ACC.main(["--out", str(out), "rounding-ablation", "--k", "4096", "--seeds", "0,1"]) == 0
    lines = out.read_text().strip().splitlines()
    assert lines[0] == "m,n,k,seed,residual_inunit_hw,residual_corrected3,residual_fp32"
    for ln in lines[1:]:
        r_in, r3, _ = (float(x) for x in ln.split(",")[4:7])
        assert r_in > 2 * r3
    rc = ACC.main(["--out", str(out), "gemm-accuracy", "--k", "1024", "--seeds", "0,1",
                   "--scheme", "tc_plain_fp16,tc_plain_tf32,markidis4,corrected4_rz"])
    assert rc == 0
    avg = {ln.split(",")[3]: float(ln.split(",")[5])
           for ln in out.read_text().splitlines() if ",avg," in ln}
    assert avg["tc_plain_fp16"] > 1e-4 and avg["markidis4"] < 1e-4


def test_underflow_closed_forms_match_reference_values():
    """analysis.py closed forms restated (P_u+gu(0) = 1/16,
    P_u(0) = 0, P_u(-1) = 1/8192)."""
    from fractions import Fraction

    from paper_2203_03341_b200 import analysis as AN

    assert AN.gradual_underflow_probability(0) == Fraction(1, 16)
    assert AN.underflow_probability(0) == 0
    assert AN.underflow_probability(-1) == Fraction(1, 8192)
    assert sum(AN.zero_run_probability(n) for n in range(14)) == 1
    assert ACC._dyadic_decimal(Fraction(91, 4)) == "22.75"


@pytest.mark.gpu
def test_split_stats_and_underflow_on_gpu():
    """GPU enumeration of all 2^23 mantissas equals the reference's
    exhaustive_length_distribution (tests/golden/split_stats_golden.json, made by
    the reference) for RN / RNA / RZ, and the exhaustive RZ underflow rates equal
    the closed forms exactly (the closed forms assume uniform mantissa bits,
    which the enumeration realises)."""
    import json
    import os
    from fractions import Fraction

    from paper_2203_03341_b200 import analysis as AN

    gold = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "split_stats_golden.json")))
    for r, dist in gold.items():
        got = AN.exhaustive_length_distribution(r).probabilities
        assert got == {int(k): Fraction(n, d) for k, (n, d) in dist.items()}, r
    for e_v in range(-30, 15):
        assert AN.exhaustive_underflow(e_v) == (AN.underflow_probability(e_v),
                                               AN.gradual_underflow_probability(e_v)), e_v
    lines = ACC.split_stats("rz")
    assert lines[-1] == "expectation,22.25"
