"""CPU checks of the C ABI boundary: the library builds, loads, exports every
symbol include/tcec.h declares, and rejects bad arguments before touching the
GPU.  No compute calls are made here."""

import ctypes
import os
import re

import pytest

from paper_2203_03341_b200 import _native as N

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "tcec.h")


@pytest.fixture(scope="module")
def lib():
    N.build()
    return N.lib()


def _declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\s*\**\s*(tcec_\w+)\s*\(", text, flags=re.M)))


def test_header_declares_expected_entry_points():
    assert _declared_functions() == sorted(N.EXPORTS)


def test_library_exports_every_declared_symbol(lib):
    for name in _declared_functions():
        assert hasattr(lib, name), name
        assert ctypes.cast(getattr(lib, name), ctypes.c_void_p).value


def test_version_and_status_strings(lib):
    assert lib.tcec_version() == 100
    for code in (N.OK, N.ERR_ARG, N.ERR_ALIGN, N.ERR_UNSUPPORTED, N.ERR_CUDA, N.ERR_ARCH):
        assert lib.tcec_status_str(code).decode()
    assert lib.tcec_status_str(12345).decode() == "unknown status"


def test_opts_struct_matches_header():
    """The ctypes mirror lists exactly the header's tcec_opts fields, in order."""
    hdr = open(HEADER).read()
    body = hdr.split("typedef struct tcec_opts {")[1].split("} tcec_opts;")[0]
    body = re.sub(r"/\*.*?\*/", "", body, flags=re.S)
    fields = re.findall(r"int32_t\s+(\w+)(?:\[(\d+)\])?;", body)
    assert [(name, int(cnt or 1)) for name, cnt in fields] == \
        [(name, getattr(typ, "_length_", 1)) for name, typ in N.TcecOpts._fields_]
    assert ctypes.sizeof(N.TcecOpts) == 4 * sum(int(cnt or 1) for _, cnt in fields)


def test_argument_validation_without_gpu(lib):
    f = lib.tcec_sgemm
    # unknown variant / negative sizes / short leading dimensions: rejected before any CUDA call
    assert f(7, 4, 4, 4, None, 4, None, 4, None, 4, None, None, None) == N.ERR_ARG
    assert f(0, -1, 4, 4, None, 4, None, 4, None, 4, None, None, None) == N.ERR_ARG
    assert f(0, 4, 4, 8, None, 4, None, 4, None, 4, None, None, None) == N.ERR_ARG
    assert f(0, 4, 8, 4, None, 4, None, 4, None, 4, None, None, None) == N.ERR_ARG
    # empty output: no-op success
    assert f(0, 0, 4, 4, None, 4, None, 4, None, 4, None, None, None) == N.OK
    assert f(1, 4, 0, 4, None, 4, None, 4, None, 4, None, None, None) == N.OK
    # unsupported option combinations
    o = N.make_opts(split_rounding=N.ROUND_RN, scale_log2=5)
    assert f(0, 4, 4, 4, None, 4, None, 4, None, 4, ctypes.byref(o), None, None) == N.ERR_UNSUPPORTED
    # drain intervals are whole MMA k-steps (16 FP16, 8 TF32)
    o = N.make_opts(drain_k=40)
    assert f(0, 4, 4, 4, None, 4, None, 4, None, 4, ctypes.byref(o), None, None) == N.ERR_UNSUPPORTED
    o = N.make_opts(drain_k=12)
    assert f(1, 4, 4, 4, None, 4, None, 4, None, 4, ctypes.byref(o), None, None) == N.ERR_UNSUPPORTED
    o = N.make_opts(drain_k=-16)
    assert f(0, 4, 4, 4, None, 4, None, 4, None, 4, ctypes.byref(o), None, None) == N.ERR_UNSUPPORTED
    # the narrow tiles drain whole operand stages; the single-CTA kernel is block_n 128 only
    o = N.make_opts(drain_k=16, block_n=192)
    assert f(0, 4, 4, 4, None, 4, None, 4, None, 4, ctypes.byref(o), None, None) == N.ERR_UNSUPPORTED
    o = N.make_opts(drain_k=16, block_n=64)
    assert f(0, 4, 4, 4, None, 4, None, 4, None, 4, ctypes.byref(o), None, None) == N.ERR_UNSUPPORTED
    o = N.make_opts(kernel_variant=1)
    assert f(0, 4, 4, 4, None, 4, None, 4, None, 4, ctypes.byref(o), None, None) == N.ERR_UNSUPPORTED
    # tile widths are 64 / 128 / 192 / 256 (0 = automatic)
    for bn in (32, 96, 320):
        o = N.make_opts(block_n=bn)
        assert f(0, 4, 4, 4, None, 4, None, 4, None, 4, ctypes.byref(o), None, None) == N.ERR_UNSUPPORTED
    o = N.make_opts(scale_log2=11)
    assert f(1, 4, 4, 4, None, 4, None, 4, None, 4, ctypes.byref(o), None, None) == N.ERR_UNSUPPORTED
    # corrected4_rn blocks are whole MMA k-steps; split_k in 0..64; kernel variants 0..4
    o = N.make_opts(scheme=4, drain_k=24)
    assert f(0, 4, 4, 4, None, 4, None, 4, None, 4, ctypes.byref(o), None, None) == N.ERR_UNSUPPORTED
    o = N.make_opts(scheme=4, drain_k=12)
    assert f(1, 4, 4, 4, None, 4, None, 4, None, 4, ctypes.byref(o), None, None) == N.ERR_UNSUPPORTED
    o = N.make_opts(split_k=-2)
    assert f(0, 4, 4, 4, None, 4, None, 4, None, 4, ctypes.byref(o), None, None) == N.ERR_UNSUPPORTED
    o = N.make_opts(split_k=65)
    assert f(0, 4, 4, 4, None, 4, None, 4, None, 4, ctypes.byref(o), None, None) == N.ERR_UNSUPPORTED
    o = N.make_opts(kernel_variant=5)
    assert f(0, 4, 4, 4, None, 4, None, 4, None, 4, ctypes.byref(o), None, None) == N.ERR_UNSUPPORTED
    o = N.make_opts(scheme=5)
    assert f(0, 4, 4, 4, None, 4, None, 4, None, 4, ctypes.byref(o), None, None) == N.ERR_UNSUPPORTED
    s = lib.tcec_split
    assert s(3, -1, -1, None, 4, None, None, None, None) == N.ERR_ARG
    assert s(0, -1, -1, None, -4, None, None, None, None) == N.ERR_ARG
    assert s(0, -1, -1, None, 0, None, None, None, None) == N.OK
    assert s(0, N.ROUND_RNA, -1, None, 4, None, None, None, None) == N.ERR_UNSUPPORTED


def test_sass_contains_tcgen05_and_tma():
    """The built library carries tcgen05 MMA (UTC*MMA), TMEM loads (LDTM) and
    TMA (UTMALDG/UTMASTG) -- the Blackwell-native path, not legacy HMMA."""
    import shutil
    import subprocess

    if shutil.which("cuobjdump") is None:
        pytest.skip("cuobjdump not available")
    N.build()
    out = subprocess.run(["cuobjdump", "-sass", N.LIB_PATH], capture_output=True, text=True,
                         check=True).stdout
    for mnem in ("UTCHMMA", "LDTM", "UTMALDG", "UTMASTG"):
        assert mnem in out, mnem
    assert re.search(r"\bHMMA\b", out) is None


def test_integration_stub_opts_match_header():
    """The ctypes stub INTEGRATION.md gives a reference maintainer declares the
    same tcec_opts fields as include/tcec.h (the C side reads the whole struct)."""
    doc = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    stub = doc.split("class _Opts(ctypes.Structure):")[1].split("]\n")[0]
    names = re.findall(r'\("(\w+)", ctypes\.c_int32(?: \* (\d+))?\)', stub)
    hdr = open(HEADER).read()
    body = re.sub(r"/\*.*?\*/", "", hdr.split("typedef struct tcec_opts {")[1].split("} tcec_opts;")[0],
                  flags=re.S)
    fields = re.findall(r"int32_t\s+(\w+)(?:\[(\d+)\])?;", body)
    assert [(n, c or "1") for n, c in names] == [(n, c or "1") for n, c in fields]


def test_torch_op_registered_with_fake_impl():
    """torch.ops.tcec.sgemm is registered; its fake implementation traces shapes
    on meta tensors (no GPU needed), and CPU tensors are refused."""
    import torch

    import paper_2203_03341_b200  # noqa: F401  (registers the op)

    a = torch.empty((64, 32), device="meta")
    b = torch.empty((32, 48), device="meta")
    c, fl = torch.ops.tcec.sgemm(a, b, 1, 0)
    assert c.shape == (64, 48) and fl.dtype == torch.int32
    with pytest.raises(Exception):
        torch.ops.tcec.sgemm(torch.zeros(4, 4), torch.zeros(4, 4), 1, 0)


def test_c_example_builds_against_the_header_and_library():
    """examples/tcec_example.c -- a plain C caller of include/tcec.h linked
    against the in-tree libtcec.so -- compiles and links (runs in the GPU suite)."""
    import subprocess

    subprocess.run(["make", "-s", "-B", "-C", os.path.join(ROOT, "examples")], check=True)
    assert os.path.exists(os.path.join(ROOT, "examples", "tcec_example"))


@pytest.mark.gpu
def test_c_example_runs():
    import subprocess

    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "examples")], check=True)
    out = subprocess.run([os.path.join(ROOT, "examples", "tcec_example"), "512"], capture_output=True,
                         text=True, timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "relres" in out.stdout


def test_scheme_routing_without_gpu():
    """Scheme objects -> (variant, rounding, scale, product schedule), and the
    drain interval each schedule asks for (no GPU needed)."""
    import paper_2203_03341_b200 as T
    from paper_2203_03341_b200 import schemes as S

    assert T.resolve_schedule("corrected3_halfhalf") == (N.TCEC_FP16, N.ROUND_RN, 11, S.SCHED_CORRECTED3)
    assert T.resolve_schedule("corrected3_tf32") == (N.TCEC_TF32, N.ROUND_RNA, 0, S.SCHED_CORRECTED3)
    assert T.resolve_schedule("markidis4")[3] == S.SCHED_INUNIT4
    assert T.resolve_schedule("corrected4_rz")[3] == S.SCHED_INUNIT4
    assert T.resolve_schedule("corrected4_rn")[3] == S.SCHED_INUNIT4_RN
    rn_tf32 = T.corrected4(T.RoundingMode.RN, T.tf32tf32())
    assert T.resolve_schedule(rn_tf32) == (N.TCEC_TF32, N.ROUND_RNA, 0, S.SCHED_INUNIT4_RN)
    assert T.resolve_schedule("tc_plain_fp16")[3] == S.SCHED_TC_PLAIN
    # no MmaConfig: the tuned default drain (corrected4_rn: the reference's block of
    # 16); an explicit MmaConfig: exactly its block_k, in whole MMA k-steps
    assert S.drain_k_for(N.TCEC_FP16, None) == 128 and S.drain_k_for(N.TCEC_TF32, None) == 64
    assert S.drain_k_for(N.TCEC_FP16, None, S.SCHED_INUNIT4_RN) == 16
    assert S.drain_k_for(N.TCEC_TF32, None, S.SCHED_INUNIT4_RN) == 16
    assert S.drain_k_for(N.TCEC_FP16, S.MmaConfig(block_k=16)) == 16
    assert S.drain_k_for(N.TCEC_TF32, S.MmaConfig(block_k=16)) == 16
    assert S.drain_k_for(N.TCEC_TF32, S.MmaConfig(block_k=8)) == 8
    assert S.drain_k_for(N.TCEC_FP16, S.default_config(T.SCHEMES_BY_NAME["corrected3_halfhalf"])) == 16
    with pytest.raises(NotImplementedError):
        S.drain_k_for(N.TCEC_FP16, S.MmaConfig(block_k=24))
    with pytest.raises(NotImplementedError):
        S.drain_k_for(N.TCEC_TF32, S.MmaConfig(block_k=12), S.SCHED_INUNIT4_RN)
    with pytest.raises(NotImplementedError):  # the emulator's accumulator width has no GPU form
        S.drain_k_for(N.TCEC_FP16, S.MmaConfig(block_k=16, acc_significand_bits=24))
    for name in ("fp64_ref", "fp32_simt", "fp32_lsbtrunc"):
        with pytest.raises(NotImplementedError):
            T.resolve_schedule(name)


def test_no_cpu_fallback_without_library(tmp_path):
    """With the CUDA library missing the product path raises -- it never routes
    through the oracle or any CPU implementation."""
    import subprocess
    import sys

    code = ("import numpy as np, paper_2203_03341_b200 as T\n"
            "a = np.ones((4, 4), np.float32)\n"
            "try:\n"
            "    T.gemm(a, a, 'corrected3_tf32')\n"
            "except RuntimeError as e:\n"
            "    print('raised:', e)\n")
    env = dict(os.environ, TCEC_LIB=str(tmp_path / "missing.so"))
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True,
                         text=True, timeout=300)
    assert "raised:" in out.stdout and "no CPU fallback" in out.stdout, out.stdout + out.stderr


def test_no_cpu_fallback_without_gpu():
    """Library present but no sm_100 device (this container): the call fails
    loudly instead of computing on the host."""
    import numpy as np
    import torch

    import paper_2203_03341_b200 as T

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    a = np.ones((4, 4), np.float32)
    with pytest.raises(Exception):
        T.gemm(a, a, "corrected3_tf32")
