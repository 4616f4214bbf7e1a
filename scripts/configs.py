"""BASELINE.json configs 1-5 on one B200: accuracy vs FP64 and throughput.

Prints one JSON object per measurement.  Inputs for the accuracy configs are
the reference's own generators (genmat.py, restated bit-exactly in the
oracle and pinned by tests/test_oracle_golden.py)."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2203_03341_b200 as T
from bench import device_matrix
from oracle import oracle as O

torch.backends.cuda.matmul.allow_tf32 = False
torch.set_float32_matmul_precision("highest")
dev = torch.device("cuda")
SCH = {"fp16": "corrected3_halfhalf", "tf32": "corrected3_tf32"}
only = set(sys.argv[1:])


def emit(d):
    print(json.dumps(d), flush=True)


def relres(c, ref):
    return float(torch.linalg.norm(ref - c.double()) / torch.linalg.norm(ref))


def timed(fn, iters=3, warm=2):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


# ---- config 1: FP16-TCEC 1024^3 urand(-1,1), seeds 0..7 (+ TF32, cuBLAS SGEMM, oracle seed 0)
if not only or "1" in only:
    rows = {"fp16": [], "fp16_block16": [], "tf32": [], "sgemm": [], "reference": []}
    exact = 0
    t_ref = 0.0
    for seed in range(8):
        a = O.urand(1024, 1024, -1, 1, seed)
        b = O.urand(1024, 1024, -1, 1, O.pair_seed(seed))
        A = torch.from_numpy(a).to(dev); B = torch.from_numpy(b).to(dev)
        ref = A.double() @ B.double()
        for v in ("fp16", "tf32"):
            rows[v].append(relres(T.gemm_device(A, B, SCH[v]), ref))
        c16 = T.gemm(A, B, SCH["fp16"], T.MmaConfig(block_k=16)).output  # the reference's schedule
        rows["fp16_block16"].append(relres(c16, ref))
        exact += int(np.array_equal(c16.cpu().numpy(), O.corrected3_hw(a, b, "fp16", drain_k=16)[0]))
        rows["sgemm"].append(relres(A @ B, ref))
        t0 = time.time()
        oc, _ = O.corrected3(a, b, "fp16", block_k=16, drain_k=16)   # the reference's algorithm
        t_ref += time.time() - t0
        rows["reference"].append(relres(torch.from_numpy(oc).to(dev), ref))
    emit({"config": 1, "desc": "FP16-TCEC 1024^3 urand(-1,1), relres vs FP64, seeds 0..7 (means)",
          "relres_fp16_tcec_mean": float(np.mean(rows["fp16"])),
          "relres_fp16_tcec_block_k16_mean": float(np.mean(rows["fp16_block16"])),
          "relres_tf32_tcec_mean": float(np.mean(rows["tf32"])),
          "relres_cublas_sgemm_mean": float(np.mean(rows["sgemm"])),
          "relres_reference_algorithm_mean": float(np.mean(rows["reference"])),
          "block_k16_bit_exact_vs_hw_oracle_seeds": exact,
          "per_seed_fp16": rows["fp16"], "per_seed_reference": rows["reference"],
          "reference_algorithm_cpu_s_total": t_ref, "host_threads": os.cpu_count()})

# ---- config 2: square sweep 1024..16384, TF32-TCEC and FP16-TCEC vs cuBLAS SGEMM, on
# the config's full-FP32-exponent-range inputs ExpRand(-50, 50) (a_max + b_max +
# log2 k < 127: no FP32 overflow), on urand(-1, 1), and for FP16-TCEC on its
# in-range band ExpRand(-15, 14) (ExpRand(-50, 50) is outside the FP16 split's
# range by design: flagged out_of_range / overflow, as the reference does)
if not only or "2" in only:
    for n in (1024, 2048, 4096, 8192, 16384):
        for dist in (("exprand", -50, 50), ("urand",), ("exprand", -15, 14)):
            g = torch.Generator(device=dev); g.manual_seed(n)
            A = device_matrix(dist, n, n, g, dev)
            B = device_matrix(dist, n, n, g, dev)
            C = torch.empty((n, n), device=dev)
            rows_idx = torch.arange(0, n, max(1, n // 256), device=dev)
            ref = A[rows_idx].double() @ B.double()
            out = {"config": 2, "n": n, "dist": "urand(-1,1)" if dist[0] == "urand"
                   else f"ExpRand({dist[1]},{dist[2]})"}
            for v in ("tf32", "fp16"):
                fl = torch.zeros(1, dtype=torch.int32, device=dev)
                T.gemm_device(A, B, SCH[v], out=C, flags=fl)
                out[f"{v}_flags"] = int(fl.item())
                out[f"{v}_relres"] = relres(C[rows_idx], ref)
                ms = timed(lambda: T.gemm_device(A, B, SCH[v], out=C), iters=5 if n <= 8192 else 3)
                out[f"{v}_tcec_tflops"] = 2 * n ** 3 / ms / 1e9
                if dist[0] == "urand":
                    ms = timed(lambda: T.gemm_device(A, B, SCH[v], out=C, split_mode=2),
                               iters=5 if n <= 8192 else 3)
                    out[f"{v}_tcec_split_once_tflops"] = 2 * n ** 3 / ms / 1e9
            ms = timed(lambda: torch.matmul(A, B, out=C), iters=3)
            out["cublas_sgemm_tflops"] = 2 * n ** 3 / ms / 1e9
            out["cublas_sgemm_relres"] = relres(C[rows_idx], ref)
            emit(out)
            del A, B, C, ref
            torch.cuda.empty_cache()

# ---- config 3: FP16-TCEC exponent sweep: ExpRand(e, e) for e in -15..15 and ExpRand(-15, 15)
if not only or "3" in only:
    m = n = 256
    k = 1024
    for e in list(range(-15, 16)) + ["spread"]:
        lo_e, hi_e = (-15, 15) if e == "spread" else (e, e)
        res = {"fp16": [], "tf32": [], "sgemm": []}
        flags = set()
        for seed in range(4):
            a = O.exprand(m, k, lo_e, hi_e, 100 + seed)
            b = O.exprand(k, n, lo_e, hi_e, O.pair_seed(100 + seed))
            A = torch.from_numpy(a).to(dev); B = torch.from_numpy(b).to(dev)
            ref = A.double() @ B.double()
            for v in ("fp16", "tf32"):
                run = T.gemm(A, B, SCH[v])
                res[v].append(relres(run.output, ref))
                if run.flags.saw_overflow:
                    flags.add(f"{v}:overflow")
                if run.flags.saw_out_of_range:
                    flags.add(f"{v}:out_of_range")
            res["sgemm"].append(relres(A @ B, ref))
        emit({"config": 3, "exponent": e, "m": m, "n": n, "k": k,
              "relres_fp16_tcec": float(np.mean(res["fp16"])), "relres_tf32_tcec": float(np.mean(res["tf32"])),
              "relres_cublas_sgemm": float(np.mean(res["sgemm"])), "flags": sorted(flags)})

# ---- config 4: rectangular / tall-skinny
if not only or "4" in only:
    for (m, n, k) in ((65536, 1024, 1024), (2048, 2048, 65536)):
        g = torch.Generator(device=dev); g.manual_seed(m + k)
        A = torch.rand((m, k), generator=g, device=dev) * 2 - 1
        B = torch.rand((k, n), generator=g, device=dev) * 2 - 1
        C = torch.empty((m, n), device=dev)
        rows_idx = torch.arange(0, m, max(1, m // 256), device=dev)
        ref = A[rows_idx].double() @ B.double()
        out = {"config": 4, "m": m, "n": n, "k": k}
        for v in ("tf32", "fp16"):
            ms = timed(lambda: T.gemm_device(A, B, SCH[v], out=C))
            out[f"{v}_tcec_tflops"] = 2 * m * n * k / ms / 1e9
            out[f"{v}_relres"] = relres(C[rows_idx], ref)
            ms = timed(lambda: T.gemm_device(A, B, SCH[v], out=C, split_mode=2))
            out[f"{v}_tcec_split_once_tflops"] = 2 * m * n * k / ms / 1e9
        ms = timed(lambda: torch.matmul(A, B, out=C))
        out["cublas_sgemm_tflops"] = 2 * m * n * k / ms / 1e9
        out["cublas_sgemm_relres"] = relres(C[rows_idx], ref)
        emit(out)
        del A, B, C, ref
        torch.cuda.empty_cache()

# ---- config 5: 65536^3 on one GPU (the N = 1 point of the row-sharded run)
if not only or "5" in only:
    n = 65536
    g = torch.Generator(device=dev); g.manual_seed(5)
    A = torch.empty((n, n), device=dev).uniform_(-1, 1, generator=g)
    B = torch.empty((n, n), device=dev).uniform_(-1, 1, generator=g)
    C = torch.empty((n, n), device=dev)
    out = {"config": 5, "m": n, "n": n, "k": n, "n_gpus": 1}
    for v in ("tf32", "fp16"):
        ms = timed(lambda: T.gemm_device(A, B, SCH[v], out=C), iters=1, warm=1)
        out[f"{v}_tcec_tflops"] = 2 * n ** 3 / ms / 1e9
        ms = timed(lambda: T.gemm_device(A, B, SCH[v], out=C, split_mode=2), iters=1, warm=1)
        out[f"{v}_tcec_split_once_tflops"] = 2 * n ** 3 / ms / 1e9
    rows_idx = torch.arange(0, n, n // 64, device=dev)
    ref = A[rows_idx].double() @ B.double()
    out["fp16_relres_64rows"] = relres(C[rows_idx], ref)
    emit(out)
