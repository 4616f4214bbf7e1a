"""B200-native error-corrected SGEMM (Ootomo & Yokota, arXiv 2203.03341).

Drop-in for the reference package's GEMM entry point on its corrected3 path
(`tcgemm.gemm(a, b, SCHEMES_BY_NAME["corrected3_halfhalf" | "corrected3_tf32"])`):
the same names and argument meanings, computed by hand-written sm_100a kernels
(libtcec.so, C ABI in include/tcec.h).
"""

from .analysis import relative_residual
from .formats import ACC25, FP16, FP32, TF32, FloatFormat, RoundingMode
from .schemes import (SCHEMES_BY_NAME, GemmKind, GemmRun, GemmScheme, MmaConfig, RunFlags,
                      corrected3, corrected4, default_config, delta_term_ablation, fp32_lsbtrunc,
                      fp32_simt, fp64_ref, gemm, gemm_device, gemm_device_multi, markidis4, resolve_schedule,
                      resolve_scheme, tc_plain)
from .splitting import (RESIDUAL_SCALE_LOG2, SplitKind, SplitMatrices, SplitScheme,
                        markidis_halfhalf, scaled_halfhalf, split_device, split_matrix, tf32tf32)

try:  # torch.ops.tcec.sgemm (registered when torch is importable)
    from . import torch_op  # noqa: F401
except ImportError:  # pragma: no cover
    torch_op = None

__version__ = "0.1.0"
