"""The PyTorch operator form of the accelerated path:

    torch.ops.tcec.sgemm(A, B, variant, drain_k) -> (C, flags)

A thin `torch.library` custom op over the C ABI (`tcec_sgemm`, via
schemes.gemm_device): CUDA float32 A (m x k) and B (k x n), `variant` 0 =
FP16-TCEC / 1 = TF32-TCEC, `drain_k` the drain interval of the main-term partial
(0 = default).  Returns C (m x n float32) and the int32 RunFlags word
(bit 0 overflow, bit 1 out_of_range, bit 2 non-finite input), both on the
device and without a host synchronisation, so the op composes with CUDA graphs
and appears as one opaque node to torch.compile.  It has a fake (meta)
implementation for tracing; there is no CPU kernel (the op raises on CPU
tensors, like every compute path of this package).
"""

from __future__ import annotations

import torch

from .schemes import gemm_device

_SCHEME = {0: "corrected3_halfhalf", 1: "corrected3_tf32"}


@torch.library.custom_op("tcec::sgemm", mutates_args=())
def sgemm(a: torch.Tensor, b: torch.Tensor, variant: int = 1,
          drain_k: int = 0) -> tuple[torch.Tensor, torch.Tensor]:
    if variant not in _SCHEME:
        raise ValueError("variant must be 0 (FP16-TCEC) or 1 (TF32-TCEC)")
    if not (a.is_cuda and b.is_cuda):
        raise ValueError("tcec::sgemm runs on CUDA tensors only (no CPU path)")
    flags = torch.zeros(1, dtype=torch.int32, device=a.device)
    c = gemm_device(a, b, _SCHEME[variant], flags=flags, drain_k=drain_k or None)
    return c.contiguous() if not c.is_contiguous() else c, flags


@sgemm.register_fake
def _(a, b, variant=1, drain_k=0):
    return (a.new_empty((a.shape[0], b.shape[1])), a.new_empty((1,), dtype=torch.int32))
