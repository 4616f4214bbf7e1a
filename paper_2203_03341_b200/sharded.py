"""Row-sharded error-corrected SGEMM over the GPUs of one node.

One process per GPU (torch.distributed, NCCL over NVLink / NVSwitch).  Every
output element depends only on its row of A and column of B (the reference
allows parallelism across output elements only), so rank r owns a
contiguous slab of A's rows, B is replicated, and the slab of C is computed
with no data-path communication.  The only collective is the optional
all-gather of C, which concatenates the row slabs in rank order (row-major,
so no re-layout).  Results are bit-identical to the single-GPU call (the
per-element arithmetic does not depend on the row offset; see the
separability tests).
"""

from __future__ import annotations

from typing import Callable, Optional


def row_slab(m: int, rank: int, world: int) -> tuple[int, int]:
    """[start, stop) of rank's rows: equal slabs of ceil(m / world) rows (the last
    ones may be short or empty), so every rank's C slab has the same padded
    shape for the all-gather."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank / world size")
    per = -(-m // world)
    start = min(m, rank * per)
    return start, min(m, start + per)


def sharded_gemm(a_slab, b, scheme="corrected3_halfhalf", *, m_total: Optional[int] = None,
                 allgather: bool = False, group=None, out=None,
                 compute: Optional[Callable] = None):
    """C_slab = A_slab @ B on this rank; optionally all-gather the full C.

    a_slab: this rank's rows of A (rows row_slab(m_total, rank, world)), b: the
    full B (replicated).  Returns C_slab, or the full (m_total x n) C when
    `allgather`.  `compute(a, b, scheme)` defaults to the sm_100a kernel
    (gemm_device); tests may substitute the CPU oracle to exercise the
    partition / gather logic on gloo without a GPU.
    """
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    if compute is None:
        from .schemes import gemm_device

        def compute(a, bb, sch):
            return gemm_device(a, bb, sch)

    c_slab = compute(a_slab, b, scheme)
    if not allgather or world == 1:
        return c_slab
    if m_total is None:
        raise ValueError("m_total is required for the all-gather")
    per = -(-m_total // world)
    n = b.shape[1]
    padded = c_slab
    if c_slab.shape[0] != per or not c_slab.is_contiguous():
        padded = torch.zeros((per, n), dtype=c_slab.dtype, device=c_slab.device)
        padded[: c_slab.shape[0]].copy_(c_slab)
    full = torch.empty((per * world, n), dtype=c_slab.dtype, device=c_slab.device)
    dist.all_gather_into_tensor(full, padded, group=group)
    result = full[:m_total]
    if out is not None:
        out.copy_(result)
        return out
    return result
