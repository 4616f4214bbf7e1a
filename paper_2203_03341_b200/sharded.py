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


def _device_compute(flags, concurrent: bool) -> Callable:
    """The sm_100a kernel, its RunFlags OR-ed into `flags` (device int32).  With
    a collective in flight on another stream the per-tile kernel is pinned
    (kernel_variant 4): the lock-step persistent kernel assumes it has every SM."""
    from .schemes import gemm_device

    def compute(a, bb, sch):
        return gemm_device(a, bb, sch, flags=flags, kernel_variant=4 if concurrent else 0)

    return compute


def _raise_on_flags(flags) -> None:
    """The reference raises ValueError for non-finite inputs (schemes.py:166-167);
    numerical anomalies only set RunFlags."""
    from . import _native as N

    if int(flags.item()) & N.FLAG_NONFINITE_INPUT:
        raise ValueError("gemm requires finite inputs")


def sharded_gemm(a_slab, b, scheme="corrected3_halfhalf", *, m_total: Optional[int] = None,
                 allgather: bool = False, group=None, out=None,
                 compute: Optional[Callable] = None, overlap_chunks: int = 1, flags=None):
    """C_slab = A_slab @ B on this rank; optionally all-gather the full C.

    a_slab: this rank's rows of A (rows row_slab(m_total, rank, world)), b: the
    full B (replicated).  Returns C_slab, or the full (m_total x n) C when
    `allgather`.  `compute(a, b, scheme)` defaults to the sm_100a kernel
    (gemm_device); tests may substitute the CPU oracle to exercise the
    partition / gather logic on gloo without a GPU.

    RunFlags: with `flags` (int32 CUDA tensor, caller-zeroed) the kernel ORs
    this rank's TCEC_FLAG_* bits into it and nothing synchronises; without it
    the call reads them once at the end and raises ValueError for non-finite
    inputs in this rank's operands, as the reference does.

    overlap_chunks > 1 (with allgather): the slab is computed in that many row
    chunks (multiples of the 256-row pair tile) and chunk i is all-gathered on
    a communication stream while chunk i + 1 computes; the gathered rows land
    directly in their final place (each rank's chunk i is a contiguous row
    block of the full C).  Same result, bit for bit.
    """
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    own_flags = None
    if compute is None:
        if flags is None:
            flags = own_flags = torch.zeros(1, dtype=torch.int32, device=b.device)
        compute = _device_compute(flags, allgather and world > 1 and overlap_chunks > 1)

    if allgather and world > 1 and overlap_chunks > 1:
        result = _gather_overlapped(a_slab, b, scheme, m_total, world, group, out, compute,
                                    overlap_chunks)
        if own_flags is not None:
            _raise_on_flags(own_flags)
        return result
    c_slab = compute(a_slab, b, scheme)
    if own_flags is not None:
        _raise_on_flags(own_flags)
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


def _gather_overlapped(a_slab, b, scheme, m_total, world, group, out, compute, chunks):
    import torch
    import torch.distributed as dist

    if m_total is None:
        raise ValueError("m_total is required for the all-gather")
    per = -(-m_total // world)
    n = b.shape[1]
    ch = max(1, -(-per // chunks))
    if ch >= 256:  # whole 256-row pair tiles per chunk
        ch = -(-ch // 256) * 256
    full = torch.empty((per * world, n), dtype=b.dtype, device=b.device)
    cuda = full.is_cuda
    comm = torch.cuda.Stream(device=full.device) if cuda else None
    main = torch.cuda.current_stream(full.device) if cuda else None
    pending = []
    for r0 in range(0, per, ch):
        rows = min(ch, per - r0)
        valid = max(0, min(rows, a_slab.shape[0] - r0))
        if valid == rows:
            c = compute(a_slab[r0:r0 + rows], b, scheme)
        else:  # short last slab: pad with zero rows
            c = torch.zeros((rows, n), dtype=b.dtype, device=b.device)
            if valid > 0:
                c[:valid].copy_(compute(a_slab[r0:r0 + valid], b, scheme))
        c = c.contiguous()
        views = [full[r * per + r0: r * per + r0 + rows] for r in range(world)]
        if cuda:
            ev = torch.cuda.Event()
            ev.record(main)
            comm.wait_event(ev)
            c.record_stream(comm)
            with torch.cuda.stream(comm):
                pending.append(dist.all_gather(views, c, group=group, async_op=True))
        else:
            dist.all_gather(views, c, group=group)
    for w in pending:
        w.wait()
    if cuda:
        main.wait_stream(comm)
    result = full[:m_total]
    if out is not None:
        out.copy_(result)
        return out
    return result


_SYMM_CACHE: dict = {}


def sharded_gemm_fused(a_slab, b, scheme="corrected3_halfhalf", *, m_total: int, group=None,
                       copy: bool = True, flags=None):
    """Row-sharded GEMM with the all-gather fused into the GEMM epilogue.

    The full C lives in symmetric memory (torch.distributed._symmetric_memory:
    one buffer per rank, every peer's buffer mapped into this GPU's address
    space over NVLink).  One kernel (tcec_sgemm_multi) computes this rank's
    slab and TMA-stores each output box into the slab's rows of every rank's
    buffer, so the gather overlaps the GEMM tile by tile with no separate
    collective; a barrier then makes the peers' stores visible.  Returns this
    rank's full (m_total x n) C.  Bit-identical to the single-GPU product.

    The symmetric buffer is cached per shape and reused: a barrier before the
    GEMM makes every rank finish with the previous call's result before any
    peer overwrites it, and the result is returned as a copy (copy=False
    returns a view of the buffer, valid until the next call with this shape).
    RunFlags as in sharded_gemm.
    """
    import torch
    import torch.distributed as dist
    import torch.distributed._symmetric_memory as symm_mem

    from .schemes import gemm_device_multi

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    if world > 8:
        raise ValueError("the fused all-gather covers at most 8 ranks (one NVLink domain)")
    per = -(-m_total // world)
    n = b.shape[1]
    ldc = max(4, (n + 3) // 4 * 4)
    grp = group if group is not None else dist.group.WORLD
    key = (per * world, ldc, str(b.device), id(grp))
    if key not in _SYMM_CACHE:  # one symmetric buffer per shape, reused across calls
        full = symm_mem.empty((per * world, ldc), dtype=torch.float32, device=b.device)
        _SYMM_CACHE[key] = (full, symm_mem.rendezvous(full, grp))
    full, hdl = _SYMM_CACHE[key]
    rows = a_slab.shape[0]
    r0 = rank * per
    # own buffer first, then the peers'
    order = [rank] + [r for r in range(world) if r != rank]
    outs = [hdl.get_buffer(r, (per * world, ldc), torch.float32)[r0:r0 + rows, :n] for r in order]
    own_flags = None
    if flags is None:
        flags = own_flags = torch.zeros(1, dtype=torch.int32, device=b.device)
    hdl.barrier()  # every rank is done with the previous result in this buffer
    if rows > 0:
        gemm_device_multi(a_slab, b, outs, scheme, flags=flags)
    hdl.barrier()  # the peers' stores into this rank's buffer are complete
    if own_flags is not None:
        _raise_on_flags(own_flags)
    result = full[:m_total, :n]
    return result.clone() if copy else result
