"""Row sharding across ranks (world size 2, gloo on CPU).

The partition and the all-gather are exercised with the CPU oracle standing in
for the kernel (test-only injection); the GPU kernel's own row-separability is
checked bit-for-bit in test_gpu_gemm.py, so the composition is exact."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as O
from paper_2203_03341_b200.sharded import row_slab, sharded_gemm


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_row_slab_partition():
    for m in (0, 1, 7, 256, 1000, 65536):
        for w in (1, 2, 3, 8):
            slabs = [row_slab(m, r, w) for r in range(w)]
            assert slabs[0][0] == 0 and slabs[-1][1] == m
            for (a, b), (c, d) in zip(slabs, slabs[1:]):
                assert b == c
            per = -(-m // w)
            assert all(b - a <= per for a, b in slabs)
    with pytest.raises(ValueError):
        row_slab(10, 2, 2)


def _oracle_compute(a, b, scheme):
    variant = "fp16" if "half" in scheme else "tf32"
    bk, d = (16, 64) if variant == "fp16" else (8, 32)
    c, _ = O.corrected3(a.numpy(), b.numpy(), variant, block_k=bk, drain_k=d)
    return torch.from_numpy(c)


def _worker(rank, world, port, m, n, k, scheme, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        a = torch.from_numpy(O.urand(m, k, -1, 1, 3))
        b = torch.from_numpy(O.urand(k, n, -1, 1, O.pair_seed(3)))
        r0, r1 = row_slab(m, rank, world)
        full = sharded_gemm(a[r0:r1], b, scheme, m_total=m, allgather=True,
                            compute=_oracle_compute)
        slab = sharded_gemm(a[r0:r1], b, scheme, compute=_oracle_compute)
        full3 = sharded_gemm(a[r0:r1], b, scheme, m_total=m, allgather=True,
                             compute=_oracle_compute, overlap_chunks=3)
        assert torch.equal(full3, full)  # chunked all-gather: same rows, same places
        if rank == 0:
            q.put((full.numpy().copy(), r0, r1, slab.numpy().copy()))
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("m", [64, 37])
@pytest.mark.parametrize("scheme", ["corrected3_halfhalf", "corrected3_tf32"])
def test_sharded_allgather_equals_single_rank(m, scheme):
    n, k = 24, 96
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, m, n, k, scheme, q)) for r in range(2)]
    for p in procs:
        p.start()
    full, r0, r1, slab = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    a = O.urand(m, k, -1, 1, 3)
    b = O.urand(k, n, -1, 1, O.pair_seed(3))
    ref = _oracle_compute(torch.from_numpy(a), torch.from_numpy(b), scheme).numpy()
    assert full.shape == (m, n)
    assert np.array_equal(full, ref)          # bit-identical to the unsharded product
    assert np.array_equal(slab, ref[r0:r1])
