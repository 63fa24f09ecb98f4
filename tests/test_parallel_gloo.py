"""Multi-process (world_size 2, gloo, CPU) tests of the sharding logic used
by the N>1 bench path: shard bounds, column all-gather assembly, NVFP4 global
amax and max-over-ranks timing.  The local GEMM is the CPU oracle here; on the
GPU box it is the tcgen05 kernel -- the collective code is identical."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2603_08713_b200 import parallel as P


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, results):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import mxq_oracle as O
        rng = np.random.Generator(np.random.PCG64(0))
        m, n, k = 16, 300, 256
        a = rng.standard_t(4, (m, k)).astype(np.float32)
        w = rng.standard_normal((n, k)).astype(np.float32)
        lo, hi = P.shard_bounds(n, world, rank)
        aq = O.dequantize(O.quantize(a, "mbs_s"))

        def gemm(x, ws):
            wd = O.dequantize(O.quantize(ws, "mbs_d"))
            return torch.from_numpy(O.matmul_blas(x, wd))

        full = P.column_sharded_linear(aq, w[lo:hi], n, gemm, world)
        want = O.matmul_blas(aq, O.dequantize(O.quantize(w, "mbs_d")))
        ok_gemm = bool(np.array_equal(full.numpy(), want))
        amax = P.global_amax(torch.tensor([float(np.abs(a[rank::world]).max())]))
        ok_amax = float(amax) == float(np.abs(a).max())
        t = P.max_over_ranks(1.0 + rank)
        results[rank] = (ok_gemm, ok_amax, t)
    finally:
        dist.destroy_process_group()


def test_column_sharded_linear_gloo_world2():
    world = 2
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), results), nprocs=world, join=True)
    for r in range(world):
        ok_gemm, ok_amax, t = results[r]
        assert ok_gemm and ok_amax
        assert t == 2.0


def test_shard_bounds_cover_and_align():
    for n in (1, 128, 300, 4096, 5760, 28672):
        for world in (1, 2, 3, 8):
            spans = [P.shard_bounds(n, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            for (a, b), (c, d) in zip(spans, spans[1:]):
                assert b == c
            for lo, hi in spans[:-1]:
                assert lo % 128 == 0 and (hi - lo) % 128 == 0 or hi == n
    assert P.layer_owner(36, 8)[0] == 0 and P.layer_owner(36, 8)[-1] == 7


def _worker_overlap(rank, world, port, results):
    """column_parallel_forward: row-blocked GEMM + all_gather + (M, N)
    assembly, against the unsharded product (bit-identical: every element is
    computed by exactly one rank with the same per-element arithmetic)."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import mxq_oracle as O
        rng = np.random.Generator(np.random.PCG64(1))
        m, n, k = 300, 700, 256
        a = rng.standard_t(4, (m, k)).astype(np.float32)
        w = rng.standard_normal((n, k)).astype(np.float32)
        lo, hi = P.shard_bounds(n, world, rank)
        wd = O.dequantize(O.quantize(w[lo:hi], "mbs_d"))

        def local_gemm(x_rows, w_shard, dst):
            xd = O.dequantize(O.quantize(x_rows.numpy(), "mbs_s"))  # per row block, as on the GPU
            dst.copy_(torch.from_numpy(O.matmul_blas(xd, w_shard)))

        out = torch.empty((m, n), dtype=torch.float32)
        P.column_parallel_forward(torch.from_numpy(a), wd, out, world, local_gemm, chunks=3)
        want = O.matmul_blas(O.dequantize(O.quantize(a, "mbs_s")), O.dequantize(O.quantize(w, "mbs_d")))
        results[rank] = bool(np.array_equal(out.numpy(), want))
    finally:
        dist.destroy_process_group()


def test_column_parallel_forward_overlap_gloo_world2():
    world = 2
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_worker_overlap, args=(world, _free_port(), results), nprocs=world, join=True)
    assert all(results[r] for r in range(world))
