"""Multi-GPU sharding of the quantize-and-GEMM path (one process per GPU).

Linear layers shard by OUTPUT COLUMN (rows of the weight W[N, K]): every rank
quantizes its own weight shard once (weights never move), quantizes the
replicated activation locally (row-independent, so every rank produces the
same bits), runs the tcgen05 GEMM on its N/world columns and -- only when the
caller needs the full product -- gathers the output shards with one NCCL
all_gather over NVLink (SURVEY §8 e, config 4).  Whole-model weight
quantization shards by layer with no collective (config 3).  NVFP4 is the
one variant whose quantization couples rows (global amax, src/quantize.py:671):
``global_amax`` is an all_reduce(MAX) of one scalar.

The collective / assembly logic is written against ``torch.distributed`` and
plain tensors so it is exercised on CPU with the gloo backend
(tests/test_parallel_gloo.py); the compute callback is the GPU GEMM in
production.
"""

from __future__ import annotations

from typing import Callable, Sequence

import torch
import torch.distributed as dist


def shard_bounds(n: int, world: int, rank: int, align: int = 128) -> tuple[int, int]:
    """[lo, hi) rows of an N-row weight owned by `rank`: contiguous, each
    shard a multiple of `align` rows except possibly the last (so the GEMM's
    128-row tiles never straddle ranks)."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    blocks = -(-n // align)
    per = blocks // world
    extra = blocks % world
    start_blk = rank * per + min(rank, extra)
    nblk = per + (1 if rank < extra else 0)
    lo = min(n, start_blk * align)
    hi = min(n, (start_blk + nblk) * align)
    return lo, hi


def layer_owner(num_layers: int, world: int) -> list[int]:
    """Layer -> rank for layer-sharded weight quantization (contiguous blocks)."""
    return [min(world - 1, (l * world) // num_layers) for l in range(num_layers)]


def gather_columns(local: torch.Tensor, n_total: int, world: int, group=None) -> torch.Tensor:
    """All-gather column shards (M, n_r) into the full (M, N) output.

    Shards follow ``shard_bounds``; unequal shards are padded to the largest
    so one ``all_gather_into_tensor`` suffices, then trimmed and concatenated.
    """
    m = local.shape[0]
    sizes = [shard_bounds(n_total, world, r)[1] - shard_bounds(n_total, world, r)[0] for r in range(world)]
    width = max(sizes)
    send = local
    if local.shape[1] != width:
        send = torch.zeros((m, width), dtype=local.dtype, device=local.device)
        send[:, : local.shape[1]] = local
    flat = torch.empty((world * m, width), dtype=local.dtype, device=local.device)
    dist.all_gather_into_tensor(flat, send.contiguous(), group=group)
    buf = flat.view(world, m, width)
    return torch.cat([buf[r, :, : sizes[r]] for r in range(world)], dim=1)


def gather_columns_into(local: torch.Tensor, out: torch.Tensor, world: int, staging: torch.Tensor = None,
                        group=None) -> torch.Tensor:
    """All-gather every rank's column shard ``local`` (m, n_r) into ``out``
    (m, N), the row-major product: one ``all_gather_into_tensor`` into a
    (world, m, width) staging buffer (shards padded to the widest), then one
    strided copy per rank into its column slice.  ``staging`` may be passed to
    reuse a buffer across calls."""
    m, n_total = out.shape
    spans = [shard_bounds(n_total, world, r) for r in range(world)]
    width = max(hi - lo for lo, hi in spans)
    send = local
    if local.shape[1] != width:
        send = torch.zeros((m, width), dtype=local.dtype, device=local.device)
        send[:, : local.shape[1]] = local
    if staging is None or staging.shape != (world, m, width):
        staging = torch.empty((world, m, width), dtype=local.dtype, device=local.device)
    dist.all_gather_into_tensor(staging.view(world * m, width), send.contiguous(), group=group)
    for r, (lo, hi) in enumerate(spans):
        out[:, lo:hi].copy_(staging[r, :, : hi - lo])
    return out


def column_parallel_forward(x: torch.Tensor, w_shard, out: torch.Tensor, world: int, local_gemm: Callable,
                            chunks: int = 4, comm_stream=None, group=None) -> torch.Tensor:
    """y = x @ W^T into ``out`` (M, N) with W row-sharded across ranks, the
    gather overlapped with compute.  x is cut into ``chunks`` row blocks;
    ``local_gemm(x_rows, w_shard, dst)`` writes the block's (rows, n_r) column
    shard into ``dst``.  Block i+1's GEMM runs on the current stream while
    block i's all_gather + (M, N) assembly run on ``comm_stream`` (CUDA; on
    CPU the blocks run one after another).  Row blocks are multiples of 128
    rows, so each is a whole number of GEMM tiles, and quantizing x block by
    block is bit-identical to one call (row partition invariance,
    /root/reference/pkg/tests/test_quantize.py:371-387).  With world == 1 the
    GEMM writes ``out`` directly."""
    m, n_total = out.shape
    if world == 1:
        local_gemm(x, w_shard, out)
        return out
    step = max(128, -(-(-(-m // chunks)) // 128) * 128)
    cuda = x.is_cuda and comm_stream is not None
    compute = torch.cuda.current_stream(x.device) if cuda else None
    lo, hi = shard_bounds(n_total, world, dist.get_rank(group))
    for r0 in range(0, m, step):
        r1 = min(m, r0 + step)
        local = torch.empty((r1 - r0, hi - lo), dtype=out.dtype, device=out.device)
        local_gemm(x[r0:r1], w_shard, local)
        if cuda:
            ev = torch.cuda.Event()
            ev.record(compute)
            with torch.cuda.stream(comm_stream):
                comm_stream.wait_event(ev)
                local.record_stream(comm_stream)
                gather_columns_into(local, out[r0:r1], world, group=group)
        else:
            gather_columns_into(local, out[r0:r1], world, group=group)
    if cuda:
        compute.wait_stream(comm_stream)
    return out


def column_sharded_linear(x, w_shard, n_total: int, gemm: Callable, world: int, gather: bool = True,
                          group=None) -> torch.Tensor:
    """y = x @ W^T with W split by rows across ranks.  `gemm(x, w_shard)`
    computes the local (M, n_r) block; the full output is gathered when
    `gather` (the only data-path collective)."""
    local = gemm(x, w_shard)
    if not gather or world == 1:
        return local
    return gather_columns(local, n_total, world, group=group)


def global_amax(local_amax: torch.Tensor, group=None) -> torch.Tensor:
    """NVFP4's tensor-wide |x| max across row shards: all_reduce(MAX)."""
    t = local_amax.clone()
    if dist.is_available() and dist.is_initialized():
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return t


def max_over_ranks(value: float, device=None, group=None) -> float:
    """Timing reduction: every multi-GPU time is the max over ranks."""
    if not (dist.is_available() and dist.is_initialized()):
        return value
    if dist.get_backend(group) == "gloo":
        device = None  # gloo reduces host tensors
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
