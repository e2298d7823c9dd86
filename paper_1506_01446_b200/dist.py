"""Partitioned (multi-GPU) bitonic sort over torch.distributed, one process per GPU.

The reference is single-device; north_star adds a 2/4/8-GPU
path.  Rank r owns the contiguous slice r of the array (the reference's
``work_slice`` partition, proj/include/bitonic/worker_pool.hpp:22-25).  The
sort is a bitonic network over the G shards in which every compare-exchange
becomes a merge-split (block 0-1 principle):

1. each rank sorts its shard locally (``sort_``, the single-GPU kernels);
2. for rank-level phase q = 1..g and step s = q..1 (g = log2 G), rank r pairs
   with r ^ 2^(s-1); the pair is ascending iff bit q of r is 0 -- the same
   direction rule as the reference's network (schedule.cpp:58-67) on shard
   indices; the lower rank of an ascending pair keeps the m smallest keys of
   the 2m union, the upper rank the m largest;
3. the exchange moves the partner's shard over NCCL (send/recv over
   NVLink/NVSwitch) and ``merge_split_`` (a merge-path kernel) keeps the
   required half.

Afterwards rank r holds global sorted positions [r*m, (r+1)*m).

The host logic here is pure torch.distributed plumbing; the two device
operations are injected (``ops``) so that the same schedule runs on CPU with
the gloo backend in the tests.  On GPU the ops are the native kernels.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, List, Tuple

import torch
import torch.distributed as dist


def network_steps(world: int) -> List[Tuple[int, int]]:
    """(phase q, step s) pairs of the rank-level bitonic network."""
    if world < 1 or world & (world - 1):
        raise ValueError("world size must be a power of two")
    g = world.bit_length() - 1
    return [(q, s) for q in range(1, g + 1) for s in range(q, 0, -1)]


def step_role(rank: int, q: int, s: int) -> Tuple[int, bool]:
    """Partner rank and whether this rank keeps the HIGH half at step (q, s)."""
    partner = rank ^ (1 << (s - 1))
    ascending = ((rank >> q) & 1) == 0
    lower = rank < partner
    keep_high = not (lower == ascending)
    return partner, keep_high


def key_xor_for(dtype, descending: bool) -> int:
    """The order transform the native kernels use: compare keys as uint32 after
    XOR with this mask (0x80000000 for int32, ~0 for descending)."""
    kx = 0x80000000 if dtype == torch.int32 else 0
    if descending:
        kx ^= 0xFFFFFFFF
    return kx


@dataclass
class Ops:
    local_sort: Callable  # (shard, descending) -> None, in place
    merge_split: Callable  # (local, partner, out, keep_high, key_xor) -> None
    exchange: Callable  # (send, recv, partner, group) -> None


def _as_wire(t):
    # NCCL/gloo have no uint32 type: move the bits as int32
    return t.view(torch.int32) if t.dtype == torch.uint32 else t


def p2p_exchange(send, recv, partner, group):
    """Swap shards with ``partner`` (paired isend/irecv; NCCL or gloo)."""
    ops = [dist.P2POp(dist.isend, _as_wire(send), partner, group),
           dist.P2POp(dist.irecv, _as_wire(recv), partner, group)]
    for req in dist.batch_isend_irecv(ops):
        req.wait()


def cuda_ops() -> Ops:
    from . import merge_split_, sort_

    def local_sort(t, descending):
        sort_(t, descending=descending)

    def merge(local, partner, out, keep_high, kx):
        merge_split_(local.view(torch.uint32), partner.view(torch.uint32),
                     out.view(torch.uint32), keep_high, kx)

    return Ops(local_sort=local_sort, merge_split=merge, exchange=p2p_exchange)


def partitioned_sort_(shard: torch.Tensor, descending: bool = False, group=None,
                      ops: Ops | None = None) -> torch.Tensor:
    """Sort the distributed array whose slice ``shard`` this rank owns.

    All ranks must pass equal-length shards of the same dtype (int32 or
    uint32).  In place: ``shard`` receives this rank's slice of the result.
    """
    ops = ops or cuda_ops()
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    ops.local_sort(shard, descending)
    if world == 1:
        return shard
    kx = key_xor_for(shard.dtype, descending)
    recv = torch.empty_like(shard)
    out = torch.empty_like(shard)
    cur = shard
    for q, s in network_steps(world):
        partner, keep_high = step_role(rank, q, s)
        ops.exchange(cur, recv, partner, group)
        ops.merge_split(cur, recv, out, keep_high, kx)
        cur, out = out, cur
    if cur is not shard:
        shard.copy_(cur)
    return shard
