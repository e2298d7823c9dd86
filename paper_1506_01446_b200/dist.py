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
3. the exchange moves, over NCCL send/recv (NVLink/NVSwitch), only the keys
   the partner keeps: the split point c (how many of the lower rank's keys
   stay low) is found with two small exchanges -- key samples every s
   positions, then one s-key window -- after which the lower rank sends its
   top m-c keys and the upper rank its bottom m-c keys (~m/2 each way on
   random data: the "half-shard" exchange), and each rank merges what it
   kept with what it received (``merge_``, a merge-path kernel).  The
   ``exchange="full"`` mode swaps whole shards instead (NCCL baseline).
4. ``exchange="peer"`` (the default on CUDA with the NCCL backend) fuses the
   exchange into the merge: every rank keeps its shard in two buffers that
   are shared with the other processes through CUDA IPC
   (``b200_bitonic_ipc_*``), and each merge-split step is ONE kernel that
   reads the partner's shard straight out of the partner GPU's memory over
   NVLink/NVSwitch -- only the part of it that lands in this rank's output
   window, ~m/2 keys on random data -- while it writes the merged output
   locally.  The steps are ordered on the device with interprocess CUDA
   events (partner's shard final before the read; read done before the
   buffer is reused); one host-only barrier per step orders the event
   records before the waits, without draining the GPUs.

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
    merge: Callable = None  # (a, b, out, key_xor) -> None (half exchange)


def _as_wire(t):
    # NCCL/gloo have no uint32 type: move the bits as int32
    return t.view(torch.int32) if t.dtype == torch.uint32 else t


def p2p_exchange(send, recv, partner, group):
    """Swap shards with ``partner`` (paired isend/irecv; NCCL or gloo)."""
    ops = [dist.P2POp(dist.isend, _as_wire(send), partner, group),
           dist.P2POp(dist.irecv, _as_wire(recv), partner, group)]
    for req in dist.batch_isend_irecv(ops):
        req.wait()


class PeerUnavailable(RuntimeError):
    """CUDA IPC peer mappings are not available on every rank."""


class PeerShards:
    """Two shard buffers per rank allocated for CUDA IPC, and every rank's
    buffers mapped into this process (the fused peer-memory exchange)."""

    def __init__(self, m: int, itemsize: int, group, rank: int, world: int):
        import ctypes
        from . import _native, _check
        self._lib = _native.lib()
        self._check = _check
        self.bytes = m * itemsize
        handles, self.local, self._opened = [], [], []
        self.ptrs = []  # ptrs[r][i]: rank r's buffer i, mapped here
        err = None
        try:
            for _ in range(2):
                ptr, h = ctypes.c_void_p(), _native.IpcHandle()
                _check(self._lib.b200_bitonic_ipc_alloc(self.bytes, ctypes.byref(ptr),
                                                        ctypes.byref(h)))
                self.local.append(ptr.value)
                handles.append(bytes(h.bytes))
        except Exception as e:  # e.g. IPC not permitted in this container
            err, handles = repr(e), []
        everyone = [None] * world
        dist.all_gather_object(everyone, handles, group=group)
        try:
            if err is not None or any(len(x) != 2 for x in everyone):
                raise RuntimeError(err or "a peer rank has no IPC buffers")
            for r in range(world):
                if r == rank:
                    self.ptrs.append(list(self.local))
                    continue
                row = []
                for hb in everyone[r]:
                    ptr, h = ctypes.c_void_p(), _native.IpcHandle()
                    ctypes.memmove(h.bytes, hb, len(hb))
                    _check(self._lib.b200_bitonic_ipc_open(ctypes.byref(h), ctypes.byref(ptr)))
                    row.append(ptr.value)
                    self._opened.append(ptr.value)
                self.ptrs.append(row)
        except Exception as e:  # e.g. no peer access / IPC not permitted here
            err = repr(e)
        # interprocess events, one per network step boundary (E[0..S]):
        # E_r[s] is recorded by rank r once its shard for step s is final
        nev = len(network_steps(world)) + 1
        self.events = []   # events[r][s], rank r's events opened here
        self._own_events, self._opened_events = [], []
        ev_handles = []
        if err is None:
            try:
                for _ in range(nev):
                    ev, h = ctypes.c_void_p(), _native.IpcHandle()
                    _check(self._lib.b200_bitonic_ipc_event_create(ctypes.byref(ev),
                                                                   ctypes.byref(h)))
                    self._own_events.append(ev.value)
                    ev_handles.append(bytes(h.bytes))
            except Exception as e:
                err = repr(e)
        everyone_ev = [None] * world
        dist.all_gather_object(everyone_ev, ev_handles, group=group)
        if err is None:
            try:
                for r in range(world):
                    if r == rank:
                        self.events.append(list(self._own_events))
                        continue
                    row = []
                    for hb in everyone_ev[r]:
                        ev, h = ctypes.c_void_p(), _native.IpcHandle()
                        ctypes.memmove(h.bytes, hb, len(hb))
                        _check(self._lib.b200_bitonic_ipc_event_open(ctypes.byref(h),
                                                                     ctypes.byref(ev)))
                        row.append(ev.value)
                        self._opened_events.append(ev.value)
                    self.events.append(row)
            except Exception as e:
                err = repr(e)
        # collective verdict: every rank mapped every peer, or nobody uses them
        oks = [None] * world
        dist.all_gather_object(oks, err is None, group=group)
        if not all(oks):
            self.close()
            raise PeerUnavailable(err or "a peer rank could not map the IPC buffers")
        # host-only barrier (orders event records before the partners' waits
        # without draining any GPU stream): the group itself when it is gloo,
        # else a gloo group over the same ranks
        backend = dist.get_backend(group)
        if backend == "gloo":
            self.host_group = group
        else:
            members = dist.get_process_group_ranks(group) if group is not None else None
            self.host_group = dist.new_group(ranks=members, backend="gloo")

    def close(self) -> None:
        import ctypes
        for p in self._opened:
            self._lib.b200_bitonic_ipc_close(ctypes.c_void_p(p))
        for p in self.local:
            self._lib.b200_bitonic_ipc_free(ctypes.c_void_p(p))
        for e in getattr(self, "_opened_events", []) + getattr(self, "_own_events", []):
            self._lib.b200_bitonic_event_destroy(ctypes.c_void_p(e))
        self._opened, self.local = [], []
        self._opened_events, self._own_events = [], []


_PEER_CACHE: dict = {}


def release_peer_buffers() -> None:
    """Unmap and free the cached IPC shard buffers (all ranks should call it
    together, after their last partitioned sort)."""
    for bufs in _PEER_CACHE.values():
        bufs.close()
    _PEER_CACHE.clear()


def _peer_shards(m, itemsize, group, rank, world, device):
    # key on the group's member ranks, not id(group): a dead group's id can be
    # reused by a new group object
    members = tuple(dist.get_process_group_ranks(group)) if group is not None else None
    key = (m, itemsize, members, rank, world, device.index)
    bufs = _PEER_CACHE.get(key)
    if bufs is None:  # collective: every rank reaches this on its first call
        bufs = PeerShards(m, itemsize, group, rank, world)
        _PEER_CACHE[key] = bufs
    return bufs


def _peer_partitioned_sort(shard, descending, group, rank, world, stats):
    """Local sort, then every merge-split step as one kernel reading the
    partner's shard through CUDA IPC peer memory.  Steps are ordered on the
    device: rank r records its interprocess event E_r[s] when its shard for
    step s is final; before step s its stream waits on the partner's E[s]
    (the partner's shard is final) and on the previous partner's E[s] (that
    rank has finished reading the buffer this step overwrites).  One
    host-only (gloo) barrier per step orders every record before the waits
    on it; the GPUs never drain between steps."""
    import ctypes
    from . import _native, _check, _stream_ptr
    lib = _native.lib()
    m = shard.numel()
    kx = key_xor_for(shard.dtype, descending)
    steps = network_steps(world)
    with torch.cuda.device(shard.device):
        stream = torch.cuda.current_stream(shard.device)
        sp = ctypes.c_void_p(_stream_ptr(stream))
        bufs = _peer_shards(m, shard.element_size(), group, rank, world, shard.device)
        ev = bufs.events
        counts = torch.zeros(len(steps), dtype=torch.int64, device=shard.device)
        cur = 0
        _check(lib.b200_bitonic_copy(ctypes.c_void_p(bufs.local[cur]),
                                     ctypes.c_void_p(shard.data_ptr()), bufs.bytes, sp))
        sort_fn = lib.b200_bitonic_sort_i32 if shard.dtype == torch.int32 \
            else lib.b200_bitonic_sort_u32
        _check(sort_fn(ctypes.c_void_p(bufs.local[cur]), m, int(bool(descending)), sp))
        _check(lib.b200_bitonic_event_record(ctypes.c_void_p(ev[rank][0]), sp))
        dist.barrier(bufs.host_group)  # every E[0] record is enqueued
        prev_partner = None
        for i, (q, s) in enumerate(steps):
            partner, keep_high = step_role(rank, q, s)
            _check(lib.b200_bitonic_stream_wait_event(sp, ctypes.c_void_p(ev[partner][i])))
            if prev_partner is not None and prev_partner != partner:
                _check(lib.b200_bitonic_stream_wait_event(
                    sp, ctypes.c_void_p(ev[prev_partner][i])))
            _check(lib.b200_bitonic_merge_split_u32_count(
                ctypes.c_void_p(bufs.local[cur]), ctypes.c_void_p(bufs.ptrs[partner][cur]),
                m, int(keep_high), ctypes.c_uint32(kx & 0xFFFFFFFF),
                ctypes.c_void_p(bufs.local[cur ^ 1]), sp,
                ctypes.c_void_p(counts.data_ptr() + 8 * i)))
            _check(lib.b200_bitonic_event_record(ctypes.c_void_p(ev[rank][i + 1]), sp))
            dist.barrier(bufs.host_group)  # every E[i+1] record is enqueued
            prev_partner = partner
            cur ^= 1
        # every rank has finished its last read of our buffers before the
        # result leaves them (and before a later call refills them)
        for r in range(world):
            if r != rank:
                _check(lib.b200_bitonic_stream_wait_event(
                    sp, ctypes.c_void_p(ev[r][len(steps)])))
        _check(lib.b200_bitonic_copy(ctypes.c_void_p(shard.data_ptr()),
                                     ctypes.c_void_p(bufs.local[cur]), bufs.bytes, sp))
    if stats is not None:
        stats["exchange"] = "peer"
        stats["steps"] = len(steps)
        stats["ordering"] = "interprocess CUDA events (device-side); gloo host barrier per step"
        # keys this rank read from its partner per step (device tensor; x4 = bytes
        # over NVLink); materialise with partner_keys.tolist() after timing
        stats["partner_keys"] = counts
    return shard


def cuda_ops() -> Ops:
    from . import merge_split_, sort_

    def local_sort(t, descending):
        sort_(t, descending=descending)

    from . import merge_

    def merge_split(local, partner, out, keep_high, kx):
        merge_split_(local.view(torch.uint32), partner.view(torch.uint32),
                     out.view(torch.uint32), keep_high, kx)

    def merge(a, b, out, kx):
        merge_(a.view(torch.uint32), b.view(torch.uint32), out.view(torch.uint32), kx)

    return Ops(local_sort=local_sort, merge_split=merge_split, exchange=p2p_exchange,
               merge=merge)


def _keys(t, kx):
    """Sort-order keys of 32-bit keys as int64 (for small sample/window math)."""
    return (t.view(torch.int32).to(torch.int64) & 0xFFFFFFFF) ^ kx


def _split_point(cur, lower, partner, kx, group, ops, s):
    """c = number of the lower rank's keys among the m smallest of the pair
    (merge path diagonal m, lower rank first on ties).  Identical on both
    ranks.  P(i) = A[i] <= B[m-1-i] (A = lower's shard, B = upper's) is
    monotone and c is its first false index: bracket c with samples A[j*s]
    and B[m-1-j*s], then evaluate P exactly on one window of < s indices."""
    m = cur.numel()
    cur = cur.view(torch.int32)  # torch has few uint32 kernels: move bits as int32
    pos = torch.arange(0, m, s, device=cur.device)
    nj = pos.numel()
    # my keys as seen from both roles: from the bottom (as A), from the top (as B)
    mine = torch.cat([cur[pos], cur[m - 1 - pos]])
    theirs = torch.empty_like(mine)
    ops.exchange(mine, theirs, partner, group)
    a_s = (mine if lower else theirs)[:nj]
    b_s = (theirs if lower else mine)[nj:]
    p = _keys(a_s, kx) <= _keys(b_s, kx)
    jstar = int(p.logical_not().to(torch.int32).argmax()) if bool((~p).any()) else nj
    lo = 0 if jstar == 0 else (jstar - 1) * s + 1
    hi = m if jstar == nj else jstar * s
    if hi <= lo:
        return lo
    # window: A[lo..hi) from the lower rank, B[m-hi..m-lo) from the upper rank
    w_mine = cur[lo:hi] if lower else cur[m - hi:m - lo]
    w_theirs = torch.empty_like(w_mine)
    ops.exchange(w_mine, w_theirs, partner, group)
    a_w = w_mine if lower else w_theirs
    b_w = (w_theirs if lower else w_mine).flip(0)  # B[m-1-i] for i = lo..hi-1
    return lo + int((_keys(a_w, kx) <= _keys(b_w, kx)).sum())


def _half_merge_split(cur, out, partner, keep_high, kx, group, ops, s):
    m = cur.numel()
    lower = not keep_high
    c = _split_point(cur, lower, partner, kx, group, ops, s)
    t = m - c  # keys crossing in each direction
    if lower:
        send, keep = cur[c:], cur[:c]
    else:
        send, keep = cur[:t], cur[t:]
    recv = torch.empty(t, dtype=cur.dtype, device=cur.device)
    if t:
        ops.exchange(send.contiguous(), recv, partner, group)
    if lower:
        ops.merge(keep, recv, out, kx)
    else:
        ops.merge(recv, keep, out, kx)
    return t


def partitioned_sort_(shard: torch.Tensor, descending: bool = False, group=None,
                      ops: Ops | None = None, exchange: str | None = None,
                      sample_stride: int = 4096, stats: dict | None = None,
                      rank: int | None = None, world: int | None = None) -> torch.Tensor:
    """Sort the distributed array whose slice ``shard`` this rank owns.

    All ranks must pass equal-length shards of the same dtype (int32 or
    uint32).  In place: ``shard`` receives this rank's slice of the result.
    ``exchange``: "peer" (one fused kernel per step reads the partner's shard
    over CUDA IPC peer memory; the default with NCCL on CUDA), "half" (NCCL
    send/recv of only the keys the partner keeps, then a merge) or "full"
    (whole shards).  ``stats`` (optional dict) receives the number of
    keys this rank sent per step.  ``rank``/``world`` override the process
    group's (in-process emulation of the ranks in tests).
    """
    from . import ConfigError
    if shard.dtype not in (torch.int32, torch.uint32):
        raise ConfigError(f"partitioned_sort_ takes int32 or uint32 shards, got {shard.dtype}")
    if not shard.is_contiguous() or shard.dim() != 1:
        raise ConfigError("the shard must be a contiguous 1-D tensor")
    if ops is None and not shard.is_cuda:
        raise ConfigError("the shard must be a CUDA tensor (CPU ops are test-only)")
    if exchange is None:
        exchange = ("peer" if shard.is_cuda and dist.is_initialized()
                    and dist.get_backend(group) == "nccl" and ops is None else "half")
    if exchange not in ("half", "full", "peer"):
        raise ValueError("exchange must be 'half', 'full' or 'peer'")
    if world is None:
        world = dist.get_world_size(group) if dist.is_initialized() else 1
    if rank is None:
        rank = dist.get_rank(group) if dist.is_initialized() else 0
    if exchange == "peer" and world > 1:
        try:
            return _peer_partitioned_sort(shard, descending, group, rank, world, stats)
        except PeerUnavailable:
            exchange = "half"  # every rank takes this branch together
            if stats is not None:
                stats["peer_fallback"] = True
    ops = ops or cuda_ops()
    ops.local_sort(shard, descending)
    if world == 1:
        return shard
    kx = key_xor_for(shard.dtype, descending)
    recv = torch.empty_like(shard)
    out = torch.empty_like(shard)
    cur = shard
    sent = []
    for q, s in network_steps(world):
        partner, keep_high = step_role(rank, q, s)
        if exchange == "half" and ops.merge is not None:
            sent.append(_half_merge_split(cur, out, partner, keep_high, kx, group, ops,
                                          sample_stride))
        else:
            ops.exchange(cur, recv, partner, group)
            ops.merge_split(cur, recv, out, keep_high, kx)
            sent.append(cur.numel())
        cur, out = out, cur
    if stats is not None:
        stats["keys_sent_per_step"] = sent
    if cur is not shard:
        shard.copy_(cur)
    return shard
