"""CPU, multi-process: the partitioned sort's rank-level schedule (dist.py)
with the gloo backend, world sizes 2 and 4.  The two device operations are
replaced by numpy equivalents here; the GPU tests cover the kernels."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1506_01446_b200 import dist as bdist


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _key(a, kx):
    return a.view(np.uint32) ^ np.uint32(kx)


def numpy_ops():
    def local_sort(t, descending):
        a = t.numpy()
        kx = bdist.key_xor_for(t.dtype, descending)
        a[:] = a[np.argsort(_key(a, kx), kind="stable")]

    def merge_split(local, partner, out, keep_high, kx):
        u = np.concatenate([local.numpy(), partner.numpy()])
        u = u[np.argsort(_key(u, kx), kind="stable")]
        m = local.numel()
        out.numpy()[:] = u[m:] if keep_high else u[:m]

    def merge(a, b, out, kx):
        u = np.concatenate([a.numpy(), b.numpy()])
        out.numpy()[:] = u[np.argsort(_key(u, kx), kind="stable")]

    return bdist.Ops(local_sort=local_sort, merge_split=merge_split,
                     exchange=bdist.p2p_exchange, merge=merge)


def _worker(rank, world, port, n, dtype_name, descending, q, exchange="half", stride=64,
            shape="random"):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(1234)
        x = rng.integers(0, 2**32, n, dtype=np.uint64).astype(np.uint32)
        x[: n // 8] = x[n // 8: n // 4]  # duplicates across shards
        if shape == "sorted":
            x = np.sort(x)
        elif shape == "reversed":
            x = np.sort(x)[::-1].copy()
        elif shape == "equal":
            x[:] = 7
        if dtype_name == "int32":
            x = x.view(np.int32)
        m = n // world
        shard = torch.from_numpy(x[rank * m:(rank + 1) * m].copy())
        stats = {}
        bdist.partitioned_sort_(shard, descending=descending, ops=numpy_ops(),
                                exchange=exchange, sample_stride=stride, stats=stats)
        wire = shard.view(torch.int32)  # gloo has no uint32 collectives
        parts = [torch.empty_like(wire) for _ in range(world)]
        dist.all_gather(parts, wire)
        if rank == 0:
            got = np.concatenate([p.numpy() for p in parts]).view(x.dtype)
            want = np.sort(x)
            if descending:
                want = want[::-1]
            q.put((bool((got == want).all()), stats.get("keys_sent_per_step")))
    finally:
        dist.destroy_process_group()


def _run(world, dtype_name, descending, exchange="half", stride=64, shape="random",
         n=1 << 12):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, dtype_name, descending, q,
                                               exchange, stride, shape))
             for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=180)
        assert p.exitcode == 0
    return q.get(timeout=5)


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("dtype_name,descending", [("uint32", False), ("int32", False),
                                                    ("uint32", True)])
def test_partitioned_sort_gloo(world, dtype_name, descending):
    ok, sent = _run(world, dtype_name, descending)
    assert ok
    # the half exchange moves about half a shard per step on random data
    m = (1 << 12) // world
    assert all(0 <= t <= m for t in sent) and sum(sent) < len(sent) * m * 0.8


@pytest.mark.parametrize("shape", ["sorted", "reversed", "equal"])
def test_partitioned_sort_gloo_adversarial(shape):
    ok, _ = _run(4, "uint32", False, shape=shape, stride=16)
    assert ok


def test_partitioned_sort_gloo_full_exchange():
    ok, sent = _run(2, "int32", True, exchange="full")
    assert ok and sent == [(1 << 12) // 2]


def test_schedule_roles():
    # every step pairs ranks symmetrically, one keeps low, one keeps high
    for world in [2, 4, 8]:
        for q, s in bdist.network_steps(world):
            for r in range(world):
                p, hi = bdist.step_role(r, q, s)
                p2, hi2 = bdist.step_role(p, q, s)
                assert p2 == r and hi != hi2
    assert len(bdist.network_steps(8)) == 6
    assert bdist.network_steps(1) == []
    with pytest.raises(ValueError):
        bdist.network_steps(3)
