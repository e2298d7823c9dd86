"""Race-check workload: every kernel family once, checked against numpy.

Run against the jitter build (tests/test_gpu_jitter.py sets
B200_BITONIC_LIB=paper_1506_01446_b200/libb200_bitonic_jitter.so, built with
-DB200_JITTER: random sleeps at every shared-memory hand-off), and meant for
compute-sanitizer (racecheck / synccheck / memcheck) where that tool is
allowed -- on this pool it is not (runs are refused, exit 86).

Runs every kernel family of the library once at small sizes -- the tile sort,
the merge passes (13/14-bit cosets and the 16-key variants), the batched
tiles, key-value and 64-bit kernels, the merge-path kernels (merge_tile /
merge_partition) and the pipelined host entry -- and checks each result
against numpy.  Usage (on the GPU box):

    B200_BITONIC_LIB=.../libb200_bitonic_jitter.so python tests/race_workload.py
    compute-sanitizer --tool racecheck python tests/race_workload.py

Exit code 0 = all results correct; the sanitizer's own summary line reports
hazards / errors.
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1506_01446_b200 as b  # noqa: E402

dev = torch.device("cuda:0")
rng = np.random.default_rng(7)
bad = []


def u32(n):
    return rng.integers(0, 2**32, n, dtype=np.uint64).astype(np.uint32)


def dev_t(x):
    t = torch.from_numpy(x.view(np.int32).copy()).to(dev)
    return t.view(torch.uint32) if x.dtype == np.uint32 else t


def host(t):
    return t.view(torch.int32).cpu().numpy().view(np.uint32) if t.dtype == torch.uint32 \
        else t.cpu().numpy()


def check(name, got, want):
    if not np.array_equal(got, want):
        bad.append(name)


ks = [int(v) for v in os.environ.get("SAN_KS", "10,13,16,18").split(",")]
for k in ks:
    x = u32(1 << k)
    t = dev_t(x)
    b.sort_(t)
    torch.cuda.synchronize()
    check(f"u32 asc 2^{k}", host(t), np.sort(x))
    xi = x.view(np.int32)
    t = dev_t(xi)
    b.sort_(t, descending=True)
    torch.cuda.synchronize()
    check(f"i32 desc 2^{k}", host(t), np.sort(xi)[::-1])
    # a second call of the same shape runs through the captured graph
    t = dev_t(x)
    b.sort_(t)
    b.sort_(t)
    torch.cuda.synchronize()
    check(f"u32 graphed 2^{k}", host(t), np.sort(x))

# 14-bit merge cosets (the k >= 24 plans) at a small size
os.environ.setdefault("B200_BITONIC_CMERGE", "14")
b.set_tuning(13, 5)
x = u32(1 << 17)
t = dev_t(x)
b.sort_(t)
torch.cuda.synchronize()
check("tile13/merge14 2^17", host(t), np.sort(x))
b.set_tuning(0, 5)

# batched tiles
x = u32(64 * 4096)
t = dev_t(x)
b.sort_batched_(t, 4096)
torch.cuda.synchronize()
check("batched 64x4096", host(t), np.sort(x.reshape(64, 4096), axis=1).reshape(-1))

# key-value
x = u32(1 << 14) % np.uint32(1000)
v = np.arange(1 << 14, dtype=np.uint32)
tk, tv = dev_t(x), dev_t(v)
b.sort_pairs_(tk, tv)
torch.cuda.synchronize()
check("pairs keys 2^14", host(tk), np.sort(x))
check("pairs perm 2^14", np.sort(host(tv)), v)

# 64-bit keys
x64 = rng.integers(-2**63, 2**63 - 1, 1 << 13, dtype=np.int64)
t = torch.from_numpy(x64.copy()).to(dev)
b.sort_(t)
torch.cuda.synchronize()
check("i64 2^13", t.cpu().numpy(), np.sort(x64))

# merge path (merge_partition + merge_tile kernels)
a = np.sort(u32(5000))
c = np.sort(u32(7001))
out = torch.empty(a.size + c.size, dtype=torch.uint32, device=dev)
b.merge_(dev_t(a), dev_t(c), out)
torch.cuda.synchronize()
check("merge 5000+7001", host(out), np.sort(np.concatenate([a, c])))

# merge-path variant: out-of-place tile sort + co-rank partitioned phases
for k in (15, 18):
    x = u32(1 << k)
    t = dev_t(x)
    b.sort_mergepath_(t)
    torch.cuda.synchronize()
    check(f"mergepath 2^{k}", host(t), np.sort(x))

# any length (padded + prefix/merge split)
x = u32((1 << 16) + 5)
t = dev_t(x)
b.sort_padded_(t)
torch.cuda.synchronize()
check("padded 2^16+5", host(t), np.sort(x))

# virtual padding (forced below its 2^26 default threshold): partial cosets
os.environ["B200_BITONIC_VIRTUAL"] = "1"
for n in [(1 << 16) - 12345, (1 << 18) - 3]:
    x = u32(n)
    t = dev_t(x)
    b.sort_padded_(t)
    torch.cuda.synchronize()
    check(f"virtual padding {n}", host(t), np.sort(x))
os.environ.pop("B200_BITONIC_VIRTUAL")

# pipelined host entry (4 chunks, merge tree, windowed D2H), pinned twice
os.environ["B200_BITONIC_HOST_CHUNKS"] = "4"
x = u32(1 << 18)
h = torch.from_numpy(x.view(np.int32).copy()).pin_memory().numpy().view(np.uint32)
for _ in range(2):
    h[:] = x
    b.sort_host(h)
    check("host entry 2^18 x4 chunks", h.copy(), np.sort(x))

print("race_workload:", "OK" if not bad else f"FAILED {bad}")
sys.exit(1 if bad else 0)
