"""Host wall time: torch copies + graphed device sort vs the host entry (probe)."""
import os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1506_01446_b200 as b

os.environ["B200_BITONIC_HOST_CHUNKS"] = "1"
n = 1 << 20
src = torch.randint(-2**31, 2**31 - 1, (n,), dtype=torch.int32).pin_memory()
work = torch.empty_like(src).pin_memory()
d = torch.empty(n, dtype=torch.int32, device="cuda")
s = torch.cuda.Stream()
arr = work.numpy()


def wall(fn, reps=20):
    ts = []
    for r in range(reps):
        work.copy_(src)
        torch.cuda.synchronize()
        c0 = time.perf_counter()
        fn()
        ts.append((time.perf_counter() - c0) * 1e6)
    ts = sorted(ts[3:])
    return ts[len(ts) // 2], ts[0]


def torch_path():
    with torch.cuda.stream(s):
        d.copy_(work, non_blocking=True)
        b.sort_(d)
        work.copy_(d, non_blocking=True)
    s.synchronize()


def copies_only():
    with torch.cuda.stream(s):
        d.copy_(work, non_blocking=True)
        work.copy_(d, non_blocking=True)
    s.synchronize()


for name, fn in (("torch copies + sort_", torch_path), ("copies only", copies_only),
                 ("host entry", lambda: b.sort_host(arr)), ("torch copies + sort_", torch_path),
                 ("host entry", lambda: b.sort_host(arr))):
    med, mn = wall(fn)
    print(f"{name:22s} med {med:6.1f} min {mn:6.1f} us", flush=True)
