"""Host-entry (sort_host) wall time vs chunk count (development probe)."""
import os, sys, time, subprocess
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1506_01446_b200 as b

for k in (20, 22, 24):
    n = 1 << k
    src = torch.randint(-2**31, 2**31 - 1, (n,), dtype=torch.int32).pin_memory()
    work = torch.empty_like(src).pin_memory()
    arr = work.numpy()
    row = []
    for g in ("1", "2", "4", "8"):
        os.environ["B200_BITONIC_HOST_CHUNKS"] = g
        ts = []
        for r in range(12):
            work.copy_(src)
            c0 = time.perf_counter()
            b.sort_host(arr)
            ts.append((time.perf_counter() - c0) * 1e6)
        ts = sorted(ts[2:])
        assert (arr[1:] >= arr[:-1]).all()
        row.append(f"G={g}: med {ts[len(ts)//2]:.0f} min {ts[0]:.0f} us")
    print(f"k={k}  " + " | ".join(row), flush=True)
