"""Python-side overhead of the host entry (development probe)."""
import ctypes, os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1506_01446_b200 as b
from paper_1506_01446_b200 import _native

n = 1 << 20
src = np.random.default_rng(1).integers(0, 2**32, n, dtype=np.uint64).astype(np.uint32)
t = torch.empty(n, dtype=torch.int32).pin_memory()
arr = t.numpy().view(np.uint32)
L = _native.lib()
ptr = ctypes.c_void_p(arr.ctypes.data)


def run(name, fn, prep):
    ts = []
    for r in range(40):
        prep()
        c0 = time.perf_counter()
        fn()
        ts.append((time.perf_counter() - c0) * 1e6)
    ts = sorted(ts[5:])
    print(f"{name:40s} median {ts[len(ts)//2]:7.1f} us  min {ts[0]:7.1f} us", flush=True)

np_prep = lambda: np.copyto(arr, src)
torch_prep = lambda: (t.copy_(torch.from_numpy(src.view(np.int32))), torch.cuda.synchronize())
run("sort_host (np prep)", lambda: b.sort_host(arr), np_prep)
run("raw ctypes (np prep)", lambda: L.b200_bitonic_sort_host_u32(ptr, n, 0), np_prep)
run("sort_host (torch prep + sync)", lambda: b.sort_host(arr), torch_prep)
run("raw ctypes (torch prep + sync)", lambda: L.b200_bitonic_sort_host_u32(ptr, n, 0), torch_prep)
