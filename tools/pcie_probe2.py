"""Repeatable breakdown of the 2^20 end-to-end step (H2D + sort + D2H)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1506_01446_b200 as b

dev = torch.device("cuda:0")
n = 1 << int(os.environ.get("K", "20"))
h = torch.randint(0, 2**31, (n,), dtype=torch.int32).pin_memory()
ho = torch.empty_like(h).pin_memory()
d = torch.empty(n, dtype=torch.int32, device=dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
cases = {
    "sort": lambda: b.sort_(d),
    "h2d": lambda: d.copy_(h, non_blocking=True),
    "d2h": lambda: ho.copy_(d, non_blocking=True),
    "h2d+sort": lambda: (d.copy_(h, non_blocking=True), b.sort_(d)),
    "sort+d2h": lambda: (b.sort_(d), ho.copy_(d, non_blocking=True)),
    "all": lambda: (d.copy_(h, non_blocking=True), b.sort_(d), ho.copy_(d, non_blocking=True)),
}
res = {c: [] for c in cases}
for pdl in (1, 0):
    b.set_tuning(0, 5 if pdl else 1005)
    res = {c: [] for c in cases}
    for rep in range(12):
        for c, fn in cases.items():
            for fl in (0, 1):
                if fl:
                    flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(); fn(); e1.record(); torch.cuda.synchronize()
                if rep >= 2:
                    res[c].append((fl, e0.elapsed_time(e1) * 1e3))
    for c, v in res.items():
        a = sorted(x for f, x in v if f == 0)
        bb = sorted(x for f, x in v if f == 1)
        print(f"pdl={pdl} {c:9s} noflush min {a[0]:7.1f} med {a[len(a)//2]:7.1f} | "
              f"flush min {bb[0]:7.1f} med {bb[len(bb)//2]:7.1f} max {bb[-1]:7.1f}", flush=True)
