"""Host<->device copy bandwidth on the box (pinned buffers), to bound e2e."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1506_01446_b200 as b

dev = torch.device("cuda:0")
s = torch.cuda.current_stream()


def t(fn, reps=20):
    ts = []
    for r in range(reps + 3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        if r >= 3:
            ts.append(e0.elapsed_time(e1))
    ts.sort()
    return ts[len(ts) // 2]


for k in (16, 20, 24, 26):
    n = 1 << k
    h = torch.randint(0, 2**31, (n,), dtype=torch.int32).pin_memory()
    ho = torch.empty_like(h).pin_memory()
    d = torch.empty(n, dtype=torch.int32, device=dev)
    th = t(lambda: d.copy_(h, non_blocking=True))
    td = t(lambda: ho.copy_(d, non_blocking=True))
    tsrt = t(lambda: (d.copy_(h, non_blocking=True), b.sort_(d), ho.copy_(d, non_blocking=True)))
    print(f"k={k} H2D {th*1e3:.1f} us ({4*n/th/1e6:.1f} GB/s)  D2H {td*1e3:.1f} us "
          f"({4*n/td/1e6:.1f} GB/s)  h2d+sort+d2h {tsrt*1e3:.1f} us", flush=True)

print("--- k=20 breakdown")
n = 1 << 20
h = torch.randint(0, 2**31, (n,), dtype=torch.int32).pin_memory()
ho = torch.empty_like(h).pin_memory()
d = torch.empty(n, dtype=torch.int32, device=dev)
for pdl in (True, False):
    b.set_tuning(0, 5 if pdl else 1005)
    print("pdl", pdl,
          "sort %.1f" % (t(lambda: b.sort_(d)) * 1e3),
          "h2d+sort %.1f" % (t(lambda: (d.copy_(h, non_blocking=True), b.sort_(d))) * 1e3),
          "sort+d2h %.1f" % (t(lambda: (b.sort_(d), ho.copy_(d, non_blocking=True))) * 1e3),
          "h2d+d2h %.1f" % (t(lambda: (d.copy_(h, non_blocking=True), ho.copy_(d, non_blocking=True))) * 1e3),
          "all %.1f" % (t(lambda: (d.copy_(h, non_blocking=True), b.sort_(d), ho.copy_(d, non_blocking=True))) * 1e3),
          flush=True)
b.set_tuning(0, 5)
import time
for _ in range(3):
    torch.cuda.synchronize(); c0 = time.perf_counter()
    for _ in range(100):
        b.sort_(d)
    c1 = time.perf_counter(); torch.cuda.synchronize(); c2 = time.perf_counter()
    print("host us per sort_ call %.1f, wall per sort %.1f" % ((c1 - c0) * 1e4, (c2 - c0) * 1e4))
