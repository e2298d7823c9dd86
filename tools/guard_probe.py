"""Out-of-bounds write check: sort views with sentinel guard regions."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1506_01446_b200 as b

dev = torch.device("cuda:0")
G = 1 << 16
bad = []
for k in list(range(1, 29)):
    n = 1 << k
    buf = torch.full((n + 2 * G,), 0x5A5A5A5A, dtype=torch.int32, device=dev)
    mid = buf[G:G + n]
    mid.random_(-2**31, 2**31 - 1)
    want = torch.sort(mid).values
    b.sort_(mid)
    torch.cuda.synchronize()
    ok = torch.equal(mid, want)
    g_ok = bool((buf[:G] == 0x5A5A5A5A).all()) and bool((buf[G + n:] == 0x5A5A5A5A).all())
    if not ok or not g_ok:
        bad.append((k, ok, g_ok))
    # merge_ of two halves into a guarded output
    if k >= 2:
        a = torch.sort(torch.randint(-2**31, 2**31 - 1, (n // 2,), dtype=torch.int32, device=dev)).values
        c = torch.sort(torch.randint(-2**31, 2**31 - 1, (n // 2,), dtype=torch.int32, device=dev)).values
        ob = torch.full((n + 2 * G,), 0x5A5A5A5A, dtype=torch.int32, device=dev)
        out = ob[G:G + n]
        b.merge_(a.view(torch.uint32), c.view(torch.uint32), out.view(torch.uint32), 0x80000000)
        torch.cuda.synchronize()
        g2 = bool((ob[:G] == 0x5A5A5A5A).all()) and bool((ob[G + n:] == 0x5A5A5A5A).all())
        ok2 = torch.equal(out, torch.sort(torch.cat([a, c])).values)
        if not (g2 and ok2):
            bad.append(("merge", k, ok2, g2))
print("bad:", bad)
