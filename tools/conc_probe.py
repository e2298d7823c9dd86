"""Concurrent sorts from several host threads on several streams (debug probe)."""
import os, sys, threading
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1506_01446_b200 as b

dev = torch.device("cuda:0")
mode = sys.argv[1]
T, k, reps = int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
n = 1 << k
full = torch.empty(T * n, dtype=torch.int32, device=dev)
errs = []


def worker(r):
    torch.cuda.set_device(0)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        x = full[r * n:(r + 1) * n]
        for i in range(reps):
            x.random_(-2**31, 2**31 - 1)
            w = torch.sort(x).values
            if mode == "sort":
                b.sort_(x)
            elif mode == "merge":
                h = n // 2
                a = torch.sort(x[:h]).values
                c = torch.sort(x[h:]).values
                b.merge_(a.view(torch.uint32), c.view(torch.uint32), x.view(torch.uint32), 0x80000000)
            s.synchronize()
            if not torch.equal(x, w):
                errs.append((r, i))

for rep in range(2):
    ts = [threading.Thread(target=worker, args=(r,)) for r in range(T)]
    for t in ts: t.start()
    for t in ts: t.join()
    torch.cuda.synchronize()
    print(mode, T, k, "round", rep, "errors", errs[:5], flush=True)
