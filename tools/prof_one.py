"""Run one sort config a few times (for ncu captures)."""
import argparse, sys, os
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1506_01446_b200 as b
ap = argparse.ArgumentParser()
ap.add_argument("--k", type=int, default=20)
ap.add_argument("--batched", type=int, default=0, help="n_per_array (0 = single array)")
ap.add_argument("--iters", type=int, default=2)
ap.add_argument("--tile", type=int, default=0)
ap.add_argument("--run", type=int, default=5)
a = ap.parse_args()
b.set_tuning(a.tile, a.run)
n = 1 << a.k
src = torch.randint(-2**31, 2**31, (n,), dtype=torch.int64, device="cuda").to(torch.int32).view(torch.uint32)
w = src.clone()
for _ in range(a.iters):
    w.copy_(src)
    if a.batched: b.sort_batched_(w, a.batched)
    else: b.sort_(w)
torch.cuda.synchronize()
ok = torch.equal(w.view(torch.int32).to(torch.int64) & 0xFFFFFFFF,
                 (torch.sort((src.view(torch.int32).to(torch.int64) & 0xFFFFFFFF).view(-1, a.batched or n), dim=1).values).view(-1))
print("ok", ok)
