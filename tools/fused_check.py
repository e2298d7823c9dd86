"""Check the cluster-fused prefix at 2^13..2^21 (debug probe)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1506_01446_b200 as b
for k in [int(x) for x in (sys.argv[1:] or ["13", "14", "15", "16", "17", "20"])]:
    n = 1 << k
    t = torch.randint(-2**31, 2**31 - 1, (n,), dtype=torch.int32, device="cuda")
    want = torch.sort(t).values
    try:
        b.sort_(t)
        torch.cuda.synchronize()
        ok = torch.equal(t, want)
        bad = (t != want).nonzero()
        print(k, "ok" if ok else f"MISMATCH {bad.numel()} first {bad[:3].flatten().tolist()}", flush=True)
    except Exception as e:
        print(k, "ERROR", repr(e)[:300], flush=True)
        break
