"""Device-timed key-value sort throughput (dev tool)."""
import sys, os, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1506_01446_b200 as b
dev = torch.device("cuda:0")
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
for k in [int(x) for x in (sys.argv[1:] or ["16", "20", "24", "28"])]:
    n = 1 << k
    ks = torch.randint(-2**31, 2**31, (n,), dtype=torch.int64, device=dev).to(torch.int32).view(torch.uint32)
    vs = torch.arange(n, dtype=torch.int32, device=dev).view(torch.uint32)
    wk, wv = ks.clone(), vs.clone()
    ts = []
    for r in range(8):
        wk.copy_(ks); wv.copy_(vs); flush.zero_()
        torch.cuda._sleep(100_000)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); b.sort_pairs_(wk, wv); e1.record(); torch.cuda.synchronize()
        if r >= 2: ts.append(e0.elapsed_time(e1))
    ok = torch.equal(ks.view(torch.int32)[wv.view(torch.int32).long()], wk.view(torch.int32))
    ms = min(ts)
    print(f"pairs k={k} passes={len(b.plan(n))} ms={ms:.4f} Gpairs/s={n/ms/1e6:.2f} ok={ok}", flush=True)
