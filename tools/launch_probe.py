"""Separate GPU execution time from host launch overhead (dev tool)."""
import sys, os, json
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1506_01446_b200 as b
dev = torch.device("cuda:0")
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
for k in [16, 20, 24]:
    n = 1 << k
    src = torch.randint(-2**31, 2**31, (n,), dtype=torch.int64, device=dev).to(torch.int32).view(torch.uint32)
    work = src.clone()
    res = {}
    for mode in ["plain", "sleep", "graph"]:
        if mode == "graph":
            s = torch.cuda.Stream()
            s.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s):
                b.sort_(work)  # warm
            torch.cuda.current_stream().wait_stream(s)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                b.sort_(work)
        ts = []
        for r in range(12):
            work.copy_(src); flush.zero_()
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            if mode == "sleep": torch.cuda._sleep(2_000_000)
            e0.record()
            if mode == "graph": g.replay()
            else: b.sort_(work)
            e1.record(); torch.cuda.synchronize()
            if r >= 2: ts.append(e0.elapsed_time(e1))
        ok = torch.equal(work.view(torch.int32).to(torch.int64) & 0xFFFFFFFF, torch.sort(src.view(torch.int32).to(torch.int64) & 0xFFFFFFFF).values)
        res[mode] = (round(min(ts)*1e3, 1), round(sorted(ts)[len(ts)//2]*1e3, 1), ok)
    print(k, json.dumps(res), flush=True)
