import sys, torch, numpy as np
sys.path.insert(0, '/root/repo')
import paper_1506_01446_b200 as b
dev = torch.device('cuda:0'); n = 1 << 20
src = torch.randint(-2**31, 2**31, (n,), dtype=torch.int64, device=dev).to(torch.int32).view(torch.uint32)
work = src.clone(); flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
s = torch.cuda.current_stream()
for mode in ["nosync_sleep", "nosync", "sync_each", "sync_sleep", "noflush"]:
    for _ in range(5): work.copy_(src); b.sort_(work)
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(20)]
    for i in range(20):
        work.copy_(src)
        if mode != "noflush": flush.zero_()
        if "sleep" in mode: torch.cuda._sleep(100_000)
        evs[i][0].record(s); b.sort_(work); evs[i][1].record(s)
        if "sync" in mode and not mode.startswith("nosync"): torch.cuda.synchronize()
    torch.cuda.synchronize()
    t = sorted(a.elapsed_time(c) * 1e3 for a, c in evs)
    print(mode, "min %.1f med %.1f max %.1f mean %.1f" % (t[0], t[10], t[-1], sum(t) / 20))
