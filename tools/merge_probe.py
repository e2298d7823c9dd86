"""Merge-path kernel throughput (merge_split_ / merge_): 8 bytes per output
key (each output key read once from A or B, written once), device-timed."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1506_01446_b200 as b  # noqa: E402

dev = torch.device("cuda:0")
for lg in [int(x) for x in os.environ.get("LOGS", "24,27,29").split(",")]:
    m = 1 << lg
    a = torch.sort(torch.randint(0, 2**31, (m,), device=dev, dtype=torch.int64)).values.to(torch.int32).view(torch.uint32)
    c = torch.sort(torch.randint(0, 2**31, (m,), device=dev, dtype=torch.int64)).values.to(torch.int32).view(torch.uint32)
    out = torch.empty(m, dtype=torch.uint32, device=dev)
    ref = torch.sort(torch.cat([a.view(torch.int32), c.view(torch.int32)])).values
    for kh in (0, 1):
        b.merge_split_(a, c, out, bool(kh))
        torch.cuda.synchronize()
        want = ref[m:] if kh else ref[:m]
        ok = torch.equal(out.view(torch.int32), want)
        ts = []
        for r in range(6):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            b.merge_split_(a, c, out, bool(kh))
            e1.record()
            torch.cuda.synchronize()
            if r:
                ts.append(e0.elapsed_time(e1))
        t = min(ts)
        print(f"merge_split m=2^{lg} keep_high={kh}: {t * 1e3:.1f} us, {8 * m / (t * 1e-3) / 1e9:.0f} GB/s, ok={ok}", flush=True)
    del a, c, out, ref
    torch.cuda.empty_cache()
