"""Per-pass device times of the sort plan (development tool).

Each pass of the plan runs back to back on one stream with an event between
consecutive passes (L2 flushed, a device sleep so the host enqueues ahead);
prints pass shape, mean microseconds and algorithmic GB/s (8 bytes per key).
    K=28 python tools/pass_times.py
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1506_01446_b200 as b  # noqa: E402

dev = torch.device("cuda:0")
k = int(os.environ.get("K", "28"))
reps = int(os.environ.get("REPS", "5"))
n = 1 << k
src = torch.randint(-2**31, 2**31, (n,), dtype=torch.int64, device=dev).to(torch.int32).view(torch.uint32)
work = src.clone()
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
plan = b.plan(n)
tot = [0.0] * len(plan)
for r in range(reps + 1):
    work.copy_(src)
    flush.zero_()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(len(plan) + 1)]
    torch.cuda._sleep(8_000_000)
    ev[0].record()
    for i in range(len(plan)):
        b.run_pass_(work, i)
        ev[i + 1].record()
    torch.cuda.synchronize()
    if r:
        for i in range(len(plan)):
            tot[i] += ev[i].elapsed_time(ev[i + 1]) / reps
ok = torch.equal(work.view(torch.int32).to(torch.int64) & 0xFFFFFFFF,
                 torch.sort(src.view(torch.int32).to(torch.int64) & 0xFFFFFFFF).values)
s = 0.0
for p, t in zip(plan, tot):
    s += t
    kind = "tile" if p.tile_sort else ("cluster" if p.cluster == 2 else "merge")
    print(f"{kind:8s} C={p.tile_bits:2d} a={p.a:2d} y={p.y:2d} SA={p.segA_hi:3d} SB={p.segB_lo:3d} "
          f"{t * 1e3:9.1f} us  {8 * n / (t * 1e-3) / 1e9:7.0f} GB/s")
print(json.dumps({"k": k, "passes": len(plan), "sum_ms": s, "ok": ok,
                  "env": {x: os.environ[x] for x in os.environ if x.startswith("B200_")}}))
