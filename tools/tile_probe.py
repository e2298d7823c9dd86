"""Time pass 0 (the tile sort) alone vs the whole sort (development probe)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1506_01446_b200 as b

dev = torch.device("cuda:0")
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
for k in [int(x) for x in sys.argv[1:]]:
    n = 1 << k
    src = torch.randint(0, 2**31, (n,), dtype=torch.int32, device=dev).view(torch.uint32)
    w = src.clone()

    def t(fn):
        ts = []
        for r in range(25):
            w.copy_(src); flush.zero_()
            torch.cuda._sleep(50_000)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); fn(); e1.record(); torch.cuda.synchronize()
            if r >= 5:
                ts.append(e0.elapsed_time(e1) * 1e3)
        ts.sort()
        return ts[len(ts) // 2]
    print(f"k={k} TILE_REGBITS={os.environ.get('B200_BITONIC_TILE_REGBITS', '-')} "
          f"tile pass {t(lambda: b.run_pass_(w, 0)):.1f} us, merge pass 1 {t(lambda: b.run_pass_(w, 1)):.1f} us, "
          f"whole sort {t(lambda: b.sort_(w)):.1f} us", flush=True)
