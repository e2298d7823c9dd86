"""Device-timed 64-bit key sort sweep (development tool, not the bench contract).
Times the interleaved int64 entry (split + planes sort + join) and the planes
entry alone, against torch.sort (CUB radix) for context."""
import argparse, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1506_01446_b200 as b

ap = argparse.ArgumentParser()
ap.add_argument("--ks", default="16,20,24,28")
ap.add_argument("--reps", type=int, default=8)
args = ap.parse_args()
dev = torch.device("cuda:0")
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)


def timeit(fn, reset, reps):
    ts = []
    for r in range(reps + 2):
        reset(); flush.zero_()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        if r >= 2:
            ts.append(e0.elapsed_time(e1) * 1e-3)
    ts.sort()
    return ts[0], ts[len(ts) // 2]


for k in [int(x) for x in args.ks.split(",")]:
    n = 1 << k
    g = torch.Generator(device=dev).manual_seed(k)
    src = torch.randint(-2**62, 2**62, (n,), dtype=torch.int64, device=dev, generator=g)
    w = src.clone()
    t64 = timeit(lambda: b.sort_(w), lambda: w.copy_(src), args.reps)
    ok = bool(torch.equal(w, torch.sort(src).values))
    hi = (src >> 32).to(torch.int32).view(torch.uint32).clone()
    lo = src.to(torch.int32).view(torch.uint32).clone()
    h, l = hi.clone(), lo.clone()
    tpl = timeit(lambda: b.sort_planes_(h, l), lambda: (h.copy_(hi), l.copy_(lo)), args.reps)
    tts = timeit(lambda: torch.sort(w), lambda: w.copy_(src), args.reps)
    print(f"k={k} int64 {t64[1]*1e3:.3f} ms ({n/t64[1]/1e9:.2f} Gkeys/s) ok={ok} | "
          f"planes {tpl[1]*1e3:.3f} ms ({n/tpl[1]/1e9:.2f}) | torch.sort {tts[1]*1e3:.3f} ms",
          flush=True)
