"""Quick device-timed sweep (development tool, not the bench contract)."""
import argparse, sys, os, json
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1506_01446_b200 as b

ap = argparse.ArgumentParser()
ap.add_argument("--ks", default="16,20,24,28")
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--tiles", default="0")
ap.add_argument("--runs", default="5")
ap.add_argument("--batched", action="store_true")
args = ap.parse_args()
dev = torch.device("cuda:0")
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
HBM = 6556.5e9
PMIN = {16: 3, 20: 7, 24: 13, 28: 21, 30: 24}

def timeit(fn, src, work, reps):
    ts = []
    for r in range(reps + 2):
        work.copy_(src); flush.zero_()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        if r >= 2: ts.append(e0.elapsed_time(e1) * 1e-3)
    return min(ts), float(np.median(ts))

res = []
for tile in [int(x) for x in args.tiles.split(",")]:
    for run in [int(x) for x in args.runs.split(",")]:
        b.set_tuning(tile, run)
        for k in [int(x) for x in args.ks.split(",")]:
            n = 1 << k
            g = torch.Generator(device=dev); g.manual_seed(1)
            src = torch.randint(-2**31, 2**31, (n,), dtype=torch.int64, device=dev, generator=g).to(torch.int32).view(torch.uint32)
            work = src.clone()
            tmin, tmed = timeit(lambda: b.sort_(work), src, work, args.reps)
            ok = bool(torch.equal(work.view(torch.int32).to(torch.int64) & 0xFFFFFFFF, torch.sort(src.view(torch.int32).to(torch.int64) & 0xFFFFFFFF).values))
            P = len(b.plan(n))
            troof = PMIN.get(k, P) * 8 * n / HBM
            r = dict(k=k, tile=tile, run=run, passes=P, ms_min=tmin*1e3, ms_med=tmed*1e3, gkeys=n/tmin/1e9, frac=troof/tmin, ok=ok,
                     gbps_design=P*8*n/tmin/1e9)
            print(json.dumps(r), flush=True); res.append(r)
        if args.batched:
            n = 1 << 24
            src = torch.randint(-2**31, 2**31, (n,), dtype=torch.int64, device=dev).to(torch.int32).view(torch.uint32)
            work = src.clone()
            tmin, tmed = timeit(lambda: b.sort_batched_(work, 4096), src, work, args.reps)
            r = dict(k="batched4096x4096", tile=tile, ms_min=tmin*1e3, ms_med=tmed*1e3, gkeys=n/tmin/1e9, frac=(8*n/HBM)/tmin)
            print(json.dumps(r), flush=True)
