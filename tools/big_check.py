"""Sort 2^30..2^32 keys on one B200 and check sortedness + multiset fingerprint."""
import sys, os, time, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1506_01446_b200 as b
dev = torch.device("cuda:0")
def fp(t):
    # chunked int64 fingerprints (sum, sum of squares, sum of a mixed hash)
    s1 = s2 = s3 = 0
    for c in t.view(torch.int32).split(1 << 27):
        v = c.to(torch.int64) & 0xFFFFFFFF
        m = (v * 0x9E3779B1 + 0x7F4A7C15) & 0xFFFFFFFF
        s1 += int(v.sum()); s2 += int((v * v).sum() & ((1 << 62) - 1)); s3 += int(m.sum())
    return s1, s2 % (1 << 62), s3
def sorted_ok(t, desc=False):
    v = t.view(torch.int32)
    ok = True
    step = 1 << 27
    for i in range(0, t.numel() - 1, step):
        a = v[i:i + step + 1].to(torch.int64) & 0xFFFFFFFF
        d = a[1:] - a[:-1]
        ok &= bool((d <= 0).all()) if desc else bool((d >= 0).all())
    return ok
for k in [int(x) for x in (sys.argv[1:] or ["30", "31", "32"])]:
    n = 1 << k
    t = torch.empty(n, dtype=torch.int32, device=dev)
    g = torch.Generator(device=dev); g.manual_seed(k)
    for c in t.split(1 << 28):
        c.copy_(torch.randint(-2**31, 2**31, (c.numel(),), dtype=torch.int64, device=dev, generator=g).to(torch.int32))
    t = t.view(torch.uint32)
    f0 = fp(t)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); b.sort_(t); e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    ok = sorted_ok(t) and fp(t) == f0
    b.sort_(t, descending=True); torch.cuda.synchronize()
    ok2 = sorted_ok(t, True) and fp(t) == f0
    print(f"k={k} passes={len(b.plan(n))} ms={ms:.1f} Gkeys/s={n/ms/1e6:.2f} asc_ok={ok} desc_ok={ok2}", flush=True)
    del t; torch.cuda.empty_cache()
