"""Long randomized cross-check of every device entry point against numpy
(development tool; run on a GPU box: python tools/fuzz.py SECONDS [SEED [KMAX]])."""
import os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1506_01446_b200 as b

dev = torch.device("cuda:0")
budget = float(sys.argv[1]) if len(sys.argv) > 1 else 120
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 7)
kmax = int(sys.argv[3]) if len(sys.argv) > 3 else 23  # largest log2 length
t0 = time.time()
n_cases = 0
fails = []


def tot64(u):
    return np.where(u >> np.uint64(63) == 1, ~u, u | np.uint64(1 << 63))


while time.time() - t0 < budget:
    kind = rng.choice(["sort", "mergepath", "padded", "batched", "pairs", "f32", "i64", "f64",
                       "planes"])
    desc = bool(rng.integers(0, 2))
    k = int(rng.integers(1, kmax + 1))
    n = 1 << k
    try:
        if kind in ("sort", "mergepath", "padded", "batched", "pairs"):
            dt = np.int32 if rng.integers(0, 2) else np.uint32
            if kind == "padded":
                n = int(rng.integers(1, 1 << 23))
            x = rng.integers(0, 2**32, n, dtype=np.uint64).astype(np.uint32)
            if rng.random() < 0.3:
                x = (x % np.uint32(rng.integers(1, 8))).astype(np.uint32)
            x = x.view(dt)
            t = torch.from_numpy(x.view(np.int32).copy()).to(dev)
            tv = t.view(torch.uint32) if dt == np.uint32 else t
            if kind == "sort":
                b.sort_(tv, descending=desc); want = np.sort(x)
            elif kind == "mergepath":
                b.sort_mergepath_(tv, descending=desc); want = np.sort(x)
            elif kind == "padded":
                b.sort_padded_(tv, descending=desc); want = np.sort(x)
            elif kind == "batched":
                per = 1 << int(rng.integers(1, k + 1))
                b.sort_batched_(tv, per, descending=desc)
                want = np.sort(x.reshape(-1, per), axis=1)
                if desc:
                    want = want[:, ::-1]
                want = want.reshape(-1)
                desc = False
            else:
                vals = torch.arange(n, dtype=torch.int32, device=dev).view(torch.uint32)
                b.sort_pairs_(tv, vals, descending=desc); want = np.sort(x)
                got_v = vals.view(torch.int32).cpu().numpy()
                if not (np.sort(got_v) == np.arange(n)).all():
                    raise AssertionError("payload not a permutation")
                if not (x[got_v] == t.cpu().numpy().view(dt)).all():
                    raise AssertionError("payload does not follow its key")
            if desc:
                want = want[::-1]
            got = t.cpu().numpy().view(dt)
        elif kind == "f32":
            x = (rng.standard_normal(n) * 10).astype(np.float32)
            t = torch.from_numpy(x.copy()).to(dev)
            b.sort_(t, descending=desc)
            u = x.view(np.uint32)
            key = u ^ np.where(u >> 31 == 1, np.uint32(0xFFFFFFFF), np.uint32(0x80000000))
            want = x[np.argsort(key, kind="stable")]
            if desc:
                want = want[::-1]
            got = t.cpu().numpy()
        else:
            k = min(k, 22); n = 1 << k
            if kind == "f64":
                x = rng.standard_normal(n) * 10
                t = torch.from_numpy(x.copy()).to(dev)
                b.sort_(t, descending=desc)
                want = x[np.argsort(tot64(x.view(np.uint64)), kind="stable")]
                got = t.cpu().numpy()
            elif kind == "i64":
                x = rng.integers(-2**63, 2**63 - 1, n, dtype=np.int64)
                t = torch.from_numpy(x.copy()).to(dev)
                b.sort_(t, descending=desc); want = np.sort(x); got = t.cpu().numpy()
            else:
                x = rng.integers(0, 2**64 - 1, n, dtype=np.uint64)
                hi = torch.from_numpy((x >> np.uint64(32)).astype(np.uint32).view(np.int32)).to(dev)
                lo = torch.from_numpy((x & np.uint64(0xFFFFFFFF)).astype(np.uint32).view(np.int32)).to(dev)
                b.sort_planes_(hi.view(torch.uint32), lo.view(torch.uint32), descending=desc)
                got = ((hi.cpu().numpy().view(np.uint32).astype(np.uint64) << np.uint64(32))
                       | lo.cpu().numpy().view(np.uint32).astype(np.uint64))
                want = np.sort(x)
            if desc:
                want = want[::-1]
        if not (np.ascontiguousarray(got).view(np.uint8) == np.ascontiguousarray(want).view(np.uint8)).all():
            fails.append((kind, n, desc))
    except Exception as e:
        fails.append((kind, n, desc, repr(e)[:120]))
    n_cases += 1
print(f"fuzz: {n_cases} cases in {time.time() - t0:.0f} s, {len(fails)} failures", fails[:10])
