"""Do two half-size sorts on two streams overlap (ALU-bound tile sort of one
with HBM-bound merges of the other)?  Development probe."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1506_01446_b200 as b

dev = torch.device("cuda:0")
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
for k in (24, 26, 28):
    n = 1 << k
    src = torch.randint(-2**31, 2**31 - 1, (n,), dtype=torch.int32, device=dev)
    w = src.clone()
    h = n // 2
    s0 = torch.cuda.current_stream()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def seq():
        b.sort_(w[:h]); b.sort_(w[h:], descending=True)

    def par():
        s1.wait_stream(s0); s2.wait_stream(s0)
        with torch.cuda.stream(s1):
            b.sort_(w[:h])
        with torch.cuda.stream(s2):
            b.sort_(w[h:], descending=True)
        s0.wait_stream(s1); s0.wait_stream(s2)

    def full():
        b.sort_(w)

    def batched():
        b.sort_batched_(w, h)

    for name, fn in (("full", full), ("2 halves seq", seq), ("2 halves par", par), ("batched x2", batched)):
        ts = []
        for r in range(8):
            w.copy_(src); flush.zero_()
            torch.cuda._sleep(100_000)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); fn(); e1.record(); torch.cuda.synchronize()
            if r >= 2:
                ts.append(e0.elapsed_time(e1))
        ts.sort()
        print(f"k={k} {name:14s} {ts[len(ts)//2]:.3f} ms", flush=True)
