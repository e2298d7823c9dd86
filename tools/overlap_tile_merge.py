"""Probe: does an ALU-bound tile sort overlap with HBM-bound merge passes?

Quarter Q0 runs its merge passes (phases 14..26 of a 2^26-key sub-sort) on
stream A while quarter Q1 runs its tile sort on stream B.  Compares the
concurrent time with the two run back to back (CUDA events, L2 flushed).
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1506_01446_b200 as b  # noqa: E402

dev = torch.device("cuda:0")
K = int(os.environ.get("K", "26"))
n = 1 << K
src = torch.randint(-2**31, 2**31, (4 * n,), dtype=torch.int64, device=dev).to(torch.int32)
work = src.clone().view(torch.uint32)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
plan = b.plan(n)
q0, q1 = work[:n], work[n:2 * n]
sa, sb = torch.cuda.Stream(), torch.cuda.Stream()


def prep():
    work.copy_(src.view(torch.uint32))
    b.run_pass_(q0, 0)  # q0's tile sort done up front
    flush.zero_()
    torch.cuda.synchronize()


def merges(t, s):
    for i in range(1, len(plan)):
        b.run_pass_(t, i, stream=s)


def timed(fn):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    cur = torch.cuda.current_stream()
    torch.cuda._sleep(2_000_000)
    e0.record(cur)
    sa.wait_stream(cur)
    sb.wait_stream(cur)
    fn()
    cur.wait_stream(sa)
    cur.wait_stream(sb)
    e1.record(cur)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


for rep in range(4):
    prep()
    t_tile = timed(lambda: b.run_pass_(q1, 0, stream=sb))
    prep()
    t_merge = timed(lambda: merges(q0, sa))
    prep()

    def both():
        b.run_pass_(q1, 0, stream=sb)
        merges(q0, sa)
    t_both = timed(both)
    prep()

    def both2():
        merges(q0, sa)
        b.run_pass_(q1, 0, stream=sb)
    t_both2 = timed(both2)
    print(f"K={K} tile {t_tile:.3f} ms  merges({len(plan) - 1}) {t_merge:.3f} ms  "
          f"serial {t_tile + t_merge:.3f}  concurrent(tile first) {t_both:.3f}  "
          f"concurrent(merges first) {t_both2:.3f}", flush=True)
