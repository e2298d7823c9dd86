"""Threaded one-GPU emulation of dist.partitioned_sort_ at given sizes (debug probe)."""
import os, sys, queue, threading
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1506_01446_b200 import dist as bdist

dev = torch.device("cuda:0")


def run(world, log2m, stride, serial_sort=False):
  m = 1 << log2m
  g = torch.Generator(device=dev).manual_seed(world)
  full = torch.randint(-2**31, 2**31, (world * m,), dtype=torch.int64, device=dev,
                       generator=g).to(torch.int32).view(torch.uint32)
  want = torch.sort(full.view(torch.int32).to(torch.int64) & 0xFFFFFFFF).values
  shards = [full[r * m:(r + 1) * m] for r in range(world)]
  boxes = {(a, b): queue.Queue() for a in range(world) for b in range(world)}
  errors = []
  lock = threading.Lock()


  def worker(r, shard):
      try:
          torch.cuda.set_device(0)
          s = torch.cuda.Stream()
          with torch.cuda.stream(s):
              def exchange(snd, rcv, partner, group):
                  s.synchronize()
                  mine = snd.clone()
                  s.synchronize()
                  boxes[(r, partner)].put(mine)
                  got = boxes[(partner, r)].get(timeout=120)
                  assert got.numel() == rcv.numel(), (r, partner, got.numel(), rcv.numel())
                  rcv.copy_(got.view(rcv.dtype))
                  s.synchronize()
              ops = bdist.cuda_ops()
              ops.exchange = exchange
              if serial_sort:
                  base = ops.local_sort
                  def ls(t, d):
                      with lock:
                          base(t, d)
                          s.synchronize()
                  ops.local_sort = ls
              bdist.partitioned_sort_(shard, ops=ops, rank=r, world=world, sample_stride=stride)
              s.synchronize()
      except Exception as e:
          errors.append((r, repr(e)[:300]))

  torch.cuda.synchronize()  # worker streams do not wait for the default stream
  ts = [threading.Thread(target=worker, args=(r, shards[r])) for r in range(world)]
  for t in ts: t.start()
  for t in ts: t.join()
  torch.cuda.synchronize()
  ok = torch.equal(full.view(torch.int32).to(torch.int64) & 0xFFFFFFFF, want)
  print(world, log2m, stride, "serial" if serial_sort else "", "ok" if ok and not errors else f"FAIL {errors[:2]}", flush=True)


for spec in sys.argv[1:]:
    parts = spec.split(",")
    run(int(parts[0]), int(parts[1]), int(parts[2]), len(parts) > 3)
