"""Debug probe: allocate/map the IPC shard buffers at a given size across
2 processes on one GPU (gloo) and report errors."""
import os, sys
import torch
import torch.distributed as dist
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1506_01446_b200 import dist as bdist

dist.init_process_group("gloo")
rank, world = dist.get_rank(), dist.get_world_size()
torch.cuda.set_device(0)
for lg in [int(x) for x in sys.argv[1:]]:
    try:
        b = bdist.PeerShards(1 << lg, 4, None, rank, world)
        print(rank, lg, "ok", flush=True)
        dist.barrier()
        b.close()
    except Exception as e:
        print(rank, lg, "FAIL", repr(e)[:300], flush=True)
    dist.barrier()
