mkdir -p gpurun_out/mp14
cat > /tmp/mp_time.py <<'PY'
import torch, numpy as np, json, sys, os
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import paper_1506_01446_b200 as b
dev = torch.device("cuda:0")
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
for k in (24, 28, 30):
    n = 1 << k
    src = torch.from_numpy(b.generate_input(n, 1).view(np.int32)).to(dev).view(torch.uint32)
    work = src.clone(); ts = []
    for r in range(8):
        work.copy_(src); flush.zero_(); torch.cuda._sleep(200000)
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); b.sort_mergepath_(work); e1.record(); torch.cuda.synchronize()
        if r >= 2: ts.append(e0.elapsed_time(e1))
    ref = torch.sort(src.view(torch.int32).to(torch.int64) & 0xFFFFFFFF).values
    ok = torch.equal(work.view(torch.int32).to(torch.int64) & 0xFFFFFFFF, ref); del ref
    print(json.dumps(dict(tr=os.environ.get("B200_BITONIC_MERGEPATH_TILE_R", "5"), tc=os.environ.get("B200_BITONIC_MERGEPATH_TILE", "14"), k=k, ms=min(ts), med=float(np.median(ts)), ok=ok)), flush=True)
PY
for TR in 5 4 6; do for TC in 14 13; do
  B200_BITONIC_MERGEPATH_TILE_R=$TR B200_BITONIC_MERGEPATH_TILE=$TC python /tmp/mp_time.py >> gpurun_out/mp14/time.log 2>&1
done; done
