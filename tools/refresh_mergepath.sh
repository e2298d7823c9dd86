#!/bin/bash
# Evidence for the merge-path variant (profiles/r2_mergepath_*): launch list
# and full ncu capture of one 2^28-key sort, and bench lines carrying the
# variant beside the headline.  Run on the GPU box through gpurun.
set -u
OUT=gpurun_out/mpref
mkdir -p $OUT
cat > /tmp/mp_once.py <<'PY'
import os, sys
import numpy as np, torch
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import paper_1506_01446_b200 as b
n = 1 << int(os.environ.get("K", "28"))
t = torch.from_numpy(b.generate_input(n, 1).view(np.int32)).cuda().view(torch.uint32)
b.sort_mergepath_(t)
torch.cuda.synchronize()
PY
python /tmp/mp_once.py || exit 1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k "regex:tile_sort|mergepath" --csv python /tmp/mp_once.py > $OUT/launches_k28.csv 2>&1
ncu --set full --clock-control none --import-source on -k regex:mergepath -s 2 -c 2 \
    -o $OUT/full_k28 python /tmp/mp_once.py > $OUT/full.log 2>&1
python bench.py > $OUT/bench_k28.json 2> $OUT/bench_k28.err
python bench.py --log2n 30 --steps 5 --no-cpu-baseline > $OUT/bench_k30.json 2> $OUT/bench_k30.err
python bench.py --log2n 24 --no-cpu-baseline > $OUT/bench_k24.json 2> $OUT/bench_k24.err
