#!/bin/bash
mkdir -p gpurun_out/shfl
for v in base shfl; do
  if [ $v = base ]; then L=""; else L="B200_BITONIC_LIB=/root/repo/build/libb200_shfl.so"; fi
  env $L ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:tile_sort_kernel" -c 1 -o gpurun_out/shfl/tile_k24_$v python tools/prof_one.py --k 24 --iters 1 > /dev/null 2>&1
  env $L ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:tile_sort_kernel" -c 1 -o gpurun_out/shfl/tile_batched_$v python tools/prof_one.py --k 24 --batched 4096 --iters 1 > /dev/null 2>&1
  env $L python tools/perf_probe.py --ks 16,20,24,28 --batched > gpurun_out/shfl/perf_$v.log 2>&1
done
python -m pytest tests/test_gpu_parity.py -x -q -k "host_entry" > gpurun_out/pytest_host.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_host.log
