#!/bin/bash
# Re-capture the profiles/ evidence on a GPU box (run via gpurun from the repo
# root).  Each ncu command runs only after the same command exited 0 without
# ncu.  Outputs land in gpurun_out/prof/; tools/ncu_summary.py and
# tools/launch_summary.py turn them into the tracked profiles/ files.
set -u
out=gpurun_out/prof
mkdir -p $out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
for cfg in "28" "24" "20" "16"; do
  cmd="python bench.py --log2n $cfg --steps 2 --warmup 3 --no-cpu-baseline --no-variants"
  if $cmd > $out/bench_k$cfg.json 2> $out/bench_k$cfg.err; then
    ncu --metrics $M --clock-control none --csv --log-file $out/launches_k$cfg.csv $cmd > /dev/null 2>&1
  fi
done
cmd="python bench.py --batched 4096 --log2n 24 --steps 2 --warmup 3 --no-cpu-baseline"
if $cmd > $out/bench_batched.json 2> $out/bench_batched.err; then
  ncu --metrics $M --clock-control none --csv --log-file $out/launches_batched.csv $cmd > /dev/null 2>&1
fi
# full captures of the dominant kernels (one launch each)
if python tools/prof_one.py --k 28 --iters 1 > /dev/null 2>&1; then
  ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
      -k "regex:merge_kernel|tile_sort_kernel" -c 6 -o $out/full_k28 python tools/prof_one.py --k 28 --iters 1 > /dev/null 2>&1
fi
if python tools/prof_one.py --k 20 --iters 1 > /dev/null 2>&1; then
  ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
      -k "regex:merge_kernel" -c 3 -o $out/full_k20_merge python tools/prof_one.py --k 20 --iters 1 > /dev/null 2>&1
fi
if python tools/prof_one.py --k 24 --batched 4096 --iters 1 > /dev/null 2>&1; then
  ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
      -k "regex:tile_sort_kernel" -c 1 -o $out/full_batched python tools/prof_one.py --k 24 --batched 4096 --iters 1 > /dev/null 2>&1
fi
if LOGS=27 python tools/merge_probe.py > /dev/null 2>&1; then
  LOGS=27 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
      -k "regex:merge_bitonic|merge_partition" -c 2 -o $out/full_mergesplit python tools/merge_probe.py > /dev/null 2>&1
fi
ls -la $out
