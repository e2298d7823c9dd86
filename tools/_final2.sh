mkdir -p gpurun_out/final2
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/final2/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/final2/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > gpurun_out/final2/smoke.log 2>&1
timeout 900 python bench.py --batched 4096 --no-cpu-baseline > gpurun_out/final2/bench_batched.log 2>&1
