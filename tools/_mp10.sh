mkdir -p gpurun_out/mp10
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/mp10/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/mp10/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > gpurun_out/mp10/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/mp10/bench.log 2>&1; echo "rc=$?" >> gpurun_out/mp10/bench.log
timeout 900 python bench.py --log2n 30 --steps 5 --no-cpu-baseline > gpurun_out/mp10/bench30.log 2>&1
timeout 900 python bench.py --log2n 24 --no-cpu-baseline > gpurun_out/mp10/bench24.log 2>&1
