export PYTHONUNBUFFERED=1
timeout 2400 python -m pytest tests -m gpu -x -q --timeout 900 > gpurun_out/final_tests.log 2>&1
echo "exit $?" >> gpurun_out/final_tests.log
timeout 900 python bench.py > gpurun_out/r2_bench.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1
TTB_SWEEP_SEEDS=1200 timeout 1800 python -m pytest tests/test_gpu_shapes.py -m gpu -q --timeout 300 -k "round_inner_norm" > gpurun_out/soak.log 2>&1
echo "exit $?" >> gpurun_out/soak.log
