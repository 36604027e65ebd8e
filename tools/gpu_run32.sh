export PYTHONUNBUFFERED=1
timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -m gpu -x -q --timeout 120 > gpurun_out/gt32.log 2>&1
echo "exit $?" >> gpurun_out/gt32.log
timeout 120 python tools/tsqr_bench.py 60 8000 60 0 60 5 > gpurun_out/tb32.log 2>&1
timeout 120 python tools/tsqr_bench.py 60 8000 30 1 30 5 >> gpurun_out/tb32.log 2>&1
timeout 120 python tools/tsqr_bench.py 16 100000 16 0 16 5 >> gpurun_out/tb32.log 2>&1
