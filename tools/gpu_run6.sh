export PYTHONUNBUFFERED=1
timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -m gpu -x -q --timeout 120 > gpurun_out/gt6.log 2>&1
echo "exit $?" >> gpurun_out/gt6.log
timeout 120 python tools/tsqr_bench.py 60 8000 60 0 60 5 > gpurun_out/tb6.log 2>&1
timeout 120 python tools/tsqr_bench.py 60 8000 30 1 30 5 >> gpurun_out/tb6.log 2>&1
TTB_LIB=scratch/wlclk.so timeout 120 python tools/wlclk.py 60 8000 60 0 > gpurun_out/clk6.log 2>&1
