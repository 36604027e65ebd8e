export PYTHONUNBUFFERED=1
timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_norm_sym.py -m gpu -x -q --timeout 120 > gpurun_out/gt34.log 2>&1
echo "exit $?" >> gpurun_out/gt34.log
TTB_LIB=scratch/dclk.so timeout 120 python tools/svdclk.py > gpurun_out/sclk34.log 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-norm > gpurun_out/bench34.log 2>&1
