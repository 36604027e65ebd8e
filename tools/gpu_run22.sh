export PYTHONUNBUFFERED=1
echo "== grp16" > gpurun_out/sclk22.log
TTB_LIB=scratch/dclk.so timeout 120 python tools/svdclk.py >> gpurun_out/sclk22.log 2>&1
echo "== grp8" >> gpurun_out/sclk22.log
TTB_LIB=scratch/dclk8.so timeout 120 python tools/svdclk.py >> gpurun_out/sclk22.log 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -m gpu -x -q --timeout 120 > gpurun_out/gt22.log 2>&1
echo "exit $?" >> gpurun_out/gt22.log
TTB_LIB=scratch/grp8.so timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q --timeout 120 -k svd >> gpurun_out/gt22.log 2>&1
echo "exit grp8 $?" >> gpurun_out/gt22.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-norm > gpurun_out/bench22.log 2>&1
TTB_LIB=scratch/grp8.so timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-norm > gpurun_out/bench22b.log 2>&1
