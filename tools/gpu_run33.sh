export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests -m gpu -x -q --timeout 300 --ignore=tests/test_gpu_fullsize.py > gpurun_out/gt33.log 2>&1
echo "exit $?" >> gpurun_out/gt33.log
TTB_LIB=scratch/dclk.so timeout 120 python tools/svdclk.py > gpurun_out/sclk33.log 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-norm > gpurun_out/bench33.log 2>&1
