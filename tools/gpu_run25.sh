export PYTHONUNBUFFERED=1
TTB_LIB=scratch/tclk2.so timeout 120 python tools/treeclk.py 60 8000 60 0 > gpurun_out/tclk25.log 2>&1
timeout 600 python -m pytest tests -m gpu -x -q --timeout 300 --ignore=tests/test_gpu_fullsize.py > gpurun_out/gt25.log 2>&1
echo "exit $?" >> gpurun_out/gt25.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-norm > gpurun_out/bench25.log 2>&1
