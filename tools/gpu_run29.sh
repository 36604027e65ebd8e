export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests -m gpu -x -q --timeout 300 --ignore=tests/test_gpu_fullsize.py > gpurun_out/gt29.log 2>&1
echo "exit $?" >> gpurun_out/gt29.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-norm > gpurun_out/bench29.log 2>&1
timeout 120 python tools/tsqr_bench.py 60 8000 60 0 60 5 > gpurun_out/tb29.log 2>&1
timeout 120 python tools/tsqr_bench.py 60 8000 30 1 30 5 >> gpurun_out/tb29.log 2>&1
