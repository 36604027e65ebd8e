export PYTHONUNBUFFERED=1
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 600 > gpurun_out/gt39.log 2>&1
echo "exit $?" >> gpurun_out/gt39.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/b39.log 2>&1
echo "exit $?" >> gpurun_out/b39.log
