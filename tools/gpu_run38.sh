export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_wide.py tests/test_gpu_errors.py -m gpu -q --timeout 300 > gpurun_out/gt38.log 2>&1
echo "exit $?" >> gpurun_out/gt38.log
