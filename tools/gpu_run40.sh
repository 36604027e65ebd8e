export PYTHONUNBUFFERED=1
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/gt40.log 2>&1
echo "exit $?" >> gpurun_out/gt40.log
