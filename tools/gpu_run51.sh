export PYTHONUNBUFFERED=1
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 --durations=25 > gpurun_out/gt51.log 2>&1
echo "exit $?" >> gpurun_out/gt51.log
