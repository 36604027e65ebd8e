export PYTHONUNBUFFERED=1
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 600 > gpurun_out/gt37.log 2>&1
echo "exit $?" >> gpurun_out/gt37.log
timeout 600 python bench.py > gpurun_out/bench37.json 2> gpurun_out/bench37.err
echo "exit $?" >> gpurun_out/bench37.err
