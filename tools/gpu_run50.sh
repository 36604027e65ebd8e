export PYTHONUNBUFFERED=1
{
echo "== staged"; timeout 300 python tools/pageable_bench.py
echo "== plain pageable copies"; TTB_HOSTIO_NOSTAGE=1 timeout 300 python tools/pageable_bench.py
} > gpurun_out/pg50.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_errors.py tests/test_gpu_multirank.py -m gpu -x -q --timeout 600 -k "host or error or multirank or nonfinite" > gpurun_out/gt50.log 2>&1
echo "exit $?" >> gpurun_out/gt50.log
