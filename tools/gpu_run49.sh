export PYTHONUNBUFFERED=1
{
echo "== register per call"; timeout 300 python tools/pageable_bench.py
echo "== plain pageable copies"; TTB_HOSTIO_NOPIN=1 timeout 300 python tools/pageable_bench.py
} > gpurun_out/pg49.log 2>&1
