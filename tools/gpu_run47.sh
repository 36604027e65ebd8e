export PYTHONUNBUFFERED=1
{
echo "== deferred T"; timeout 300 python tools/tsqr_bench.py 60 8000 60 0 60 5
} > gpurun_out/tb47.log 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/b47.log 2>&1
