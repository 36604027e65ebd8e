export PYTHONUNBUFFERED=1
{
echo "== b=30 480000 rows"; timeout 300 python tools/tsqr_bench.py 60 8000 30 0 30 5
echo "== b=32 480000 rows"; timeout 300 python tools/tsqr_bench.py 60 8000 32 0 32 5
echo "== b=16 480000 rows"; timeout 300 python tools/tsqr_bench.py 60 8000 16 0 16 5
echo "== b=15 480000 rows"; timeout 300 python tools/tsqr_bench.py 60 8000 15 0 15 5
echo "== b=60 480000 rows"; timeout 300 python tools/tsqr_bench.py 60 8000 60 0 60 5
} > gpurun_out/tb44.log 2>&1
