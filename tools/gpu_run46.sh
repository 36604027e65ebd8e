export PYTHONUNBUFFERED=1
{
echo "== deferred T"; timeout 300 python tools/tsqr_bench.py 60 8000 60 0 60 5
echo "== inline T"; TTB_LEAF_T=inline timeout 300 python tools/tsqr_bench.py 60 8000 60 0 60 5
echo "== deferred T b=30"; timeout 300 python tools/tsqr_bench.py 60 8000 30 0 30 5
echo "== inline T b=30"; TTB_LEAF_T=inline timeout 300 python tools/tsqr_bench.py 60 8000 30 0 30 5
} > gpurun_out/tb46.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_multirank.py -m gpu -x -q --timeout 600 > gpurun_out/gt46.log 2>&1
echo "exit $?" >> gpurun_out/gt46.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/b46.log 2>&1
TTB_LEAF_T=inline timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/b46i.log 2>&1
