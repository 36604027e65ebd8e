export PYTHONUNBUFFERED=1
{
echo "== V 480000x60"; timeout 300 python tools/tsqr_bench.py 60 8000 60 0 60 5
echo "== H^T 240000x60"; timeout 300 python tools/tsqr_bench.py 60 8000 30 1 30 5
echo "== V 480000x30"; timeout 300 python tools/tsqr_bench.py 60 8000 30 0 30 5
echo "== V 480000x16"; timeout 300 python tools/tsqr_bench.py 60 8000 16 0 16 5
} > gpurun_out/try.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_multirank.py -m gpu -x -q --timeout 600 > gpurun_out/try_t.log 2>&1
echo "exit $?" >> gpurun_out/try_t.log
