export PYTHONUNBUFFERED=1
{
echo "== V 480000x60 k=60"; timeout 300 python tools/tsqr_bench.py 60 8000 60 0 60 5
echo "== H^T 240000x60 k=30"; timeout 300 python tools/tsqr_bench.py 60 8000 30 1 30 5
echo "== V 480000x30"; timeout 300 python tools/tsqr_bench.py 60 8000 30 0 30 5
echo "== V 1600000x16"; timeout 300 python tools/tsqr_bench.py 16 100000 16 0 16 5
} > gpurun_out/try2.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q --timeout 600 --deselect tests/test_gpu_fullsize.py > gpurun_out/try2_t.log 2>&1
echo "exit $?" >> gpurun_out/try2_t.log
