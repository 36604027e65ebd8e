export PYTHONUNBUFFERED=1
timeout 1200 python -m pytest tests -m gpu -x -q --timeout 600 --deselect tests/test_gpu_fullsize.py > gpurun_out/try2_t.log 2>&1
echo "exit $?" >> gpurun_out/try2_t.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/try2_b.log 2>&1
