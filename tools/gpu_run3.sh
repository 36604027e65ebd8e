timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q --timeout 60 > gpurun_out/gt3a.log 2>&1
echo "exit $?" >> gpurun_out/gt3a.log
timeout 600 python -m pytest tests -m gpu -q --timeout 120 --ignore=tests/test_gpu_fullsize.py > gpurun_out/gt3b.log 2>&1
echo "exit $?" >> gpurun_out/gt3b.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-norm > gpurun_out/bench3.log 2>&1
echo "bench exit $?" >> gpurun_out/bench3.log
