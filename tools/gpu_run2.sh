timeout 900 python -m pytest tests -m gpu -x -q --ignore=tests/test_gpu_fullsize.py > gpurun_out/gputest2.log 2>&1
echo "pytest exit $?" >> gpurun_out/gputest2.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-norm > gpurun_out/bench2.log 2>&1
echo "bench exit $?" >> gpurun_out/bench2.log
