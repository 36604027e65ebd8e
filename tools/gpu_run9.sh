export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -m gpu -q --timeout 300 --ignore=tests/test_gpu_fullsize.py > gpurun_out/gt9.log 2>&1
echo "exit $?" >> gpurun_out/gt9.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/bench9.log 2>&1
echo "bench exit $?" >> gpurun_out/bench9.log
timeout 600 python tools/sanitize_case.py > gpurun_out/san_plain.log 2>&1
timeout 900 compute-sanitizer --tool memcheck --leak-check no python tools/sanitize_case.py > gpurun_out/san_memcheck.log 2>&1
echo "exit $?" >> gpurun_out/san_memcheck.log
timeout 1200 compute-sanitizer --tool racecheck --racecheck-report all python tools/sanitize_case.py > gpurun_out/san_racecheck.log 2>&1
echo "exit $?" >> gpurun_out/san_racecheck.log
timeout 900 compute-sanitizer --tool synccheck python tools/sanitize_case.py > gpurun_out/san_synccheck.log 2>&1
echo "exit $?" >> gpurun_out/san_synccheck.log
