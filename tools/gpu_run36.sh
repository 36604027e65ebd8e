export PYTHONUNBUFFERED=1
timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -m gpu -x -q --timeout 120 > gpurun_out/gt36.log 2>&1
echo "exit $?" >> gpurun_out/gt36.log
timeout 900 python profiles/measure_configs.py > gpurun_out/cfg36.txt 2>&1
for a in "16 100000 16 0 16 5" "16 100000 16 1 16 5"; do timeout 120 python tools/tsqr_bench.py $a >> gpurun_out/tb36.log 2>&1; TTB_WLEAF=1 timeout 120 python tools/tsqr_bench.py $a >> gpurun_out/tb36.log 2>&1; done
