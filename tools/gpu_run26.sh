export PYTHONUNBUFFERED=1
for v in tclk2 tx0 tx0r16; do echo "== $v" >> gpurun_out/tclk26.log; TTB_LIB=scratch/$v.so timeout 120 python tools/treeclk.py 60 8000 60 0 2>&1 | head -4 >> gpurun_out/tclk26.log; done
TTB_LIB=scratch/tx0b.so timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multirank.py -m gpu -x -q --timeout 120 > gpurun_out/gt26.log 2>&1
echo "exit $?" >> gpurun_out/gt26.log
TTB_LIB=scratch/tx0r16b.so timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multirank.py -m gpu -x -q --timeout 120 >> gpurun_out/gt26.log 2>&1
echo "exit $?" >> gpurun_out/gt26.log
