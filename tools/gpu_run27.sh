export PYTHONUNBUFFERED=1
for v in tx0; do echo "== $v" >> gpurun_out/tclk27.log; TTB_LIB=scratch/$v.so timeout 120 python tools/treeclk.py 60 8000 60 0 2>&1 | head -4 >> gpurun_out/tclk27.log; done
TTB_LIB=scratch/tx0b.so timeout 600 python -m pytest tests -m gpu -x -q --timeout 300 --ignore=tests/test_gpu_fullsize.py > gpurun_out/gt27.log 2>&1
echo "exit $?" >> gpurun_out/gt27.log
TTB_LIB=scratch/tx0b.so timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-norm > gpurun_out/bench27.log 2>&1
