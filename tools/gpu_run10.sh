export PYTHONUNBUFFERED=1
TTB_LIB=scratch/tclk2.so timeout 120 python tools/treeclk.py 60 8000 60 0 > gpurun_out/tclk10.log 2>&1
TTB_LIB=scratch/tclk2.so timeout 120 python tools/treeclk.py 60 8000 30 1 >> gpurun_out/tclk10.log 2>&1
timeout 120 python tools/tsqr_bench.py 60 8000 60 0 60 5 > gpurun_out/tb10.log 2>&1
TTB_LIB=scratch/tc16.so timeout 120 python tools/tsqr_bench.py 60 8000 60 0 60 5 >> gpurun_out/tb10.log 2>&1
