export PYTHONUNBUFFERED=1
TTB_LIB=scratch/wlclk.so timeout 120 python tools/wlclk.py 60 8000 60 0 > gpurun_out/clk5.log 2>&1
timeout 120 python tools/tsqr_bench.py 60 8000 60 0 60 5 > gpurun_out/tb5.log 2>&1
TTB_LIB=scratch/wlring1.so timeout 120 python tools/tsqr_bench.py 60 8000 60 0 60 5 >> gpurun_out/tb5.log 2>&1
