export PYTHONUNBUFFERED=1
TTB_LIB=scratch/dclk.so timeout 120 python tools/leafclk.py 60 8000 60 0 > gpurun_out/lclk12.log 2>&1
