export PYTHONUNBUFFERED=1
TTB_LIB=scratch/tclk2.so timeout 120 python tools/treeclk.py 60 8000 60 0 > gpurun_out/tclk24.log 2>&1
