export PYTHONUNBUFFERED=1
TTB_LIB=scratch/dclk.so timeout 120 python tools/svdclk.py > gpurun_out/sclk21.log 2>&1
