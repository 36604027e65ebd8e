export PYTHONUNBUFFERED=1
TTB_LIB=scratch/dtile.so timeout 120 python tools/tileclk.py 60 8000 60 0 > gpurun_out/tile13.log 2>&1
TTB_LIB=scratch/dtile.so timeout 120 python tools/tileclk.py 60 8000 30 1 >> gpurun_out/tile13.log 2>&1
