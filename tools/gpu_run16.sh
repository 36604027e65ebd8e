export PYTHONUNBUFFERED=1
echo "== new load" > gpurun_out/tile16.log
TTB_LIB=scratch/dtile.so timeout 120 python tools/tileclk.py 60 8000 60 0 >> gpurun_out/tile16.log 2>&1
echo "== old load" >> gpurun_out/tile16.log
TTB_LIB=scratch/varA.so timeout 120 python tools/tileclk.py 60 8000 60 0 >> gpurun_out/tile16.log 2>&1
