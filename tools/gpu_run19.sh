export PYTHONUNBUFFERED=1
echo "== fence" > gpurun_out/tclk19.log
TTB_LIB=scratch/tclk2.so timeout 120 python tools/treeclk.py 60 8000 60 0 >> gpurun_out/tclk19.log 2>&1
echo "== nofence" >> gpurun_out/tclk19.log
TTB_LIB=scratch/tclk2nf.so timeout 120 python tools/treeclk.py 60 8000 60 0 >> gpurun_out/tclk19.log 2>&1
