export PYTHONUNBUFFERED=1
timeout 120 python tools/tsqr_bench.py 60 8000 60 0 60 5 > gpurun_out/tb4.log 2>&1
timeout 120 python tools/tsqr_bench.py 60 8000 30 1 30 5 >> gpurun_out/tb4.log 2>&1
TTB_WLEAF_OFF=1 timeout 120 python tools/tsqr_bench.py 60 8000 60 0 60 5 >> gpurun_out/tb4.log 2>&1
TTB_WLEAF_OFF=1 timeout 120 python tools/tsqr_bench.py 60 8000 30 1 30 5 >> gpurun_out/tb4.log 2>&1
timeout 300 ncu --set full --import-source on -k regex:wleaf -c 1 -o gpurun_out/wleaf1 python tools/tsqr_bench.py 60 8000 60 0 60 1 > gpurun_out/ncu4.log 2>&1
echo "ncu exit $?" >> gpurun_out/ncu4.log
