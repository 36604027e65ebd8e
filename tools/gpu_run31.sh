export PYTHONUNBUFFERED=1
timeout 120 python tools/tsqr_bench.py 60 8000 30 1 30 2 > gpurun_out/plain31.log 2>&1 && \
timeout 300 ncu --set full --import-source on --clock-control none -k regex:tsqr_product -s 2 -c 1 -o gpurun_out/prod31 python tools/tsqr_bench.py 60 8000 30 1 30 2 > gpurun_out/ncu31.log 2>&1
