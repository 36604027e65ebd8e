export PYTHONUNBUFFERED=1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:wleaf -c 1 -o gpurun_out/wleaf2 python tools/tsqr_bench.py 60 8000 60 0 60 1 > gpurun_out/ncu7.log 2>&1
echo "ncu exit $?" >> gpurun_out/ncu7.log
