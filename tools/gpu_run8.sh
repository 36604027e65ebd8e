export PYTHONUNBUFFERED=1
for args in "1 8000 60 0 60 5" "60 8000 1 1 60 5" "30 8000 60 0 30 5" "1 2000 20 0 20 5" "20 2000 20 0 20 5" "16 100000 16 0 16 5" "60 8000 60 0 60 3"; do
  echo "== new $args" >> gpurun_out/tb8.log
  timeout 120 python tools/tsqr_bench.py $args >> gpurun_out/tb8.log 2>&1
  echo "== old $args" >> gpurun_out/tb8.log
  TTB_WLEAF_OFF=1 timeout 120 python tools/tsqr_bench.py $args >> gpurun_out/tb8.log 2>&1
done
