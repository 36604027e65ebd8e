export PYTHONUNBUFFERED=1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tsqr_product -s 2 -c 1 -o gpurun_out/r2_product python tools/tsqr_bench.py 60 8000 60 0 60 2 > gpurun_out/ncu_product.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fold_kernel -s 2 -c 1 -o gpurun_out/r2_fold python profiles/round_once.py 1 > gpurun_out/ncu_fold.log 2>&1
