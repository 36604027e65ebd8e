export PYTHONUNBUFFERED=1
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r2_bench.log 2>&1
timeout 1200 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2_bench_reference.log 2>&1
