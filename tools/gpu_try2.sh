export PYTHONUNBUFFERED=1
timeout 900 python profiles/measure_configs.py > gpurun_out/r2_configs.txt 2>&1
