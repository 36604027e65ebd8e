# round-2 measurement set: bench line, reference arm, launch list, leaf ncu, per-kernel roofline capture
export PYTHONUNBUFFERED=1
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r2_bench.log 2>&1
timeout 1200 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2_bench_reference.log 2>&1
timeout 300 python profiles/round_once.py 2 > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches.csv python profiles/round_once.py 2 > gpurun_out/ncu_ll.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tsqr_leaf -s 30 -c 1 -o gpurun_out/r2_leaf python profiles/round_once.py 2 > gpurun_out/ncu_leaf.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:'gram|tsqr|jacobi|skinny|fold|hadamard|add_kernel' -c 16 -o gpurun_out/r2_kr python profiles/kernel_roofline.py > gpurun_out/ncu_kr.log 2>&1
echo done > gpurun_out/prof_done.txt
timeout 900 python profiles/measure_configs.py > gpurun_out/r2_configs.txt 2>&1
