export PYTHONUNBUFFERED=1
{
echo "== default leaf"; timeout 300 python tools/tsqr_bench.py 60 8000 60 0 60 5
echo "== leaf3 V"; TTB_LEAF3=1 timeout 300 python tools/tsqr_bench.py 60 8000 60 0 60 5
echo "== leaf3 H^T"; TTB_LEAF3=1 timeout 300 python tools/tsqr_bench.py 60 8000 30 1 30 5
echo "== default H^T"; timeout 300 python tools/tsqr_bench.py 60 8000 30 1 30 5
echo "== leaf3 small"; TTB_LEAF3=1 timeout 300 python tools/tsqr_bench.py 7 300 40 0 40 2
} > gpurun_out/tb41.log 2>&1
TTB_LEAF3=1 timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -m gpu -x -q --timeout 600 > gpurun_out/gt41.log 2>&1
echo "exit $?" >> gpurun_out/gt41.log
{
echo "== lf3 clk V 480000x60"; TTB_LIB=scratch/lf3clk.so TTB_LEAF3=1 timeout 300 python tools/lf3clk.py 60 8000 60 0
} > gpurun_out/clk41.log 2>&1
