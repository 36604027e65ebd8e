export PYTHONUNBUFFERED=1
{
echo "== lf3 clk V 480000x60"; TTB_LIB=scratch/lf3clk.so TTB_LEAF3=1 timeout 300 python tools/lf3clk.py 60 8000 60 0 | tail -4
echo "== leaf3 V"; TTB_LEAF3=1 timeout 300 python tools/tsqr_bench.py 60 8000 60 0 60 5
echo "== leaf3 H^T"; TTB_LEAF3=1 timeout 300 python tools/tsqr_bench.py 60 8000 30 1 30 5
} > gpurun_out/clk43.log 2>&1
