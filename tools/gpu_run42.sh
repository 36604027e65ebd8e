export PYTHONUNBUFFERED=1
{
echo "== lf3 clk V 480000x60"; TTB_LIB=scratch/lf3clk.so TTB_LEAF3=1 timeout 300 python tools/lf3clk.py 60 8000 60 0
} > gpurun_out/clk42.log 2>&1
