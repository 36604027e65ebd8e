export PYTHONUNBUFFERED=1
{
echo "== lf3 clk V 480000x60"; TTB_LIB=scratch/lf3clk.so TTB_LEAF3=1 timeout 300 python tools/lf3clk.py 60 8000 60 0 | tail -3
echo "== lf3 NOT clk V 480000x60"; TTB_LIB=scratch/lf3not.so TTB_LEAF3=1 timeout 300 python tools/lf3clk.py 60 8000 60 0 | tail -3
echo "== leaf3 V"; TTB_LEAF3=1 timeout 300 python tools/tsqr_bench.py 60 8000 60 0 60 5
echo "== leaf3 NOT V (apply wrong: no T)"; TTB_LIB=scratch/lf3not.so TTB_LEAF3=1 timeout 300 python tools/tsqr_bench.py 60 8000 60 0 60 5
} > gpurun_out/clk45.log 2>&1
