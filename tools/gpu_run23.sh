export PYTHONUNBUFFERED=1
for v in dclk dclk_noupd dclk_nodot; do
echo "== $v" >> gpurun_out/lclk23.log
TTB_LIB=scratch/$v.so timeout 120 python tools/leafclk.py 60 8000 60 0 2>&1 | head -4 >> gpurun_out/lclk23.log
done
