export PYTHONUNBUFFERED=1
TTB_LEAF3=1 timeout 1200 python -m pytest tests -m gpu -q --timeout 600 --deselect tests/test_gpu_fullsize.py > gpurun_out/opt_leaf3.log 2>&1
echo "exit $?" >> gpurun_out/opt_leaf3.log
TTB_LEAF_T=defer timeout 1200 python -m pytest tests -m gpu -q --timeout 600 --deselect tests/test_gpu_fullsize.py > gpurun_out/opt_defer.log 2>&1
echo "exit $?" >> gpurun_out/opt_defer.log
TTB_FULLSIZE= timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/final_default.log 2>&1
echo "exit $?" >> gpurun_out/final_default.log
