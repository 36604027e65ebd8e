export PYTHONUNBUFFERED=1
timeout 2400 python -m pytest tests -m gpu -x -q --timeout 900 > gpurun_out/final_tests.log 2>&1
echo "exit $?" >> gpurun_out/final_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1
echo "exit $?" >> gpurun_out/final_smoke.log
bash tools/gpu_prof_r2.sh
