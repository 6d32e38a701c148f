timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/s2_all_gpu_tests.log 2>&1; echo "tests rc=$?"; tail -6 gpurun_out/s2_all_gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s2_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/s2_smoke.log
