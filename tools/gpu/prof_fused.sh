mkdir -p gpurun_out/prof
timeout 600 python -m pytest tests/test_fused_gpu.py -m gpu -x -q > gpurun_out/prof/tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/prof/tests.log
B="python bench.py --no-cpu-baseline --no-secondary --steps 3 --warmup 3"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ck_kernel -s 2 -c 1 \
  -o gpurun_out/prof/ck_fused_b10 $B --workload cfg2_treelstm_b10 > gpurun_out/prof/ncu.log 2>&1
ls -la gpurun_out/prof
