timeout 900 python -m pytest tests/test_bf16_dispatch_gpu.py tests/test_forward_gpu.py -m gpu -q -x > gpurun_out/fc_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/fc_tests.log
for wl in cfg3_treefc_b1 cfg3_treefc_b10; do
  timeout 300 python bench.py --steps 100 --warmup 10 --no-secondary --no-cpu-baseline --dtype bf16 --workload $wl > gpurun_out/fc_$wl.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/fc_$wl.json'));print('$wl bf16 step', round(d['latency_us'],1), d['launch'])"
done
