timeout 900 python -m pytest tests/test_linearize_gpu.py tests/test_fused_gpu.py -m gpu -q -x > gpurun_out/warp_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/warp_tests.log
timeout 300 python bench.py --steps 200 --warmup 10 --no-secondary --no-cpu-baseline --workload cfg1_treernn > gpurun_out/warp_cfg1.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/warp_cfg1.json'));print('cfg1 step', round(d['latency_us'],2), 'mean', round(d['ms_per_step']*1e3,2), 'lin', round(d['linearize_us'],2))"
CX_TRACE=1 timeout 120 python tools/trace_single.py cfg1_treernn
