timeout 900 python -m pytest tests/test_linearize_gpu.py -m gpu -q -x > gpurun_out/lin_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/lin_tests.log
CX_TRACE=1 timeout 120 python tools/trace_lin.py cfg5_treelstm_b4096 | tail -12
timeout 300 python bench.py --steps 50 --warmup 5 --no-secondary --no-cpu-baseline --workload cfg5_treelstm_b4096 --dtype bf16 > gpurun_out/lin_b4096.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/lin_b4096.json'));print('b4096 bf16 step', round(d['latency_us'],1), 'lin', round(d['linearize_us'],1))"
