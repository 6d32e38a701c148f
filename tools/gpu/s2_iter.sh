# iteration check: parity debug (push/pull x fused/separate), fused+forward GPU tests, bench, trace timeline
set -x
timeout 300 python tools/dbg_push.py cfg2_treelstm_b10 > gpurun_out/it_dbg.txt 2>&1; echo "dbg rc=$?"; tail -6 gpurun_out/it_dbg.txt
timeout 300 python tools/dbg_push.py cfg2_treelstm_b1 > gpurun_out/it_dbg1.txt 2>&1; echo "dbg1 rc=$?"; tail -6 gpurun_out/it_dbg1.txt
timeout 900 python -m pytest tests/test_fused_gpu.py tests/test_forward_gpu.py -m gpu -x -q > gpurun_out/it_tests.log 2>&1; echo "tests rc=$?"
tail -5 gpurun_out/it_tests.log
timeout 300 python bench.py --steps 50 --warmup 5 --no-secondary --no-cpu-baseline > gpurun_out/it_bench.json 2>gpurun_out/it_bench.err; echo "bench rc=$?"
python -c "import json;d=json.load(open('gpurun_out/it_bench.json'));print('LAT', d['latency_us'], d['forward_us'], d['linearize_us'], d['two_launch_latency_us'])"
tail -3 gpurun_out/it_bench.err
CX_TRACE=1 timeout 120 python tools/trace_cluster.py cfg2_treelstm_b10 fused > gpurun_out/it_trace.txt 2>&1
head -32 gpurun_out/it_trace.txt
