# round 2 session 2 baseline: push-mode check, all GPU tests, bench, trace
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python tools/dbg_push.py cfg2_treelstm_b10 > gpurun_out/s2_dbg.txt 2>&1; echo "dbg rc=$?"
cat gpurun_out/s2_dbg.txt | tail -8
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/s2_gpu_tests.log 2>&1; echo "tests rc=$?"
tail -15 gpurun_out/s2_gpu_tests.log
timeout 300 python bench.py --steps 50 --warmup 5 --no-secondary --no-cpu-baseline > gpurun_out/s2_bench.json 2>gpurun_out/s2_bench.err; echo "bench rc=$?"
python -c "import json;d=json.load(open('gpurun_out/s2_bench.json'));print('LAT', d['latency_us'], d['forward_us'], d['linearize_us'], d['two_launch_latency_us'])"
tail -3 gpurun_out/s2_bench.err
timeout 120 python tools/trace_cluster.py cfg2_treelstm_b10 fused > gpurun_out/s2_trace.txt 2>&1
head -40 gpurun_out/s2_trace.txt
