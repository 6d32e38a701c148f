CX_TRACE=1 timeout 120 python tools/trace_cluster.py ${1:-cfg2_treelstm_b10} fused > gpurun_out/it_trace.txt 2>&1
cat gpurun_out/it_trace.txt | head -45
timeout 300 python bench.py --steps 50 --warmup 5 --no-secondary --no-cpu-baseline --workload ${1:-cfg2_treelstm_b10} > gpurun_out/it_bench.json 2>gpurun_out/it_bench.err; echo "bench rc=$?"
python -c "import json;d=json.load(open('gpurun_out/it_bench.json'));print('LAT', d['latency_us'], d['forward_us'], d['linearize_us'], d['two_launch_latency_us'])"
