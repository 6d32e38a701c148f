set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2_base_gpu_tests.log 2>&1; echo "tests rc=$?"
timeout 300 python bench.py --steps 50 --warmup 5 --no-secondary --no-cpu-baseline > gpurun_out/r2_base_bench.json 2>gpurun_out/r2_base_bench.err; echo "bench rc=$?"
timeout 120 python tools/trace_cluster.py cfg2_treelstm_b10 fused > gpurun_out/r2_base_trace.txt 2>&1
tail -3 gpurun_out/r2_base_gpu_tests.log; cat gpurun_out/r2_base_bench.json | head -c 600
