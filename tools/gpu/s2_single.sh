set -x
timeout 900 python -m pytest tests/test_fused_gpu.py -m gpu -x -q > gpurun_out/sc_tests.log 2>&1; echo "tests rc=$?"; tail -5 gpurun_out/sc_tests.log
for u in 1 2; do
  CX_UNROLL=$u timeout 300 python bench.py --steps 200 --warmup 10 --no-secondary --no-cpu-baseline --workload cfg1_treernn > gpurun_out/sc_cfg1_u$u.json 2>>gpurun_out/sc_bench.err
  python -c "import json;d=json.load(open('gpurun_out/sc_cfg1_u$u.json'));print('cfg1 unroll=$u step', round(d['latency_us'],2), 'launches', d['gpu_launches']/d['steps'], 'Tcp', round(d['roofline']['critical_path']['T_cp_us'],2), d['launch'])"
done
CX_FUSED=0 timeout 300 python bench.py --steps 200 --warmup 10 --no-secondary --no-cpu-baseline --workload cfg1_treernn > gpurun_out/sc_cfg1_twolaunch.json 2>>gpurun_out/sc_bench.err
python -c "import json;d=json.load(open('gpurun_out/sc_cfg1_twolaunch.json'));print('cfg1 two-launch step', round(d['latency_us'],2))"
tail -3 gpurun_out/sc_bench.err
CX_TRACE=1 timeout 120 python tools/trace_single.py cfg1_treernn
