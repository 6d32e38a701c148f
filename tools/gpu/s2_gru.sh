# f3: GRU cells under both schedules: parity tests, then latency per schedule
set -x
#timeout 900 python -m pytest tests/test_gru_gpu.py -m gpu -x -q > gpurun_out/gru_tests.log 2>&1; echo "tests rc=$?"; tail -5 gpurun_out/gru_tests.log
for sched in 0 1; do
for wl in ${WLS:-cfg3_treegru_b10 cfg3_treegru_b1 f3_simpletreegru_b10 f3_simpletreegru_b1 f4_gru_seq100_b10}; do
  CX_GRU_REFACTOR=$sched timeout 300 python bench.py --steps 100 --warmup 10 --no-secondary --no-cpu-baseline --workload $wl > gpurun_out/gru_${wl}_r${sched}.json 2>>gpurun_out/gru_bench.err
  python -c "import json,sys;d=json.load(open('gpurun_out/gru_${wl}_r${sched}.json'));print('$wl refactor=$sched', 'step', round(d['latency_us'],1), 'fwd', round(d['forward_us'],1), 'Tcp', round(d['roofline']['critical_path']['T_cp_us'],1))"
done; done
tail -3 gpurun_out/gru_bench.err
