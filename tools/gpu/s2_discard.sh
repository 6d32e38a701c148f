timeout 900 python -m pytest tests/test_forward_tc_gpu.py tests/test_bf16_dispatch_gpu.py -m gpu -q -x > gpurun_out/discard_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/discard_tests.log
timeout 900 python -m pytest tests/test_shard_gpu.py -m gpu -q -x -k b4096 > gpurun_out/discard_shard.log 2>&1; echo "shard rc=$?"; tail -2 gpurun_out/discard_shard.log
for d in 0 1; do
  CX_DISCARD=$d timeout 300 python bench.py --steps 100 --warmup 10 --no-secondary --no-cpu-baseline --dtype bf16 --workload cfg5_treelstm_b4096 > gpurun_out/discard_$d.json 2>>gpurun_out/discard.err
  python -c "import json;d=json.load(open('gpurun_out/discard_$d.json'));print('discard=$d step', round(d['latency_us'],1), 'fwd', round(d['forward_us'],1))"
  CX_DISCARD=$d timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:tc_kernel -s 2 -c 1 --csv python bench.py --steps 3 --warmup 3 --no-secondary --no-cpu-baseline --dtype bf16 --workload cfg5_treelstm_b4096 > gpurun_out/discard_ncu_$d.csv 2>/dev/null
  grep -E "dram__bytes|gpu__time|tensor" gpurun_out/discard_ncu_$d.csv | awk -F'","' '{print $(NF-2), $(NF-1), $NF}'
done
