#!/bin/bash
# ncu evidence for profiles/: launch lists (cold, serialised) of the default
# bench and of the bf16 b4096 step, and full captures of the top kernels.
mkdir -p gpurun_out/prof
B="python bench.py --no-cpu-baseline --no-secondary --steps 3 --warmup 3"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
  --log-file gpurun_out/prof/launches_b10_f32.csv $B --workload cfg2_treelstm_b10 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
  --log-file gpurun_out/prof/launches_b4096_bf16.csv $B --workload cfg5_treelstm_b4096 --dtype bf16 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_kernel -s 3 -c 1 \
  -o gpurun_out/prof/tc_b4096 $B --workload cfg5_treelstm_b4096 --dtype bf16 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ck_kernel -s 3 -c 1 \
  -o gpurun_out/prof/ck_b10 $B --workload cfg2_treelstm_b10 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:lin_kernel -s 3 -c 1 \
  -o gpurun_out/prof/lin_b4096 $B --workload cfg5_treelstm_b4096 --dtype bf16 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_kernel -s 3 -c 1 \
  -o gpurun_out/prof/tc_dag_b4096 $B --workload cfg5_dagrnn_b4096 --dtype bf16 > /dev/null 2>&1
ls -la gpurun_out/prof
