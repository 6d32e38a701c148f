#!/bin/bash
# ncu evidence for the fused (cx_linearize_forward) default bench step: the
# launch list (cold, serialised) and a full capture of the fused kernel.
mkdir -p gpurun_out/prof
B="python bench.py --no-cpu-baseline --no-secondary --steps 3 --warmup 3"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv \
  --log-file gpurun_out/prof/launches_b10_fused.csv $B --workload cfg2_treelstm_b10 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ck_kernel -s 2 -c 1 \
  -o gpurun_out/prof/ck_fused_b10 $B --workload cfg2_treelstm_b10 > /dev/null 2>&1
ls -la gpurun_out/prof
