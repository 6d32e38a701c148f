#!/bin/bash
# DRAM bytes of the forward launch per workload (ncu, third launch of tools/one_forward.py)
mkdir -p gpurun_out/traffic
for a in "cfg5_treelstm_b4096 f32" "cfg5_dagrnn_b4096 f32" "cfg3_treefc_b10 f32" "cfg5_treelstm_b4096 bf16" "cfg5_dagrnn_b4096 bf16" "cfg2_treelstm_b10 f32"; do
  set -- $a
  python tools/one_forward.py $1 $2 > gpurun_out/traffic/plain_$1_$2.log 2>&1 && \
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"tc_kernel|ck_kernel|rw_kernel" -s 2 -c 1 --csv python tools/one_forward.py $1 $2 > gpurun_out/traffic/ncu_$1_$2.csv 2>&1
  echo "$1 $2 rc=$?"
done
