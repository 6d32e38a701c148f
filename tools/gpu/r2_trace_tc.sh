#!/bin/bash
mkdir -p gpurun_out/trace_tc
for a in "cfg5_treelstm_b4096 bf16" "cfg5_treelstm_b4096 f32" "cfg5_dagrnn_b4096 f32" "cfg3_treefc_b10 f32" "cfg3_treefc_b10 bf16"; do
  set -- $a
  CX_TRACE=1 timeout 300 python tools/trace_tc.py $1 $2 > gpurun_out/trace_tc/$1_$2.txt 2>&1
done
tail -n +1 gpurun_out/trace_tc/*.txt | grep -v "stage\|tile" | head -150
