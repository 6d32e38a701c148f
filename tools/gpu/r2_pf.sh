#!/bin/bash
timeout 900 python -m pytest tests/test_forward_tc32_gpu.py tests/test_forward_tc_gpu.py -q -x 2>&1 | tail -2
b() { python bench.py --workload $1 --dtype $2 --no-cpu-baseline --no-secondary --steps 50 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print('$3', '$1', '$2', round(d['ms_per_step']*1e3,1), 'fwd', round(d['forward_us'],1))"; }
for a in "cfg5_treelstm_b4096 f32" "cfg5_treelstm_b4096 bf16" "cfg3_treefc_b10 f32"; do
  set -- $a
  b $1 $2 pf4
  CX_LIB=paper_2011_01383_b200/variants/libcx_pf0.so b $1 $2 pf0
  CX_LIB=paper_2011_01383_b200/variants/libcx_pf8.so b $1 $2 pf8
done
