#!/bin/bash
b() { python bench.py --workload $1 --no-cpu-baseline --no-secondary --steps 300 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print('$2', '$1', round(d['ms_per_step']*1e3,2), round(d['latency_us'],2))"; }
for rep in 1 2; do
  CX_LIB=paper_2011_01383_b200/variants/libcx_head.so b cfg2_treelstm_b10 head
  b cfg2_treelstm_b10 conc12
  CX_LIN_CONC=0 b cfg2_treelstm_b10 serial
  CX_LIB=paper_2011_01383_b200/variants/libcx_lw8.so b cfg2_treelstm_b10 conc8
done
