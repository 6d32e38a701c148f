#!/bin/bash
# fused TreeLSTM: concurrent linearizer (default 12 leaf warps), 8 leaf warps, serial (CX_LIN_CONC=0)
timeout 600 python -m pytest tests/test_fused_gpu.py tests/test_workspace_gpu.py -q -x 2>&1 | tail -2
b() { python bench.py --workload $1 --no-cpu-baseline --no-secondary --steps 300 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print('$2', '$1', round(d['ms_per_step']*1e3,2), round(d['latency_us'],2))"; }
for w in cfg2_treelstm_b10 cfg2_treelstm_b1 f4_lstm_seq100_b10; do
  b $w conc12
  CX_LIN_CONC=0 b $w serial
  CX_LIB=paper_2011_01383_b200/variants/libcx_lw8.so b $w conc8
done
