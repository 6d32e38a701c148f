#!/bin/bash
timeout 900 python -m pytest tests/test_forward_tc32_gpu.py tests/test_forward_tc_gpu.py tests/test_workspace_gpu.py -q -x -k "dag or DAG or b4096 or workspace" 2>&1 | tail -3
b() { python bench.py --workload $1 --dtype $2 --no-cpu-baseline --no-secondary --steps 50 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print('$3', '$1', '$2', round(d['ms_per_step']*1e3,1), 'fwd', round(d['forward_us'],1))"; }
for dt in f32 bf16; do
  b cfg5_dagrnn_b4096 $dt hoist
  CX_TC_HOIST=0 b cfg5_dagrnn_b4096 $dt nohoist
done
