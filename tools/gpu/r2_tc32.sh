#!/bin/bash
# split-fp32 tensor-core path: parity tests, then bench lines of the fp32
# workloads it takes (and the FMA kernels they replaced, forced with CX_TC_F32_MIN_N)
mkdir -p gpurun_out/tc32
timeout 900 python -m pytest tests/test_forward_tc32_gpu.py -x -q > gpurun_out/tc32/tests.log 2>&1
tail -3 gpurun_out/tc32/tests.log
for w in cfg5_treelstm_b4096 cfg5_dagrnn_b4096 cfg3_treefc_b10; do
  timeout 300 python bench.py --workload $w --no-cpu-baseline --no-secondary --steps 50 > gpurun_out/tc32/$w.json 2> gpurun_out/tc32/$w.err
  python -c "import json;d=json.loads(open('gpurun_out/tc32/$w.json').read().strip().splitlines()[-1]);print('$w', d['ms_per_step']*1e3, 'us', d['value'], d.get('launch'))" || tail -5 gpurun_out/tc32/$w.err
done
REPEATS=200 timeout 300 python tools/determinism.py cfg3_treegru_b10 2>&1 | tail -2
