#!/bin/bash
# bench the tensor-core kernel variants (tools/build_variant.sh) on the b4096 workloads
mkdir -p gpurun_out/var
for v in default bshare s4; do
  for a in "cfg5_treelstm_b4096 bf16" "cfg5_treelstm_b4096 f32" "cfg5_dagrnn_b4096 f32" "cfg5_dagrnn_b4096 bf16"; do
    set -- $a
    if [ $v = default ]; then unset CX_LIB; else export CX_LIB=paper_2011_01383_b200/variants/libcx_$v.so; fi
    timeout 300 python bench.py --workload $1 --dtype $2 --no-cpu-baseline --no-secondary --steps 30 > gpurun_out/var/$v_$1_$2.json 2> gpurun_out/var/err.txt
    python -c "import json;d=json.loads(open('gpurun_out/var/$v_$1_$2.json').read().strip().splitlines()[-1]);print('$v $1 $2', round(d['ms_per_step']*1e3,1), 'us fwd', round(d['forward_us'],1), d['launch'])" || tail -3 gpurun_out/var/err.txt
  done
done
