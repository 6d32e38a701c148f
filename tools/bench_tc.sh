#!/bin/bash
# bf16 tensor-core path: bench lines for every config the path covers, plus
# the ncu launch list and one full capture of tc_kernel at batch 4096.
mkdir -p gpurun_out/tc
for w in cfg5_treelstm_b4096 cfg5_dagrnn_b4096 cfg3_treefc_b10 cfg2_treelstm_b10 cfg2_treelstm_b1 cfg5_dagrnn_b10; do
  timeout 300 python bench.py --workload $w --dtype bf16 --no-cpu-baseline --steps 200 > gpurun_out/tc/bench_$w.json 2> gpurun_out/tc/bench_$w.err
done
if [ "$1" = "ncu" ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv \
    --log-file gpurun_out/tc/launches_b4096.csv python bench.py --workload cfg5_treelstm_b4096 --dtype bf16 --no-cpu-baseline --steps 5 --warmup 3 > /dev/null 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_kernel -s 2 -c 1 \
    -o gpurun_out/tc/prof_tc_b4096 python bench.py --workload cfg5_treelstm_b4096 --dtype bf16 --no-cpu-baseline --steps 3 --warmup 3 > /dev/null 2>&1
fi
cat gpurun_out/tc/bench_*.json | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); r=d['roofline']
    print(d['config']['workload'], d['dtype'], 'lat_us %.1f fwd_us %.1f lin_us %.1f trees/s %.0f frac %.3f hbm_frac %.3f e2e %.0f' % (d['latency_us'], d['forward_us'], d['linearize_us'], d['value'], r['frac'], r.get('hbm_frac',0), d['e2e']['value']))
"
