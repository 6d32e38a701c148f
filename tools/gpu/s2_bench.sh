set -x
timeout 300 python tools/sync_costs.py > gpurun_out/r02_sync_costs.json 2>gpurun_out/sync.err; echo "sync rc=$?"; cat gpurun_out/r02_sync_costs.json | head -40; tail -3 gpurun_out/sync.err
timeout 600 python bench.py > gpurun_out/r02_bench_default.json 2>gpurun_out/r02_bench_default.err; echo "bench rc=$?"
tail -3 gpurun_out/r02_bench_default.err
python -c "
import json;d=json.load(open('gpurun_out/r02_bench_default.json'))
print('LAT',d['latency_us'],'value',d['value'],'e2e',d['e2e']['value'], d['e2e']['roots_only'])
print(json.dumps(d['roofline'],indent=1)); print(json.dumps(d['cpu_baseline'],indent=1)); print(d['launch'])"
