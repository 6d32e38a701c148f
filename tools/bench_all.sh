#!/bin/bash
# Every BASELINE.json workload through bench.py (fp32, and bf16 where the
# tensor-core path covers the cell), one JSON line each under gpurun_out/all/,
# then a summary table.
mkdir -p gpurun_out/all
for w in cfg2_treelstm_b10 cfg2_treelstm_b1 cfg3_treegru_b10 cfg3_treegru_b1 f3_simpletreegru_b10 f3_simpletreegru_b1 cfg3_treefc_b10 cfg3_treefc_b1 cfg4_mvrnn_b10 cfg5_dagrnn_b10 cfg5_dagrnn_b1 cfg1_treernn f4_lstm_seq100_b10 f4_gru_seq100_b10 cfg5_treelstm_b4096 cfg5_dagrnn_b4096; do
  timeout 300 python bench.py --workload $w --no-cpu-baseline --no-secondary --steps 200 > gpurun_out/all/f32_$w.json 2> gpurun_out/all/f32_$w.err
done
for w in cfg2_treelstm_b10 cfg2_treelstm_b1 cfg3_treefc_b10 cfg3_treefc_b1 cfg5_dagrnn_b10 cfg5_dagrnn_b1 cfg5_treelstm_b4096 cfg5_dagrnn_b4096; do
  timeout 300 python bench.py --workload $w --dtype bf16 --no-cpu-baseline --no-secondary --steps 200 > gpurun_out/all/bf16_$w.json 2> gpurun_out/all/bf16_$w.err
done
python - <<'PY'
import glob, json
rows = []
for f in sorted(glob.glob("gpurun_out/all/*.json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "FAILED", e); continue
    r = d["roofline"]
    cp = r.get("critical_path", {})
    rows.append((d["config"]["workload"], d["dtype"], d["ms_per_step"] * 1e3, d.get("fused"), d["linearize_us"], d["forward_us"], d["value"], r["frac"], r["bound"], r.get("binding"), r.get("binding_frac"), cp.get("T_cp_us"), d["launch"].get("ctas"), d["launch"].get("cluster"), d["e2e"]["value"], d["clocks"]["sm_mhz"]))
print("| workload | dtype | step µs (mean) | launches | linearize µs | forward µs | trees/s | binding (frac) | T_cp µs | ALU/tensor frac | grid x cluster | e2e trees/s | SM MHz |")
print("|---|---|---|---|---|---|---|---|---|---|---|---|---|")
for w, dt, lat, fu, lin, fwd, v, fr, b, bind, bfr, tcp, ctas, clu, e2e, mhz in rows:
    print(f"| {w} | {dt} | {lat:.1f} | {1 if fu else 2} | {lin:.1f} | {fwd:.1f} | {v:,.0f} | {bind} ({bfr:.3f}) | {tcp:.1f} | {fr:.3f} ({b}) | {ctas} x {clu} | {e2e:,.0f} | {mhz} |")
PY
