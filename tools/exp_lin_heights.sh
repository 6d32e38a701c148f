# A/B of the single-CTA height modes (CX_LIN_JACOBI: 0 async, 1 rounds, 2 walk-up)
for J in 0 1 2; do
  export CX_LIN_JACOBI=$J
  echo "== CX_LIN_JACOBI=$J"
  for w in cfg2_treelstm_b10 cfg2_treelstm_b1 cfg5_dagrnn_b10 f4_lstm_seq100_b10; do python tools/trace_lin.py $w 2>&1 | head -4; done
  python bench.py --no-secondary --no-cpu-baseline --steps 300 --warmup 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('bench', d['latency_us'], d['linearize_us'], d['two_launch_latency_us'])"
done
