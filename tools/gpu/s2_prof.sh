# ncu full capture of the fused cluster kernel (push mode) at cfg2 b10
mkdir -p gpurun_out/prof
B="python bench.py --no-cpu-baseline --no-secondary --steps 3 --warmup 3"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ck_kernel -s 2 -c 1 \
  -o gpurun_out/prof/ck_push_b10 $B --workload cfg2_treelstm_b10 > gpurun_out/prof/ncu.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/prof/ncu.log
ls -la gpurun_out/prof
