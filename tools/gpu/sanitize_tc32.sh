# compute-sanitizer memcheck / racecheck / synccheck on the split-fp32 tensor-core cases
mkdir -p gpurun_out/sanitizer
CS=/usr/local/cuda/bin/compute-sanitizer
for c in tc32_lstm tc32_dag tc32_dag_nohoist tc32_fc; do
  python tools/sanitize_case.py $c || { echo "$c plain run failed"; continue; }
  for tool in memcheck racecheck synccheck; do
    timeout 600 $CS --tool $tool --error-exitcode 9 --print-limit 20 python tools/sanitize_case.py $c > gpurun_out/sanitizer/${c}_${tool}.log 2>&1
    rc=$?
    echo "$c $tool rc=$rc $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/sanitizer/${c}_${tool}.log | tail -1)"
  done
done
