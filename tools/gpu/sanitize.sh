# compute-sanitizer memcheck / racecheck / synccheck on one small case per kernel family
mkdir -p gpurun_out/sanitizer
CS=/usr/local/cuda/bin/compute-sanitizer
for c in lin_multi cluster_lstm_fused cluster_lstm cluster_dag_fused rw_gru rw_fc smem_lstm big_lstm mvrnn tc_lstm tc_dag single_rnn; do
  for tool in memcheck racecheck synccheck; do
    timeout 600 $CS --tool $tool --error-exitcode 9 --print-limit 20 python tools/sanitize_case.py $c > gpurun_out/sanitizer/${c}_${tool}.log 2>&1
    rc=$?
    echo "$c $tool rc=$rc $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/sanitizer/${c}_${tool}.log | tail -1)"
  done
done
