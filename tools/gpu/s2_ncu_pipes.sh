# ncu metrics (time, DRAM bytes, FMA / tensor pipe activity, L2 bytes) for one launch of
# every kernel family at its representative workload
mkdir -p gpurun_out/ncu_pipes
ncu --query-metrics --chip gb100 2>/dev/null | grep -E "^sm__pipe_(fma|fmaheavy|alu|tensor|shared|fp)|^sm__inst_executed_pipe_(fma|tensor|uniform)" | head -40 > gpurun_out/ncu_pipes/metric_names.txt
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active,smsp__warps_issue_stalled_barrier_per_warp_active.pct,launch__registers_per_thread,launch__grid_size,launch__block_size,launch__cluster_dim_x
run() {  # name kernel-regex env workload dtype
  env $3 timeout 600 ncu --metrics $M --clock-control none -k regex:"$2" -s 2 -c 1 --csv \
    python bench.py --steps 3 --warmup 3 --no-secondary --no-cpu-baseline --workload $4 --dtype $5 \
    > gpurun_out/ncu_pipes/$1.csv 2> gpurun_out/ncu_pipes/$1.err
  echo "$1 rc=$? $(grep -c gpu__time gpurun_out/ncu_pipes/$1.csv)"
}
run cluster_fused_lstm_b10 ck_kernel X=1 cfg2_treelstm_b10 f32
run cluster_fused_lstm_b10_bf16 ck_kernel X=1 cfg2_treelstm_b10 bf16
run cluster_fused_dag_b10 ck_kernel X=1 cfg5_dagrnn_b10 f32
run rw_treegru_b10 rw_kernel X=1 cfg3_treegru_b10 f32
run rw_treefc_b10 rw_kernel X=1 cfg3_treefc_b10 f32
run mvrnn_b10 mvrnn_kernel X=1 cfg4_mvrnn_b10 f32
run single_treernn_cfg1 sc_kernel X=1 cfg1_treernn f32
run smem_treernn_cfg1 fwd_kernel CX_FUSED=0 cfg1_treernn f32
run lin_single_b10 lin_single_kernel CX_FUSED=0 cfg2_treelstm_b10 f32
run lin_multi_b4096 lin_kernel X=1 cfg5_treelstm_b4096 f32
run big_treelstm_b4096 big_kernel X=1 cfg5_treelstm_b4096 f32
run big_dagrnn_b4096 big_kernel X=1 cfg5_dagrnn_b4096 f32
run tc_treelstm_b4096 tc_kernel X=1 cfg5_treelstm_b4096 bf16
run tc_dagrnn_b4096 tc_kernel X=1 cfg5_dagrnn_b4096 bf16
run tc_treefc_b10 tc_kernel X=1 cfg3_treefc_b10 bf16
