# Tensor-pipe / TMEM / L2 / TMA counters of every kernel of one training step (eager
# launches), for the GEMM roofline analysis.  Run after the same workload exited 0 without
# ncu.   usage: bash tools/gpu_ncu_gemm.sh WORKLOAD [PRECISION]
set -x
W=${1:-alexnet}
M=gpu__time_duration.sum,sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_tc.sum,lts__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_bytes.sum,l1tex__m_xbar2l1tex_read_bytes_pipe_tma.sum,l1tex__data_pipe_tc_wavefronts.avg.pct_of_peak_sustained_elapsed,l1tex__data_pipe_tc_wavefronts_mem_shared_op_utcmma_matrix_a.sum,l1tex__data_pipe_tc_wavefronts_mem_shared_op_utcmma_matrix_b_scope_1cta.sum,l1tex__data_pipe_tc_wavefronts_mem_shared_op_utcmma_matrix_b_scope_2cta.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed
PSG_EAGER=1 timeout 1200 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/gemm_metrics_$W.csv \
  python tools/op_traffic.py run --workload $W --precision ${2:-tf32} --ops gpurun_out/ops_$W.json > gpurun_out/ncu_gemm_$W.log 2>&1
echo ncu rc $?
tail -3 gpurun_out/ncu_gemm_$W.log
