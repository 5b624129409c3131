set -x
tools/ubench_lds_patterns > gpurun_out/ubench_lds2.txt 2>&1
M=gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,smsp__inst_executed_op_shared_ld.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,l1tex__throughput.avg.pct_of_peak_sustained_elapsed,smsp__inst_executed.sum,sm__cycles_elapsed.avg,l1tex__data_pipe_lsu_wavefronts.sum,smsp__average_warp_latency_issue_stalled_mio_throttle.ratio,smsp__average_warp_latency_issue_stalled_short_scoreboard.ratio
for OT in 64 32; do
SWEEP="[{\"LMKAN_B200_OT\":\"$OT\",\"LMKAN_B200_MODE\":\"staged\",\"LMKAN_B200_RT\":\"16\"}]" timeout 300 ncu --metrics $M -k regex:fwd_fused -s 2 -c 1 --csv python tools/sweep.py 2 > gpurun_out/ncu_ot$OT.csv 2>&1
done
