set -x
O=gpurun_out/s3p; mkdir -p $O
M=gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,l1tex__throughput.avg.pct_of_peak_sustained_elapsed,smsp__inst_executed.sum,sm__cycles_elapsed.avg,l1tex__m_xbar2l1tex_read_bytes.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_pipe_lsu_wavefronts.sum,smsp__pcsamp_warps_issue_stalled_short_scoreboard,smsp__pcsamp_warps_issue_stalled_barrier,smsp__pcsamp_warps_issue_stalled_mio_throttle,smsp__pcsamp_warps_issue_stalled_long_scoreboard,smsp__pcsamp_warps_issue_stalled_wait,smsp__pcsamp_warps_issue_stalled_lg_throttle
for OT in 64 32; do
SWEEP="[{\"LMKAN_B200_OT\":\"$OT\"}]" timeout 300 ncu --metrics $M --clock-control none -k regex:fwd_fused -s 2 -c 1 --csv python tools/sweep.py 2 > $O/ncu_ot$OT.csv 2>&1
done
