cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 tools/sweep/sha_sweep > gpurun_out/sweep5.log 2>&1
timeout 600 ncu --clock-control none --metrics sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fmaheavy.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,gpu__time_duration.sum,smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio,smsp__warps_active.avg.per_cycle_active,smsp__thread_inst_executed_per_inst_executed.ratio --csv -k regex:l32r -c 14 tools/sweep/sha_sweep > gpurun_out/sweep5_ncu.csv 2>&1
echo done
