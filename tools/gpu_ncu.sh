#!/bin/bash
# ncu evidence at the bench configuration (C5 workload, 296 filters = one
# workspace slot per resident CTA, 2 warm-up steps, 1 profiled step).
# Application replay: the program is rerun per pass (kernel replay would
# save/restore ~80 GB of workspaces per pass).
set -x
mkdir -p gpurun_out
M=gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fp64.sum,sm__inst_executed_pipe_tensor_subpipe_dmma.sum,sm__inst_executed.sum,sm__issue_active.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio,smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio,smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio,smsp__average_warps_issue_stalled_wait_per_issue_active.ratio,smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio,smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio,smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio,smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio,smsp__average_warps_issue_stalled_branch_resolving_per_issue_active.ratio,smsp__average_warps_issue_stalled_sleeping_per_issue_active.ratio
timeout 2400 ncu --replay-mode application --profile-from-start off -k regex:k_items --clock-control none --metrics $M --csv --log-file gpurun_out/r02_ncu_c5_metrics.csv python tools/prof_run.py --batch 296 --warmup 2 --steps 1 > gpurun_out/r02_ncu_c5_metrics.log 2>&1; echo NCU_M_RC=$?
timeout 2400 ncu --replay-mode application --profile-from-start off -k regex:k_items --clock-control none --section SourceCounters --section WarpStateStats --import-source on -f -o gpurun_out/r02_ncu_c5_source python tools/prof_run.py --batch 296 --warmup 2 --steps 1 > gpurun_out/r02_ncu_c5_source.log 2>&1; echo NCU_S_RC=$?
