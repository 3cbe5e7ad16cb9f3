timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
for t in auto 48,38 64,30 80,22 160,22; do
  FUSEPLAN_FAST_TILE=$t timeout 120 python scripts/tile_sweep.py 800 600 300 2>&1 | tail -1
done
FUSEPLAN_FAST_TILE=64,30 timeout 600 ncu --metrics l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,smsp__inst_executed.sum,gpu__time_duration.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio,smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio,smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio,smsp__average_warps_issue_stalled_wait_per_issue_active.ratio,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio -k regex:k_chain_fast -c 1 python scripts/tile_sweep.py 800 600 300 2>&1 | grep -E "conflicts|wavefronts|inst_executed|duration|issue_active|stalled"
