# strip-kernel bring-up: fast-path parity, nw sweep, ncu counters
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "fast or state_carry or smoke or golden_partitions" 2>&1 | tail -4
for nw in auto 9 8 7 6; do
  if [ $nw = auto ]; then unset FUSEPLAN_STRIP_NW; else export FUSEPLAN_STRIP_NW=$nw; fi
  timeout 120 python scripts/tile_sweep.py 800 600 300 2>&1 | tail -1
done
unset FUSEPLAN_STRIP_NW
FUSEPLAN_VARIANT=fast_tile timeout 120 python scripts/tile_sweep.py 800 600 300 2>&1 | tail -1
timeout 600 ncu --metrics l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,smsp__inst_executed.sum,gpu__time_duration.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio,smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio,smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio,smsp__average_warps_issue_stalled_wait_per_issue_active.ratio,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio,smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio,smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio,smsp__average_warps_issue_stalled_dispatch_stall_per_issue_active.ratio,dram__bytes_read.sum,dram__bytes_write.sum -k regex:k_chain_strip -c 1 python scripts/tile_sweep.py 800 600 300 2>&1 | grep -E "conflicts|wavefronts|inst_executed|duration|issue_active|stalled|dram"
