# ncu evidence for every kernel class besides the headline (north star:
# achieved HBM GB/s, shared-memory bank conflicts, occupancy per kernel):
# the exact frame-pair pipeline, the small-frame (config 1) certified launch,
# the unfused stages and the two-fusion F12 / F345 kernels at 800x600.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,launch__grid_size,launch__block_size,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active
run() { timeout 600 ncu --metrics $M --clock-control none --csv "$@" 2>/dev/null | grep -E '^"[0-9]'; }
{
FUSEPLAN_VARIANT=exact run -k regex:k_chain_pair -c 1 python scripts/tile_sweep.py 800 600 1000
run -k regex:"k_chain_pair|k_verify" -c 3 python scripts/small_frames.py 192 432 600
run -k regex:"k_rgba2gray|k_iir|k_gaussian|k_gradient|k_pointwise" -c 5 python scripts/unfused_launches.py 1000
run -k regex:"k_gray_iir|k_chain_pipe" -c 2 python scripts/time_partition.py 800 600 1000 "1-2,3-5"
FUSEPLAN_VARIANT=exact run -k regex:"k_chain_pair" -c 1 python scripts/time_partition.py 800 600 1000 "1-2,3-5"
} > gpurun_out/kernels_ncu.csv
wc -l gpurun_out/kernels_ncu.csv
python scripts/ncu_kernels_table.py gpurun_out/kernels_ncu.csv > gpurun_out/kernels_ncu.txt
cat gpurun_out/kernels_ncu.txt
