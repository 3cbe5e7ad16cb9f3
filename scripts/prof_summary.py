"""Key counters of an ncu raw-page CSV export (one kernel)."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
h, v = rows[0], rows[2]
keys = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'smsp__issue_active.avg.pct_of_peak_sustained_active', 'smsp__inst_executed.sum',
        'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum',
        'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'launch__registers_per_thread',
        'sm__cycles_elapsed.avg.per_second']
for i, n in enumerate(h):
    if n in keys or (n.startswith('smsp__average_warps_issue_stalled') and
                     n.endswith('per_issue_active.ratio') and float(v[i] or 0) > 0.05):
        print(f"{n:80s} {v[i]}")
