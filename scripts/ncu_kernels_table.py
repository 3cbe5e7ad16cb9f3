"""Formats scripts/gpu_ncu_kernels.sh's ncu --csv metric rows into one line
per launch (profiles/r02_kernels_ncu.txt)."""
import collections, csv, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if r and r[0].isdigit()]
by = collections.OrderedDict()
for r in rows:
    # "ID","Process ID","Process Name","Host Name","Kernel Name",...,"Metric Name","Metric Unit","Metric Value"
    key = (r[0], r[4])
    by.setdefault(key, {})[r[-3]] = (r[-2], r[-1].replace(",", ""))
def val(m, name, unit_to=None):
    u, v = m.get(name, ("", "nan"))
    x = float(v)
    if unit_to == "GB":
        x *= {"byte": 1e-9, "Kbyte": 1e-6, "KB": 1e-6, "Mbyte": 1e-3, "MB": 1e-3,
              "Gbyte": 1.0, "GB": 1.0}.get(u, 1.0)
    if unit_to == "us":
        x *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3,
              "ms": 1e3}.get(u, 1.0)
    return x
for (i, name), m in by.items():
    t = val(m, "gpu__time_duration.sum", "us")
    dr = val(m, "dram__bytes_read.sum", "GB") + val(m, "dram__bytes_write.sum", "GB")
    bc = val(m, "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum")
    wf = val(m, "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum")
    print(f"{name[:56]:56s} {t:9.1f} us  DRAM {dr:6.3f} GB {dr / t * 1e6 if t else 0:7.0f} GB/s  "
          f"smem conflicts {100 * bc / wf if wf else 0:5.1f} %  "
          f"warps {val(m, 'sm__warps_active.avg.pct_of_peak_sustained_active'):5.1f} %  "
          f"regs {val(m, 'launch__registers_per_thread'):3.0f}  "
          f"fma {val(m, 'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active'):5.1f} %  "
          f"fp64 {val(m, 'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active'):5.1f} %  "
          f"issue {val(m, 'smsp__issue_active.avg.pct_of_peak_sustained_active'):5.1f} %")
